LIBS="cur=tools/exp/lib_cur2.so,exp2=tools/exp/lib_exp2.so" timeout 1200 python tools/ab_libs.py 3 3,300 | tail -8
