LIBS="cur=tools/exp/lib_cur.so,xcall=tools/exp/lib_xcall.so" timeout 1200 python tools/ab_libs.py 2 3,300 | tail -8
