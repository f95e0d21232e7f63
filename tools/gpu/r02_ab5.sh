LIBS="cur=tools/exp/lib_cur2.so,nt192=tools/exp/lib_nt192.so|WB_KSTEP_VARIANT=11,nt128=tools/exp/lib_nt192.so" timeout 1200 python tools/ab_libs.py 2 3,300 | tail -10
