LIBS="ysm=tools/exp/lib_ysm.so,xdiv=tools/exp/lib_xdiv.so,det64=tools/exp/lib_l128.so,l128=tools/exp/lib_l128.so|WB_ROWS=128" timeout 1200 python tools/ab_libs.py 2 3,300 | tail -14
