LIBS="clamp=tools/exp/lib_clamp.so,rnl=tools/exp/lib_rnl.so,yid=tools/exp/lib_yid.so" timeout 1500 python tools/ab_libs.py 3 3,300 | tail -10
