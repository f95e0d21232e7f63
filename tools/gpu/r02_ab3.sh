LIBS="ysm=tools/exp/lib_ysm.so,rot=tools/exp/lib_rot.so,rotq=tools/exp/lib_rotq.so" timeout 1200 python tools/ab_libs.py 3 3,300 | tail -10
