LIBS="upd=tools/exp/lib_upd2.so,clamp=tools/exp/lib_clamp.so" timeout 1500 python tools/ab_libs.py 3 3,300 | tail -8
WB_LIB_PATH=tools/exp/lib_clamp.so timeout 300 python tools/replay_census.py 300 2>&1 | grep ^step
