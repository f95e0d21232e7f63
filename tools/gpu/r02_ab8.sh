LIBS="rm=tools/exp/lib_rm.so,upd=tools/exp/lib_upd.so" timeout 1500 python tools/ab_libs.py 2 3,300 | tail -8
WB_LIB_PATH=tools/exp/lib_upd.so timeout 300 python tools/replay_census.py 300 2>&1 | grep ^step
