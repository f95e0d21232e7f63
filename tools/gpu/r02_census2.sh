# lane-level vs warp-level replay counts at steps 3..300 of the bench slab
timeout 600 python tools/replay_census.py 300 2>&1 | grep ^step
WB_LIB_PATH=tools/exp/lib_wrep.so timeout 600 python tools/replay_census.py 300 2>&1 | grep ^step
