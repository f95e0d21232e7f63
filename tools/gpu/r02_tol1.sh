LIBS="base=tools/exp/lib_base.so,tol1=tools/exp/lib_tol1.so" timeout 900 python tools/ab_libs.py 2 3,300
WB_LIB_PATH=tools/exp/lib_tol1.so timeout 300 python tools/replay_census.py 300 2>&1 | grep ^step
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
