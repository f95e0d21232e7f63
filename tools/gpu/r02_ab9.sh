LIBS="upd=tools/exp/lib_upd.so,tait=tools/exp/lib_tait.so" timeout 1500 python tools/ab_libs.py 3 3,300 | tail -8
