LIBS="upd=tools/exp/lib_upd2.so,nsel=tools/exp/lib_nsel.so" timeout 1500 python tools/ab_libs.py 3 3,300 | tail -8
