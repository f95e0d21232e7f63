# bound on the developed-flow gain of deferring face replays: rejected faces not replayed (not exact)
LIBS="cur=tools/exp/lib_cur.so,norep=tools/exp/lib_norep.so,nochk=tools/exp/lib_nochk.so" timeout 1500 python tools/ab_libs.py 2 3,300 | tail -10
