# IEEE division of the replays out of line (smaller replay code)
LIBS="cur=tools/exp/lib_cur.so,divcall=tools/exp/lib_divcall.so" timeout 1500 python tools/ab_libs.py 3 3,300 | tail -8
