# y-face exact replay with the Romberg node loop rolled (smaller replay code)
LIBS="cur=tools/exp/lib_cur.so,yr=tools/exp/lib_yr.so" timeout 1500 python tools/ab_libs.py 2 3,300 | tail -8
