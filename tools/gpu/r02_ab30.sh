# x-face D- exchange by shuffles + pair barriers instead of the second CTA barrier
LIBS="cur=tools/exp/lib_cur.so,xs=tools/exp/lib_xs.so" timeout 1500 python tools/ab_libs.py 3 3,300 | tail -8
