# x-face (speculative + replay) out of line: smaller row loop
LIBS="cur=tools/exp/lib_cur.so,xool=tools/exp/lib_xool.so" timeout 1500 python tools/ab_libs.py 3 3,300 | tail -8
