# rows per CTA: wave quantisation of 34 strips x ceil(16384 / L) CTAs over 148 x 3 slots
LIBS="L64=tools/exp/lib_cur.so,L63=tools/exp/lib_cur.so|WB_ROWS=63,L62=tools/exp/lib_cur.so|WB_ROWS=62,L60=tools/exp/lib_cur.so|WB_ROWS=60,L56=tools/exp/lib_cur.so|WB_ROWS=56" timeout 1500 python tools/ab_libs.py 2 3 | tail -7
