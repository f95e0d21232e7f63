LIBS="exp2=tools/exp/lib_exp2.so,bpair=tools/exp/lib_bpair.so,rmode=tools/exp/lib_rmode.so,both=tools/exp/lib_both.so" timeout 1500 python tools/ab_libs.py 2 3,300 | tail -12
