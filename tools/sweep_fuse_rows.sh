for F in 0 1; do for R in 16 32 64; do echo "fuse=$F rows=$R"; WB_FUSE_DETECT=$F WB_ROWS=$R python tools/config_sweep.py 20 2>&1 | grep -E "C1|C2|C3|C5"; done; done
