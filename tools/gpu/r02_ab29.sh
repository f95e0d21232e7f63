# Phys for the replays from constant memory by slot (no per-thread stack copy at kernel entry)
LIBS="cur=tools/exp/lib_cur.so,cs2=tools/exp/lib_cs2.so" timeout 1500 python tools/ab_libs.py 2 3,300 | tail -8
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
WB_LIB_PATH=tools/exp/lib_cs2.so timeout 600 ncu --metrics $M --clock-control none -k regex:k_step -s 3 -c 1 --csv python bench.py --steps 4 --warmup 3 --no-cpu --no-developed 2>/dev/null | grep -o '"dram__bytes_[a-z]*.sum","byte","[0-9]*"\|"gpu__time_duration.sum","ns","[0-9]*"'
