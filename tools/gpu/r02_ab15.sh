# lane rotation A/B, the check-free build at step 300 (replay cost bound), and
# the store/load sector counts of k_step with and without the rotation
LIBS="norot=tools/exp/lib_norot.so,rot=tools/exp/lib_rot.so,nochk=tools/exp/lib_nochk.so" timeout 1500 python tools/ab_libs.py 2 3,300 | tail -12
M=dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_l1tex2xbar_write_sectors_mem_lg_op_st.sum,l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum,l1tex__m_xbar2l1tex_read_sectors_mem_global_op_tma_ld.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
for v in norot rot; do
WB_LIB_PATH=tools/exp/lib_$v.so timeout 600 ncu --metrics $M --clock-control none -k regex:k_step -s 3 -c 1 --csv python bench.py --steps 4 --warmup 3 --no-cpu --no-developed > gpurun_out/r02_mem_$v.csv 2> gpurun_out/r02_mem_$v.err
done
