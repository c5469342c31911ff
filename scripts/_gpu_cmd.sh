L=$PWD/paper_1603_02297_b200/_lib
P="kern=smem;kx=2;ky=2;tx=64;ty=64;order=1;occ=0;st=2"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,lts__t_sectors_srcunit_tex_op_write_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum
for c in p_t00_a79 p_t00_a80; do
TTB_LIB_PATH=$L/libttb_noload.so timeout 120 python scripts/run_case.py $c --plan "$P" --iters 3 > gpurun_out/p_$c.log 2>&1 && TTB_LIB_PATH=$L/libttb_noload.so timeout 600 ncu --metrics $M --clock-control none -k regex:dense_kernel -s 2 -c 1 --csv --log-file gpurun_out/m_$c.csv python scripts/run_case.py $c --plan "$P" --iters 3 > gpurun_out/ncu_$c.log 2>&1
done
