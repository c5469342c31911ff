for k in "c1|kern=smem;kx=1;ky=1;tx=128;ty=32;order=0;occ=0;st=2;bp=1;vec=1" "c1|kern=rt;mx=4;my=4;lx=8;kx=1;ky=1;order=0;occ=0" "c5_t21|kern=smem;kx=2;ky=1;tx=32;ty=64;order=0;occ=0;st=3;bp=1;vec=1" "c1|kern=smem;kx=1;ky=1;tx=64;ty=64;order=0;occ=0;st=3;bp=1;vec=0"; do
row=${k%%|*}; plan=${k#*|}; tag=$(echo "$row$plan" | md5sum | cut -c1-6)
timeout 300 ncu --set full --clock-control none -k regex:'^(tile|dense|vtile|copy|copy_rows|rt|smem)_kernel' -c 1 -f --export /tmp/p_$tag python scripts/run_case.py $row --iters 1 --plan "$plan" > /dev/null 2>&1
echo "== $row $plan" >> gpurun_out/ncu_cmp2.log
python scripts/ncu_summary.py /tmp/p_$tag.ncu-rep --json gpurun_out/cmp2_$tag.json >> gpurun_out/ncu_cmp2.log 2>&1
ncu -i /tmp/p_$tag.ncu-rep --page raw --csv --metrics dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__sectors_read.sum,dram__sectors_write.sum,lts__average_gcomp_input_sector_success_rate.pct,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum.per_second,dram__bytes_write.sum.per_second > gpurun_out/raw2_$tag.csv 2>&1
done
