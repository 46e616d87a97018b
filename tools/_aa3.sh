mkdir -p gpurun_out
for c in channel128 ras256_phi02; do
  SPLBM_SINGLE_COPY=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,smsp__inst_executed.sum,launch__registers_per_thread --clock-control none -k regex:t2c_ -c 4 --csv python tools/profile_case.py $c 6 > gpurun_out/aa3_$c.csv 2>&1; echo ncu=$?
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,smsp__inst_executed.sum --clock-control none -k regex:t2c_ -c 2 --csv python tools/profile_case.py channel128 4 > gpurun_out/aa3_two.csv 2>&1
