mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_device_single_copy.py -q -x > gpurun_out/aa2_test.log 2>&1; echo test=$?
tail -3 gpurun_out/aa2_test.log
for c in channel128 ras256_phi02; do
  SPLBM_SINGLE_COPY=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:t2c_ -c 8 --csv python tools/profile_case.py $c 8 > gpurun_out/aa2_$c.csv 2>&1; echo ncu=$?
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:t2c_ -c 4 --csv python tools/profile_case.py $c 8 > gpurun_out/aa2_two_$c.csv 2>&1; echo ncu=$?
done
