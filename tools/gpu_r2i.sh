mkdir -p gpurun_out
ONLY_L2=1 timeout 120 ./tools/pair_probe 1024 32 > gpurun_out/l2_probe.txt 2>&1; echo probe=$?
# DRAM bytes of the pair sequence (C=1 hints) vs the one-step pair: first 2 + 40 launches
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --cache-control none -c 120 --csv ./tools/pair_probe 1024 32 > gpurun_out/pair_probe_ncu.csv 2>&1; echo ncu=$?
