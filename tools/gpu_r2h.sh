mkdir -p gpurun_out
timeout 300 ./tools/pair_probe 1024 32 > gpurun_out/pair_probe.txt 2>&1; echo probe=$?
timeout 300 ./tools/pair_probe 4096 64 > gpurun_out/pair_probe_256.txt 2>&1; echo probe2=$?
for i in 1 2 3 4 5 6; do timeout 600 python -m pytest tests/test_slab_mp_gpu.py tests/test_slab_gpu.py -q -x -p no:cacheprovider > gpurun_out/flake_$i.log 2>&1; echo "loop$i=$? $(tail -1 gpurun_out/flake_$i.log)"; done
