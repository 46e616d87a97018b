mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench2.log 2>&1; echo bench=$?
tail -c 6000 gpurun_out/bench2.log
