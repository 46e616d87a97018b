#!/bin/bash
# Round 2: the runtime-specialised MRT step (NVRTC) — parity vs oracle and vs the generic kernel,
# interleaved A/B, bench other_configs.
O=gpurun_out/r2cc
mkdir -p $O
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests/test_mrt.py tests/test_dropin_cpp.py tests/test_device_fullsize.py -q -x > $O/pytest.log 2>&1; echo pytest=$?; tail -2 $O/pytest.log
V='{"jit": {"SPLBM_MODEL": "mrt"}, "generic": {"SPLBM_MODEL": "mrt", "SPLBM_MRT_JIT": "0"}}'
timeout 1500 python tools/ab.py "$V" channel128 ras256_phi05 full256 cavity2d_4096_a4 --rounds 11 --steps 128 > $O/ab.txt 2>&1; echo ab=$?
head -4 $O/ab.txt
timeout 900 python bench.py --no-cpu --no-configs4 --no-sweep > $O/bench.json 2>$O/bench.err; echo bench=$?
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['value'], [(o['config'][:40], o['us_per_step'], o['frac_of_measured_peak']) for o in d['other_configs'] if 'MRT' in o['config']])"
