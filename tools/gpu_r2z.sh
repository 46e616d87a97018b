#!/bin/bash
# Round 2: bench other_configs (MRT rows) with the 10-CTA MRT step; MRT parity tests.
O=gpurun_out/r2z
mkdir -p $O
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_mrt.py tests/test_device_fullsize.py tests/test_dropin_cpp.py -q -x -k "mrt or MRT or dropin" > $O/pytest.log 2>&1; echo pytest=$?; tail -1 $O/pytest.log
timeout 900 python bench.py --no-cpu --no-configs4 --no-sweep > $O/bench.json 2>$O/bench.err; echo bench=$?
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['value'], [(o['config'][:45], o['us_per_step'], o['frac_of_measured_peak']) for o in d['other_configs']])"
