mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t6_test.log 2>&1; echo test=$?
tail -3 gpurun_out/t6_test.log
timeout 900 python bench.py --no-cpu > gpurun_out/t6_bench.log 2>&1; echo bench=$?
python3 -c "
import json; d=json.loads(open('gpurun_out/t6_bench.log').read().strip().splitlines()[-1])
print(d['value'], d['roofline'])
for r in d['porosity_sweep']: print(r['phi'], r['mlups'], r['frac_of_measured_peak'])
for r in d['other_configs']: print(r['config'][:60], r['us_per_step'], r['mlups'])
print(d['e2e'])"
