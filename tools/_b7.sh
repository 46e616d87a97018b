mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/b7.log 2>&1; echo bench=$?
python3 -c "
import json; d=json.loads(open('gpurun_out/b7.log').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['overhead'])
for r in d['porosity_sweep']: print(r['phi'], r['mlups'], r['frac_of_measured_peak'], r['overhead'])
print(d['cpu_baseline'])
for r in d['other_configs']: print(r['config'][:60], r['us_per_step'], r['mlups'])"
