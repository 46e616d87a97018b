#!/bin/bash
# Round 2: 3D step in 128-thread CTAs (default) vs 64 (variant), bench-level, alternating twice.
O=gpurun_out/r2vv
mkdir -p $O
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in t128 t64; do
    if [ $v = t64 ]; then L=variants/lib_t64.so; else L=; fi
    SPLBM_LIB=$L timeout 600 python bench.py --no-cpu --no-configs4 > $O/bench_${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/bench_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', $rep, d['ms_per_step'], [s['mlups'] for s in d['porosity_sweep']], [o['us_per_step'] for o in d['other_configs'][:4]])"
  done
done
