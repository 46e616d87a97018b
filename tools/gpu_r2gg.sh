#!/bin/bash
# Round 2: bench headline + sweep with 64- vs 128-thread 3D step CTAs, alternating twice.
O=gpurun_out/r2gg
mkdir -p $O
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in t64 t128; do
    if [ $v = t128 ]; then L=variants/lib_t128.so; else L=; fi
    SPLBM_LIB=$L timeout 600 python bench.py --no-cpu --no-configs4 --no-other > $O/bench_${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/bench_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', $rep, d['ms_per_step'], [s['mlups'] for s in d['porosity_sweep']])"
  done
done
