#!/bin/bash
# Round 2: store-address re-derivation as the in-tree default vs the old build (reverse A/B) + bench.
O=gpurun_out/r2x
mkdir -p $O
cd "$(dirname "$0")/.."
V='{"rec": {}, "norec": {"LIB": "variants/lib_norec.so"}}'
timeout 1500 python tools/ab.py "$V" channel128 ras256_phi02 ras256_phi05 full256 --rounds 15 --steps 192 > $O/ab.txt 2>&1; echo ab=$?
head -4 $O/ab.txt
timeout 900 python bench.py --no-cpu --no-configs4 > $O/bench.json 2>$O/bench.err; echo bench=$?
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], [ (s['phi'], s['mlups']) for s in d['porosity_sweep']], [(o['config'][:30], o['us_per_step']) for o in d['other_configs']])"
