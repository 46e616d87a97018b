#!/bin/bash
# Round 2: z-range L2 prefetch under the 1024^3 power cap (fewer DRAM bytes -> less power?):
# alternating runs, RAS 1024^3 phi 0.2 two copies.
O=gpurun_out/r2ll
mkdir -p $O
cd "$(dirname "$0")/.."
for rep in 1 2 3; do
  for v in 0 1; do
    SPLBM_PF_RANGE=$v timeout 600 python tools/size_probe.py 1024 1024 1024 0.2 --steps 100 --warmup 10 | sed "s/^/range=$v /"
  done
done > $O/probe.txt 2>&1
cat $O/probe.txt
