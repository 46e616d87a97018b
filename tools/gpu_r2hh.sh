#!/bin/bash
# Round 2: sanitizer round incl. the specialised MRT step and the D2Q9 f64 two-node step; GPU suite.
O=gpurun_out/r2hh
mkdir -p $O
cd "$(dirname "$0")/.."
bash tools/sanitize_round.sh > $O/sanitizer.txt 2>&1; echo san=$?
grep -c "rc=0" $O/sanitizer.txt; grep -v "rc=0" $O/sanitizer.txt | head
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest=$?; tail -1 $O/pytest.log
