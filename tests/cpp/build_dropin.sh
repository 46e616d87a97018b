#!/usr/bin/env bash
# TEST INFRASTRUCTURE: builds oracle/_ref/dropin_test from tests/cpp/dropin_test.cpp against the
# UNMODIFIED reference headers/sources (in place under /root/reference) and libsplbm_b200.so.
set -euo pipefail
root="$(cd "$(dirname "$0")/../.." && pwd)"
ref="${SPLBM_REFERENCE:-/root/reference/proj}"
[ -d "$ref/include/splbm" ] || { echo "reference absent; skipping drop-in build" >&2; exit 0; }
mkdir -p "$root/oracle/_ref"
g++ -std=c++20 -O2 -DNDEBUG -pthread -I "$root/oracle/eigen_shim" -I "$ref/include" -I "$ref/tests" \
  -I "$root/include" "$root/tests/cpp/dropin_test.cpp" "$ref/src/lattice.cpp" "$ref/src/collision.cpp" \
  "$ref/src/geometry.cpp" "$ref/src/tiling.cpp" \
  -L "$root/paper_1703_08015_b200" -l:libsplbm_b200.so \
  -Wl,-rpath,'$ORIGIN/../../paper_1703_08015_b200' -o "$root/oracle/_ref/dropin_test"
echo "built $root/oracle/_ref/dropin_test"
