#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Compiles the UNMODIFIED reference solver in place from
# /root/reference/proj (no sources are copied) plus oracle/ref_capi.cpp into
#   oracle/_ref/libsplbm_ref.so       bitwise oracle: the reference's CMake Release flags
#                                     (-O3 -DNDEBUG, baseline x86-64 => no FMA contraction)
#   oracle/_ref/libsplbm_ref_fast.so  CPU timing baseline: same sources, -march=x86-64-v3
#                                     (AVX2+FMA; FMA contraction changes bits ~1e-15)
#   oracle/_ref/libsplbm_ref_v4.so    CPU timing baseline for AVX-512 hosts, -march=x86-64-v4
# (-march=native is not an option: the GPU box has no /root/reference to compile from, so the
# timing builds are the portable ISA levels; bench.py loads the highest one the host supports.)
# Eigen3 is absent from the image; oracle/eigen_shim provides the subset the reference uses.
# vtk.cpp/config.cpp (output, CLI plumbing) are not needed by the hot path and not built.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${SPLBM_REFERENCE:-/root/reference/proj}"
out="$here/_ref"
if [ ! -d "$ref/include/splbm" ]; then
  echo "reference tree not found at $ref; skipping oracle/_ref build" >&2
  exit 0
fi
mkdir -p "$out"
srcs=("$ref/src/lattice.cpp" "$ref/src/collision.cpp" "$ref/src/geometry.cpp"
      "$ref/src/tiling.cpp" "$ref/src/overhead.cpp" "$here/ref_capi.cpp")
common=(-std=c++20 -DNDEBUG -fPIC -shared -pthread -I "$here/eigen_shim" -I "$ref/include" -I "$ref/tests")
g++ -O3 -ffp-contract=off "${common[@]}" "${srcs[@]}" -o "$out/libsplbm_ref.so.tmp"
mv "$out/libsplbm_ref.so.tmp" "$out/libsplbm_ref.so"
g++ -O3 -march=x86-64-v3 "${common[@]}" "${srcs[@]}" -o "$out/libsplbm_ref_fast.so.tmp"
mv "$out/libsplbm_ref_fast.so.tmp" "$out/libsplbm_ref_fast.so"
g++ -O3 -march=x86-64-v4 -mprefer-vector-width=512 "${common[@]}" "${srcs[@]}" -o "$out/libsplbm_ref_v4.so.tmp"
mv "$out/libsplbm_ref_v4.so.tmp" "$out/libsplbm_ref_v4.so"
echo "built $out/libsplbm_ref.so, libsplbm_ref_fast.so and libsplbm_ref_v4.so"
