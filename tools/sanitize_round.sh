#!/bin/bash
# compute-sanitizer memcheck / racecheck / initcheck over the step paths (two copies, single copy,
# f32, pow2 and generic kernels, the resident multi-step kernel) and the device RAS generator;
# summary table on stdout.
mkdir -p gpurun_out/san
cd "$(dirname "$0")/.."
run() {  # name env case
  local name=$1; shift; local envs=$1; shift; local case=$1
  for t in memcheck racecheck initcheck; do
    env $envs timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/profile_case.py $case 3 > gpurun_out/san/${t}_$name.log 2>&1
    echo "$name $t rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${t}_$name.log | tail -1)"
  done
}
run ras48_f64 "SPLBM_PRECISION=f64" ras48_periodic
run ras48_single_copy "SPLBM_SINGLE_COPY=1" ras48_periodic
run ras48_f32 "SPLBM_PRECISION=f32" ras48_periodic
run channel_single_copy_f32 "SPLBM_SINGLE_COPY=1 SPLBM_PRECISION=f32" channel3d_small
run cavity2d_a16_single_copy "SPLBM_SINGLE_COPY=1" cavity2d_64_a16
run random_a3_generic "SPLBM_PRECISION=f64" random_a3
run ras48_mrt "SPLBM_MODEL=mrt" ras48_periodic
run ras_device_generator "SPLBM_PRECISION=f64" ras_device_generator
# round 2: the resident multi-step kernel (small domains: cooperative grid, neighbour-CTA flags)
run cavity2d_256_resident "SPLBM_PRECISION=f64" cavity2d_256_a4
run cavity2d_256_resident_f32 "SPLBM_PRECISION=f32" cavity2d_256_a4
run channel3d_small_resident "SPLBM_PRECISION=f64" channel3d_small
run channel3d_small_streamed "SPLBM_RESIDENT=0" channel3d_small
# round 2: the MRT step specialised through NVRTC, the D2Q9 f64 two-nodes-per-thread step
run ras48_mrt_specialised "SPLBM_MODEL=mrt" ras48_periodic
run ras48_single_copy_mrt_specialised "SPLBM_MODEL=mrt SPLBM_SINGLE_COPY=1" ras48_periodic
run cavity2d_512_x2 "SPLBM_PRECISION=f64" cavity2d_512_a4
