// Runtime-specialised MRT step: the power-of-two step kernel (step_pow2.cuh)
// compiled through NVRTC for one relaxation operator K, with K's constants folded into the code
// and the products K_ij * delta_j computed once per distinct value of column j (the rows whose
// K_ij are bitwise equal share them; each row still accumulates in the reference's j order, so
// the result is bit-identical to the generic kernel). D3Q19 with default rates at tau 0.8: 139
// instead of 361 products per node.
#pragma once
#include <string>
#include <vector>

namespace splbm_host {

// Source of the collide_mrt_gen<D, INC, R> specialisation for operator K (row-major q x q doubles,
// rounded to float first when f32) — exposed for tests and diagnostics.
std::string mrt_collision_source(int d, bool incompressible, bool f32, const std::vector<double>& K,
                                 int* products_out);

// The kernels compiled for one operator: the two-copy step and the two single-copy (AA) phases.
struct MrtJitKernels {
  const void* step = nullptr;                // t2c_step_pow2_kernel<..., GEN = true>
  const void* aa[2] = {nullptr, nullptr};    // t2c_aa_kernel<..., PHASE 1 / 2, ..., GEN = true>
};

// NVRTC compilation only (no device needed): one cubin with the three kernels and their lowered
// names (step, AA phase 1, AA phase 2).
bool mrt_jit_cubin(int d, int loga, bool incompressible, bool f32, const std::vector<double>& K,
                   std::vector<char>* cubin, std::vector<std::string>* lowered_names, std::string* why);

// The specialised kernels (cudaKernel_t handles, usable as the `func` of cudaLaunchKernelExC) for
// a power-of-two tile edge 2^loga; false with *why set when NVRTC is missing or fails. Compiled
// once per distinct operator in the process.
bool mrt_jit_kernels(int d, int loga, bool incompressible, bool f32, const std::vector<double>& K,
                     MrtJitKernels* out, std::string* why);

}  // namespace splbm_host
