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

// NVRTC compilation only (no device needed): the cubin and the kernel's lowered name.
bool mrt_jit_cubin(int d, int loga, bool incompressible, bool f32, const std::vector<double>& K,
                   std::vector<char>* cubin, std::string* lowered_name, std::string* why);

// The specialised step kernel (a cudaKernel_t, usable as the `func` of cudaLaunchKernelExC) for a
// power-of-two tile edge 2^loga, or nullptr with *why set (NVRTC missing, compile error, ...).
// Compiled once per distinct source in the process.
const void* mrt_jit_kernel(int d, int loga, bool incompressible, bool f32, const std::vector<double>& K,
                           std::string* why);

}  // namespace splbm_host
