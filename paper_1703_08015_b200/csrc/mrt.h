// MRT collision operator matrix for the device kernels (reference collision.cpp:11-113).
#pragma once
#include <vector>

namespace splbm_host {

// K = M^-1 S M, row-major q x q, with M the orthogonal moment basis (Lallemand-Luo D2Q9,
// d'Humieres D3Q19), M^-1 = M^T diag(1/|row|^2) and S = diag(rates). `rates` has q entries or is
// null for the default (0 on the conserved moments, 1/tau elsewhere). Products are evaluated in
// the order of the reference's dense matrix products (sum over k ascending, from 0.0), so K is
// bit-identical to CollisionOperator<double>::kernel_ of the oracle build.
std::vector<double> mrt_kernel(int d, double tau, const double* rates);

}  // namespace splbm_host
