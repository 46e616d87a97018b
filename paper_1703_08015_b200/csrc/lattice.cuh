// Lattice constants and the per-node physics of the T2C step, shared by all device kernels.
//
// Directions follow the reference order exactly (lattice.cpp:18-25 D2Q9, 33-42 D3Q19): rest,
// axes, planar diagonals, opposite directions in adjacent pairs. Components are packed two bits
// per direction so every lookup folds to an immediate in the unrolled loops.
//
// Arithmetic contract: every floating-point operation is an explicit
// round-to-nearest intrinsic (__dadd_rn/__dmul_rn/__ddiv_rn, __fadd_rn/... for the f32 engine) in
// the reference's operation order, all in the engine's real type R (the reference's T: double or
// float, lattice.hpp:72-112), so nvcc cannot contract to FMA and results are bit-identical to the
// reference built with its CMake Release flags. Products by a zero direction component are omitted: x + (+-0) == x for
// x != 0 and a zero sum starts from +0, so the omitted terms never change a finite result (the
// only difference is on states that already fail the step's finite check).
#pragma once
#ifndef __CUDACC_RTC__
#include <cstdint>
#endif

namespace splbm_dev {

template <int D>
struct Lat;

// (e+1) packed 2 bits per direction, direction 0 in the low bits.
__host__ __device__ constexpr uint64_t pack_dirs(const int* v, int q) {
  uint64_t r = 0;
  for (int i = q - 1; i >= 0; --i) r = (r << 2) | static_cast<uint64_t>(v[i] + 1);
  return r;
}

template <>
struct Lat<2> {
  static constexpr int Q = 9;
  static constexpr int ex_[9] = {0, 1, -1, 0, 0, 1, -1, 1, -1};
  static constexpr int ey_[9] = {0, 0, 0, 1, -1, 1, -1, -1, 1};
  static constexpr int ez_[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  static constexpr uint64_t EX = pack_dirs(ex_, 9);
  static constexpr uint64_t EY = pack_dirs(ey_, 9);
  static constexpr uint64_t EZ = pack_dirs(ez_, 9);
  __host__ __device__ static constexpr double w(int i) {
    return i == 0 ? 4.0 / 9.0 : (i <= 4 ? 1.0 / 9.0 : 1.0 / 36.0);
  }
};

template <>
struct Lat<3> {
  static constexpr int Q = 19;
  static constexpr int ex_[19] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0};
  static constexpr int ey_[19] = {0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1};
  static constexpr int ez_[19] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1};
  static constexpr uint64_t EX = pack_dirs(ex_, 19);
  static constexpr uint64_t EY = pack_dirs(ey_, 19);
  static constexpr uint64_t EZ = pack_dirs(ez_, 19);
  __host__ __device__ static constexpr double w(int i) {
    return i == 0 ? 1.0 / 3.0 : (i <= 6 ? 1.0 / 18.0 : 1.0 / 36.0);
  }
};

template <int D>
__host__ __device__ constexpr int ex(int i) {
  return static_cast<int>((Lat<D>::EX >> (2 * i)) & 3ull) - 1;
}
template <int D>
__host__ __device__ constexpr int ey(int i) {
  return static_cast<int>((Lat<D>::EY >> (2 * i)) & 3ull) - 1;
}
template <int D>
__host__ __device__ constexpr int ez(int i) {
  return static_cast<int>((Lat<D>::EZ >> (2 * i)) & 3ull) - 1;
}
// opposite pairs are adjacent (lattice.cpp:65-74 finds exactly this)
__host__ __device__ constexpr int opp(int i) { return i == 0 ? 0 : ((i & 1) ? i + 1 : i - 1); }

// Round-to-nearest arithmetic in the engine's real type (overloads; never mix with a double
// literal — every constant below is R(...), as the reference writes T(...)).
//
// SPLBM_FMA=1 (experiment / tolerance-mode builds only, never the parity library): plain operators,
// so nvcc contracts multiply-adds into FMA (the reference built with -march=native does the same
// on the CPU: <= 1.1e-13 after 1000 steps), and the velocity division becomes a
// reciprocal multiply (the paper's GPU kernels).
#ifndef SPLBM_FMA
#define SPLBM_FMA 0
#endif
#if SPLBM_FMA
__device__ __forceinline__ double dadd(double a, double b) { return a + b; }
__device__ __forceinline__ double dsub(double a, double b) { return a - b; }
__device__ __forceinline__ double dmul(double a, double b) { return a * b; }
__device__ __forceinline__ double ddiv(double a, double b) { return a / b; }
__device__ __forceinline__ float dadd(float a, float b) { return a + b; }
__device__ __forceinline__ float dsub(float a, float b) { return a - b; }
__device__ __forceinline__ float dmul(float a, float b) { return a * b; }
__device__ __forceinline__ float ddiv(float a, float b) { return a / b; }
#else
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float dadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float dsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float dmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float ddiv(float a, float b) { return __fdiv_rn(a, b); }
#endif
__device__ __forceinline__ bool finite(double v) { return isfinite(v); }
__device__ __forceinline__ bool finite(float v) { return isfinite(v); }

#ifndef SPLBM_FAST_DIV
#define SPLBM_FAST_DIV 1
#endif

// u_k = m_k / rho for the three momenta, each correctly rounded (IEEE division, as the reference
// computes mom.u /= mom.rho, collision.hpp:48). Fast path: one correctly rounded reciprocal
// y = RN(1/rho) shared by the three quotients, then Markstein's correction per quotient:
//   q0 = RN(m*y) (within 1 ulp of m/rho), r = fma(-rho, q0, m) (exact), q = RN(q0 + r*y) = RN(m/rho)
// (Markstein's theorem; Handbook of Floating-Point Arithmetic, Th. 8.10). It holds while no
// intermediate leaves the normal range, which the exponent guard ensures; zeros keep their sign
// via m*y; anything else takes the full IEEE division.
__device__ __forceinline__ bool div_safe(double v) {
  const double av = fabs(v);
  return av == 0.0 || (av >= 0x1p-480 && av <= 0x1p480);
}
__device__ __forceinline__ void divide3(double& m0, double& m1, double& m2, double rho) {
#if SPLBM_FMA
  const double y = 1.0 / rho;
  m0 *= y;
  m1 *= y;
  m2 *= y;
  return;
#endif
#if SPLBM_FAST_DIV
  const double ar = fabs(rho);
  if (ar >= 0x1p-480 && ar <= 0x1p480 && div_safe(m0) && div_safe(m1) && div_safe(m2)) {
    const double y = __drcp_rn(rho);
    auto q = [&](double m) {
      const double q0 = __dmul_rn(m, y);
      if (m == 0.0) return q0;
      const double r = __fma_rn(-rho, q0, m);
      return __fma_rn(r, y, q0);
    };
    m0 = q(m0);
    m1 = q(m1);
    m2 = q(m2);
    return;
  }
#endif
  m0 = ddiv(m0, rho);
  m1 = ddiv(m1, rho);
  m2 = ddiv(m2, rho);
}
// f32 engine: the same shared correctly rounded reciprocal + Markstein correction in binary32
// (the theorem is format-independent); the guard keeps every intermediate normal (|q| within
// 2^+-100, the residual above 2^-126), anything else takes IEEE __fdiv_rn. Besides saving two
// reciprocals, it keeps zero momenta (a domain started from rest) off __fdiv_rn's slow path.
__device__ __forceinline__ bool div_safe(float v) {
  const float av = fabsf(v);
  return av == 0.0f || (av >= 0x1p-50f && av <= 0x1p50f);
}
__device__ __forceinline__ void divide3(float& m0, float& m1, float& m2, float rho) {
#if SPLBM_FMA
  const float y = 1.0f / rho;
  m0 *= y;
  m1 *= y;
  m2 *= y;
  return;
#endif
#if SPLBM_FAST_DIV
  const float ar = fabsf(rho);
  if (ar >= 0x1p-50f && ar <= 0x1p50f && div_safe(m0) && div_safe(m1) && div_safe(m2)) {
    const float y = __frcp_rn(rho);
    auto q = [&](float m) {
      const float q0 = __fmul_rn(m, y);
      if (m == 0.0f) return q0;
      const float r = __fmaf_rn(-rho, q0, m);
      return __fmaf_rn(r, y, q0);
    };
    m0 = q(m0);
    m1 = q(m1);
    m2 = q(m2);
    return;
  }
#endif
  m0 = ddiv(m0, rho);
  m1 = ddiv(m1, rho);
  m2 = ddiv(m2, rho);
}

// sum_i e_ik * f_i in direction order, zero components omitted (moments<T>, lattice.hpp:97-102)
template <int D, int K, class R>
__device__ __forceinline__ R momentum(const R* f) {
  R m = R(0);
#pragma unroll
  for (int i = 0; i < Lat<D>::Q; ++i) {
    const int e = K == 0 ? ex<D>(i) : (K == 1 ? ey<D>(i) : ez<D>(i));
    if (e > 0) m = dadd(m, f[i]);
    if (e < 0) m = dsub(m, f[i]);
  }
  return m;
}

template <int D, class R>
__device__ __forceinline__ R density(const R* f) {
  R r = R(0);
#pragma unroll
  for (int i = 0; i < Lat<D>::Q; ++i) r = dadd(r, f[i]);
  return r;
}

// e_i . u in the order (e0 u0 + e1 u1) + e2 u2 with zero terms omitted (lattice.hpp:82)
template <int D, class R>
__device__ __forceinline__ R edotu(int i, R u0, R u1, R u2) {
  const int a = ex<D>(i), b = ey<D>(i), c = ez<D>(i);
  R cu = R(0);
  bool first = true;
  if (a != 0) {
    cu = a > 0 ? u0 : -u0;
    first = false;
  }
  if (b != 0) {
    const R t = b > 0 ? u1 : -u1;
    cu = first ? t : dadd(cu, t);
    first = false;
  }
  if (c != 0) {
    const R t = c > 0 ? u2 : -u2;
    cu = first ? t : dadd(cu, t);
  }
  return cu;
}

// T(lat.w[i]): the double weight rounded to the engine's type (lattice.hpp:86-88)
template <int D, class R>
__device__ __forceinline__ constexpr R weight(int i) {
  return static_cast<R>(Lat<D>::w(i));
}

// equilibrium<T> (lattice.hpp:72-91); uu = (u0^2 + u1^2) + u2^2 (oracle Eigen-shim order).
template <int D, bool INC, class R>
__device__ __forceinline__ R feq(int i, R rho, R u0, R u1, R u2, R uu) {
  const R cu = edotu<D>(i, u0, u1, u2);
  const R shape = dsub(dadd(dmul(cu, R(3)), dmul(dmul(cu, cu), R(4.5))), dmul(uu, R(1.5)));
  const R w = weight<D, R>(i);
  return INC ? dmul(w, dadd(rho, shape)) : dmul(dmul(w, rho), dadd(R(1), shape));
}

// The equilibria of an opposite pair (i, opp(i) = i + 1, i odd) at once. Negation is exact and
// round-to-nearest is sign-symmetric, so with cu' = -cu: cu'*3 = -(cu*3), cu'*cu' = cu*cu and
// (-(cu*3)) + q = q - cu*3 — the pair shares e.u, cu*3 and (cu*cu)*4.5 and each value is still
// bit-identical to feq() (the reference's per-direction formula, lattice.hpp:78-89).
template <int D, bool INC, class R>
__device__ __forceinline__ void feq_pair(int i, R rho, R u0, R u1, R u2, R uu15, R& fp, R& fm) {
  const R cu = edotu<D>(i, u0, u1, u2);
  const R c3 = dmul(cu, R(3));
  const R q = dmul(dmul(cu, cu), R(4.5));
  const R sp = dsub(dadd(c3, q), uu15);
  const R sm = dsub(dsub(q, c3), uu15);
  const R w = weight<D, R>(i);
  if (INC) {
    fp = dmul(w, dadd(rho, sp));
    fm = dmul(w, dadd(rho, sm));
  } else {
    const R wr = dmul(w, rho);
    fp = dmul(wr, dadd(R(1), sp));
    fm = dmul(wr, dadd(R(1), sm));
  }
}

template <class R>
__device__ __forceinline__ R sqnorm(R u0, R u1, R u2) {
  return dadd(dadd(dmul(u0, u0), dmul(u1, u1)), dmul(u2, u2));
}

template <int D, bool INC, class R>
__device__ __forceinline__ void equilibrium(R rho, R u0, R u1, R u2, R* out) {
  const R uu = sqnorm(u0, u1, u2);
  const R uu15 = dmul(uu, R(1.5));
  out[0] = feq<D, INC>(0, rho, u0, u1, u2, uu);
#pragma unroll
  for (int i = 1; i < Lat<D>::Q; i += 2) feq_pair<D, INC>(i, rho, u0, u1, u2, uu15, out[i], out[i + 1]);
}

// CollisionOperator<T>::operator() BGK branch (collision.hpp:35-65). Returns
// finite_moments(m) (engine.hpp:96-102); on a broken quasi-compressible density f is left
// untouched and the step fails (collision.hpp:44-47). inv_tau = T(1.0 / tau) (collision.cpp:93).
template <int D, bool INC, class R>
__device__ __forceinline__ bool collide_bgk(R* f, R inv_tau) {
  const R rho = density<D>(f);
  R u0 = momentum<D, 0>(f);
  R u1 = momentum<D, 1>(f);
  R u2 = momentum<D, 2>(f);
  if (!INC) {
    if (!(rho > R(0)) || !finite(rho)) return false;
    divide3(u0, u1, u2, rho);
  }
  const R uu = sqnorm(u0, u1, u2);
  const R uu15 = dmul(uu, R(1.5));
  f[0] = dadd(f[0], dmul(inv_tau, dsub(feq<D, INC>(0, rho, u0, u1, u2, uu), f[0])));
#pragma unroll
  for (int i = 1; i < Lat<D>::Q; i += 2) {
    R fp, fm;
    feq_pair<D, INC>(i, rho, u0, u1, u2, uu15, fp, fm);
    f[i] = dadd(f[i], dmul(inv_tau, dsub(fp, f[i])));
    f[i + 1] = dadd(f[i + 1], dmul(inv_tau, dsub(fm, f[i + 1])));
  }
  return finite(rho) && finite(u0) && finite(u1) && finite(u2);
}

// CollisionOperator<T>::operator() MRT branch (collision.hpp:54-63): the same moments and
// equilibrium as BGK, then f_i += sum_j K_ij (feq_j - f_j) with the q x q operator K = M^-1 S M
// (row-major, T(kernel(i, j)), a __grid_constant__ kernel parameter: the constants feed the
// multiplies directly).
template <int D, bool INC, class R>
__device__ __forceinline__ bool collide_mrt(R* f, const R* K) {
  constexpr int Q = Lat<D>::Q;
  const R rho = density<D>(f);
  R u0 = momentum<D, 0>(f);
  R u1 = momentum<D, 1>(f);
  R u2 = momentum<D, 2>(f);
  if (!INC) {
    if (!(rho > R(0)) || !finite(rho)) return false;
    divide3(u0, u1, u2, rho);
  }
  R delta[Q];
  equilibrium<D, INC>(rho, u0, u1, u2, delta);
#pragma unroll
  for (int i = 0; i < Q; ++i) delta[i] = dsub(delta[i], f[i]);
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    R acc = R(0);
#pragma unroll
    for (int j = 0; j < Q; ++j) acc = dadd(acc, dmul(K[i * Q + j], delta[j]));
    f[i] = dadd(f[i], acc);
  }
  return finite(rho) && finite(u0) && finite(u1) && finite(u2);
}

struct BcParams {
  double u0, u1, u2;
  double rho;
};

// apply_boundary<T> (engine.hpp:32-65). type 2 = VelocityBC, 3 = PressureBC. The BC velocity and
// density are the doubles of BcParams rounded to T (bc.velocity.cast<T>(), T(bc.density)).
template <int D, bool INC, class R>
__device__ __forceinline__ bool apply_boundary(R* f, int type, bool rho_underdetermined,
                                               const BcParams bc) {
  if (type == 2) {
    R rho = R(1);
    if (!rho_underdetermined) {
      rho = density<D>(f);
      if (!(rho > R(0)) || !finite(rho)) rho = R(1);
    }
    const R b0 = static_cast<R>(bc.u0), b1 = static_cast<R>(bc.u1), b2 = static_cast<R>(bc.u2);
    equilibrium<D, INC>(rho, b0, b1, b2, f);
    return finite(rho) && finite(b0) && finite(b1) && finite(b2);
  }
  const R rho = density<D>(f);
  const R m0 = momentum<D, 0>(f), m1 = momentum<D, 1>(f), m2 = momentum<D, 2>(f);
  R u0 = R(0), u1 = R(0), u2 = R(0);
  if (!INC) {
    if (rho > R(0)) {
      u0 = m0;
      u1 = m1;
      u2 = m2;
      divide3(u0, u1, u2, rho);
    }
  } else {
    u0 = m0;
    u1 = m1;
    u2 = m2;
  }
  const R rb = static_cast<R>(bc.rho);
  equilibrium<D, INC>(rb, u0, u1, u2, f);
  return finite(rb) && finite(u0) && finite(u1) && finite(u2);
}

}  // namespace splbm_dev
