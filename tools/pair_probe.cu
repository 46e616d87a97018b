// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pair_probe tools/pair_probe.cu
// Feasibility probe for two-step temporal blocking of the T2C step on B200 (DESIGN.md (f)2): can
// an L2-resident ring of intermediate tile planes (step s+1) survive the streaming traffic of the
// step-s reads and step-s+2 writes, and what does a fused launch sequence cost?
//   one-step:  every tile: 19 x 64 doubles read from src, written to dst (the T2C step's bytes;
//              no cross-tile gathers — this measures the memory system, not the stencil)
//   pair:      launches X(0..J): X(j) = B over plane chunk j-1 (ring -> dst) and A over plane
//              chunk j+1 (src -> ring, one plane ahead); ring slot = plane mod R, R = 2C + 2
// Variants: hint 0 = plain loads/stores, 1 = L2 cache-policy hints (src/dst evict_first, ring
// evict_last), 2 = persisting access-policy window on the ring. Prints us per two steps.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int Q = 19, NTN = 64;
constexpr size_t TILE = size_t(Q) * NTN;  // doubles per tile

__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <int H>
__device__ __forceinline__ double ld(const double* a, uint64_t pol) {
  double v;
  if (H == 1)
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  else
    asm volatile("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(a));
  return v;
}
template <int H>
__device__ __forceinline__ void st(double* a, double v, uint64_t pol) {
  if (H == 1)
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
  else
    asm volatile("st.global.f64 [%0], %1;" ::"l"(a), "d"(v) : "memory");
}

template <int H>
__device__ __forceinline__ void tile_op(const double* in, double* out, bool in_ring, bool out_ring) {
  const int p = threadIdx.x;
  const uint64_t pin = in_ring ? pol_last() : pol_first();
  const uint64_t pout = out_ring ? pol_last() : pol_first();
  double f[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) f[i] = ld<H>(in + i * NTN + p, pin);
  double s = 0;
#pragma unroll
  for (int i = 0; i < Q; ++i) s += f[i];
#pragma unroll
  for (int i = 0; i < Q; ++i) st<H>(out + i * NTN + p, f[i] * 0.999 + s * 1e-3, pout);
}

template <int H>
__global__ void __launch_bounds__(64) one_step(const double* src, double* dst) {
  const size_t t = blockIdx.x;
  tile_op<H>(src + t * TILE, dst + t * TILE, false, false);
}

// CTAs [0, nb): B part (ring plane -> dst), the rest: A part (src -> ring plane)
template <int H>
__global__ void __launch_bounds__(64) x_step(const double* src, double* ring, double* dst, int tpp,
                                              int b_plane0, int nb, int a_plane0, int R, int interleave) {
  int b = blockIdx.x;
  bool isB;
  int k;
  if (interleave) {  // alternate B and A CTAs while both have work
    const int na = gridDim.x - nb;
    const int m = nb < na ? nb : na;
    if (b < 2 * m) { isB = (b & 1) == 0; k = b >> 1; }
    else { isB = nb > na; k = b - m; }
  } else {
    isB = b < nb;
    k = isB ? b : b - nb;
  }
  const int plane = (isB ? b_plane0 : a_plane0) + k / tpp;
  const size_t local = k % tpp;
  double* rp = ring + (size_t(plane % R) * tpp + local) * TILE;
  const size_t gt = size_t(plane) * tpp + local;
  if (isB) tile_op<H>(rp, dst + gt * TILE, true, false);
  else tile_op<H>(src + gt * TILE, rp, false, true);
}

int main(int argc, char** argv) {
  const int tpp = argc > 1 ? atoi(argv[1]) : 1024;  // tiles per plane (128^2 cross-section)
  const int nz = argc > 2 ? atoi(argv[2]) : 32;
  const int reps = 20;
  const size_t n = size_t(tpp) * nz * TILE;
  double *src, *dst;
  cudaMalloc(&src, n * 8);
  cudaMalloc(&dst, n * 8);
  cudaMemset(src, 0, n * 8);
  cudaMemset(dst, 0, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaStream_t s;
  cudaStreamCreate(&s);
  int dev;
  cudaGetDevice(&dev);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  printf("L2 %d B, persisting max %d B, window max %d B\n", prop.l2CacheSize, prop.persistingL2CacheMaxSize,
         prop.accessPolicyMaxWindowSize);
  auto time_it = [&](auto&& body) {
    for (int w = 0; w < 3; ++w) body();
    cudaEventRecord(e0, s);
    for (int r = 0; r < reps; ++r) body();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3 / reps;
  };
  const double pair_bytes = 2.0 * 2.0 * n * 8;  // two steps, read + write each
  {
    double us = time_it([&] {
      one_step<0><<<tpp * nz, 64, 0, s>>>(src, dst);
      one_step<0><<<tpp * nz, 64, 0, s>>>(dst, src);
    });
    printf("one-step x2: %.1f us per two steps (%.0f GB/s)\n", us, pair_bytes / us * 1e-3);
  }
  for (int mb : {8, 16, 32, 48, 64}) {  // L2-resident copy bandwidth (read + write bytes)
    const int nt = int(size_t(mb) * 1000000 / (TILE * 8));
    double us = time_it([&] {
      for (int k = 0; k < 8; ++k) {
        one_step<0><<<nt, 64, 0, s>>>(src, dst);
        one_step<0><<<nt, 64, 0, s>>>(dst, src);
      }
    });
    printf("L2-resident copy %d MB x2: %.1f GB/s\n", mb, 16.0 * 2 * nt * TILE * 8 / us * 1e-3);
  }
  if (getenv("ONLY_L2")) return 0;
  for (int C : {1, 2, 3, 4, 6}) {
    const int R = 2 * C + 2;
    double* ring;
    cudaMalloc(&ring, size_t(R) * tpp * TILE * 8);
    cudaMemset(ring, 0, size_t(R) * tpp * TILE * 8);
    const int nchunk = (nz + C - 1) / C;
    for (int H : {0, 1, 2}) {
      for (int il : {0, 1}) {
        if (H == 2) {
          cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prop.persistingL2CacheMaxSize);
          cudaStreamAttrValue v = {};
          v.accessPolicyWindow.base_ptr = ring;
          v.accessPolicyWindow.num_bytes = std::min<size_t>(size_t(R) * tpp * TILE * 8, prop.accessPolicyMaxWindowSize);
          v.accessPolicyWindow.hitRatio = 1.0f;
          v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
          v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
          cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
        }
        auto launch = [&](int j) {  // X(j): B over chunk j-1, A over planes (j*C, (j+1)*C] (X(0): [0, C])
          int b0 = (j - 1) * C, nbp = j >= 1 ? std::min(C, nz - b0) : 0;
          int a0 = j == 0 ? 0 : j * C + 1;
          int a1 = std::min((j + 1) * C + 1, nz);
          int nap = a1 > a0 ? a1 - a0 : 0;
          int grid = (nbp + nap) * tpp;
          if (grid == 0) return;
          if (H == 1)
            x_step<1><<<grid, 64, 0, s>>>(src, ring, dst, tpp, b0, nbp * tpp, a0, R, il);
          else
            x_step<0><<<grid, 64, 0, s>>>(src, ring, dst, tpp, b0, nbp * tpp, a0, R, il);
        };
        double us = time_it([&] {
          for (int j = 0; j <= nchunk; ++j) launch(j);
        });
        printf("pair C=%d R=%d ring %.0f MB hint=%d interleave=%d: %.1f us per two steps (%.0f GB/s DRAM-equivalent of one-step bytes)\n",
               C, R, R * tpp * TILE * 8 / 1e6, H, il, us, pair_bytes / us * 1e-3);
        if (H == 2) {
          cudaStreamAttrValue v = {};
          v.accessPolicyWindow.num_bytes = 0;
          cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
          cudaCtxResetPersistingL2Cache();
        }
      }
    }
    cudaFree(ring);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
