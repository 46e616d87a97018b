// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/barrier_probe tools/barrier_probe.cu
// Cost of one grid-wide barrier on B200 for the resident multi-step kernel (t2c_resident_kernel):
// G CTAs x T threads, N barriers back to back, optionally with a store + L2 load per thread
// between barriers (a step's memory traffic in miniature). Variants:
//   0 counter: atomicAdd arrival + acquire spin on a generation word (the kernel's barrier)
//   1 counter + __nanosleep backoff in the spin
//   2 flags: every CTA release-stores its epoch in its own 128-B slot, CTA 0's threads gather
//     them with acquire loads and release the generation; the others spin on it
//   3 cooperative_groups grid.sync()
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int V>
__device__ __forceinline__ void barrier(unsigned* bar, unsigned* flags, unsigned epoch) {
  if (V == 3) {
    cg::this_grid().sync();
    return;
  }
  __syncthreads();
  if (V == 2) {
    if (threadIdx.x == 0) {
      __threadfence();
      st_rel(flags + blockIdx.x * 32, epoch);
    }
    if (blockIdx.x == 0) {
      for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
        while (ld_acq(flags + b * 32) < epoch) {
        }
      __syncthreads();
      if (threadIdx.x == 0) st_rel(bar + 1, epoch);
    } else if (threadIdx.x == 0) {
      while (ld_acq(bar + 1) < epoch) {
      }
    }
    __syncthreads();
    return;
  }
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acq(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      st_rel(bar + 1, gen + 1);
    } else {
      while (ld_acq(bar + 1) == gen) {
        if (V == 1) __nanosleep(32);
      }
    }
  }
  __syncthreads();
}

template <int V, bool WORK>
__global__ void probe(unsigned* bar, unsigned* flags, double* buf, int n, unsigned epoch0) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const size_t total = static_cast<size_t>(gridDim.x) * blockDim.x;
  double acc = 0;
  for (int s = 0; s < n; ++s) {
    if (WORK) {
      double v;
      asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(buf + ((i + 977 * (s + 1)) % total)) : "memory");
      acc += v;
      buf[total + i] = acc;
    }
    barrier<V>(bar, flags, epoch0 + s + 1);
  }
  if (acc == 12345.0) buf[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *bar, *flags;
  double* buf;
  cudaMalloc(&bar, 8);
  cudaMalloc(&flags, 4096 * 128);
  cudaMalloc(&buf, 2 * 1024 * 1024 * 8);
  cudaMemset(buf, 0, 2 * 1024 * 1024 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int N = 2000;
  unsigned epoch = 0;
  auto run = [&](auto kern, const char* name, int G, int T) {
    cudaMemset(bar, 0, 8);
    cudaMemset(flags, 0, 4096 * 128);
    epoch = 0;
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaMemset(bar, 0, 8);
      cudaMemset(flags, 0, 4096 * 128);
      int n = N;
      unsigned e0 = 0;
      void* args[] = {&bar, &flags, &buf, &n, &e0};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)kern, G, T, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("%-28s G=%4d T=%4d: %.3f us per barrier (%s)\n", name, G, T, best * 1e3 / N, cudaGetErrorString(e));
  };
  for (int T : {256, 448, 1024}) {
    run(probe<0, false>, "counter", sms, T);
    run(probe<1, false>, "counter+nanosleep", sms, T);
    run(probe<2, false>, "flags", sms, T);
    run(probe<3, false>, "cg grid.sync", sms, T);
    run(probe<0, true>, "counter +ld/st", sms, T);
    run(probe<2, true>, "flags +ld/st", sms, T);
    run(probe<3, true>, "cg grid.sync +ld/st", sms, T);
  }
  run(probe<0, false>, "counter", 64, 448);
  run(probe<2, false>, "flags", 64, 448);
  run(probe<0, false>, "counter", 32, 1024);
  run(probe<2, false>, "flags", 32, 1024);
  return 0;
}
