// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
// Probe for the sparse-medium design question: when only part of every 128-B line is needed (a
// partially solid tile layer), (1) how many DRAM bytes does a bulk copy (cp.async.bulk, the
// TMA engine, completed on an mbarrier) of B bytes per line fetch, and (2) what useful bandwidth
// does it sustain, compared with per-thread loads of the same bytes? Run under ncu with
// gpu__time_duration.sum,dram__bytes_read.sum. Kernel template arguments carry the flavour:
//   tma_lines<B, SEG>: SEG bulk copies of B bytes per 128-B line (SEG = 1: offset 0; SEG = 2:
//                      offsets 0 and 64), 64 lines per pipeline stage, 8 stages per CTA
//   ld_lines<F, B>:    the same bytes by per-thread 8-B loads (F 0 = ld.global.nc,
//                      F 5 = ld.global.nc.L2::64B), B/8 threads per line
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kLinesPerStage = 64;
constexpr int kStages = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int B, int SEG>
__global__ void __launch_bounds__(128) tma_lines(const char* __restrict__ in, double* out, size_t n_lines) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[kStages];
  const size_t n_chunks = n_lines / kLinesPerStage;
  const size_t per_cta = (n_chunks + gridDim.x - 1) / gridDim.x;
  const size_t c0 = blockIdx.x * per_cta;
  const size_t c1 = c0 + per_cta < n_chunks ? c0 + per_cta : n_chunks;
  constexpr uint32_t stage_bytes = kLinesPerStage * SEG * B;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](size_t c, int s) {
    mbar_expect_tx(&full[s], stage_bytes);
    char* dst = smem + s * stage_bytes;
    for (int l = 0; l < kLinesPerStage; ++l)
      for (int g = 0; g < SEG; ++g)
        bulk_g2s(dst + (l * SEG + g) * B, in + (c * kLinesPerStage + l) * 128 + g * 64, B, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < kStages && c0 + s < c1; ++s) issue(c0 + s, s);
  double acc = 0;
  for (size_t c = c0; c < c1; ++c) {
    const int s = static_cast<int>((c - c0) % kStages);
    const uint32_t parity = static_cast<uint32_t>(((c - c0) / kStages) & 1);
    mbar_wait(&full[s], parity);
    const double* v = reinterpret_cast<const double*>(smem + s * stage_bytes);
    for (uint32_t k = threadIdx.x; k < stage_bytes / 8; k += blockDim.x) acc += v[k];
    __syncthreads();
    if (threadIdx.x == 0 && c + kStages < c1) issue(c + kStages, s);
  }
  if (acc == 1234.5) out[0] = acc;
}

template <int F>
__device__ __forceinline__ double ld(const double* p) {
  double v;
  if constexpr (F == 0) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if constexpr (F == 5) asm volatile("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int F, int B>
__global__ void ld_lines(const double* __restrict__ in, double* out, size_t n_lines) {
  constexpr int per = B / 8;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  double acc = 0;
  for (; i < n_lines * per; i += (size_t)gridDim.x * blockDim.x) acc += ld<F>(in + (i / per) * 16 + i % per);
  if (acc == 1234.5) out[0] = acc;
}

template <class K>
void launch_tma(K k, int smem, const char* in, double* out, size_t n, int grid) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<grid, 128, smem>>>(in, out, n);
}

int main() {
  const size_t bytes = size_t(4) << 30;
  char* in;
  double* out;
  cudaMalloc(&in, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(in, 0, bytes);
  const size_t n = bytes / 128;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 2; ++rep) {
    launch_tma(tma_lines<32, 1>, kStages * kLinesPerStage * 32, in, out, n, sms * 8);
    launch_tma(tma_lines<64, 1>, kStages * kLinesPerStage * 64, in, out, n, sms * 4);
    launch_tma(tma_lines<128, 1>, kStages * kLinesPerStage * 128, in, out, n, sms * 2);
    launch_tma(tma_lines<32, 2>, kStages * kLinesPerStage * 64, in, out, n, sms * 4);
    ld_lines<0, 32><<<sms * 8, 256>>>(reinterpret_cast<const double*>(in), out, n);
    ld_lines<5, 32><<<sms * 8, 256>>>(reinterpret_cast<const double*>(in), out, n);
    ld_lines<5, 64><<<sms * 8, 256>>>(reinterpret_cast<const double*>(in), out, n);
    ld_lines<0, 128><<<sms * 8, 256>>>(reinterpret_cast<const double*>(in), out, n);
  }
  cudaDeviceSynchronize();
  printf("done: %s (lines %zu)\n", cudaGetErrorString(cudaGetLastError()), n);
  return 0;
}
