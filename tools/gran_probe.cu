// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gran_probe tools/gran_probe.cu
// Probe: DRAM bytes and L2 sectors fetched when one 32-B sector out of every 128 B is read, per
// load flavour (does an L1 miss request 32 B or the whole 128-B line?). Run under ncu with
// dram__bytes_read.sum and lts__t_sectors_srcunit_tex_op_read.sum; the kernel name carries the
// flavour: 0 __ldg (ld.global.nc), 1 ld.global (ca), 2 ld.global.cg, 3 ld.global.nc.L1::no_allocate,
// 4 ld.global.cv, 5 ld.global.nc.L2::64B, 6 ld.global.lu, 7 ld.global.cs
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
template <int F>
__device__ __forceinline__ double ld(const double* p) {
  double v;
  if constexpr (F == 0) v = __ldg(p);
  if constexpr (F == 1) asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if constexpr (F == 2) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if constexpr (F == 3) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if constexpr (F == 4) asm volatile("ld.global.cv.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if constexpr (F == 5) asm volatile("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if constexpr (F == 6) asm volatile("ld.global.lu.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if constexpr (F == 7) asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
// 4 consecutive threads read the 4 doubles of one sector; sectors 128 B apart (like one fluid
// row per 4-row line of a sparse tile).
template <int F>
__global__ void probe(const double* __restrict__ in, double* out, size_t n_sectors) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  double acc = 0;
  for (; i < n_sectors * 4; i += (size_t)gridDim.x * blockDim.x) {
    const size_t sector = i / 4, lane = i % 4;
    acc += ld<F>(in + sector * 16 + lane);
  }
  if (acc == 1234.5) out[0] = acc;
}
int main(int argc, char** argv) {
  if (argc > 1) {  // cudaLimitMaxL2FetchGranularity in bytes
    const size_t g = static_cast<size_t>(atoi(argv[1]));
    printf("set MaxL2FetchGranularity %zu: %s\n", g,
           cudaGetErrorString(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g)));
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
    printf("limit now %zu\n", got);
  }
  const size_t bytes = size_t(2) << 30;
  double *in, *out;
  cudaMalloc(&in, bytes); cudaMalloc(&out, 8);
  cudaMemset(in, 0, bytes);
  const size_t ns = bytes / 128;
  probe<0><<<148 * 8, 256>>>(in, out, ns);
  probe<1><<<148 * 8, 256>>>(in, out, ns);
  probe<2><<<148 * 8, 256>>>(in, out, ns);
  probe<3><<<148 * 8, 256>>>(in, out, ns);
  probe<4><<<148 * 8, 256>>>(in, out, ns);
  probe<5><<<148 * 8, 256>>>(in, out, ns);
  probe<6><<<148 * 8, 256>>>(in, out, ns);
  probe<7><<<148 * 8, 256>>>(in, out, ns);
  cudaDeviceSynchronize();
  printf("done: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
