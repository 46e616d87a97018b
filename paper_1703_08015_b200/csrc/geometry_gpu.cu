// Geometry input side on the device: the random-sphere (RAS) generator of the
// reference (generate_ras, geometry.cpp:251-326) run on a B200, raster bit-identical to the host
// restatement (csrc/geometry.cpp) and therefore to the reference.
//
// The reference inserts periodic spheres one by one until phi <= target + 0.01, each candidate's
// acceptance depending on the porosity left by all earlier ones — an inherently sequential loop.
// What parallelises is the work per candidate: counting (and then marking) the nodes of a ~d^3
// bounding box. The RNG stream is independent of the decisions (every candidate consumes exactly
// three canonical() draws, geometry.cpp:302-304), so the host draws the candidate centres with the
// same mt19937_64 and one persistent thread-block cluster (16 CTAs x 1024 threads on 16 SMs) runs
// the accept/skip/retry loop on the device: each CTA counts its share of the box, the 16 partial
// counts are exchanged through distributed shared memory around one cluster barrier per pass,
// every CTA takes the reference's decision on the same total, and the marking pass follows.
// Until the first skip (near the end, and only when one sphere moves phi by ~0.02 or more) every
// candidate is accepted, so batches of candidates are first painted in parallel (see the batch
// fast path below): 1024^3 in 0.3-1.0 s instead of 2.5-4 s.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "common.h"
#include "splbm_b200.h"

using namespace splbm_host;

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(SPLBM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ck((x), #x)

constexpr int kRasThreads = 1024;
constexpr uint8_t kSolid = 0, kFluid = 1;

struct RasState {
  unsigned long long solid;  // nodes marked solid so far
  int skips;
  int done;                  // porosity reached
  double best_err, best[3];
  unsigned long long consumed;  // candidates used from the current batch
};

struct RasArgs {
  uint8_t* t;
  int dims[3];
  unsigned long long n_total;
  double r, r2, upper, lower, target;
  const double* cand;  // 3 per candidate
  unsigned long long n_cand;
  RasState* st;
};

namespace cg = cooperative_groups;

__device__ __forceinline__ int wrap(int v, int n) { return ((v % n) + n) % n; }

// Count (commit == false) or mark (commit == true) the nodes of the sphere at c, as mark_sphere
// (geometry.cpp:267-291). Block-wide; returns the count on every thread. `serial` handles boxes
// wider than the domain (a wrapped node visited twice): the reference's sequential order decides.
__device__ unsigned long long sphere_pass(const RasArgs& a, const double* c, bool commit,
                                          unsigned long long* s_red, unsigned long long* s_part,
                                          int& parity) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  const int nranks = static_cast<int>(cluster.num_blocks());
  const int x0 = static_cast<int>(floor(__dsub_rn(c[0], a.r))), x1 = static_cast<int>(ceil(__dadd_rn(c[0], a.r)));
  const int y0 = static_cast<int>(floor(__dsub_rn(c[1], a.r))), y1 = static_cast<int>(ceil(__dadd_rn(c[1], a.r)));
  const int z0 = static_cast<int>(floor(__dsub_rn(c[2], a.r))), z1 = static_cast<int>(ceil(__dadd_rn(c[2], a.r)));
  const int nx = x1 - x0 + 1, ny = y1 - y0 + 1, nz = z1 - z0 + 1;
  const bool serial = commit && (nx > a.dims[0] || ny > a.dims[1] || nz > a.dims[2]);
  unsigned long long cnt = 0;
  const long long box = static_cast<long long>(nx) * ny * nz;
  if (!serial) {
    for (long long k = static_cast<long long>(rank) * kRasThreads + threadIdx.x; k < box;
         k += static_cast<long long>(nranks) * kRasThreads) {
      const int x = x0 + static_cast<int>(k % nx);
      const int y = y0 + static_cast<int>((k / nx) % ny);
      const int z = z0 + static_cast<int>(k / (static_cast<long long>(nx) * ny));
      const double dx = __dsub_rn(static_cast<double>(x), c[0]);
      const double dy = __dsub_rn(static_cast<double>(y), c[1]);
      const double dz = __dsub_rn(static_cast<double>(z), c[2]);
      const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      if (d2 > a.r2) continue;
      uint8_t* p = a.t + (static_cast<size_t>(wrap(z, a.dims[2])) * a.dims[1] + wrap(y, a.dims[1])) *
                             static_cast<size_t>(a.dims[0]) + wrap(x, a.dims[0]);
      if (*p != kSolid) {
        ++cnt;
        if (commit) *p = kSolid;
      }
    }
  } else if (threadIdx.x == 0 && rank == 0) {  // reference loop order z, y, x
    for (int z = z0; z <= z1; ++z) {
      const double dz = __dsub_rn(static_cast<double>(z), c[2]);
      for (int y = y0; y <= y1; ++y) {
        const double dy = __dsub_rn(static_cast<double>(y), c[1]);
        for (int x = x0; x <= x1; ++x) {
          const double dx = __dsub_rn(static_cast<double>(x), c[0]);
          const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
          if (d2 > a.r2) continue;
          uint8_t* p = a.t + (static_cast<size_t>(wrap(z, a.dims[2])) * a.dims[1] + wrap(y, a.dims[1])) *
                                 static_cast<size_t>(a.dims[0]) + wrap(x, a.dims[0]);
          if (*p != kSolid) {
            ++cnt;
            *p = kSolid;
          }
        }
      }
    }
  }
  // block reduction (deterministic: integer counts)
  for (int off = 16; off > 0; off >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, off);
  __syncthreads();  // s_red reuse across calls
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned long long v = s_red[threadIdx.x];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (threadIdx.x == 0) s_part[parity] = v;
  }
  // The marks of this pass and the partial count are published to the whole cluster (release /
  // acquire barrier); every CTA then sums the same partials in the same order. s_part is double
  // buffered by pass parity: a slot is rewritten two passes later, after every CTA has passed the
  // next pass's barrier, i.e. after it read this pass's values.
  __threadfence();
  cluster.sync();
  if (threadIdx.x == 0) {
    unsigned long long tot = 0;
    for (int r = 0; r < nranks; ++r) tot += *cluster.map_shared_rank(&s_part[parity], r);
    s_red[32] = tot;
  }
  __syncthreads();
  const unsigned long long total = s_red[32];
  parity ^= 1;
  return total;
}

// The accept/skip/retry loop of generate_ras (geometry.cpp:296-324) over one batch of candidates.
__global__ void __launch_bounds__(kRasThreads, 1) ras_kernel(RasArgs a) {
  __shared__ unsigned long long s_red[33];
  __shared__ unsigned long long s_part[2];
  int parity = 0;
  RasState s = *a.st;
  unsigned long long k = 0;
  while (static_cast<double>(a.n_total - s.solid) / static_cast<double>(a.n_total) > a.upper) {
    if (k == a.n_cand) break;  // batch exhausted: the host draws more candidates
    const double* c = a.cand + 3 * k;
    ++k;
    const unsigned long long newly = sphere_pass(a, c, false, s_red, s_part, parity);
    const double phi_after = static_cast<double>(a.n_total - s.solid - newly) / static_cast<double>(a.n_total);
    if (phi_after >= a.lower || s.skips >= 2000) {
      s.solid += sphere_pass(a, c, true, s_red, s_part, parity);
      s.skips = 0;
      s.best_err = 2.0;
      continue;
    }
    const double err = fabs(__dsub_rn(phi_after, a.target));
    if (err < s.best_err) {
      s.best_err = err;
      s.best[0] = c[0];
      s.best[1] = c[1];
      s.best[2] = c[2];
    }
    if (++s.skips == 2000) {
      s.solid += sphere_pass(a, s.best, true, s_red, s_part, parity);
      s.skips = 0;
      s.best_err = 2.0;
    }
  }
  if (threadIdx.x == 0 && cg::this_cluster().block_rank() == 0) {
    s.done = static_cast<double>(a.n_total - s.solid) / static_cast<double>(a.n_total) <= a.upper;
    s.consumed = k;
    *a.st = s;
  }
  cg::this_cluster().sync();  // no CTA leaves while another may still read its shared memory
}

// ---- batch fast path -----------------------------------------------------------------------
// While every candidate is accepted (the reference skips one only when it would push phi below
// target - 0.01, i.e. near the end and only if one sphere moves phi by more than that), the
// raster after candidate j is the union of spheres 0..j and candidate j's count is the number of
// still-fluid nodes it covers that no earlier sphere covers. A batch is therefore painted in
// parallel: every fluid node inside sphere j takes owner = min(j) (atomicMin), a histogram of
// owners gives each candidate's count, the host replays the reference's decisions on those counts
// and the accepted prefix is marked. At the first skip the sequential cluster loop takes over with
// the identical state. Requires boxes no wider than the domain (no node visited twice).
__global__ void __launch_bounds__(256) paint_kernel(RasArgs a, uint32_t* owner) {
  const unsigned long long j = blockIdx.x;
  const double* c = a.cand + 3 * j;
  const int x0 = static_cast<int>(floor(__dsub_rn(c[0], a.r))), x1 = static_cast<int>(ceil(__dadd_rn(c[0], a.r)));
  const int y0 = static_cast<int>(floor(__dsub_rn(c[1], a.r))), y1 = static_cast<int>(ceil(__dadd_rn(c[1], a.r)));
  const int z0 = static_cast<int>(floor(__dsub_rn(c[2], a.r))), z1 = static_cast<int>(ceil(__dadd_rn(c[2], a.r)));
  const int nx = x1 - x0 + 1, ny = y1 - y0 + 1, nz = z1 - z0 + 1;
  const long long box = static_cast<long long>(nx) * ny * nz;
  for (long long k = threadIdx.x; k < box; k += blockDim.x) {
    const int x = x0 + static_cast<int>(k % nx);
    const int y = y0 + static_cast<int>((k / nx) % ny);
    const int z = z0 + static_cast<int>(k / (static_cast<long long>(nx) * ny));
    const double dx = __dsub_rn(static_cast<double>(x), c[0]);
    const double dy = __dsub_rn(static_cast<double>(y), c[1]);
    const double dz = __dsub_rn(static_cast<double>(z), c[2]);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    if (d2 > a.r2) continue;
    const size_t idx = (static_cast<size_t>(wrap(z, a.dims[2])) * a.dims[1] + wrap(y, a.dims[1])) *
                           static_cast<size_t>(a.dims[0]) + wrap(x, a.dims[0]);
    if (a.t[idx] != kSolid) atomicMin(owner + idx, static_cast<uint32_t>(j));
  }
}

__global__ void owner_hist_kernel(const uint32_t* owner, size_t n, uint32_t* hist) {
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint32_t o = owner[i];
    if (o != 0xffffffffu) atomicAdd(hist + o, 1u);
  }
}

__global__ void owner_mark_kernel(uint8_t* t, const uint32_t* owner, size_t n, uint32_t accepted) {
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    if (owner[i] < accepted) t[i] = kSolid;
}

// One cluster of 16 CTAs (non-portable size; 8, then 1, if the device refuses it).
void launch_cluster(const RasArgs& a) {
  static int size = 0;
  if (size == 0) {
    cudaFuncSetAttribute(ras_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    size = 16;
  }
  for (;;) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(size);
    cfg.blockDim = dim3(kRasThreads);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = size;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, ras_kernel, a);
    if (e == cudaSuccess) return;
    cudaGetLastError();  // clear, retry smaller
    if (size == 1) CK(e);
    size = size > 8 ? 8 : 1;
  }
}

}  // namespace

extern "C" int splbm_generate_device(int kind, const splbm_generate_params* p, int device,
                                     uint8_t* types_out, int* d_out, double bc_velocity_out[3],
                                     double* bc_density_out) {
  if (kind != SPLBM_GEOM_RAS3D)  // the other generators are O(N) host fills
    return splbm_generate(kind, p, types_out, d_out, bc_velocity_out, bc_density_out);
  return guarded([&] {
    if (!p || !types_out) throw config_error("null argument");
    const int dims[3] = {p->dims[0], p->dims[1], p->dims[2]};
    for (int k = 0; k < 3; ++k)
      if (dims[k] <= 0) throw config_error("dimensions must be positive");
    const int min_dim = std::min({dims[0], dims[1], dims[2]});  // geometry.cpp:253-261
    if (p->sphere_diameter < 2) throw config_error("sphere diameter must be at least 2");
    if (p->sphere_diameter >= min_dim)
      throw config_error("sphere diameter must be smaller than the smallest dimension");
    if (!(p->target_porosity > 0.0 && p->target_porosity < 1.0))
      throw config_error("target porosity must lie in (0, 1)");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(SPLBM_ERR_CUDA, "no CUDA device available");
    CK(cudaSetDevice(device));
    const size_t n = static_cast<size_t>(dims[0]) * dims[1] * dims[2];
    RasArgs a{};
    for (int k = 0; k < 3; ++k) a.dims[k] = dims[k];
    a.n_total = n;
    a.r = p->sphere_diameter / 2.0;
    a.r2 = a.r * a.r;
    a.target = p->target_porosity;
    a.upper = p->target_porosity + 0.01;
    a.lower = p->target_porosity - 0.01;
    uint8_t* t = nullptr;
    double* cand = nullptr;
    RasState* st = nullptr;
    uint32_t* owner = nullptr;
    uint32_t* hist = nullptr;
    auto cleanup = [&] {
      cudaFree(t);
      cudaFree(cand);
      cudaFree(st);
      cudaFree(owner);
      cudaFree(hist);
    };
    try {
      CK(cudaMalloc(&t, n));
      CK(cudaMemset(t, kFluid, n));
      CK(cudaMalloc(&st, sizeof(RasState)));
      RasState s0{};
      s0.best_err = 2.0;
      CK(cudaMemcpy(st, &s0, sizeof(s0), cudaMemcpyHostToDevice));
      // candidate batches from the reference's RNG stream (canonical, geometry.cpp:195-197)
      std::mt19937_64 rng(p->seed);
      const double vol = 4.0 / 3.0 * 3.141592653589793 * a.r * a.r * a.r;
      const double est = std::max(1.0, -std::log(std::max(p->target_porosity, 1e-3)) * n / vol);
      size_t batch = static_cast<size_t>(std::min(8.0e6, est * 1.3 + 4096.0));
      std::vector<double> host(3 * batch);
      CK(cudaMalloc(&cand, host.size() * sizeof(double)));
      a.st = st;
      a.t = t;
      a.cand = cand;
      // batch fast path while no box can wrap onto itself (SPLBM_RAS_SEQ=1: sequential only)
      bool fast = p->sphere_diameter + 2 <= min_dim && std::getenv("SPLBM_RAS_SEQ") == nullptr;
      unsigned long long solid = 0;
      std::vector<uint32_t> hist_h;
      if (fast) {
        CK(cudaMalloc(&owner, n * sizeof(uint32_t)));
        CK(cudaMalloc(&hist, batch * sizeof(uint32_t)));
        hist_h.resize(batch);
      }
      int sms = 148;
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
      const unsigned sweep_blocks = static_cast<unsigned>(sms) * 8;
      for (;;) {
        for (size_t k = 0; k < batch; ++k)
          for (int c = 0; c < 3; ++c)
            host[3 * k + c] = static_cast<double>(rng() >> 11) * 0x1.0p-53 * dims[c];
        CK(cudaMemcpy(cand, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice));
        size_t start = 0;
        if (fast) {
          a.cand = cand;
          a.n_cand = batch;
          CK(cudaMemset(owner, 0xff, n * sizeof(uint32_t)));
          CK(cudaMemset(hist, 0, batch * sizeof(uint32_t)));
          paint_kernel<<<static_cast<unsigned>(batch), 256>>>(a, owner);
          CK(cudaGetLastError());
          owner_hist_kernel<<<sweep_blocks, 256>>>(owner, n, hist);
          CK(cudaGetLastError());
          CK(cudaMemcpy(hist_h.data(), hist, batch * sizeof(uint32_t), cudaMemcpyDeviceToHost));
          // the reference's loop (geometry.cpp:296-324) on the counts; skips == 0 throughout
          size_t accepted = 0;
          bool done = false, skip = false;
          for (; accepted < batch; ++accepted) {
            if (!(static_cast<double>(n - solid) / static_cast<double>(n) > a.upper)) {
              done = true;
              break;
            }
            const unsigned long long newly = hist_h[accepted];
            const double phi_after = static_cast<double>(n - solid - newly) / static_cast<double>(n);
            if (!(phi_after >= a.lower)) {
              skip = true;
              break;
            }
            solid += newly;
          }
          owner_mark_kernel<<<sweep_blocks, 256>>>(t, owner, n, static_cast<uint32_t>(accepted));
          CK(cudaGetLastError());
          if (!done && !skip && !(static_cast<double>(n - solid) / static_cast<double>(n) > a.upper)) done = true;
          if (done) break;
          if (!skip) continue;
          // first skip: the sequential loop resumes at this candidate with the same state
          fast = false;
          RasState s1{};
          s1.solid = solid;
          s1.best_err = 2.0;
          CK(cudaMemcpy(st, &s1, sizeof(s1), cudaMemcpyHostToDevice));
          start = accepted;
        }
        a.cand = cand + 3 * start;
        a.n_cand = batch - start;
        launch_cluster(a);
        RasState s{};
        CK(cudaMemcpy(&s, st, sizeof(s), cudaMemcpyDeviceToHost));
        if (s.done) break;
        if (s.consumed != batch - start) throw Error(SPLBM_ERR_CUDA, "RAS generator stopped early");
      }
      CK(cudaMemcpy(types_out, t, n, cudaMemcpyDeviceToHost));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
    if (d_out) *d_out = 3;
    if (bc_velocity_out)
      for (int k = 0; k < 3; ++k) bc_velocity_out[k] = 0.0;
    if (bc_density_out) *bc_density_out = 1.0;
  });
}
