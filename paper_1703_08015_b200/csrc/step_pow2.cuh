// The power-of-two T2C step kernel and the device helpers it uses (gather loads, streaming
// stores, traversal order, L2 prefetch). Included by kernels.cu (ahead of time, every variant) and
// compiled at run time by mrt_jit.cpp through NVRTC, with collide_mrt_gen<> defined for one MRT
// operator (GEN = true). Must therefore stay free of host-only headers.
#pragma once
#include "lattice.cuh"
#include "step_args.h"

namespace splbm_dev {

constexpr uint32_t kEmpty = 0xffffffffu;
constexpr int kThreads = 256;
#ifndef SPLBM_STEP_THREADS
#define SPLBM_STEP_THREADS 64  // CTA size of the 3D power-of-two step kernel (128: BGK +0.2-0.7 %, MRT -1 %, round 2)
#endif
#ifndef SPLBM_AA_THREADS
#define SPLBM_AA_THREADS 128  // CTA size of the single-copy (AA) kernels (two 4^3 tiles: RAS phi 0.2 -2.7 % vs 64)
#endif
#ifndef SPLBM_STEP_THREADS2
#define SPLBM_STEP_THREADS2 64  // CTA size of the 2D power-of-two step kernel
#endif
// the CTA size of a power-of-two step: 64 threads (one 4^3 tile; four 4x4 2D tiles) measured
// 6-12 % faster than 256 (interleaved A/B); never below one tile (a CTA owns whole tiles)
template <int D, int NTN>
__host__ __device__ constexpr int step_threads() {
  return (D == 3 ? SPLBM_STEP_THREADS : SPLBM_STEP_THREADS2) > NTN ? (D == 3 ? SPLBM_STEP_THREADS : SPLBM_STEP_THREADS2) : NTN;
}
// Device neighbour table: the 27 cells of engine.hpp:446-463 in 3D; in 2D only the dz = 0 slice
// (cells 9..17) is ever addressed, so it is stored compactly with 9 entries per tile.
template <int D>
__host__ __device__ constexpr int nb_stride() { return D == 3 ? 27 : 9; }
template <int D>
__host__ __device__ constexpr int nb_offset() { return D == 3 ? 0 : 9; }
#ifndef SPLBM_MINB3
#define SPLBM_MINB3 4  // resident 256-thread CTAs per SM the 3D step is budgeted for
#endif
#ifndef SPLBM_MINB2
#define SPLBM_MINB2 6  // resident 256-thread CTAs per SM the 2D step is budgeted for
#endif
#ifndef SPLBM_MINB3F
#define SPLBM_MINB3F 5  // the f32 engine: 48 registers, 20 CTAs/SM (+3-4 % vs 16, A/B)
#endif
#ifndef SPLBM_MINB2F
#define SPLBM_MINB2F 6
#endif
#ifndef SPLBM_X2_THREADS
#define SPLBM_X2_THREADS 64  // two-nodes-per-thread step (f32): CTA size
#endif
#ifndef SPLBM_X2_MINB
#define SPLBM_X2_MINB 16     // ... and resident CTAs per SM (64 registers)
#endif
#ifndef SPLBM_MINB_MRT
#define SPLBM_MINB_MRT 3  // the 3D MRT step when SPLBM_CTAS_MRT3 = 0: 80 registers (+4-9 % vs 2, round 1)
#endif
#ifndef SPLBM_MINB_MRT2
#define SPLBM_MINB_MRT2 4  // the 2D MRT step: +12 % vs 2 (interleaved A/B)
#endif
#ifndef SPLBM_AA1_MINB
#define SPLBM_AA1_MINB 4  // single-copy phase 1: 256-thread CTA equivalents per SM (64 registers)
#endif
#ifndef SPLBM_CTAS3
#define SPLBM_CTAS3 0  // experiment: resident 64-thread CTAs/SM budgeted for the 3D f64 BGK step (0 = SPLBM_MINB3)
#endif
#ifndef SPLBM_CTAS_MRT3
#define SPLBM_CTAS_MRT3 10  // 3D MRT step: 640 resident threads/SM (10 x 64) = 94 registers, no spills
                            // (12 CTAs: 80 registers + 144 B of spills, 2-3 % slower, round 2 A/B)
#endif
#ifndef SPLBM_ZERO_FILL
#define SPLBM_ZERO_FILL 1  // write 0.0 to solid slots sharing a 32-B sector with fluid slots
#endif
#ifndef SPLBM_PDL
#define SPLBM_PDL 1  // programmatic dependent launch between consecutive step kernels
#endif
#ifndef SPLBM_STORE_CS
#define SPLBM_STORE_CS 1  // evict-first stores: the written copy is not re-read this step
#endif

__device__ __forceinline__ void st_stream(double* p, double v) {
#if SPLBM_STORE_CS
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
#else
  *p = v;
#endif
}
__device__ __forceinline__ void st_stream(float* p, float v) {
#if SPLBM_STORE_CS
  asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
#else
  *p = v;
#endif
}

// PDF gather load. B200 measurement (tools/gran_probe.cu): a plain or .nc global load that misses
// fetches the whole 128-B line from DRAM; the .L2::64B prefetch-size qualifier limits that to
// 64 B (the device limit cudaLimitMaxL2FetchGranularity has no effect): +1-3 % on every workload
// (interleaved A/B), most on sparse media. SPLBM_LD_64B=0 builds the plain __ldg variant.
#ifndef SPLBM_LD_64B
#define SPLBM_LD_64B 1
#endif
__device__ __forceinline__ double ld_pdf(const double* p) {
#if SPLBM_LD_64B
  double v;
  asm volatile("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ float ld_pdf(const float* p) {
#if SPLBM_LD_64B
  float v;
  asm volatile("ld.global.nc.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

// Coherent variant for the single-copy (AA) kernels, which read and write the same array in one
// launch: `.nc` is only defined for data that stays read-only for the whole kernel, so these keep
// the L2::64B fetch size but go through the coherent path.
__device__ __forceinline__ double ld_pdf_rw(const double* p) {
  double v;
  asm volatile("ld.global.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_pdf_rw(const float* p) {
  float v;
  asm volatile("ld.global.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

// Stored tile of the k-th stepped tile of a launch: the column traversal order when set (large
// whole-domain engines, StepArgs::order), else the range [t0, ...) with the optional skip.
__device__ __forceinline__ uint64_t tile_of(const StepArgs& a, uint64_t k) {
  if (a.order) return __ldg(a.order + k);
  return a.t0 + k + (k >= a.skip_at ? a.skip_by : 0);
}

// L2 prefetch of a future CTA's read blocks (the CTA StepArgs::l2pf CTAs ahead, about half a
// wave): one bulk request per tile block (Q*NTN doubles, contiguous) holds no registers, so more
// DRAM reads are in flight than the gather alone keeps. Whole blocks measured faster than
// per-direction or non-solid-row requests even on sparse media.
template <int Q, int NTN, int TILES, class R>
__device__ __forceinline__ void l2_prefetch_blocks(const R* pdf, uint64_t tile, bool valid) {
  if (threadIdx.x < TILES && valid)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pdf + tile * Q * NTN),
                 "r"(static_cast<uint32_t>(Q * NTN * sizeof(R))) : "memory");
}

// The MRT collision with the operator's constants folded in and the products K_ij * delta_j
// shared between the rows whose K_ij are equal (defined only in the runtime-specialised source).
template <int D, bool INC, class R>
__device__ bool collide_mrt_gen(R* f);

// Resident CTAs per SM the power-of-two step is budgeted for (the registers follow): SPLBM_CTAS3 /
// SPLBM_CTAS_MRT3 count 64-thread CTA equivalents, SPLBM_MINB* 256-thread ones.
template <int D, int NTN, bool MRT, class R>
__host__ __device__ constexpr int step_min_blocks() {
  constexpr int T = step_threads<D, NTN>();
  return (SPLBM_CTAS3 && D == 3 && !MRT && sizeof(R) == 8) ? SPLBM_CTAS3 * 64 / T
         : (SPLBM_CTAS_MRT3 && D == 3 && MRT)             ? SPLBM_CTAS_MRT3 * 64 / T
         : (MRT ? (D == 3 ? SPLBM_MINB_MRT : SPLBM_MINB_MRT2)
                : (D == 3 ? (sizeof(R) == 4 ? SPLBM_MINB3F : SPLBM_MINB3) : (sizeof(R) == 4 ? SPLBM_MINB2F : SPLBM_MINB2))) *
               256 / T;
}

// Fast path for power-of-two tiles of at most 256 nodes (a = 4 in 3D, a <= 16 in 2D): a CTA owns
// kThreads / n_tn whole tiles. The 27 neighbour-tile base pointers of each tile are staged in
// shared memory once per CTA (one coalesced read of nb, overlapped with the gather-word load), so
// the per-direction source address is pure integer arithmetic on compile-time lattice constants
// plus one shared-memory lookup and two selects — no divergent branches, no dependent global load
// before the PDF gather.
template <int D, int LOGA, bool INC, bool PEER, bool MRT, class R, bool GEN = false>
__global__ void __launch_bounds__((step_threads<D, (D == 3 ? (1 << (3 * LOGA)) : (1 << (2 * LOGA)))>()),
                                  (step_min_blocks<D, (D == 3 ? (1 << (3 * LOGA)) : (1 << (2 * LOGA))), MRT, R>()))
    t2c_step_pow2_kernel(StepArgs args, const __grid_constant__ MrtMatrix<R, (MRT && !GEN) ? Lat<D>::Q : 1> mrt) {
  constexpr int Q = Lat<D>::Q;
  const R* const rd = static_cast<const R*>(args.read);
  constexpr int A = 1 << LOGA;
  constexpr int NTN = D == 3 ? A * A * A : A * A;
  constexpr int TILES = step_threads<D, NTN>() / NTN;
  constexpr uint64_t STRIDE = static_cast<uint64_t>(Q) * NTN;
  constexpr int NBS = nb_stride<D>();
  __shared__ const R* s_base[TILES][NBS];

  const uint64_t n_tiles = args.n_nodes / NTN;
  const uint64_t tile_blk = static_cast<uint64_t>(blockIdx.x) * TILES;
  for (int k = threadIdx.x; k < TILES * NBS; k += step_threads<D, NTN>()) {
    const int tl = k / NBS, dd = k % NBS;
    const uint64_t tt = tile_blk + tl;
    const R* b = nullptr;
    if (tt < n_tiles) {
      const uint32_t s = __ldg(args.nb + tile_of(args, tt) * NBS + dd);
      b = s == kEmpty ? nullptr : rd + static_cast<uint64_t>(s) * STRIDE;
    }
    s_base[tl][dd] = b;
  }
  const int tl = threadIdx.x / NTN;
  const int p = threadIdx.x % NTN;
  const uint64_t tloc = tile_blk + tl;
  const bool live = tloc < n_tiles;
  const uint64_t t = live ? tile_of(args, tloc) : 0;
  const uint32_t info = live ? __ldg(args.info + t * NTN + p) : 0u;
  const uint64_t pf = tile_blk + static_cast<uint64_t>(args.l2pf) * TILES + threadIdx.x;
  __syncthreads();
#if SPLBM_PDL
  // Everything above reads only static tables (nb, info); the PDFs of the previous step are
  // touched only after its grid has completed and its writes are visible.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  l2_prefetch_blocks<Q, NTN, TILES>(rd, (args.l2pf && pf < n_tiles && threadIdx.x < TILES) ? tile_of(args, pf) : 0,
                                    args.l2pf && pf < n_tiles);
  const int type = (info >> 24) & 3;
  R* wr = static_cast<R*>(args.write) + t * STRIDE + p;
  if (type == 0) {
    if (info & (1u << 27)) {
#pragma unroll
      for (int i = 0; i < Q; ++i) st_stream(wr + i * NTN, R(0));
    }
    return;
  }
  const int lx = p & (A - 1);
  const int ly = (p >> LOGA) & (A - 1);
  const int lz = D == 3 ? (p >> (2 * LOGA)) : 0;
  const R* own = rd + t * STRIDE;
  const R* const* nbp = s_base[tl];

  R f[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    const int vx = lx - ex<D>(i), vy = ly - ey<D>(i), vz = lz - ez<D>(i);
    const int dx = ex<D>(i) ? (vx >> LOGA) : 0;  // arithmetic shift: -1, 0 or +1
    const int dy = ey<D>(i) ? (vy >> LOGA) : 0;
    const int dz = (D == 3 && ez<D>(i)) ? (vz >> LOGA) : 0;
    const int sp = (vx & (A - 1)) | ((vy & (A - 1)) << LOGA) | (D == 3 ? ((vz & (A - 1)) << (2 * LOGA)) : 0);
    const int delta = 13 + dx + 3 * dy + 9 * dz;
    const R* src = (delta == 13 ? own : nbp[delta - nb_offset<D>()]) + (i * NTN + sp);
    const R* bb = own + (opp(i) * NTN + p);  // half-way bounce-back (engine.hpp:498-500)
    f[i] = ld_pdf(((info >> i) & 1u) ? bb : src);
  }

  bool good;
  if (type == 1) {
    if constexpr (MRT && GEN) {
      good = collide_mrt_gen<D, INC, R>(f);  // runtime-specialised operator (mrt_jit.cpp)
    } else if constexpr (MRT) {
      good = collide_mrt<D, INC>(f, mrt.K);
    } else {
      good = collide_bgk<D, INC>(f, static_cast<R>(args.inv_tau));
    }
  } else {
    good = apply_boundary<D, INC>(f, type, (info >> 26) & 1u, args.bc);
  }
  if (!good) atomicMin(args.failed, static_cast<unsigned long long>(*args.step_base + args.rel + 1));
  if constexpr (!PEER) {
    // Only f[] stays live through the collision: the store address is re-derived from opaque
    // reads of the CTA/thread index (as in t2c_aa_kernel phase 1) — 64 registers without spills
    // (8 B of spills otherwise); within ±0.3 % in the bench, −2…−4 % in interleaved A/B.
    uint32_t bx, tx;
    asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(bx));
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tx));
    R* wr2 = static_cast<R*>(args.write) +
             tile_of(args, static_cast<uint64_t>(bx) * TILES + tx / NTN) * STRIDE + tx % NTN;
#pragma unroll
    for (int i = 0; i < Q; ++i) st_stream(wr2 + i * NTN, f[i]);
  } else {
#pragma unroll
  for (int i = 0; i < Q; ++i) st_stream(wr + i * NTN, f[i]);

  // Slab faces straight into the neighbours' halo tiles over NVLink (fused with the step): the
  // neighbour gathers exactly these slots (layer a-1 / 0, directions crossing the face).
  if constexpr (sizeof(R) == 8) {
  const int lslab = D == 3 ? lz : ly;
  if (args.peer_up && t >= args.top_begin && lslab == A - 1) {
    double* dst = args.peer_up + (t - args.top_begin) * STRIDE + p;
#pragma unroll
    for (int i = 0; i < Q; ++i)
      if ((D == 3 ? ez<D>(i) : ey<D>(i)) > 0) dst[i * NTN] = f[i];
  }
  if (args.peer_down && t >= args.bot_begin && t < args.bot_end && lslab == 0) {
    double* dst = args.peer_down + (t - args.bot_begin) * STRIDE + p;
#pragma unroll
    for (int i = 0; i < Q; ++i)
      if ((D == 3 ? ez<D>(i) : ey<D>(i)) < 0) dst[i * NTN] = f[i];
  }
  }
  }
}

}  // namespace splbm_dev
