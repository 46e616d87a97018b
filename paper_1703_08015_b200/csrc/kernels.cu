// sm_100a kernels of the T2C time-step path (arXiv 1703.08015; reference engine.hpp:311-551).
//
// HBM layout: per-tile structure of arrays, slot (t*q + i)*n_tn + p exactly as
// the reference (engine.hpp:397-399), two copies (read/write swapped per step). Per tile node a
// 32-bit gather word `info` replaces the reference's per-direction node-type lookups:
//   bits 0..q-1  direction i is blocked (own solid source, EMPTY neighbour tile or solid
//                neighbour source) -> half-way bounce-back from the own opposite slot
//   bits 24..25  NodeType; bit 26 bc_degenerate (engine.hpp:409-417)
//   bit 27       solid node whose 32-B sector holds a non-solid node: written (as 0.0) so
//                every store sector is whole (no L2 partial-write fills); never read.
// One thread per tile node (two in the f32 and D2Q9 f64 steps), 64-thread CTAs for the
// power-of-two tile kernels (one 4^3 tile per CTA; 256 for the generic and auxiliary kernels),
// consecutive threads = consecutive p so all q stores of a warp are 256-B coalesced runs; the
// gather reads the own tile and the face-adjacent neighbour tiles (L2 hits: neighbours are near in
// the compact z-major order, and the tile blocks two CTAs per SM ahead are bulk-prefetched into
// L2). The power-of-two two-copy step and the single-copy phases live in step_pow2.cuh /
// step_aa.cuh, which mrt_jit.cpp also compiles at run time (NVRTC) for each MRT operator; small
// whole domains run batches of steps in the resident multi-step kernel below.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "lattice.cuh"
#include "kernels.h"
#include "step_pow2.cuh"
#include "step_aa.cuh"

namespace splbm_dev {

// Slot the natural-state gather of direction i reads for node (t, p) (engine.hpp:485-501): the
// source x - e_i in its tile, or the own opposite slot when the direction is blocked. Generic
// tile edge; the neighbour tile comes from the stored nb table.
template <int D>
__device__ __forceinline__ uint64_t gather_slot(const uint32_t* nb, uint32_t info, int a, int n_tn,
                                                uint64_t t, int p, int i) {
  constexpr uint64_t Q = Lat<D>::Q;
  if ((info >> i) & 1u) return (t * Q + opp(i)) * n_tn + p;
  int sx = p % a - ex<D>(i), sy = (p / a) % a - ey<D>(i), sz = (D == 3 ? p / (a * a) : 0) - ez<D>(i);
  int dx = 0, dy = 0, dz = 0;
  if (sx < 0) { dx = -1; sx += a; } else if (sx >= a) { dx = 1; sx -= a; }
  if (sy < 0) { dy = -1; sy += a; } else if (sy >= a) { dy = 1; sy -= a; }
  if (D == 3) {
    if (sz < 0) { dz = -1; sz += a; } else if (sz >= a) { dz = 1; sz -= a; }
  }
  const int delta = (dx + 1) + 3 * ((dy + 1) + 3 * (dz + 1));
  const uint64_t u = delta == 13 ? t : nb[t * nb_stride<D>() + delta - nb_offset<D>()];
  return (u * Q + i) * n_tn + (sx + a * (sy + a * sz));
}

// The post-collision PDFs S[x][.] of node (t, p) in the current state (StateView).
template <int D, class R>
__device__ __forceinline__ void load_state(const R* pdf, uint32_t info, const StateView& v,
                                           int n_tn, uint64_t t, int p, R* f) {
  constexpr int Q = Lat<D>::Q;
#pragma unroll
  for (int i = 0; i < Q; ++i)
    f[i] = v.swapped ? pdf[gather_slot<D>(v.nb, info, v.a, n_tn, t, p, opp(i))]
                     : pdf[(t * Q + i) * static_cast<uint64_t>(n_tn) + p];
}

// ---------------------------------------------------------------------------------------------
// The fused gather-propagation + BGK/boundary + store step (engine.hpp:466-514, collision.hpp:35-65,
// engine.hpp:32-65). A > 0 is a compile-time tile edge; A == 0 reads a_rt.
template <int D, int A, bool INC, bool MRT, class R>
__global__ void __launch_bounds__(kThreads)
    t2c_step_kernel(StepArgs args, const __grid_constant__ MrtMatrix<R, MRT ? Lat<D>::Q : 1> mrt) {
  constexpr int Q = Lat<D>::Q;
  const R* const rd = static_cast<const R*>(args.read);
  const int a = A > 0 ? A : args.a;
  const int az = D == 3 ? a : 1;
  const int n_tn = a * a * az;
  const uint64_t g = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
  if (g >= args.n_nodes) return;
  uint64_t tord = g / static_cast<uint64_t>(n_tn);
  if (tord >= args.skip_at) tord += args.skip_by;
  const uint64_t t = args.t0 + tord;
  const int p = static_cast<int>(g % static_cast<uint64_t>(n_tn));
  const uint64_t node = t * n_tn + p;
  const uint32_t info = __ldg(args.info + node);
  const int type = (info >> 24) & 3;
  const uint64_t tile_stride = static_cast<uint64_t>(Q) * n_tn;
  R* wr = static_cast<R*>(args.write) + t * tile_stride + p;
  if (type == 0) {
    if (info & (1u << 27)) {
#pragma unroll
      for (int i = 0; i < Q; ++i) st_stream(wr + i * n_tn, R(0));
    }
    return;
  }
  const int lx = p % a;
  const int ly = (p / a) % a;
  const int lz = D == 3 ? p / (a * a) : 0;
  const R* own = rd + t * tile_stride;
  const uint32_t* nbt = args.nb + t * nb_stride<D>() - nb_offset<D>();

  R f[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    // source node x - e_i (engine.hpp:421-445): local coordinates and neighbour cell offset
    int sx = lx - ex<D>(i), sy = ly - ey<D>(i), sz = lz - ez<D>(i);
    int dx = 0, dy = 0, dz = 0;
    if (ex<D>(i) != 0) {
      if (sx < 0) { dx = -1; sx += a; } else if (sx >= a) { dx = 1; sx -= a; }
    }
    if (ey<D>(i) != 0) {
      if (sy < 0) { dy = -1; sy += a; } else if (sy >= a) { dy = 1; sy -= a; }
    }
    if (D == 3 && ez<D>(i) != 0) {
      if (sz < 0) { dz = -1; sz += a; } else if (sz >= a) { dz = 1; sz -= a; }
    }
    const int delta = (dx + 1) + 3 * ((dy + 1) + 3 * (dz + 1));
    const int sp = sx + a * (sy + a * sz);
    const bool blocked = (info >> i) & 1u;
    const R* src;
    if (blocked) {
      src = own + opp(i) * n_tn + p;  // half-way bounce-back (engine.hpp:498-500)
    } else if (delta == 13) {
      src = own + i * n_tn + sp;
    } else {
      const uint64_t s = __ldg(nbt + delta);
      src = rd + s * tile_stride + i * n_tn + sp;
    }
    f[i] = ld_pdf(src);
  }

  bool good;
  if (type == 1) {
    if constexpr (MRT)
      good = collide_mrt<D, INC>(f, mrt.K);
    else
      good = collide_bgk<D, INC>(f, static_cast<R>(args.inv_tau));
  } else {
    good = apply_boundary<D, INC>(f, type, (info >> 26) & 1u, args.bc);
  }
  if (!good) atomicMin(args.failed, static_cast<unsigned long long>(*args.step_base + args.rel + 1));
#pragma unroll
  for (int i = 0; i < Q; ++i) st_stream(wr + i * n_tn, f[i]);
}

// Two nodes per thread (the f32 engine, and D2Q9 in f64): a float gather moves half the bytes of a
// double one (a D2Q9 node has 9 instead of 19 values), so one node per thread leaves too few bytes
// in flight; here thread j of a tile's half takes nodes j and j + NTN/2 and issues both gathers
// (2 x q loads) before either collision: +7-13 % over one node per thread for f32, +5 % for D2Q9
// f64 (interleaved A/B). Same addressing, slots and arithmetic as t2c_step_pow2_kernel (BGK, no
// slab peer stores).
template <int D, int LOGA, bool INC, class R, bool O32>
__global__ void __launch_bounds__(SPLBM_X2_THREADS, SPLBM_X2_MINB)
    t2c_step_x2_kernel(StepArgs args, const __grid_constant__ MrtMatrix<R, 1> mrt) {
  constexpr int Q = Lat<D>::Q;
  const R* const rd = static_cast<const R*>(args.read);
  constexpr int A = 1 << LOGA;
  constexpr int NTN = D == 3 ? A * A * A : A * A;
  constexpr int HALF = NTN / 2;                 // threads per tile
  constexpr int TILES = SPLBM_X2_THREADS / HALF;
  constexpr uint64_t STRIDE = static_cast<uint64_t>(Q) * NTN;
  constexpr int NBS = nb_stride<D>();
  __shared__ const R* s_base[TILES][O32 ? 1 : NBS];
  __shared__ uint32_t s_off[TILES][O32 ? NBS : 1];  // O32: neighbour tile offsets in elements

  const uint64_t n_tiles = args.n_nodes / NTN;
  const uint64_t tile_blk = static_cast<uint64_t>(blockIdx.x) * TILES;
  for (int k = threadIdx.x; k < TILES * NBS; k += SPLBM_X2_THREADS) {
    const int tl = k / NBS, dd = k % NBS;
    const uint64_t tt = tile_blk + tl;
    const R* b = nullptr;
    if (tt < n_tiles) {
      const uint32_t s = __ldg(args.nb + (args.t0 + tt) * NBS + dd);
      b = s == kEmpty ? nullptr : rd + static_cast<uint64_t>(s) * STRIDE;
      if constexpr (O32) s_off[tl][dd] = s == kEmpty ? 0u : s * static_cast<uint32_t>(STRIDE);
    }
    if constexpr (!O32) s_base[tl][dd] = b;
  }
  const int tl = threadIdx.x / HALF;
  const int j = threadIdx.x % HALF;
  const uint64_t tloc = tile_blk + tl;
  const bool live = tloc < n_tiles;
  const uint64_t t = args.t0 + tloc;
  uint32_t info[2];
  info[0] = live ? __ldg(args.info + t * NTN + j) : 0u;
  info[1] = live ? __ldg(args.info + t * NTN + j + HALF) : 0u;
  const uint64_t pf = tile_blk + static_cast<uint64_t>(args.l2pf) * TILES + threadIdx.x;
  __syncthreads();
#if SPLBM_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  l2_prefetch_blocks<Q, NTN, TILES>(rd, args.t0 + pf, args.l2pf && pf < n_tiles);
  const R* own = rd + t * STRIDE;
  const uint32_t own_off = static_cast<uint32_t>(t * STRIDE);
  const R* const* nbp = s_base[tl];
  R f[2][Q];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int p = j + u * HALF;
    const int lx = p & (A - 1);
    const int ly = (p >> LOGA) & (A - 1);
    const int lz = D == 3 ? (p >> (2 * LOGA)) : 0;
    const bool act = ((info[u] >> 24) & 3) != 0;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      const int vx = lx - ex<D>(i), vy = ly - ey<D>(i), vz = lz - ez<D>(i);
      const int dx = ex<D>(i) ? (vx >> LOGA) : 0;
      const int dy = ey<D>(i) ? (vy >> LOGA) : 0;
      const int dz = (D == 3 && ez<D>(i)) ? (vz >> LOGA) : 0;
      const int sp = (vx & (A - 1)) | ((vy & (A - 1)) << LOGA) | (D == 3 ? ((vz & (A - 1)) << (2 * LOGA)) : 0);
      const int delta = 13 + dx + 3 * dy + 9 * dz;
      if constexpr (O32) {  // 32-bit element offsets: one select and one wide add per load
        const uint32_t so = (delta == 13 ? own_off : s_off[tl][delta - nb_offset<D>()]) + (i * NTN + sp);
        const uint32_t bo = own_off + (opp(i) * NTN + p);
        f[u][i] = act ? ld_pdf(rd + (((info[u] >> i) & 1u) ? bo : so)) : R(0);
      } else {
        const R* src = (delta == 13 ? own : nbp[delta - nb_offset<D>()]) + (i * NTN + sp);
        const R* bb = own + (opp(i) * NTN + p);
        f[u][i] = act ? ld_pdf(((info[u] >> i) & 1u) ? bb : src) : R(0);
      }
    }
  }
  R* wr0 = static_cast<R*>(args.write) + t * STRIDE + j;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    R* wr = wr0 + u * HALF;
    const int type = (info[u] >> 24) & 3;
    if (type == 0) {
      if (info[u] & (1u << 27)) {
#pragma unroll
        for (int i = 0; i < Q; ++i) st_stream(wr + i * NTN, R(0));
      }
      continue;
    }
    bool good;
    if (type == 1)
      good = collide_bgk<D, INC>(f[u], static_cast<R>(args.inv_tau));
    else
      good = apply_boundary<D, INC>(f[u], type, (info[u] >> 26) & 1u, args.bc);
    if (!good) atomicMin(args.failed, static_cast<unsigned long long>(*args.step_base + args.rel + 1));
#pragma unroll
    for (int i = 0; i < Q; ++i) st_stream(wr + i * NTN, f[u][i]);
  }
}

// Advances the step counter the failure stamps are relative to (one per enqueued batch).
__global__ void bump_kernel(long long* step_base, long long by) { *step_base += by; }

// ---------------------------------------------------------------------------------------------
// Resident multi-step kernel for small domains (whole domain on one CTA per SM, e.g. BASELINE
// configs[0], 65 K nodes: the per-step launch gap is the step time there). One cooperative grid
// runs a whole batch of steps; every thread keeps its node for the batch, its q gather slots
// (the natural-state gather of engine.hpp:485-501, blocked directions included) are resolved once
// into shared memory, and consecutive steps are separated by a neighbour-CTA flag sync. The PDF gathers go
// through L2 only (ld.global.cg): a copy written by other CTAs in step s is read in step s+1 of
// the same kernel, so the non-coherent L1 path of the streamed kernels is not allowed here. Same
// slots, same arithmetic, same zero-fill: bit-identical to the one-launch-per-step path.
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double ld_l2(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float ld_l2(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}

// Between steps a CTA waits only for the CTAs that own tiles next to its own (the only ones whose
// step-s values it gathers in step s+1, and the only ones that gathered its step-s inputs, which
// step s+1 overwrites): each CTA release-stores its step epoch into its own flag word, then its
// threads poll the neighbour CTAs' flags with acquire loads, one flag per thread. Measured on B200
// (tools/barrier_probe.cu): a grid-wide barrier costs 1.2-2 us per step, more than the step.
__device__ __forceinline__ void neighbour_sync(unsigned* flags, unsigned epoch, const uint16_t* nbr,
                                               int n_nbr) {
  __syncthreads();
  if (threadIdx.x == 0) st_release_gpu(flags + blockIdx.x * 32, epoch);  // cumulative over the CTA
  for (int j = threadIdx.x; j < n_nbr; j += blockDim.x)
    while (static_cast<int>(ld_acquire_gpu(flags + nbr[j] * 32) - epoch) < 0) {
    }
  __syncthreads();
}

// Largest CTA of the resident kernel: 1024 threads (64 registers) except D3Q19 in f64, whose 19
// doubles spill at 64 (and at 80) registers: 512 threads.
template <int D, class R>
__host__ __device__ constexpr int resident_threads_max() { return D == 3 && sizeof(R) == 8 ? 512 : 1024; }

template <int D, bool INC, class R>
__global__ void __launch_bounds__(resident_threads_max<D, R>(), 1) t2c_resident_kernel(ResidentArgs ra) {
  constexpr int Q = Lat<D>::Q;
  extern __shared__ uint32_t s_src[];  // [Q][blockDim.x] gather slot of direction i
  const StepArgs& a = ra.s;
  const int n_tn = a.a * a.a * (D == 3 ? a.a : 1);
  const uint64_t k = static_cast<uint64_t>(blockIdx.x) * ra.tiles_per_cta * n_tn + threadIdx.x;
  const bool live = threadIdx.x < static_cast<unsigned>(ra.tiles_per_cta * n_tn) && k < a.n_nodes;
  const uint64_t t = a.t0 + (live ? k / n_tn : 0);
  const int p = live ? static_cast<int>(k % n_tn) : 0;
  const uint32_t info = live ? __ldg(a.info + t * n_tn + p) : 0u;
  const int type = (info >> 24) & 3;
  const bool zero_fill = live && type == 0 && (info & (1u << 27));
  const uint32_t own = static_cast<uint32_t>(t * Q * n_tn + p);  // slot (t, 0, p): < 2^32 (engine)
  const unsigned bd = blockDim.x;
#pragma unroll
  for (int i = 0; i < Q; ++i)
    s_src[i * bd + threadIdx.x] =
        type != 0 ? static_cast<uint32_t>(gather_slot<D>(a.nb, info, a.a, n_tn, t, p, i)) : 0u;
  // the CTAs owning the neighbour tiles of this CTA's tiles (kResidentMaxCtas bits)
  __shared__ unsigned s_bits[kResidentMaxCtas / 32];
  __shared__ uint16_t s_nbr[kResidentMaxCtas];
  __shared__ int s_n_nbr;
  for (int w = threadIdx.x; w < kResidentMaxCtas / 32; w += bd) s_bits[w] = 0u;
  if (threadIdx.x == 0) s_n_nbr = 0;
  __syncthreads();
  if (live && p == 0) {
    constexpr int NBS = D == 3 ? 27 : 9;
    for (int c = 0; c < NBS; ++c) {
      const uint32_t u = __ldg(a.nb + t * NBS + c);
      if (u == kEmpty || u < a.t0) continue;
      const uint64_t owner = (u - a.t0) / ra.tiles_per_cta;
      if (owner < gridDim.x && owner != blockIdx.x) atomicOr(&s_bits[owner / 32], 1u << (owner % 32));
    }
  }
  __syncthreads();
  for (unsigned c = threadIdx.x; c < gridDim.x; c += bd)
    if (s_bits[c / 32] & (1u << (c % 32))) s_nbr[atomicAdd(&s_n_nbr, 1)] = static_cast<uint16_t>(c);
  __syncthreads();
  const int n_nbr = s_n_nbr;
  const long long base = *a.step_base;
  const R inv_tau = static_cast<R>(a.inv_tau);
  for (int s = 0; s < ra.nsteps; ++s) {
    const int rd = (ra.rd0 + s) & 1;
    const R* src = static_cast<const R*>(rd ? ra.pdf1 : ra.pdf0);
    R* dst = static_cast<R*>(rd ? ra.pdf0 : ra.pdf1) + own;
    if (type != 0) {
      R f[Q];
#pragma unroll
      for (int i = 0; i < Q; ++i) f[i] = ld_l2(src + s_src[i * bd + threadIdx.x]);
      const bool good = type == 1 ? collide_bgk<D, INC>(f, inv_tau)
                                  : apply_boundary<D, INC>(f, type, (info >> 26) & 1u, a.bc);
      if (!good) atomicMin(a.failed, static_cast<unsigned long long>(base + s + 1));
#pragma unroll
      for (int i = 0; i < Q; ++i) dst[i * n_tn] = f[i];
    } else if (zero_fill) {
#pragma unroll
      for (int i = 0; i < Q; ++i) dst[i * n_tn] = R(0);
    }
    if (s + 1 < ra.nsteps) neighbour_sync(ra.flags, ra.epoch0 + s + 1, s_nbr, n_nbr);
  }
}

// Slab halo-arrival wait (p2p transport): one thread polls the "faces arrived" flags with
// system-scope acquire loads until both reach `seq`. The neighbours publish a flag only after
// their boundary planes (whose peer stores into my halo tiles precede it: stream write-value with
// its default system-scope fence); the acquire makes those remote stores visible here, and the
// boundary-plane kernel that follows in stream order reads them. This is the PTX memory-model
// release/acquire pattern, valid also when the receiving GPU reorders remote writes (the reason a
// plain cuStreamWaitValue64 would need CU_STREAM_WAIT_VALUE_FLUSH).
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__global__ void wait_flags_kernel(const unsigned long long* f0, const unsigned long long* f1,
                                  unsigned long long seq) {
  unsigned ns = 32;
  for (const unsigned long long* f : {f0, f1}) {
    if (!f) continue;
    while (ld_acquire_sys(f) < seq) {
      __nanosleep(ns);
      ns = ns < 1024 ? 2 * ns : ns;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Gather words (see file header). Mirrors the blocked test of the sweep (engine.hpp:485-500).
template <int D>
__global__ void node_info_kernel(NodeInfoArgs args) {
  constexpr int Q = Lat<D>::Q;
  const int a = args.a;
  const int az = D == 3 ? a : 1;
  const int n_tn = a * a * az;
  const uint64_t node = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (node >= args.n_stored * n_tn) return;
  const uint64_t t = node / n_tn;
  const int p = static_cast<int>(node % n_tn);
  const uint8_t own_byte = args.types[node];
  const int type = own_byte & 3;
  uint32_t info = static_cast<uint32_t>(type) << 24;
  if (own_byte & 4) info |= 1u << 26;
  if (type == 0) {
    // the 32-B store sector holds `sector` consecutive slots (4 doubles / 8 floats)
    const int g = args.sector;
    if (SPLBM_ZERO_FILL && n_tn % g == 0) {
      const uint8_t* grp = args.types + (node - node % g);
      uint8_t any = 0;
      for (int k = 0; k < g; ++k) any |= grp[k];
      if (any & 3) info |= 1u << 27;
    }
    args.info[node] = info;
    return;
  }
  const int lx = p % a, ly = (p / a) % a, lz = D == 3 ? p / (a * a) : 0;
  for (int i = 0; i < Q; ++i) {
    int sx = lx - ex<D>(i), sy = ly - ey<D>(i), sz = lz - ez<D>(i);
    int dx = 0, dy = 0, dz = 0;
    if (sx < 0) { dx = -1; sx += a; } else if (sx >= a) { dx = 1; sx -= a; }
    if (sy < 0) { dy = -1; sy += a; } else if (sy >= a) { dy = 1; sy -= a; }
    if (D == 3) {
      if (sz < 0) { dz = -1; sz += a; } else if (sz >= a) { dz = 1; sz -= a; }
    }
    const int delta = (dx + 1) + 3 * ((dy + 1) + 3 * (dz + 1));
    const int sp = sx + a * (sy + a * sz);
    bool blocked;
    if (delta == 13) {
      blocked = (args.types[t * n_tn + sp] & 3) == 0;
    } else {
      const uint32_t s = args.nb[t * nb_stride<D>() + delta - nb_offset<D>()];
      // a neighbour outside the stored range (slab mode edge) counts as EMPTY
      blocked = s == kEmpty || (args.types[static_cast<uint64_t>(s) * n_tn + sp] & 3) == 0;
    }
    if (blocked) info |= 1u << i;
  }
  args.info[node] = info;
}

// ---------------------------------------------------------------------------------------------
// TileEngineT2C::initialize (engine.hpp:336-352): equilibrium<T>(T(rho), u.cast<T>()) of per-node
// (rho, u) into both copies (one in single-copy mode).
template <int D, bool INC, class R>
__global__ void init_kernel(InitArgs args) {
  constexpr int Q = Lat<D>::Q;
  const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= args.count) return;
  const uint64_t node = args.node0 + k;
  const uint64_t t = node / args.n_tn;
  const int p = static_cast<int>(node % args.n_tn);
  double rho, u0, u1, u2;
  if (args.rho) {
    rho = args.rho[k];
    u0 = args.ux[k];
    u1 = args.uy[k];
    u2 = args.uz[k];
  } else {
    rho = args.rho0;
    u0 = args.u0[0];
    u1 = args.u0[1];
    u2 = args.u0[2];
  }
  const R r = static_cast<R>(rho);
  if (!INC && !(r > R(0))) atomicOr(args.domain_error, 1);  // lattice.hpp:76-78
  R f[Q];
  equilibrium<D, INC>(r, static_cast<R>(u0), static_cast<R>(u1), static_cast<R>(u2), f);
  const uint64_t base = t * static_cast<uint64_t>(Q) * args.n_tn + p;
  R* p0 = static_cast<R*>(args.pdf0);
  R* p1 = static_cast<R*>(args.pdf1);
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    p0[base + static_cast<uint64_t>(i) * args.n_tn] = f[i];
    if (p1) p1[base + static_cast<uint64_t>(i) * args.n_tn] = f[i];
  }
}

// ---------------------------------------------------------------------------------------------
// fields(): moments<T> (lattice.hpp:94-112) of every non-solid stored node, written as
// static_cast<double>(m) (engine.hpp:383-386) at its raster index in the FieldData frame slice.
template <int D, bool INC, class R>
__global__ void __launch_bounds__(256) frame_kernel(FrameArgs args) {
  constexpr int Q = Lat<D>::Q;
  const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= args.n_tiles * args.n_tn) return;
  const uint64_t t = args.tile0 + k / args.n_tn;
  const int p = static_cast<int>(k % args.n_tn);
  const uint64_t node = t * args.n_tn + p;
  const uint32_t inf = args.info[node];
  if (((inf >> 24) & 3) == 0) return;
  const uint32_t c = args.cells[k / args.n_tn];
  const int a = args.a;
  const int x = static_cast<int>(c % args.gx) * a + p % a;
  const int y = static_cast<int>((c / args.gx) % args.gy) * a + (p / a) % a;
  const int z = D == 3 ? static_cast<int>(c / (static_cast<uint32_t>(args.gx) * args.gy)) * a + p / (a * a) : 0;
  const uint64_t o = static_cast<uint64_t>(x) +
                     static_cast<uint64_t>(args.dims[0]) * (y + static_cast<uint64_t>(args.dims[1]) * z) - args.base;
  R f[Q];
  load_state<D>(static_cast<const R*>(args.pdf), inf, args.view, args.n_tn, t, p, f);
  const R r = density<D>(f);
  R m0 = momentum<D, 0>(f), m1 = momentum<D, 1>(f), m2 = momentum<D, 2>(f);
  if (!INC) {
    if (r == R(0)) {
      atomicOr(args.domain_error, 1);  // lattice.hpp:105-108
    } else {
      divide3(m0, m1, m2, r);
    }
  }
  if (args.rho) args.rho[o] = static_cast<double>(r);
  if (args.ux) args.ux[o] = static_cast<double>(m0);
  if (args.uy) args.uy[o] = static_cast<double>(m1);
  if (args.uz) args.uz[o] = static_cast<double>(m2);
  if (args.mask) args.mask[o] = 1;
}

// ---------------------------------------------------------------------------------------------
// Deterministic reduction over owned non-solid nodes: fixed per-block tree, then one block.
// Moments in the engine's type, accumulated in double.
template <int D, bool INC, class R>
__global__ void __launch_bounds__(kThreads) reduce_partial_kernel(ReduceArgs args) {
  constexpr int Q = Lat<D>::Q;
  __shared__ double s_mass[kThreads];
  __shared__ double s_umax[kThreads];
  __shared__ double s_bad[kThreads];
  double mass = 0.0, umax = 0.0, bad = 0.0;
  const uint64_t n = args.n_nodes;
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; k < n;
       k += static_cast<uint64_t>(gridDim.x) * kThreads) {
    const uint64_t node = args.node0 + k;
    const int type = (args.info[node] >> 24) & 3;
    if (type == 0) continue;
    const uint64_t t = node / args.n_tn;
    const int p = static_cast<int>(node % args.n_tn);
    R f[Q];
    load_state<D>(static_cast<const R*>(args.pdf), args.info[node], args.view, args.n_tn, t, p, f);
    const R rr = density<D>(f);
    R v0 = momentum<D, 0>(f), v1 = momentum<D, 1>(f), v2 = momentum<D, 2>(f);
    if (!INC && rr != R(0)) {
      v0 = ddiv(v0, rr);
      v1 = ddiv(v1, rr);
      v2 = ddiv(v2, rr);
    }
    const double r = static_cast<double>(rr);
    const double sp = sqrt(sqnorm(static_cast<double>(v0), static_cast<double>(v1),
                                  static_cast<double>(v2)));
    if (!(isfinite(r) && isfinite(sp))) {
      bad += 1.0;
    } else {
      mass += r;
      umax = fmax(umax, sp);
    }
  }
  s_mass[threadIdx.x] = mass;
  s_umax[threadIdx.x] = umax;
  s_bad[threadIdx.x] = bad;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s_mass[threadIdx.x] += s_mass[threadIdx.x + w];
      s_umax[threadIdx.x] = fmax(s_umax[threadIdx.x], s_umax[threadIdx.x + w]);
      s_bad[threadIdx.x] += s_bad[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    args.partial[3 * blockIdx.x + 0] = s_mass[0];
    args.partial[3 * blockIdx.x + 1] = s_umax[0];
    args.partial[3 * blockIdx.x + 2] = s_bad[0];
  }
}

__global__ void reduce_final_kernel(const double* partial, int n, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double m = 0.0, u = 0.0, b = 0.0;
  for (int i = 0; i < n; ++i) {
    m += partial[3 * i];
    u = fmax(u, partial[3 * i + 1]);
    b += partial[3 * i + 2];
  }
  out[0] = m;
  out[1] = u;
  out[2] = b;
}

// ---------------------------------------------------------------------------------------------
// Slab-mode halo faces: copy the lz == a-1 (high face) or lz == 0 (low face) layer of
// the directions crossing that face, for a contiguous range of tiles, to/from a packed buffer.
// Packed order: [tile k][direction j of the face set][a*a face nodes], all contiguous runs.
template <int D>
__global__ void halo_copy_kernel(HaloArgs args) {
  constexpr int Q = Lat<D>::Q;
  const int a = args.a;
  const int n_tn = D == 3 ? a * a * a : a * a;
  const int face = n_tn / a;  // one layer normal to the slab axis (z in 3D, y in 2D)
  const uint64_t per_tile = static_cast<uint64_t>(args.n_dirs) * face;
  const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= args.n_tiles * per_tile) return;
  const uint64_t tk = k / per_tile;
  const int rem = static_cast<int>(k % per_tile);
  const int j = rem / face;
  const int fnode = rem % face;
  const int dir = args.dirs[j];
  const uint64_t slot = ((args.tile0 + tk) * Q + dir) * static_cast<uint64_t>(n_tn) +
                        static_cast<uint64_t>(args.layer) * face + fnode;
  if (args.pack) {
    args.buf[k] = args.pdf[slot];
  } else {
    if (args.info) {  // single-copy backward unpack: only slots the neighbour's scatter wrote
      const uint32_t w = args.info[(args.tile0 + tk) * n_tn + static_cast<uint64_t>(args.layer) * face + fnode];
      if (((w >> 24) & 3u) == 0u || ((w >> opp(dir)) & 1u)) return;
    }
    args.pdf[slot] = args.buf[k];
  }
}

// Natural-layout copy of a tile range of the current state (parity dumps of a swapped AA state).
template <int D, class R>
__global__ void unswap_kernel(const R* pdf, const uint32_t* info, StateView v, int n_tn,
                              uint64_t tile0, uint64_t n_tiles, R* out) {
  constexpr int Q = Lat<D>::Q;
  const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n_tiles * n_tn) return;
  const uint64_t t = tile0 + k / n_tn;
  const int p = static_cast<int>(k % n_tn);
  const uint32_t w = info[t * n_tn + p];
  R f[Q];
  if (((w >> 24) & 3) == 0) {  // solid slots are not part of the state: copied as stored
#pragma unroll
    for (int i = 0; i < Q; ++i) f[i] = pdf[(t * Q + i) * static_cast<uint64_t>(n_tn) + p];
  } else {
    load_state<D>(pdf, w, v, n_tn, t, p, f);
  }
  R* o = out + (k / n_tn) * Q * n_tn + p;
#pragma unroll
  for (int i = 0; i < Q; ++i) o[static_cast<uint64_t>(i) * n_tn] = f[i];
}

// Self-test of the shared-reciprocal division against IEEE division (tests/test_device_division.py).
template <class R>
__global__ void divide_selftest_kernel(uint64_t n, const R* m, const R* rho, R* out) {
  const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  R a = m[3 * k], b = m[3 * k + 1], c = m[3 * k + 2];
  divide3(a, b, c, rho[k]);
  out[3 * k] = a;
  out[3 * k + 1] = b;
  out[3 * k + 2] = c;
}

// ---------------------------------------------------------------------------------------------
// Launchers (host side of this translation unit)
// T(kernel(i, j)): the double MRT operator rounded to the engine's type (collision.cpp:108-111)
template <class R, int Q>
static MrtMatrix<R, Q> mrt_param(const double* K) {
  MrtMatrix<R, Q> m;
  for (int i = 0; i < Q * Q; ++i) m.K[i] = static_cast<R>(K[i]);
  return m;
}

template <class Kern, class M>
static void launch_maybe_pdl(Kern kern, unsigned blocks, cudaStream_t st, const StepArgs& a, const M& m,
                             int threads = kThreads) {
#if SPLBM_PDL
  // Overlap the next step's launch and static-table prologue with this step's tail; below a few
  // waves (launch-latency-bound domains) the plain launch measured faster.
  if (static_cast<uint64_t>(blocks) * threads >= a.pdl_min_threads) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a, m);
    return;
  }
#endif
  kern<<<blocks, threads, 0, st>>>(a, m);
}

template <int D, int LOGA, bool INC, int PHASE, class R>
static void launch_aa(const StepArgs& a, unsigned blocks, cudaStream_t st) {
  if constexpr (PHASE == 1 && std::is_same<R, double>::value) {
    if (!a.mrt_K && (a.peer_up || a.peer_down)) {  // slab boundary planes, p2p single copy
      t2c_aa_kernel<D, LOGA, INC, false, 1, R, true>
          <<<blocks, aa_threads<D, LOGA>(), 0, st>>>(a, MrtMatrix<R, 1>{});
      return;
    }
  }
  if (a.mrt_K && a.jit) {  // the phase kernel specialised for this engine's operator (mrt_jit.cpp)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(aa_threads<D, LOGA>());
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
#if SPLBM_PDL
    if (static_cast<uint64_t>(blocks) * aa_threads<D, LOGA>() >= a.pdl_min_threads) {
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
    }
#endif
    StepArgs args = a;
    MrtMatrix<R, 1> k{};
    void* params[] = {&args, &k};
    cudaLaunchKernelExC(&cfg, a.jit, params);
  } else if (a.mrt_K)
    launch_maybe_pdl(t2c_aa_kernel<D, LOGA, INC, true, PHASE, R>, blocks, st, a,
                     mrt_param<R, Lat<D>::Q>(a.mrt_K), aa_threads<D, LOGA>());
  else
    launch_maybe_pdl(t2c_aa_kernel<D, LOGA, INC, false, PHASE, R>, blocks, st, a, MrtMatrix<R, 1>{},
                     aa_threads<D, LOGA>());
}

template <int D, int LOGA, bool INC, class R>
static void launch_pow2(const StepArgs& a, cudaStream_t st) {
  constexpr int NTN = D == 3 ? (1 << (3 * LOGA)) : (1 << (2 * LOGA));
  constexpr int TILES = step_threads<D, NTN>() / NTN;
  const uint64_t tiles = a.n_nodes / NTN;
  const unsigned blocks = static_cast<unsigned>((tiles + TILES - 1) / TILES);
  const MrtMatrix<R, 1> none{};
  if (a.aa) {
    constexpr int ATILES = aa_threads<D, LOGA>() / NTN;
    const unsigned ablocks = static_cast<unsigned>((tiles + ATILES - 1) / ATILES);
    if (a.aa == 1) launch_aa<D, LOGA, INC, 1, R>(a, ablocks, st);
    else launch_aa<D, LOGA, INC, 2, R>(a, ablocks, st);
    return;
  }
  if (a.mrt_K) {
    if (a.jit) {  // specialised for this engine's operator (mrt_jit.cpp; same template, GEN = true)
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(blocks);
      cfg.blockDim = dim3(step_threads<D, NTN>());
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
#if SPLBM_PDL
      if (static_cast<uint64_t>(blocks) * step_threads<D, NTN>() >= a.pdl_min_threads) {
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
      }
#endif
      StepArgs args = a;
      MrtMatrix<R, 1> k{};
      void* params[] = {&args, &k};
      cudaLaunchKernelExC(&cfg, a.jit, params);
      return;
    }
    launch_maybe_pdl(t2c_step_pow2_kernel<D, LOGA, INC, false, true, R>, blocks, st, a,
                     mrt_param<R, Lat<D>::Q>(a.mrt_K), step_threads<D, NTN>());
    return;
  }
  if constexpr (std::is_same<R, double>::value) {
    if (a.peer_up || a.peer_down) {  // slab boundary planes with NVLink peer stores
      t2c_step_pow2_kernel<D, LOGA, INC, true, false, R><<<blocks, step_threads<D, NTN>(), 0, st>>>(a, none);
      return;
    }
  }
  // f32, and D2Q9 in f64 (18 values per thread fit 64 registers: vessel tree / dense 4096^2 -5 %,
  // profiles/ab_x2_2d_r2.txt); D3Q19 f64 would need 128 registers and measured 5-11 % slower
  if constexpr ((sizeof(R) == 4 || D == 2) && NTN >= 16 && (SPLBM_X2_THREADS % (NTN / 2)) == 0) {
    if (a.x2 && a.skip_by == 0) {  // two nodes per thread
      constexpr int XT = SPLBM_X2_THREADS / (NTN / 2);
      const unsigned xb = static_cast<unsigned>((tiles + XT - 1) / XT);
      if (a.off32)
        launch_maybe_pdl(t2c_step_x2_kernel<D, LOGA, INC, R, true>, xb, st, a, none, SPLBM_X2_THREADS);
      else
        launch_maybe_pdl(t2c_step_x2_kernel<D, LOGA, INC, R, false>, xb, st, a, none, SPLBM_X2_THREADS);
      return;
    }
  }
  launch_maybe_pdl(t2c_step_pow2_kernel<D, LOGA, INC, false, false, R>, blocks, st, a, none,
                   step_threads<D, NTN>());
}

template <int D, int A, bool INC, class R>
static void launch_generic(const StepArgs& a, unsigned blocks, cudaStream_t st) {
  if (a.aa) return;  // the engine rejects single-copy mode for non-power-of-two tiles
  if (a.mrt_K)
    t2c_step_kernel<D, A, INC, true, R><<<blocks, kThreads, 0, st>>>(a, mrt_param<R, Lat<D>::Q>(a.mrt_K));
  else
    t2c_step_kernel<D, A, INC, false, R><<<blocks, kThreads, 0, st>>>(a, MrtMatrix<R, 1>{});
}

template <int D, bool INC, class R>
static cudaError_t launch_step_d(const StepArgs& a, cudaStream_t st) {
  const unsigned blocks = static_cast<unsigned>((a.n_nodes + kThreads - 1) / kThreads);
  if (blocks == 0) return cudaSuccess;
  if constexpr (D == 3) {
    switch (a.a) {
      case 2: launch_pow2<D, 1, INC, R>(a, st); break;
      case 4: launch_pow2<D, 2, INC, R>(a, st); break;
      case 8: launch_generic<D, 8, INC, R>(a, blocks, st); break;
      default: launch_generic<D, 0, INC, R>(a, blocks, st); break;
    }
  } else {
    switch (a.a) {
      case 2: launch_pow2<D, 1, INC, R>(a, st); break;
      case 4: launch_pow2<D, 2, INC, R>(a, st); break;
      case 8: launch_pow2<D, 3, INC, R>(a, st); break;
      case 16: launch_pow2<D, 4, INC, R>(a, st); break;
      default: launch_generic<D, 0, INC, R>(a, blocks, st); break;
    }
  }
  return cudaGetLastError();
}

// Dispatch on (dimension, compressibility, real type) for the per-type launchers below.
template <template <int, bool, class> class F, class... Args>
static cudaError_t dispatch(int d, bool inc, bool f32, Args&&... args) {
  if (d == 2) {
    if (f32) return inc ? F<2, true, float>::run(args...) : F<2, false, float>::run(args...);
    return inc ? F<2, true, double>::run(args...) : F<2, false, double>::run(args...);
  }
  if (f32) return inc ? F<3, true, float>::run(args...) : F<3, false, float>::run(args...);
  return inc ? F<3, true, double>::run(args...) : F<3, false, double>::run(args...);
}

template <int D, bool INC, class R>
struct StepL {
  static cudaError_t run(const StepArgs& a, cudaStream_t st) { return launch_step_d<D, INC, R>(a, st); }
};
template <int D, bool INC, class R>
struct InitL {
  static cudaError_t run(const InitArgs& a, cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>((a.count + 255) / 256);
    if (blocks) init_kernel<D, INC, R><<<blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
  }
};
template <int D, bool INC, class R>
struct FrameL {
  static cudaError_t run(const FrameArgs& a, cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>((a.n_tiles * a.n_tn + 255) / 256);
    if (blocks) frame_kernel<D, INC, R><<<blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
  }
};
template <int D, bool INC, class R>
struct ReduceL {
  static cudaError_t run(const ReduceArgs& a, int blocks, double* out, cudaStream_t st) {
    reduce_partial_kernel<D, INC, R><<<blocks, kThreads, 0, st>>>(a);
    reduce_final_kernel<<<1, 32, 0, st>>>(a.partial, blocks, out);
    return cudaGetLastError();
  }
};
template <int D, bool INC, class R>
struct UnswapL {
  static cudaError_t run(const void* pdf, const uint32_t* info, StateView v, int n_tn,
                         uint64_t tile0, uint64_t n_tiles, void* out, cudaStream_t st) {
    const uint64_t n = n_tiles * n_tn;
    const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
    if (blocks)
      unswap_kernel<D, R><<<blocks, 256, 0, st>>>(static_cast<const R*>(pdf), info, v, n_tn, tile0,
                                                  n_tiles, static_cast<R*>(out));
    return cudaGetLastError();
  }
};

cudaError_t launch_step(int d, bool inc, bool f32, const StepArgs& a, cudaStream_t st) {
  return dispatch<StepL>(d, inc, f32, a, st);
}

template <int D, bool INC, class R>
struct ResidentL {
  static cudaError_t run(const ResidentArgs& ra, unsigned blocks, unsigned threads, cudaStream_t st,
                         bool probe) {
    auto kern = t2c_resident_kernel<D, INC, R>;
    const size_t smem = static_cast<size_t>(Lat<D>::Q) * threads * sizeof(uint32_t);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    if (probe) {  // `blocks` CTAs of this size resident per SM?
      if (threads > static_cast<unsigned>(resident_threads_max<D, R>())) return cudaErrorInvalidValue;
      int occ = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, static_cast<int>(threads), smem);
      if (e != cudaSuccess) return e;
      return occ >= static_cast<int>(blocks) ? cudaSuccess : cudaErrorCooperativeLaunchTooLarge;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, ra);
  }
};

cudaError_t launch_resident(int d, bool inc, bool f32, const ResidentArgs& ra, unsigned blocks,
                            unsigned threads, cudaStream_t st) {
  return dispatch<ResidentL>(d, inc, f32, ra, blocks, threads, st, false);
}

cudaError_t resident_fits(int d, bool inc, bool f32, unsigned threads, unsigned per_sm) {
  return dispatch<ResidentL>(d, inc, f32, ResidentArgs{}, per_sm, threads, cudaStream_t{}, true);
}

cudaError_t launch_bump(long long* step_base, long long by, cudaStream_t st) {
  bump_kernel<<<1, 1, 0, st>>>(step_base, by);
  return cudaGetLastError();
}

cudaError_t launch_wait_flags(const unsigned long long* f0, const unsigned long long* f1,
                              unsigned long long seq, cudaStream_t st) {
  wait_flags_kernel<<<1, 1, 0, st>>>(f0, f1, seq);
  return cudaGetLastError();
}

cudaError_t launch_node_info(int d, const NodeInfoArgs& a, cudaStream_t st) {
  const int n_tn = a.a * a.a * (d == 3 ? a.a : 1);
  const uint64_t n = a.n_stored * n_tn;
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  if (blocks == 0) return cudaSuccess;
  if (d == 2)
    node_info_kernel<2><<<blocks, 256, 0, st>>>(a);
  else
    node_info_kernel<3><<<blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_init(int d, bool inc, bool f32, const InitArgs& a, cudaStream_t st) {
  return dispatch<InitL>(d, inc, f32, a, st);
}

cudaError_t launch_frame(int d, bool inc, bool f32, const FrameArgs& a, cudaStream_t st) {
  return dispatch<FrameL>(d, inc, f32, a, st);
}

cudaError_t launch_reduce(int d, bool inc, bool f32, const ReduceArgs& a, int blocks, double* out,
                          cudaStream_t st) {
  return dispatch<ReduceL>(d, inc, f32, a, blocks, out, st);
}

cudaError_t launch_unswap(int d, bool f32, const void* pdf, const uint32_t* info, StateView v,
                          int n_tn, uint64_t tile0, uint64_t n_tiles, void* out, cudaStream_t st) {
  return dispatch<UnswapL>(d, false, f32, pdf, info, v, n_tn, tile0, n_tiles, out, st);
}

cudaError_t launch_divide_selftest(uint64_t n, const double* m, const double* rho, double* out,
                                   cudaStream_t st) {
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  if (blocks) divide_selftest_kernel<double><<<blocks, 256, 0, st>>>(n, m, rho, out);
  return cudaGetLastError();
}

cudaError_t launch_divide_selftest_f32(uint64_t n, const float* m, const float* rho, float* out,
                                       cudaStream_t st) {
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  if (blocks) divide_selftest_kernel<float><<<blocks, 256, 0, st>>>(n, m, rho, out);
  return cudaGetLastError();
}

cudaError_t launch_halo(int d, const HaloArgs& a, cudaStream_t st) {
  const uint64_t n = a.n_tiles * static_cast<uint64_t>(a.n_dirs) * (d == 3 ? a.a * a.a : a.a);
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  if (blocks == 0) return cudaSuccess;
  if (d == 2)
    halo_copy_kernel<2><<<blocks, 256, 0, st>>>(a);
  else
    halo_copy_kernel<3><<<blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace splbm_dev
