// The single-copy (AA) step kernels. Included by kernels.cu (ahead of time) and compiled at run
// time by mrt_jit.cpp through NVRTC for single-copy MRT engines (GEN = true, the operator's
// specialised collide_mrt_gen<>). Must stay free of host-only headers.
#pragma once
#include "step_pow2.cuh"

namespace splbm_dev {

// Single-copy propagation (the AA access pattern on the reference's tile layout). One
// PDF array, updated in place; results are bit-identical to the two-copy T2C step because every
// node applies the same arithmetic to the same incoming values. With addr(i) = the slot the
// natural gather of direction i reads (source x - e_i, or the own opposite slot if blocked):
//   PHASE 1 (natural state):  f_i = *addr(i); collide; *addr(opp(i)) = f*_i   -> swapped state
//   PHASE 2 (swapped state):  f_i = own[opp(i)];  collide; own[i] = f*_i       -> natural state
// Each node reads and writes exactly the slots of its own set, so the in-place update is race
// free; phase 2 touches only the node's own slots (no neighbour tables, no cross-tile reads).
// Register budget: phase 1 keeps only the q values live through the collision and re-derives the
// scatter addresses afterwards (64 registers, no spills, 16 CTAs of 64 threads per SM).
template <int D, int LOGA>
__host__ __device__ constexpr int aa_threads() {
  return SPLBM_AA_THREADS > (D == 3 ? (1 << (3 * LOGA)) : (1 << (2 * LOGA))) ? SPLBM_AA_THREADS
                                                                             : (D == 3 ? (1 << (3 * LOGA)) : (1 << (2 * LOGA)));
}
template <int D, int LOGA, bool INC, bool MRT, int PHASE, class R, bool PEER = false, bool GEN = false>
__global__ void __launch_bounds__(aa_threads<D, LOGA>(),
                                  (MRT ? 2 : (D == 3 ? (PHASE == 1 ? SPLBM_AA1_MINB : SPLBM_MINB3) : SPLBM_MINB2)) * 256 / aa_threads<D, LOGA>())
    t2c_aa_kernel(StepArgs args, const __grid_constant__ MrtMatrix<R, (MRT && !GEN) ? Lat<D>::Q : 1> mrt) {
  constexpr int Q = Lat<D>::Q;
  constexpr int A = 1 << LOGA;
  constexpr int NTN = D == 3 ? A * A * A : A * A;
  constexpr int TILES = aa_threads<D, LOGA>() / NTN;
  constexpr uint64_t STRIDE = static_cast<uint64_t>(Q) * NTN;
  constexpr int NBS = nb_stride<D>();
  __shared__ R* s_base[PHASE == 1 ? TILES : 1][NBS];

  R* const pdf = static_cast<R*>(args.write);
  const uint64_t n_tiles = args.n_nodes / NTN;
  const uint64_t tile_blk = static_cast<uint64_t>(blockIdx.x) * TILES;
  if constexpr (PHASE == 1) {
    for (int k = threadIdx.x; k < TILES * NBS; k += aa_threads<D, LOGA>()) {
      const int tl = k / NBS, dd = k % NBS;
      const uint64_t tt = tile_blk + tl;
      R* b = nullptr;
      if (tt < n_tiles) {
        const uint32_t s = __ldg(args.nb + tile_of(args, tt) * NBS + dd);
        if (s == kEmpty) b = nullptr;
        // slab p2p, phase 1: the slots of halo nodes are read and written in place in the
        // neighbour's owned tiles over NVLink (each slot is touched by exactly one node, this one)
        else if (PEER && s < args.halo_lo_end) b = reinterpret_cast<R*>(args.peer_down) + static_cast<uint64_t>(s) * STRIDE;
        else if (PEER && s >= args.halo_hi_begin) b = reinterpret_cast<R*>(args.peer_up) + static_cast<uint64_t>(s - args.halo_hi_begin) * STRIDE;
        else b = pdf + static_cast<uint64_t>(s) * STRIDE;
      }
      s_base[tl][dd] = b;
    }
  }
  const int tl = threadIdx.x / NTN;
  const int p = threadIdx.x % NTN;
  const uint64_t tloc = tile_blk + tl;
  const uint64_t t = tloc < n_tiles ? tile_of(args, tloc) : 0;
  const uint32_t info = tloc < n_tiles ? __ldg(args.info + t * NTN + p) : 0u;
  if constexpr (PHASE == 1) __syncthreads();
#if SPLBM_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  {
    const uint64_t pf = tile_blk + static_cast<uint64_t>(args.l2pf) * TILES + threadIdx.x;
    l2_prefetch_blocks<Q, NTN, TILES>(pdf, (args.l2pf && pf < n_tiles && threadIdx.x < TILES) ? tile_of(args, pf) : 0,
                                      args.l2pf && pf < n_tiles);
  }
  const int type = (info >> 24) & 3;
  R* own = pdf + t * STRIDE;
  if (type == 0) {  // solid slots are never read: whole store sectors (see file header)
    if (info & (1u << 27)) {
#pragma unroll
      for (int i = 0; i < Q; ++i) st_stream(own + i * NTN + p, R(0));
    }
    return;
  }
  const int lx = p & (A - 1);
  const int ly = (p >> LOGA) & (A - 1);
  const int lz = D == 3 ? (p >> (2 * LOGA)) : 0;
  R* const* nbp = s_base[PHASE == 1 ? tl : 0];
  auto addr = [&](int i) -> R* {  // PHASE 1 only
    const int vx = lx - ex<D>(i), vy = ly - ey<D>(i), vz = lz - ez<D>(i);
    const int dx = ex<D>(i) ? (vx >> LOGA) : 0;
    const int dy = ey<D>(i) ? (vy >> LOGA) : 0;
    const int dz = (D == 3 && ez<D>(i)) ? (vz >> LOGA) : 0;
    const int sp = (vx & (A - 1)) | ((vy & (A - 1)) << LOGA) | (D == 3 ? ((vz & (A - 1)) << (2 * LOGA)) : 0);
    const int delta = 13 + dx + 3 * dy + 9 * dz;
    R* src = (delta == 13 ? own : nbp[delta - nb_offset<D>()]) + (i * NTN + sp);
    R* bb = own + (opp(i) * NTN + p);
    return ((info >> i) & 1u) ? bb : src;
  };

  R f[Q];
#pragma unroll
  for (int i = 0; i < Q; ++i) f[i] = ld_pdf_rw(PHASE == 1 ? addr(i) : own + (opp(i) * NTN + p));

  bool good;
  if (type == 1) {
    if constexpr (MRT && GEN)
      good = collide_mrt_gen<D, INC, R>(f);  // runtime-specialised operator (mrt_jit.cpp)
    else if constexpr (MRT)
      good = collide_mrt<D, INC>(f, mrt.K);
    else
      good = collide_bgk<D, INC>(f, static_cast<R>(args.inv_tau));
  } else {
    good = apply_boundary<D, INC>(f, type, (info >> 26) & 1u, args.bc);
  }
  if (!good) atomicMin(args.failed, static_cast<unsigned long long>(*args.step_base + args.rel + 1));
  if constexpr (PHASE == 1) {
    // Nothing but f[] stays live through the collision: the node's tile, position and gather word
    // are re-derived from opaque reads of the CTA/thread index (the compiler cannot keep the old
    // values instead) and the scatter addresses recomputed from the shared-memory bases. 64
    // registers without spills (80 with 28 B of spills otherwise): channel / RAS phi 0.5 / 2D
    // -3 / -6 / -3 % per single-copy step (interleaved A/B, profiles/ab_aa1_r2.txt).
    uint32_t bx, tx;
    asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(bx));
    asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tx));
    const int tl2 = static_cast<int>(tx) / NTN;
    const int p2 = static_cast<int>(tx) % NTN;
    const uint64_t t2 = tile_of(args, static_cast<uint64_t>(bx) * TILES + tl2);
    uint32_t info2;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(info2) : "l"(args.info + t2 * NTN + p2));
    R* own2 = pdf + t2 * STRIDE;
    R* const* nbp2 = s_base[tl2];
    const int lx2 = p2 & (A - 1), ly2 = (p2 >> LOGA) & (A - 1), lz2 = D == 3 ? (p2 >> (2 * LOGA)) : 0;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      const int j = opp(i);
      const int vx = lx2 - ex<D>(j), vy = ly2 - ey<D>(j), vz = lz2 - ez<D>(j);
      const int dx = ex<D>(j) ? (vx >> LOGA) : 0;
      const int dy = ey<D>(j) ? (vy >> LOGA) : 0;
      const int dz = (D == 3 && ez<D>(j)) ? (vz >> LOGA) : 0;
      const int sp = (vx & (A - 1)) | ((vy & (A - 1)) << LOGA) | (D == 3 ? ((vz & (A - 1)) << (2 * LOGA)) : 0);
      const int delta = 13 + dx + 3 * dy + 9 * dz;
      R* dst = (delta == 13 ? own2 : nbp2[delta - nb_offset<D>()]) + (j * NTN + sp);
      st_stream(((info2 >> j) & 1u) ? own2 + (i * NTN + p2) : dst, f[i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < Q; ++i) st_stream(own + (i * NTN + p), f[i]);
  }
}

}  // namespace splbm_dev
