// Kernel-argument structs of the step kernels, shared by the ahead-of-time build (kernels.cu) and
// the runtime-specialised MRT step (mrt_jit.cpp compiles step_pow2.cuh with NVRTC): plain data,
// no CUDA runtime headers.
#pragma once
#include "lattice.cuh"

namespace splbm_dev {

// PDF arrays are `void*` here: the engine's real type (double for TileEngineT2C<double>, float
// for TileEngineT2C<float>) selects the kernel instantiation (launch_* `f32`).
struct StepArgs {
  const void* read;
  void* write;
  const uint32_t* info;  // per stored tile node gather word
  const uint32_t* nb;    // stored tiles x 27 (3D) / 9 (2D, dz = 0 slice), local indices
  uint64_t t0;           // first stepped tile (stored index)
  uint64_t n_nodes;      // stepped tiles * n_tn
  uint64_t skip_at;      // stepped-tile ordinal from which `skip_by` tiles are jumped (two ranges
  uint64_t skip_by;      // in one launch: a slab's bottom and top planes); skip_by = 0 = one range
  int a;
  double inv_tau;  // T(1.0 / tau) (collision.cpp:93), exact in double for either T
  const double* mrt_K;  // MRT operator (q x q, HOST memory, rounded to T and copied into the
                        // launch); nullptr = BGK
  BcParams bc;
  unsigned long long* failed;  // min failing step number (ULLONG_MAX = none)
  const long long* step_base;  // steps completed before this batch
  int rel;                     // step index within the batch
  uint32_t l2pf;               // pow2 kernel: bulk-prefetch the read blocks of the CTA this many
                               // CTAs ahead into L2 (0 = off)
  // Single-copy (AA) propagation, read == write: 0 = two copies (the reference T2C scheme);
  // 1 = the step from the natural state (gather from x - e_i, scatter to x + e_i);
  // 2 = the step from the swapped state (own node only: read slot opp(i), write slot i).
  int aa;
  uint64_t pdl_min_threads;  // programmatic dependent launch from this grid size on
  int x2;  // f32 power-of-two BGK step: two nodes per thread (t2c_step_x2_kernel)
  int off32;  // every stored slot index fits 32 bits: 32-bit gather offsets (x2 kernel)
  // Slab mode, NVLink peer stores (power-of-two tile kernel only): the face layer of my top
  // plane tiles [top_begin, ...) is also stored, for the directions leaving upwards, into the
  // upper neighbour's next copy at its low halo tiles (peer_up = that copy's first halo tile);
  // likewise the bottom plane [bot_begin, bot_end) into the lower neighbour's high halo tiles.
  // Single copy (aa = 1, phase 1) in slab p2p mode: stored tiles below halo_lo_end are the lower
  // neighbour's top-plane tiles (peer_down = its first one), tiles from halo_hi_begin on are the
  // upper neighbour's bottom-plane tiles (peer_up = its first one): read and written in place.
  double* peer_up;
  double* peer_down;
  uint64_t top_begin, bot_begin, bot_end;
  uint64_t halo_lo_end, halo_hi_begin;
  // Traversal order (power-of-two 3D kernels, whole-domain engines): the k-th stepped tile is
  // order[k] (tiling_gpu.h build_column_order); nullptr = the compact order t0 + k.
  const uint32_t* order;
  // MRT engines: the step kernel specialised for this engine's operator (a cudaKernel_t from
  // mrt_jit.cpp, launched instead of the generic MRT instantiation); nullptr = generic
  const void* jit;
};

// The MRT operator as a kernel parameter (constant bank): the unrolled K_ij * delta_j products
// read it as immediate constant operands instead of 361 loads per node.
template <class R, int Q>
struct MrtMatrix {
  R K[Q * Q];
};

}  // namespace splbm_dev
