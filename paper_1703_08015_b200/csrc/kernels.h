// Launch interface between the host runtime (engine.cpp) and the sm_100a kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "lattice.cuh"
#include "step_args.h"

namespace splbm_dev {

struct NodeInfoArgs {
  const uint8_t* types;  // stored tiles x n_tn: bits 0-1 NodeType, bit 2 bc_degenerate
  const uint32_t* nb;
  uint32_t* info;
  uint64_t n_stored;
  int a;
  int sector;  // PDF slots per 32-B sector (4 doubles, 8 floats): the zero-fill group
};

struct InitArgs {
  void* pdf0;
  void* pdf1;
  const double* rho;  // nullptr -> uniform (rho0, u0)
  const double* ux;
  const double* uy;
  const double* uz;
  double rho0;
  double u0[3];
  uint64_t node0, count;
  int n_tn;
  int* domain_error;
};

// Where the post-collision value S[x][i] of the current state lives (single copy):
// two-copy / natural state -> slot (t, i, p); swapped state (after an odd number of AA steps) ->
// the slot the natural-state gather of direction opp(i) reads (x + e_i, or own slot i if blocked).
struct StateView {
  const uint32_t* nb;  // stored tiles x 27 (3D) / 9 (2D); only read when swapped
  int a;
  int swapped;
};

// FieldData frame (engine.hpp:516-534) written on the device: moments of stored tiles
// [tile0, tile0 + n_tiles) scattered to raster order, relative to raster node `base`. The frame
// slice must be zero-filled beforehand; solid and padding nodes are left untouched.
struct FrameArgs {
  const void* pdf;
  const uint32_t* info;
  StateView view;
  const uint32_t* cells;  // cell index (cx + gx (cy + gy cz)) of stored tile tile0 + i
  uint64_t tile0, n_tiles;
  int n_tn, a;
  int gx, gy;
  int dims[3];
  uint64_t base;
  double* rho;
  double* ux;
  double* uy;
  double* uz;
  uint8_t* mask;
  int* domain_error;
};

struct ReduceArgs {
  const void* pdf;
  const uint32_t* info;
  StateView view;
  uint64_t node0, n_nodes;
  int n_tn;
  double* partial;  // 3 per block
};

struct HaloArgs {
  double* pdf;
  double* buf;
  uint64_t tile0, n_tiles;
  int a;
  int layer;  // local coordinate along the slab axis of the face layer
  int n_dirs;
  const int* dirs;  // device array of direction indices
  int pack;         // 1: pdf -> buf, 0: buf -> pdf
  // unpack only: when set, a slot (x, dir) is written only if x is non-solid and x's gather of
  // opp(dir) is not blocked (the single-copy backward exchange: the downstream node x + e_dir
  // exists and is non-solid, so the neighbour's scatter wrote it)
  const uint32_t* info;
};

// Resident multi-step batch (small whole-domain two-copy BGK engines): one cooperative grid of
// `blocks` (<= kResidentMaxCtas) CTAs x `threads` (tiles_per_cta whole tiles each) runs `nsteps`
// steps from copy rd0; between steps each CTA waits for the CTAs owning its neighbour tiles
// (per-CTA epoch flags). StepArgs::read/write are unused (pdf0/pdf1 alternate).
constexpr int kResidentMaxCtas = 512;
struct ResidentArgs {
  StepArgs s;
  void* pdf0;
  void* pdf1;
  int rd0;
  int nsteps;
  int tiles_per_cta;
  unsigned* flags;  // blocks x 32 words: CTA c's step epoch at flags[32 c]; zero at creation
  unsigned epoch0;  // resident steps completed before this launch (engine counter)
};
cudaError_t launch_resident(int d, bool inc, bool f32, const ResidentArgs& a, unsigned blocks,
                            unsigned threads, cudaStream_t st);
// cudaSuccess when `per_sm` CTAs of `threads` threads of the resident kernel fit an SM.
cudaError_t resident_fits(int d, bool inc, bool f32, unsigned threads, unsigned per_sm = 1);
cudaError_t launch_step(int d, bool inc, bool f32, const StepArgs& a, cudaStream_t st);
cudaError_t launch_bump(long long* step_base, long long by, cudaStream_t st);
// Slab p2p: wait (system-scope acquire polling) until the non-null flags reach seq.
cudaError_t launch_wait_flags(const unsigned long long* f0, const unsigned long long* f1,
                              unsigned long long seq, cudaStream_t st);
cudaError_t launch_node_info(int d, const NodeInfoArgs& a, cudaStream_t st);
cudaError_t launch_init(int d, bool inc, bool f32, const InitArgs& a, cudaStream_t st);
cudaError_t launch_frame(int d, bool inc, bool f32, const FrameArgs& a, cudaStream_t st);
cudaError_t launch_reduce(int d, bool inc, bool f32, const ReduceArgs& a, int blocks, double* out,
                          cudaStream_t st);
cudaError_t launch_halo(int d, const HaloArgs& a, cudaStream_t st);
// Natural-layout copy of tiles [tile0, tile0 + n_tiles) of a (possibly swapped) state into out.
cudaError_t launch_unswap(int d, bool f32, const void* pdf, const uint32_t* info, StateView v,
                          int n_tn, uint64_t tile0, uint64_t n_tiles, void* out, cudaStream_t st);
cudaError_t launch_divide_selftest(uint64_t n, const double* m, const double* rho, double* out,
                                   cudaStream_t st);
cudaError_t launch_divide_selftest_f32(uint64_t n, const float* m, const float* rho, float* out,
                                       cudaStream_t st);

}  // namespace splbm_dev
