// GPU tile builder (tiling_gpu.cu): the host builder's outputs for a whole-domain engine.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace splbm_dev {

struct TileBuildOut {
  uint64_t n_tiles = 0, fluid_nodes = 0;
  uint32_t* tile_map = nullptr;     // [C] compact tile index or kEmptyTile, cells x fastest
  uint32_t* cell_of = nullptr;      // [T] cell index of each tile
  uint32_t* fluid_count = nullptr;  // [T]
  uint8_t* types = nullptr;         // [T * n_tn] NodeType, x-fastest local, padding Solid
  uint8_t* types_bc = nullptr;      // [T * n_tn] NodeType | bc_degenerate << 2 (node_info input)
  uint32_t* nb = nullptr;           // [T * 27] (3D) / [T * 9] (2D, the dz = 0 slice)
};

// `types` is the device raster (x fastest). Synchronises `st`; on error nothing stays allocated.
cudaError_t build_tiles_device(const uint8_t* types, int d, const int dims[3], int a, int periodic,
                               const int grid_dims[3], cudaStream_t st, TileBuildOut* out);
void free_tile_build(TileBuildOut* o);

// Step traversal order for domains whose tile planes outgrow L2: the non-empty tiles listed column
// by column — (x, y) columns of BX x BY cells, each walked z-major (then y, then x) — so a tile's
// +-z neighbours are stepped one column-plane (BX*BY cells) apart instead of one full plane. The
// PDF layout keeps the reference's compact order; only the CTA -> tile mapping changes.
cudaError_t build_column_order(const uint32_t* tile_map, const int grid_dims[3], int BX, int BY,
                               uint64_t n_tiles, uint32_t* order, cudaStream_t st);

}  // namespace splbm_dev
