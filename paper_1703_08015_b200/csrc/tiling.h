// Host tile map (TileGrid's tile-cover part, reference tiling.hpp:50-115).
#pragma once
#include <cstdint>
#include <vector>

namespace splbm_host {

constexpr uint32_t kEmpty = 0xffffffffu;  // kEmptyTile (tiling.hpp:16)

struct TileMap {
  int d = 2, a = 4, n_tn = 16, periodic = 0;
  int dims[3] = {0, 0, 1};
  int grid_dims[3] = {0, 0, 1};
  int padded_dims[3] = {0, 0, 1};
  uint64_t n_tiles = 0;
  std::vector<uint32_t> tile_map;    // grid cells, x fastest
  std::vector<int32_t> origins;      // T x 3
  std::vector<uint8_t> types;        // T x n_tn, x-fastest local, padding Solid
  std::vector<uint32_t> fluid_count; // T
};

// Multi-GPU slab of the tile planes [z0, z1) along the last axis (z in 3D, y in 2D), SURVEY §8e.
// Stored tiles = [low halo plane][owned planes][high halo plane], each group in compact order
// (a z-slab is a contiguous range of the z-major compact index).
struct SlabLayout {
  int axis = 2, z0 = 0, z1 = 0, zl = -1, zh = -1;
  uint64_t n_low = 0, n_own = 0, n_high = 0;
  uint64_t g_low0 = 0, g_own0 = 0, g_high0 = 0;
  uint64_t send_low_tiles = 0, send_high_tiles = 0;  // tiles of the bottom / top owned plane
  uint64_t stored() const { return n_low + n_own + n_high; }
  uint64_t global_of(uint64_t s) const {
    if (s < n_low) return g_low0 + s;
    if (s < n_low + n_own) return g_own0 + (s - n_low);
    return g_high0 + (s - n_low - n_own);
  }
  uint32_t to_local(uint32_t g) const;
};

void validate_tiling(int d, const int* dims, int a, int periodic);
std::vector<uint64_t> plane_tile_counts(const TileMap& tm);
SlabLayout slab_layout(const TileMap& tm, int z0, int z1);
// Local 27-neighbour table (global ids outside the stored set -> kEmpty) and local tile node
// types (bits 0-1 NodeType, bit 2 bc_degenerate) of the stored tiles.
void slab_tables(const TileMap& tm, const SlabLayout& sl, const std::vector<uint32_t>& nb_global,
                 const std::vector<uint8_t>& deg, std::vector<uint32_t>& nb_local,
                 std::vector<uint8_t>& types_local);
void tile_dims(int d, const int* dims, int a, int* gd, int* pd);
TileMap build_tile_map(const uint8_t* types, int d, const int* dims, int a, int periodic);
uint32_t tile_at(const TileMap& tm, int cx, int cy, int cz);
std::vector<uint32_t> neighbour_table(const TileMap& tm);
std::vector<uint8_t> degenerate_mask(const uint8_t* types, int d, const int* dims, int periodic);

}  // namespace splbm_host
