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

void validate_tiling(int d, const int* dims, int a, int periodic);
void tile_dims(int d, const int* dims, int a, int* gd, int* pd);
TileMap build_tile_map(const uint8_t* types, int d, const int* dims, int a, int periodic);
uint32_t tile_at(const TileMap& tm, int cx, int cy, int cz);
std::vector<uint32_t> neighbour_table(const TileMap& tm);
std::vector<uint8_t> degenerate_mask(const uint8_t* types, int d, const int* dims, int periodic);

}  // namespace splbm_host
