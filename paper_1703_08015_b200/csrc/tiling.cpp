// Integer tile-map builder (host, multithreaded over tile planes), bit-exact with the
// reference's build_tile_grid tile-cover pass (tiling.cpp:85-141), its tile_at wrap rule
// (tiling.hpp:93-102), the T2C 27-neighbour table (engine.hpp:446-463) and the degenerate
// boundary mask (engine.hpp:110-140). The ghost-buffer topology of the TGB scheme
// (tiling.cpp:143-212) is not needed by this path and is not built.
#include <cstring>
#include <numeric>

#include "common.h"
#include "tiling.h"

namespace splbm_host {

static const int kE2[9][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},
                              {1, 1, 0},  {-1, -1, 0}, {1, -1, 0}, {-1, 1, 0}};
static const int kE3[19][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0},  {0, 1, 0},  {0, -1, 0},
                               {0, 0, 1},  {0, 0, -1},  {1, 1, 0},   {-1, -1, 0}, {1, -1, 0},
                               {-1, 1, 0}, {1, 0, 1},   {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
                               {0, 1, 1},  {0, -1, -1}, {0, 1, -1},  {0, -1, 1}};

void validate_tiling(int d, const int* dims, int a, int periodic) {
  if (d != 2 && d != 3) throw config_error("dimension must be 2 or 3");
  for (int k = 0; k < 3; ++k)
    if (dims[k] <= 0) throw config_error("dimensions must be positive");
  if (d == 2 && dims[2] != 1) throw config_error("2D geometry requires nz = 1");
  if (a < 2) throw config_error("tile edge must be at least 2");  // tiling.cpp:87
  for (int k = 0; k < d; ++k)                                        // tiling.cpp:89-93
    if (((periodic >> k) & 1) && dims[k] % a != 0)
      throw config_error("periodic axes require dimensions divisible by the tile edge");
}

void tile_dims(int d, const int* dims, int a, int* gd, int* pd) {
  for (int k = 0; k < 3; ++k) {  // tiling.cpp:103-108
    const int extent = (k == 2 && d == 2) ? 1 : dims[k];
    const int te = (k == 2 && d == 2) ? 1 : a;
    gd[k] = (extent + te - 1) / te;
    pd[k] = gd[k] * te;
  }
}

// Per-cell non-solid counts; planes in parallel.
static std::vector<uint32_t> cell_fluid_counts(const uint8_t* types, int d, const int* dims, int a,
                                               const int* gd) {
  const int az = d == 3 ? a : 1;
  std::vector<uint32_t> fc(static_cast<std::size_t>(gd[0]) * gd[1] * gd[2], 0);
  parallel_for(static_cast<std::size_t>(gd[2]) * gd[1], [&](std::size_t b, std::size_t e) {
    for (std::size_t row = b; row < e; ++row) {
      const int cy = static_cast<int>(row % gd[1]), cz = static_cast<int>(row / gd[1]);
      for (int lz = 0; lz < az; ++lz) {
        const int z = cz * az + lz;
        if (z >= dims[2]) break;
        for (int ly = 0; ly < a; ++ly) {
          const int y = cy * a + ly;
          if (y >= dims[1]) break;
          const uint8_t* rowp = types + raster_index(dims, 0, y, z);
          uint32_t* out = fc.data() + row * gd[0];
          for (int x = 0; x < dims[0]; ++x) out[x / a] += rowp[x] != 0;
        }
      }
    }
  });
  return fc;
}

TileMap build_tile_map(const uint8_t* types, int d, const int* dims, int a, int periodic) {
  validate_tiling(d, dims, a, periodic);
  TileMap tm;
  tm.d = d;
  tm.a = a;
  tm.periodic = periodic;
  for (int k = 0; k < 3; ++k) tm.dims[k] = dims[k];
  tile_dims(d, dims, a, tm.grid_dims, tm.padded_dims);
  tm.n_tn = a * a * (d == 3 ? a : 1);
  const std::vector<uint32_t> fc = cell_fluid_counts(types, d, dims, a, tm.grid_dims);
  // compact index in cz -> cy -> cx order (tiling.cpp:113-141)
  const std::size_t C = fc.size();
  tm.tile_map.resize(C);
  uint64_t T = 0;
  for (std::size_t c = 0; c < C; ++c) tm.tile_map[c] = fc[c] > 0 ? static_cast<uint32_t>(T++) : kEmpty;
  if (T >= kEmpty) throw config_error("too many non-empty tiles for 32-bit tile indices");
  tm.n_tiles = T;
  tm.origins.resize(T * 3);
  tm.fluid_count.resize(T);
  tm.types.assign(T * tm.n_tn, 0);  // padding is Solid
  const int az = d == 3 ? a : 1;
  const int* gd = tm.grid_dims;
  parallel_for(C, [&](std::size_t b, std::size_t e) {
    for (std::size_t c = b; c < e; ++c) {
      const uint32_t t = tm.tile_map[c];
      if (t == kEmpty) continue;
      const int cx = static_cast<int>(c % gd[0]);
      const int cy = static_cast<int>((c / gd[0]) % gd[1]);
      const int cz = static_cast<int>(c / (static_cast<std::size_t>(gd[0]) * gd[1]));
      const int o[3] = {cx * a, cy * a, cz * az};
      for (int k = 0; k < 3; ++k) tm.origins[3 * static_cast<std::size_t>(t) + k] = o[k];
      tm.fluid_count[t] = fc[c];
      uint8_t* tt = tm.types.data() + static_cast<std::size_t>(t) * tm.n_tn;
      for (int lz = 0; lz < az; ++lz) {
        const int z = o[2] + lz;
        if (z >= dims[2]) continue;
        for (int ly = 0; ly < a; ++ly) {
          const int y = o[1] + ly;
          if (y >= dims[1]) continue;
          for (int lx = 0; lx < a; ++lx) {
            const int x = o[0] + lx;
            if (x >= dims[0]) continue;
            tt[lx + a * (ly + a * lz)] = types[raster_index(dims, x, y, z)];
          }
        }
      }
    }
  }, 4096);
  return tm;
}

uint32_t tile_at(const TileMap& tm, int cx, int cy, int cz) {  // tiling.hpp:93-102
  int c[3] = {cx, cy, cz};
  for (int k = 0; k < 3; ++k) {
    if (c[k] < 0 || c[k] >= tm.grid_dims[k]) {
      if (!((tm.periodic >> k) & 1)) return kEmpty;
      c[k] = ((c[k] % tm.grid_dims[k]) + tm.grid_dims[k]) % tm.grid_dims[k];
    }
  }
  return tm.tile_map[raster_index(tm.grid_dims, c[0], c[1], c[2])];
}

std::vector<uint32_t> neighbour_table(const TileMap& tm) {  // engine.hpp:446-463
  std::vector<uint32_t> nb(tm.n_tiles * 27, kEmpty);
  parallel_for(tm.n_tiles, [&](std::size_t b, std::size_t e) {
    for (std::size_t t = b; t < e; ++t) {
      const int* o = &tm.origins[3 * t];
      const int az = tm.d == 3 ? tm.a : 1;
      const int cx = o[0] / tm.a, cy = o[1] / tm.a, cz = o[2] / az;
      for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx)
            nb[t * 27 + (dx + 1) + 3 * ((dy + 1) + 3 * (dz + 1))] =
                tile_at(tm, cx + dx, cy + dy, cz + dz);
    }
  }, 1024);
  return nb;
}

std::vector<uint8_t> degenerate_mask(const uint8_t* types, int d, const int* dims, int periodic) {
  const int q = d == 2 ? 9 : 19;
  const int(*e)[3] = d == 2 ? kE2 : kE3;
  std::vector<uint8_t> mask(static_cast<std::size_t>(dims[0]) * dims[1] * dims[2], 0);
  parallel_for(static_cast<std::size_t>(dims[1]) * dims[2], [&](std::size_t b, std::size_t en) {
    for (std::size_t row = b; row < en; ++row) {
      const int y = static_cast<int>(row % dims[1]), z = static_cast<int>(row / dims[1]);
      for (int x = 0; x < dims[0]; ++x) {
        const uint8_t t = types[raster_index(dims, x, y, z)];
        if (t != 2 && t != 3) continue;
        bool degenerate = false;
        for (int i = 1; i < q && !degenerate; ++i) {
          int s[3] = {x - e[i][0], y - e[i][1], z - e[i][2]};
          bool outside = false;
          for (int k = 0; k < 3; ++k) {
            if (s[k] < 0 || s[k] >= dims[k]) {
              if ((periodic >> k) & 1) {
                s[k] = ((s[k] % dims[k]) + dims[k]) % dims[k];
              } else {
                outside = true;
                break;
              }
            }
          }
          degenerate = outside || types[raster_index(dims, s[0], s[1], s[2])] == 0;
        }
        if (degenerate) mask[raster_index(dims, x, y, z)] = 1;
      }
    }
  }, 64);
  return mask;
}

std::vector<uint64_t> plane_tile_counts(const TileMap& tm) {
  const int ax = tm.d == 3 ? 2 : 1;
  const int L = tm.grid_dims[ax];
  const uint64_t plane_cells = static_cast<uint64_t>(tm.grid_dims[0]) * (tm.d == 3 ? tm.grid_dims[1] : 1);
  std::vector<uint64_t> cnt(static_cast<std::size_t>(L), 0);
  for (int z = 0; z < L; ++z) {
    const uint32_t* row = tm.tile_map.data() + static_cast<uint64_t>(z) * plane_cells;
    for (uint64_t c = 0; c < plane_cells; ++c) cnt[z] += row[c] != kEmpty;
  }
  return cnt;
}

uint32_t SlabLayout::to_local(uint32_t g) const {
  if (g == kEmpty) return kEmpty;
  if (g >= g_own0 && g < g_own0 + n_own) return static_cast<uint32_t>(n_low + (g - g_own0));
  if (n_low && g >= g_low0 && g < g_low0 + n_low) return static_cast<uint32_t>(g - g_low0);
  if (n_high && g >= g_high0 && g < g_high0 + n_high)
    return static_cast<uint32_t>(n_low + n_own + (g - g_high0));
  return kEmpty;
}

SlabLayout slab_layout(const TileMap& tm, int z0, int z1) {
  SlabLayout sl;
  sl.axis = tm.d == 3 ? 2 : 1;
  const int L = tm.grid_dims[sl.axis];
  if (z0 == 0 && z1 == 0) z1 = L;
  if (z0 < 0 || z1 > L || z0 >= z1) throw config_error("invalid slab range");
  sl.z0 = z0;
  sl.z1 = z1;
  const std::vector<uint64_t> cnt = plane_tile_counts(tm);
  std::vector<uint64_t> F(static_cast<std::size_t>(L) + 1, 0);  // first compact index of plane z
  for (int z = 0; z < L; ++z) F[z + 1] = F[z] + cnt[z];
  const bool whole = (z0 == 0 && z1 == L);
  const bool per_ax = (tm.periodic >> sl.axis) & 1;
  if (!whole) {
    if (z0 > 0) sl.zl = z0 - 1; else if (per_ax) sl.zl = L - 1;
    if (z1 < L) sl.zh = z1; else if (per_ax) sl.zh = 0;
    if ((sl.zl >= z0 && sl.zl < z1) || (sl.zh >= z0 && sl.zh < z1) || (sl.zl >= 0 && sl.zl == sl.zh))
      throw config_error("slab too thick for its periodic halo planes");
  }
  sl.g_own0 = F[z0];
  sl.n_own = F[z1] - F[z0];
  sl.g_low0 = sl.zl >= 0 ? F[sl.zl] : 0;
  sl.n_low = sl.zl >= 0 ? F[sl.zl + 1] - F[sl.zl] : 0;
  sl.g_high0 = sl.zh >= 0 ? F[sl.zh] : 0;
  sl.n_high = sl.zh >= 0 ? F[sl.zh + 1] - F[sl.zh] : 0;
  sl.send_low_tiles = whole ? 0 : F[z0 + 1] - F[z0];
  sl.send_high_tiles = whole ? 0 : F[z1] - F[z1 - 1];
  return sl;
}

void slab_tables(const TileMap& tm, const SlabLayout& sl, const std::vector<uint32_t>& nb_global,
                 const std::vector<uint8_t>& deg, std::vector<uint32_t>& nb_local,
                 std::vector<uint8_t>& types_local) {
  const uint64_t S = sl.stored();
  const int n_tn = tm.n_tn, a = tm.a;
  nb_local.assign(S * 27, kEmpty);
  types_local.assign(S * n_tn, 0);
  parallel_for(S, [&](std::size_t b, std::size_t en) {
    for (std::size_t s = b; s < en; ++s) {
      const uint64_t g = sl.global_of(s);
      for (int k = 0; k < 27; ++k) nb_local[s * 27 + k] = sl.to_local(nb_global[g * 27 + k]);
      const int32_t* o = &tm.origins[3 * g];
      for (int p = 0; p < n_tn; ++p) {
        uint8_t t = tm.types[g * n_tn + p];
        if (t == 2 || t == 3) {  // bc_degenerate(t, p) (engine.hpp:409-417)
          const int x = o[0] + p % a, y = o[1] + (p / a) % a, z = o[2] + (tm.d == 3 ? p / (a * a) : 0);
          if (deg[raster_index(tm.dims, x, y, z)]) t |= 4;
        }
        types_local[s * n_tn + p] = t;
      }
    }
  }, 1024);
}

}  // namespace splbm_host

using namespace splbm_host;

extern "C" {

int splbm_tile_dims(int d, const int dims[3], int a, int grid_dims_out[3], int padded_dims_out[3]) {
  return guarded([&] {
    if (a < 2) throw config_error("tile edge must be at least 2");
    tile_dims(d, dims, a, grid_dims_out, padded_dims_out);
  });
}

int splbm_count_tiles(const uint8_t* types, int d, const int dims[3], int a, int periodic,
                      uint64_t* n_tiles_out) {
  return guarded([&] {
    validate_tiling(d, dims, a, periodic);
    int gd[3], pd[3];
    tile_dims(d, dims, a, gd, pd);
    const auto fc = cell_fluid_counts(types, d, dims, a, gd);
    uint64_t T = 0;
    for (uint32_t v : fc) T += v > 0;
    *n_tiles_out = T;
  });
}

int splbm_build_tile_map(const uint8_t* types, int d, const int dims[3], int a, int periodic,
                         uint32_t* tile_map, int32_t* origins, uint8_t* tile_types,
                         uint32_t* fluid_count, uint32_t* nb) {
  return guarded([&] {
    const TileMap tm = build_tile_map(types, d, dims, a, periodic);
    if (tile_map) std::memcpy(tile_map, tm.tile_map.data(), tm.tile_map.size() * 4);
    if (origins) std::memcpy(origins, tm.origins.data(), tm.origins.size() * 4);
    if (tile_types) std::memcpy(tile_types, tm.types.data(), tm.types.size());
    if (fluid_count) std::memcpy(fluid_count, tm.fluid_count.data(), tm.fluid_count.size() * 4);
    if (nb) {
      const auto n = neighbour_table(tm);
      std::memcpy(nb, n.data(), n.size() * 4);
    }
  });
}

int splbm_plane_tile_counts(const uint8_t* types, int d, const int dims[3], int a, int periodic,
                            uint64_t* counts_out) {
  return guarded([&] {
    const TileMap tm = build_tile_map(types, d, dims, a, periodic);
    const auto c = plane_tile_counts(tm);
    std::memcpy(counts_out, c.data(), c.size() * sizeof(uint64_t));
  });
}

int splbm_slab_layout(const uint8_t* types, int d, const int dims[3], int a, int periodic, int z0,
                      int z1, splbm_slab_layout_t* out, uint32_t* nb_local, uint8_t* types_local) {
  return guarded([&] {
    if (!out) throw config_error("null argument");
    const TileMap tm = build_tile_map(types, d, dims, a, periodic);
    const SlabLayout sl = slab_layout(tm, z0, z1);
    out->axis = sl.axis;
    out->z0 = sl.z0;
    out->z1 = sl.z1;
    out->zl = sl.zl;
    out->zh = sl.zh;
    out->n_low = sl.n_low;
    out->n_own = sl.n_own;
    out->n_high = sl.n_high;
    out->g_low0 = sl.g_low0;
    out->g_own0 = sl.g_own0;
    out->g_high0 = sl.g_high0;
    out->send_low_tiles = sl.send_low_tiles;
    out->send_high_tiles = sl.send_high_tiles;
    if (nb_local || types_local) {
      std::vector<uint32_t> nbl;
      std::vector<uint8_t> tl;
      slab_tables(tm, sl, neighbour_table(tm), degenerate_mask(types, d, dims, periodic), nbl, tl);
      if (nb_local) std::memcpy(nb_local, nbl.data(), nbl.size() * 4);
      if (types_local) std::memcpy(types_local, tl.data(), tl.size());
    }
  });
}

int splbm_degenerate_bc_mask(const uint8_t* types, int d, const int dims[3], int periodic,
                             uint8_t* mask_out) {
  return guarded([&] {
    const auto m = degenerate_mask(types, d, dims, periodic);
    std::memcpy(mask_out, m.data(), m.size());
  });
}

}  // extern "C"
