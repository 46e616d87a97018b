// Tile cover, neighbour table and BC-degenerate flags built on the GPU (the tile
// builder for 1024^3). Produces exactly the host builder's outputs (tiling.cpp build_tile_map,
// neighbour_table, degenerate_mask + slab_tables for the whole-domain case), which follow the
// reference: uniform a^d cover from node (0,0,0), solid padding, tiles with fluid_count == 0
// dropped, compact index in cz -> cy -> cx order (reference tiling.cpp:85-141), neighbours by
// tile_at with periodic wrap (tiling.hpp:93-102, engine.hpp:446-463), degenerate BC nodes as in
// engine.hpp:110-140. The compaction is an exclusive scan over the cell flags, so the order is the
// host loop's order.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <cstdint>

#include "lattice.cuh"
#include "tiling_gpu.h"

namespace splbm_dev {

namespace {

constexpr uint32_t kEmptyTile = 0xffffffffu;

struct Grid {
  int d, a, az, n_tn, periodic;
  int dims[3];
  int gd[3];
};

__device__ __forceinline__ uint64_t raster(const Grid& g, int x, int y, int z) {
  return static_cast<uint64_t>(x) + static_cast<uint64_t>(g.dims[0]) * (y + static_cast<uint64_t>(g.dims[1]) * z);
}

// Non-solid nodes per cell (one thread per cell; a warp reads 32 adjacent cells' rows) and the
// non-empty flag; the block's fluid total goes to *fluid.
__global__ void cell_count_kernel(Grid g, const uint8_t* types, uint32_t* counts, uint32_t* flags,
                                  unsigned long long* fluid) {
  const uint64_t C = static_cast<uint64_t>(g.gd[0]) * g.gd[1] * g.gd[2];
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t n = 0;
  if (c < C) {
    const int cx = static_cast<int>(c % g.gd[0]);
    const int cy = static_cast<int>((c / g.gd[0]) % g.gd[1]);
    const int cz = static_cast<int>(c / (static_cast<uint64_t>(g.gd[0]) * g.gd[1]));
    const int x0 = cx * g.a, x1 = min(x0 + g.a, g.dims[0]);
    for (int lz = 0; lz < g.az; ++lz) {
      const int z = cz * g.az + lz;
      if (z >= g.dims[2]) break;
      for (int ly = 0; ly < g.a; ++ly) {
        const int y = cy * g.a + ly;
        if (y >= g.dims[1]) break;
        const uint8_t* row = types + raster(g, 0, y, z);
        for (int x = x0; x < x1; ++x) n += row[x] != 0;
      }
    }
    counts[c] = n;
    flags[c] = n > 0;
  }
  const unsigned s = __reduce_add_sync(0xffffffffu, n);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(fluid, static_cast<unsigned long long>(s));
}

__global__ void tile_map_kernel(uint64_t C, const uint32_t* counts, const uint32_t* flags,
                                const uint32_t* idx, uint32_t* tile_map, uint32_t* cell_of,
                                uint32_t* fluid_count) {
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= C) return;
  if (flags[c]) {
    const uint32_t t = idx[c];
    tile_map[c] = t;
    cell_of[t] = static_cast<uint32_t>(c);
    fluid_count[t] = counts[c];
  } else {
    tile_map[c] = kEmptyTile;
  }
}

// Per tile node: the NodeType (padding Solid) and, for BC nodes, bc_degenerate (any upstream
// neighbour x - e_i solid, or outside a non-periodic edge; engine.hpp:110-140) in bit 2.
template <int D>
__global__ void tile_types_kernel(Grid g, const uint8_t* types, const uint32_t* cell_of, uint64_t T,
                                  uint8_t* tile_types, uint8_t* tile_types_bc) {
  const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= T * g.n_tn) return;
  const uint64_t t = k / g.n_tn;
  const int p = static_cast<int>(k % g.n_tn);
  const uint32_t c = cell_of[t];
  const int x = static_cast<int>(c % g.gd[0]) * g.a + p % g.a;
  const int y = static_cast<int>((c / g.gd[0]) % g.gd[1]) * g.a + (p / g.a) % g.a;
  const int z = D == 3 ? static_cast<int>(c / (static_cast<uint32_t>(g.gd[0]) * g.gd[1])) * g.a + p / (g.a * g.a) : 0;
  uint8_t ty = 0;
  if (x < g.dims[0] && y < g.dims[1] && z < g.dims[2]) ty = types[raster(g, x, y, z)];
  uint8_t bc = ty;
  if (ty == 2 || ty == 3) {
    bool degenerate = false;
    for (int i = 1; i < Lat<D>::Q && !degenerate; ++i) {
      int s[3] = {x - ex<D>(i), y - ey<D>(i), z - ez<D>(i)};
      bool outside = false;
      for (int a = 0; a < 3; ++a) {
        if (s[a] < 0 || s[a] >= g.dims[a]) {
          if ((g.periodic >> a) & 1) {
            s[a] = ((s[a] % g.dims[a]) + g.dims[a]) % g.dims[a];
          } else {
            outside = true;
            break;
          }
        }
      }
      degenerate = outside || types[raster(g, s[0], s[1], s[2])] == 0;
    }
    if (degenerate) bc |= 4;
  }
  tile_types[k] = ty;
  tile_types_bc[k] = bc;
}

// nb[t][k]: tile_at(c + (dx, dy, dz)); 3D keeps all 27 (k = (dx+1) + 3(dy+1) + 9(dz+1)), 2D the
// dz = 0 slice (9 entries), the engine's device layouts.
__global__ void neighbour_kernel(Grid g, const uint32_t* tile_map, const uint32_t* cell_of, uint64_t T,
                                 uint32_t* nb) {
  const int nbs = g.d == 3 ? 27 : 9;
  const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= T * nbs) return;
  const uint64_t t = k / nbs;
  const int j = static_cast<int>(k % nbs) + (g.d == 3 ? 0 : 9);
  const uint32_t c = cell_of[t];
  int cc[3] = {static_cast<int>(c % g.gd[0]) + j % 3 - 1,
               static_cast<int>((c / g.gd[0]) % g.gd[1]) + (j / 3) % 3 - 1,
               static_cast<int>(c / (static_cast<uint32_t>(g.gd[0]) * g.gd[1])) + j / 9 - 1};
  uint32_t r = 0;
  bool empty = false;
  for (int a = 0; a < 3; ++a) {
    if (cc[a] < 0 || cc[a] >= g.gd[a]) {
      if (!((g.periodic >> a) & 1)) {
        empty = true;
        break;
      }
      cc[a] = ((cc[a] % g.gd[a]) + g.gd[a]) % g.gd[a];
    }
  }
  if (empty) {
    r = kEmptyTile;
  } else {
    r = tile_map[static_cast<uint64_t>(cc[0]) + static_cast<uint64_t>(g.gd[0]) * (cc[1] + static_cast<uint64_t>(g.gd[1]) * cc[2])];
  }
  nb[k] = r;
}

unsigned blocks_for(uint64_t n, unsigned threads) { return static_cast<unsigned>((n + threads - 1) / threads); }

// Cell of position j of the block-column traversal: columns of BX x BY cells in (x, y) (the last
// ones ragged), column-major over (by, bx), inside a column z-major, then y, then x. BX = gx gives
// row bands (each (band, plane) piece is one contiguous run of the compact order).
__device__ __forceinline__ uint64_t column_cell(uint64_t j, const int* gd, int BX, int BY) {
  const uint64_t gx = gd[0], gy = gd[1], gz = gd[2];
  const uint64_t full_rows = gy / BY;  // column rows of height BY (the last one may be shorter)
  const uint64_t row_cells = gx * static_cast<uint64_t>(BY) * gz;
  uint64_t br = j / row_cells;
  if (br > full_rows) br = full_rows;
  uint64_t r = j - br * row_cells;
  const uint64_t h = (br < full_rows) ? static_cast<uint64_t>(BY) : gy - full_rows * BY;
  // inside a column row: columns bx of width BX (the last one ragged), each BX * h * gz cells
  const uint64_t col_cells = static_cast<uint64_t>(BX) * h * gz;
  uint64_t bx = r / col_cells;
  const uint64_t full_cols = gx / BX;
  if (bx > full_cols) bx = full_cols;
  r -= bx * col_cells;
  const uint64_t w = (bx < full_cols) ? static_cast<uint64_t>(BX) : gx - full_cols * BX;
  const uint64_t cz = r / (w * h);
  const uint64_t rr = r % (w * h);
  const uint64_t cy = br * BY + rr / w;
  const uint64_t cx = bx * BX + rr % w;
  return cx + gx * (cy + gy * cz);
}

__global__ void column_flags_kernel(uint64_t C, Grid g, int BX, int BY, const uint32_t* tile_map, uint32_t* flags) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= C) return;
  flags[j] = tile_map[column_cell(j, g.gd, BX, BY)] != kEmptyTile;
}

__global__ void column_order_kernel(uint64_t C, Grid g, int BX, int BY, const uint32_t* tile_map,
                                    const uint32_t* pos, uint32_t* order) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= C) return;
  const uint32_t t = tile_map[column_cell(j, g.gd, BX, BY)];
  if (t != kEmptyTile) order[pos[j]] = t;
}

}  // namespace

cudaError_t build_column_order(const uint32_t* tile_map, const int grid_dims[3], int BX, int BY,
                               uint64_t n_tiles, uint32_t* order, cudaStream_t st) {
  Grid g{};
  for (int k = 0; k < 3; ++k) g.gd[k] = grid_dims[k];
  const uint64_t C = static_cast<uint64_t>(g.gd[0]) * g.gd[1] * g.gd[2];
  if (!C || !n_tiles) return cudaSuccess;
  uint32_t *flags = nullptr, *pos = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  cudaError_t err = cudaSuccess;
  auto ok = [&](cudaError_t e) {
    if (err == cudaSuccess) err = e;
    return err == cudaSuccess;
  };
  do {
    if (!ok(cudaMalloc(&flags, C * 4)) || !ok(cudaMalloc(&pos, C * 4))) break;
    column_flags_kernel<<<blocks_for(C, 256), 256, 0, st>>>(C, g, BX, BY, tile_map, flags);
    if (!ok(cudaGetLastError())) break;
    if (!ok(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, flags, pos, static_cast<int>(C), st))) break;
    if (!ok(cudaMalloc(&temp, temp_bytes))) break;
    if (!ok(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, flags, pos, static_cast<int>(C), st))) break;
    column_order_kernel<<<blocks_for(C, 256), 256, 0, st>>>(C, g, BX, BY, tile_map, pos, order);
    if (!ok(cudaGetLastError())) break;
    ok(cudaStreamSynchronize(st));
  } while (false);
  for (void* p : {static_cast<void*>(flags), static_cast<void*>(pos), temp})
    if (p) cudaFree(p);
  return err;
}

void free_tile_build(TileBuildOut* o) {
  for (void* p : {static_cast<void*>(o->tile_map), static_cast<void*>(o->cell_of),
                  static_cast<void*>(o->fluid_count), static_cast<void*>(o->types),
                  static_cast<void*>(o->types_bc), static_cast<void*>(o->nb)})
    if (p) cudaFree(p);
  *o = TileBuildOut{};
}

cudaError_t build_tiles_device(const uint8_t* types, int d, const int dims[3], int a, int periodic,
                               const int grid_dims[3], cudaStream_t st, TileBuildOut* out) {
  *out = TileBuildOut{};
  Grid g{};
  g.d = d;
  g.a = a;
  g.az = d == 3 ? a : 1;
  g.n_tn = a * a * g.az;
  g.periodic = periodic;
  for (int k = 0; k < 3; ++k) {
    g.dims[k] = dims[k];
    g.gd[k] = grid_dims[k];
  }
  const uint64_t C = static_cast<uint64_t>(g.gd[0]) * g.gd[1] * g.gd[2];
  if (C >= kEmptyTile) return cudaErrorInvalidValue;  // 32-bit cell and tile indices
  uint32_t *counts = nullptr, *flags = nullptr, *idx = nullptr;
  unsigned long long* fluid = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  cudaError_t err = cudaSuccess;
  auto ok = [&](cudaError_t e) {
    if (err == cudaSuccess) err = e;
    return err == cudaSuccess;
  };
  uint32_t tail[2] = {0, 0};
  unsigned long long fluid_h = 0;
  do {
    if (!ok(cudaMalloc(&counts, C * 4)) || !ok(cudaMalloc(&flags, C * 4)) || !ok(cudaMalloc(&idx, C * 4)) ||
        !ok(cudaMalloc(&fluid, 8)) || !ok(cudaMalloc(&out->tile_map, C * 4)))
      break;
    if (!ok(cudaMemsetAsync(fluid, 0, 8, st))) break;
    cell_count_kernel<<<blocks_for(C, 256), 256, 0, st>>>(g, types, counts, flags, fluid);
    if (!ok(cudaGetLastError())) break;
    if (!ok(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, flags, idx, static_cast<int>(C), st))) break;
    if (!ok(cudaMalloc(&temp, temp_bytes))) break;
    if (!ok(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, flags, idx, static_cast<int>(C), st))) break;
    if (!ok(cudaMemcpyAsync(&tail[0], idx + C - 1, 4, cudaMemcpyDeviceToHost, st)) ||
        !ok(cudaMemcpyAsync(&tail[1], flags + C - 1, 4, cudaMemcpyDeviceToHost, st)) ||
        !ok(cudaMemcpyAsync(&fluid_h, fluid, 8, cudaMemcpyDeviceToHost, st)) || !ok(cudaStreamSynchronize(st)))
      break;
    const uint64_t T = static_cast<uint64_t>(tail[0]) + tail[1];
    out->n_tiles = T;
    out->fluid_nodes = fluid_h;
    const uint64_t Tn = T ? T : 1;
    const int nbs = d == 3 ? 27 : 9;
    if (!ok(cudaMalloc(&out->cell_of, Tn * 4)) || !ok(cudaMalloc(&out->fluid_count, Tn * 4)) ||
        !ok(cudaMalloc(&out->types, Tn * g.n_tn)) || !ok(cudaMalloc(&out->types_bc, Tn * g.n_tn)) ||
        !ok(cudaMalloc(&out->nb, Tn * nbs * 4)))
      break;
    tile_map_kernel<<<blocks_for(C, 256), 256, 0, st>>>(C, counts, flags, idx, out->tile_map, out->cell_of,
                                                       out->fluid_count);
    if (!ok(cudaGetLastError())) break;
    if (T) {
      if (d == 3)
        tile_types_kernel<3><<<blocks_for(T * g.n_tn, 256), 256, 0, st>>>(g, types, out->cell_of, T, out->types,
                                                                          out->types_bc);
      else
        tile_types_kernel<2><<<blocks_for(T * g.n_tn, 256), 256, 0, st>>>(g, types, out->cell_of, T, out->types,
                                                                          out->types_bc);
      if (!ok(cudaGetLastError())) break;
      neighbour_kernel<<<blocks_for(T * nbs, 256), 256, 0, st>>>(g, out->tile_map, out->cell_of, T, out->nb);
      if (!ok(cudaGetLastError())) break;
    }
    ok(cudaStreamSynchronize(st));
  } while (false);
  for (void* p : {static_cast<void*>(counts), static_cast<void*>(flags), static_cast<void*>(idx),
                  static_cast<void*>(fluid), temp})
    if (p) cudaFree(p);
  if (err != cudaSuccess) free_tile_build(out);
  return err;
}

}  // namespace splbm_dev
