"""Tile map of the T2C path (reference proj/include/splbm/tiling.hpp:13-138, tiling.cpp:85-141).

`build_tile_grid` runs the native multithreaded builder (csrc/tiling.cpp); its output is
bit-exact with the reference (tile_map, compact order, origins, tile node types, fluid counts).
The TGB ghost-buffer topology (tiling.cpp:143-212) is not part of this path and is not built.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .geometry import Geometry

kEmptyTile = 0xFFFFFFFF  # tiling.hpp:16


@dataclass
class Periodicity:  # tiling.hpp:19-24
    x: bool = False
    y: bool = False
    z: bool = False

    def axis(self, k: int) -> bool:
        return (self.x, self.y, self.z)[k]

    def mask(self) -> int:
        return (1 if self.x else 0) | (2 if self.y else 0) | (4 if self.z else 0)

    @classmethod
    def of(cls, p) -> "Periodicity":
        if isinstance(p, Periodicity):
            return p
        if p is None:
            return cls()
        if isinstance(p, int):
            return cls(bool(p & 1), bool(p & 2), bool(p & 4))
        t = (tuple(p) + (False, False, False))[:3]
        return cls(bool(t[0]), bool(t[1]), bool(t[2]))


@dataclass
class TileGrid:  # tiling.hpp:59-115 (tile cover part)
    a: int
    d: int
    n_tn: int
    periodic: Periodicity
    geo_dims: tuple
    padded_dims: tuple
    grid_dims: tuple
    tile_map: np.ndarray          # uint32[cells], x fastest
    origins: np.ndarray           # int32[T, 3]
    types: np.ndarray             # uint8[T, n_tn], x-fastest local, padding Solid
    fluid_count: np.ndarray       # uint32[T]
    nb: np.ndarray = field(default=None)  # uint32[T, 27] (engine.hpp:446-463)

    def cell_count(self) -> int:
        return int(self.grid_dims[0]) * int(self.grid_dims[1]) * int(self.grid_dims[2])

    tile_count = cell_count

    def fluid_tile_count(self) -> int:
        return int(self.origins.shape[0])

    def cell_index(self, cx, cy, cz):
        return cx + self.grid_dims[0] * (cy + self.grid_dims[1] * cz)

    def node_offset(self, lx, ly, lz):
        return lx + self.a * (ly + self.a * lz)

    def tile_at(self, cx: int, cy: int, cz: int) -> int:  # tiling.hpp:93-102
        c = [cx, cy, cz]
        for k in range(3):
            if c[k] < 0 or c[k] >= self.grid_dims[k]:
                if not self.periodic.axis(k):
                    return kEmptyTile
                c[k] %= self.grid_dims[k]
        return int(self.tile_map[self.cell_index(*c)])


def tile_dims(d: int, dims, a: int):
    gd = np.zeros(3, np.int32)
    pd = np.zeros(3, np.int32)
    _native.check(_native.lib().splbm_tile_dims(d, np.asarray(dims, np.int32), a, gd, pd))
    return tuple(int(v) for v in gd), tuple(int(v) for v in pd)


def build_tile_grid(g: Geometry, a: int, periodic=None, with_neighbours: bool = True) -> TileGrid:
    """build_tile_grid(g, a, lat, periodic) tile cover (tiling.cpp:85-141), native + bit-exact."""
    L = _native.lib()
    per = Periodicity.of(periodic)
    dims = np.asarray(g.dims, np.int32)
    types = np.ascontiguousarray(g.types, np.uint8)
    gd, pd = tile_dims(g.d, dims, a) if a >= 2 else ((0, 0, 0), (0, 0, 0))
    T = C.c_uint64()
    _native.check(L.splbm_count_tiles(types, g.d, dims, a, per.mask(), C.byref(T)))
    T = T.value
    n_tn = a * a * (a if g.d == 3 else 1)
    ncell = gd[0] * gd[1] * gd[2]
    tile_map = np.empty(ncell, np.uint32)
    origins = np.empty(max(T, 1) * 3, np.int32)
    ttypes = np.empty(max(T, 1) * n_tn, np.uint8)
    fc = np.empty(max(T, 1), np.uint32)
    nb = np.empty(max(T, 1) * 27, np.uint32) if with_neighbours else None
    _native.check(L.splbm_build_tile_map(types, g.d, dims, a, per.mask(), tile_map, origins, ttypes,
                                         fc, _native.ptr(nb)))
    return TileGrid(a, g.d, n_tn, per, tuple(g.dims), pd, gd, tile_map,
                    origins[:3 * T].reshape(T, 3), ttypes[:T * n_tn].reshape(T, n_tn), fc[:T],
                    nb[:27 * T].reshape(T, 27) if nb is not None else None)


@dataclass
class TileStats:  # tiling.hpp:126-136 (T2C-relevant members)
    phi_t: float = 0.0
    eta_t: float = 0.0
    ratio_tiles: float = 0.0
    n_tiles: int = 0
    n_ftiles: int = 0
    # alpha_M / alpha_B describe TGB ghost buffers (tiling.cpp:229-247), not built on this path
    alpha_m: float | None = None
    alpha_b: float | None = None


def tile_stats(tg: TileGrid) -> TileStats:  # tiling.cpp:216-227
    st = TileStats(n_tiles=tg.tile_count(), n_ftiles=tg.fluid_tile_count())
    if st.n_ftiles == 0:
        return st
    fluid = int(tg.fluid_count.astype(np.uint64).sum())
    st.phi_t = float(fluid) / (float(st.n_ftiles) * tg.n_tn)
    st.eta_t = 1.0 - st.phi_t
    st.ratio_tiles = float(st.n_tiles) / float(st.n_ftiles)
    return st


def degenerate_bc_mask(g: Geometry, periodic=None) -> np.ndarray:
    """detail::degenerate_bc_mask (engine.hpp:110-140)."""
    out = np.empty(g.node_count(), np.uint8)
    _native.check(_native.lib().splbm_degenerate_bc_mask(
        np.ascontiguousarray(g.types, np.uint8), g.d, np.asarray(g.dims, np.int32),
        Periodicity.of(periodic).mask(), out))
    return out

