"""TEST INFRASTRUCTURE ONLY: ctypes front-end of the C oracle (oracle/splbm_oracle.c).

A CPU restatement of the reference T2C path, pinned against the reference itself
(oracle/_ref) and the golden digests (tests/golden/).  Only tests/, smoke() and the
bench's cpu_baseline / reference legs may use it; the product never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
_L = None

_dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u32 = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")

EMPTY = 0xFFFFFFFF
FNV_OFFSET = 1469598103934665603


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB


def lib():
    global _L
    if _L is not None:
        return _L
    if not os.path.exists(_LIB):
        build()
    L = C.CDLL(_LIB)
    L.oracle_tile_dims.argtypes = [C.c_int, _i32, C.c_int, _i32, _i32]
    L.oracle_build_tiles.argtypes = [_u8, C.c_int, _i32, C.c_int, C.c_int, _u32, _i32, _u8, _u32]
    L.oracle_build_tiles.restype = C.c_int64
    L.oracle_nb_table.argtypes = [_i32, C.c_int, _u32, _u32]
    L.oracle_degenerate_mask.argtypes = [_u8, C.c_int, _i32, C.c_int, _u8]
    L.oracle_t2c_initialize.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, _dp, _dp, _dp, _dp,
                                        _dp, _dp]
    L.oracle_t2c_step.argtypes = [C.c_int, C.c_int, C.c_int64, _u8, _u32, _u8, _dp, _dp,
                                  C.c_double, C.c_int, _dp, C.c_double, C.c_int, C.c_void_p]
    L.oracle_mrt_kernel.argtypes = [C.c_int, C.c_double, C.c_void_p, _dp]
    # host model of the product's single-copy (AA) ordering (slab-exchange tests)
    L.oracle_aa_step.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, _u8, _u32, _u8, _dp,
                                 C.c_int, C.c_double, C.c_int, _dp, C.c_double]
    L.oracle_aa_step.restype = C.c_int
    L.oracle_t2c_step.restype = C.c_int
    L.oracle_fields.argtypes = [C.c_int, C.c_int, C.c_int64, _i32, _u8, _i32, _dp, C.c_int, _dp,
                                _dp, _dp, _dp, _u8]
    L.oracle_total_mass.argtypes = [C.c_size_t, _dp, _u8]
    L.oracle_total_mass.restype = C.c_double
    L.oracle_tilemap_digest.argtypes = [C.c_size_t, _u32, C.c_int64, C.c_int, _i32, _u8]
    L.oracle_tilemap_digest.restype = C.c_uint64
    L.oracle_fields_digest.argtypes = [C.c_size_t, _u8, _dp, _dp, _dp, _dp]
    L.oracle_fields_digest.restype = C.c_uint64
    L.oracle_wavy.argtypes = [C.c_size_t, _i32, _i32, _i32, _dp, _dp, _dp, _dp]
    # TileEngineT2C<float> instance of the same restatement (oracle/t2c_real.inc)
    L.oracle_t2c_initialize_f32.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, _dp, _dp, _dp,
                                            _dp, _fp, _fp]
    L.oracle_t2c_step_f32.argtypes = [C.c_int, C.c_int, C.c_int64, _u8, _u32, _u8, _fp, _fp,
                                      C.c_float, C.c_int, _fp, C.c_float, C.c_int, C.c_void_p]
    L.oracle_t2c_step_f32.restype = C.c_int
    L.oracle_fields_f32.argtypes = [C.c_int, C.c_int, C.c_int64, _i32, _u8, _i32, _fp, C.c_int,
                                    _dp, _dp, _dp, _dp, _u8]
    _L = L
    return L


def _pmask(periodic) -> int:
    if isinstance(periodic, int):
        return periodic
    x, y, z = (tuple(periodic) + (False, False, False))[:3]
    return (1 if x else 0) | (2 if y else 0) | (4 if z else 0)


def build_tiles(types, d, dims, a, periodic=0):
    """tiling.cpp:85-141 — returns dict(grid_dims, padded_dims, tile_map, origins, types, fc)."""
    L = lib()
    dims = np.asarray(list(dims) + [1] * (3 - len(dims)), np.int32)
    gd = np.zeros(3, np.int32)
    pd = np.zeros(3, np.int32)
    L.oracle_tile_dims(d, dims, a, gd, pd)
    ncell = int(gd[0]) * int(gd[1]) * int(gd[2])
    n_tn = a * a * (a if d == 3 else 1)
    tile_map = np.empty(ncell, np.uint32)
    origins = np.empty(ncell * 3, np.int32)
    ttypes = np.empty(ncell * n_tn, np.uint8)
    fc = np.empty(ncell, np.uint32)
    T = L.oracle_build_tiles(np.ascontiguousarray(types, np.uint8), d, dims, a, _pmask(periodic),
                             tile_map, origins, ttypes, fc)
    if T < 0:
        raise ValueError("oracle: invalid tiling configuration")
    return dict(grid_dims=tuple(int(v) for v in gd), padded_dims=tuple(int(v) for v in pd),
                n_tn=n_tn, tile_map=tile_map, origins=origins[:3 * T].reshape(T, 3).copy(),
                types=ttypes[:T * n_tn].reshape(T, n_tn).copy(), fluid_count=fc[:T].copy())


def nb_table(grid_dims, periodic, tile_map, T):
    nb = np.full(max(T, 1) * 27, EMPTY, np.uint32)
    lib().oracle_nb_table(np.asarray(grid_dims, np.int32), _pmask(periodic), tile_map, nb)
    return nb[:T * 27].reshape(T, 27)


def degenerate_mask(types, d, dims, periodic=0):
    dims = np.asarray(list(dims) + [1] * (3 - len(dims)), np.int32)
    out = np.empty(int(np.prod(dims)), np.uint8)
    lib().oracle_degenerate_mask(np.ascontiguousarray(types, np.uint8), d, dims,
                                 _pmask(periodic), out)
    return out


def tilemap_digest(tiles) -> int:
    T = tiles["origins"].shape[0]
    return lib().oracle_tilemap_digest(tiles["tile_map"].size, tiles["tile_map"], T,
                                       tiles["n_tn"],
                                       np.ascontiguousarray(tiles["origins"]).ravel(),
                                       np.ascontiguousarray(tiles["types"]).ravel())


def fields_digest(f) -> int:
    return lib().oracle_fields_digest(f["rho"].size, f["mask"], f["rho"], f["ux"], f["uy"],
                                      f["uz"])


def wavy(x, y, z):
    """wavy_init (tests/test_util.hpp:39-46) on integer coordinate arrays, via glibc."""
    x = np.ascontiguousarray(x, np.int32).ravel()
    y = np.ascontiguousarray(y, np.int32).ravel()
    z = np.ascontiguousarray(z, np.int32).ravel()
    n = x.size
    out = [np.empty(n) for _ in range(4)]
    lib().oracle_wavy(n, x, y, z, *out)
    return out


def mrt_kernel(d, tau, rates=None):
    """K = M^-1 S M of CollisionOperator (collision.cpp:86-113), restated in C."""
    q = 9 if d == 2 else 19
    out = np.empty(q * q)
    r = None if rates is None else np.ascontiguousarray(rates, np.float64)
    lib().oracle_mrt_kernel(d, tau, None if r is None else r.ctypes.data, out)
    return out.reshape(q, q)


def tile_node_coords(origins, a, d):
    """node_coords(tile, p) for every tile node (engine.hpp:401-407) -> x, y, z [T*n_tn]."""
    n_tn = a * a * (a if d == 3 else 1)
    p = np.arange(n_tn)
    lx, ly, lz = p % a, (p // a) % a, p // (a * a)
    x = (origins[:, 0:1] + lx[None, :]).ravel()
    y = (origins[:, 1:2] + ly[None, :]).ravel()
    z = (origins[:, 2:3] + lz[None, :]).ravel()
    return x.astype(np.int32), y.astype(np.int32), z.astype(np.int32)


class OracleT2C:
    """TileEngineT2C<T> restated in C (engine.hpp:311-551), BGK or MRT; T = double, or float
    with precision="f32" (constants, BC values, 1/tau and the MRT operator rounded to float as
    the reference's T(...) casts do, collision.cpp:93, 108-111; engine.hpp:54-63)."""

    def __init__(self, types, d, dims, a=4, tau=0.8, incompressible=False, periodic=0,
                 bc_velocity=(0.0, 0.0, 0.0), bc_density=1.0, threads=1, mrt=False,
                 mrt_rates=None, precision="f64"):
        if not tau > 0.5:
            raise ValueError("relaxation time tau must be > 0.5")
        self.d, self.a = d, a
        self.dims = tuple(list(dims) + [1] * (3 - len(dims)))
        self.q = 9 if d == 2 else 19
        self.periodic = _pmask(periodic)
        self.incompressible = int(bool(incompressible))
        self.f32 = precision == "f32"
        self.dtype = np.float32 if self.f32 else np.float64
        self.inv_tau = 1.0 / tau
        self.bc_u = np.asarray(bc_velocity, self.dtype)
        self.bc_rho = float(bc_density)
        self.threads = threads
        self.K = (np.ascontiguousarray(mrt_kernel(d, tau, mrt_rates)).ravel().astype(self.dtype)
                  if mrt else None)
        self.tiles = build_tiles(types, d, self.dims, a, self.periodic)
        self.T = self.tiles["origins"].shape[0]
        self.n_tn = self.tiles["n_tn"]
        self.nb = np.ascontiguousarray(nb_table(self.tiles["grid_dims"], self.periodic,
                                                self.tiles["tile_map"], self.T)).ravel()
        deg = degenerate_mask(types, d, self.dims, self.periodic)
        x, y, z = tile_node_coords(self.tiles["origins"], a, d)
        inside = (x < self.dims[0]) & (y < self.dims[1]) & (z < self.dims[2])
        idx = np.where(inside, x + self.dims[0] * (y + self.dims[1] * z), 0)
        self.bcdeg = np.where(inside, deg[idx], 0).astype(np.uint8)
        self.ttypes = np.ascontiguousarray(self.tiles["types"]).ravel()
        n = self.T * self.q * self.n_tn
        self.pdf = [np.zeros(max(n, 1), self.dtype), np.zeros(max(n, 1), self.dtype)]
        self.read = 0
        self.step_count = 0

    def node_coords(self):
        return tile_node_coords(self.tiles["origins"], self.a, self.d)

    def initialize_arrays(self, rho, ux, uy, uz):
        c = lambda v: np.ascontiguousarray(v, np.float64).ravel()
        fn = lib().oracle_t2c_initialize_f32 if self.f32 else lib().oracle_t2c_initialize
        fn(self.d, self.T, self.n_tn, self.incompressible, c(rho), c(ux), c(uy), c(uz),
           self.pdf[0], self.pdf[1])
        self.read = 0
        self.step_count = 0

    def initialize_uniform(self, rho=1.0, u=(0.0, 0.0, 0.0)):
        n = self.T * self.n_tn
        self.initialize_arrays(np.full(n, rho), np.full(n, u[0]), np.full(n, u[1]),
                               np.full(n, u[2]))

    def initialize_wavy(self):
        self.initialize_arrays(*wavy(*self.node_coords()))

    def step(self, n=1):
        """Returns (ok, failed_step) like the C-ABI."""
        for _ in range(n):
            fn = lib().oracle_t2c_step_f32 if self.f32 else lib().oracle_t2c_step
            # the f32 arguments are rounded by ctypes' c_float: T(1.0 / tau), T(bc.density)
            ok = fn(self.d, self.a, self.T, self.ttypes, self.nb, self.bcdeg, self.pdf[self.read],
                    self.pdf[1 - self.read], self.inv_tau, self.incompressible, self.bc_u,
                    self.bc_rho, self.threads, None if self.K is None else self.K.ctypes.data)
            self.read = 1 - self.read
            self.step_count += 1
            if not ok:
                return False, self.step_count
        return True, 0

    def current_pdf(self):
        return self.pdf[self.read][: self.T * self.q * self.n_tn]

    def fields(self):
        n = self.dims[0] * self.dims[1] * self.dims[2]
        rho, ux, uy, uz = (np.empty(n) for _ in range(4))
        mask = np.empty(n, np.uint8)
        fn = lib().oracle_fields_f32 if self.f32 else lib().oracle_fields
        rc = fn(self.d, self.a, self.T,
                                 np.ascontiguousarray(self.tiles["origins"]).ravel(), self.ttypes,
                                 np.asarray(self.dims, np.int32), self.pdf[self.read],
                                 self.incompressible, rho, ux, uy, uz, mask)
        if rc != 0:
            raise ZeroDivisionError("moments: zero density under the quasi-compressible model")
        mass = lib().oracle_total_mass(n, rho, mask)
        return dict(rho=rho, ux=ux, uy=uy, uz=uz, mask=mask, mass=mass)
