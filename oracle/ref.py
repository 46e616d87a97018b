"""TEST INFRASTRUCTURE ONLY: ctypes access to the UNMODIFIED reference solver.

`oracle/_ref/libsplbm_ref.so` is the reference C++ code (/root/reference/proj/src +
headers) compiled in place by `oracle/build_ref.sh` behind the thin C shim
`oracle/ref_capi.cpp`.  Only tests/, `__graft_entry__.smoke()` and bench.py's
reference/cpu_baseline legs may use this module — never the product.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")
_libs: dict[str, C.CDLL] = {}

KIND = {"cavity2d": 0, "cavity3d": 1, "channel2d": 2, "ras3d": 3}
METHOD = {"dense": 0, "t2c": 1, "tgb": 2}

_dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32 = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def available(fast=False) -> bool:
    return os.path.exists(_path(fast))


def _path(fast) -> str:
    """fast: False = the bitwise oracle build; True / "v3" = -march=x86-64-v3; "v4" = x86-64-v4."""
    name = {False: "libsplbm_ref.so", True: "libsplbm_ref_fast.so", "v3": "libsplbm_ref_fast.so",
            "v4": "libsplbm_ref_v4.so"}[fast]
    return os.path.join(REF_DIR, name)


def best_timing_build():
    """The highest ISA-level timing build of the reference this host can run (None = only the
    baseline-x86-64 oracle build): x86-64-v4 needs AVX-512 F/BW/CD/DQ/VL, v3 needs AVX2+FMA."""
    try:
        flags = set(open("/proc/cpuinfo").read().split())
    except OSError:
        flags = set()
    if {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"} <= flags and available("v4"):
        return "v4"
    if {"avx2", "fma", "bmi2"} <= flags and available("v3"):
        return "v3"
    return None


def lib(fast=False) -> C.CDLL:
    key = {False: "exact", True: "v3", "v3": "v3", "v4": "v4"}[fast]
    if key in _libs:
        return _libs[key]
    L = C.CDLL(_path(fast))
    vp = C.c_void_p
    L.ref_last_error.restype = C.c_char_p
    L.ref_generate.argtypes = [C.c_int] * 4 + [C.c_double] * 3 + [C.c_int, C.c_double,
                                                                    C.c_uint64, C.POINTER(vp)]
    L.ref_geometry_from_raster.argtypes = [C.c_int, _i32, _u8, _dp, C.c_double, C.POINTER(vp)]
    L.ref_geometry_load.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.ref_geometry_save.argtypes = [vp, C.c_char_p, C.c_int]
    L.ref_geometry_info.argtypes = [vp, C.POINTER(C.c_int), _i32, _dp, C.POINTER(C.c_double)]
    L.ref_geometry_types.argtypes = [vp, _u8]
    L.ref_geometry_free.argtypes = [vp]
    L.ref_tile_grid.argtypes = [vp, C.c_int, C.c_int, C.POINTER(vp)]
    L.ref_tile_grid_info.argtypes = [vp, _i32, _i32, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
    L.ref_tile_grid_arrays.argtypes = [vp, _u32, _i32, _u8, _u32]
    L.ref_tile_grid_nb.argtypes = [vp, _u32]
    L.ref_tile_stats.argtypes = [vp, _dp]
    L.ref_tile_grid_free.argtypes = [vp]
    L.ref_degenerate_mask.argtypes = [vp, C.c_int, _u8]
    L.ref_engine_create.argtypes = [vp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.POINTER(vp)]
    L.ref_engine_create_p.argtypes = [vp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                      C.c_int, C.c_int, C.POINTER(vp)]
    L.ref_engine_initialize.argtypes = [vp, C.c_int, C.c_double, _dp]
    L.ref_engine_initialize_fields.argtypes = [vp, _i32, _dp, _dp, _dp, _dp]
    L.ref_engine_step.argtypes = [vp, C.c_long, C.POINTER(C.c_int), C.POINTER(C.c_long),
                                  C.POINTER(C.c_double)]
    L.ref_engine_current_step.argtypes = [vp]
    L.ref_engine_current_step.restype = C.c_long
    L.ref_engine_tile_visits.argtypes = [vp]
    L.ref_engine_tile_visits.restype = C.c_uint64
    L.ref_engine_padded_dims.argtypes = [vp, _i32]
    L.ref_engine_fields.argtypes = [vp, _dp, _dp, _dp, _dp, _u8, C.POINTER(C.c_double)]
    L.ref_engine_pdf.argtypes = [vp, C.c_void_p]
    L.ref_engine_pdf.restype = C.c_uint64
    L.ref_engine_free.argtypes = [vp]
    L.ref_run_simulation.argtypes = [vp, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                     C.c_int, C.c_long, C.c_int, _dp, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p]
    L.ref_overhead_t2c.argtypes = [C.c_int, C.c_int] + [C.c_double] * 7 + [_dp]
    L.ref_bandwidth_utilization.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double,
                                            C.POINTER(C.c_double)]
    L.ref_hardware_threads.restype = C.c_int
    L.ref_mrt_kernel.argtypes = [C.c_int, C.c_double, C.c_void_p, C.c_int, _dp]
    _libs[key] = L
    return L


def _check(L, rc):
    if rc != 0:
        raise RefError(rc, L.ref_last_error().decode())


def per_mask(periodic) -> int:
    if isinstance(periodic, int):
        return periodic
    x, y, z = (tuple(periodic) + (False, False, False))[:3]
    return (1 if x else 0) | (2 if y else 0) | (4 if z else 0)


class RefGeometry:
    def __init__(self, handle, L):
        self._h = handle
        self._L = L

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.ref_geometry_free(self._h)
            self._h = None

    @classmethod
    def generate(cls, kind, dims, lid=0.05, inlet=0.05, outlet=1.0, diameter=40, target=0.9,
                 seed=0, fast=False):
        L = lib(fast)
        h = C.c_void_p()
        dims = list(dims) + [1] * (3 - len(dims))
        _check(L, L.ref_generate(KIND[kind], dims[0], dims[1], dims[2], lid, inlet, outlet,
                                 diameter, target, seed, C.byref(h)))
        return cls(h, L)

    @classmethod
    def from_raster(cls, d, dims, types, bc_velocity=(0.0, 0.0, 0.0), bc_density=1.0, fast=False):
        L = lib(fast)
        h = C.c_void_p()
        dims = np.asarray(list(dims) + [1] * (3 - len(dims)), np.int32)
        _check(L, L.ref_geometry_from_raster(d, dims, np.ascontiguousarray(types, np.uint8),
                                             np.asarray(bc_velocity, np.float64), bc_density,
                                             C.byref(h)))
        return cls(h, L)

    @classmethod
    def load(cls, path, fast=False):
        L = lib(fast)
        h = C.c_void_p()
        _check(L, L.ref_geometry_load(path.encode(), C.byref(h)))
        return cls(h, L)

    def save(self, path, binary=True):
        _check(self._L, self._L.ref_geometry_save(self._h, path.encode(), int(binary)))

    def info(self):
        d = C.c_int()
        dims = np.zeros(3, np.int32)
        vel = np.zeros(3)
        rho = C.c_double()
        self._L.ref_geometry_info(self._h, C.byref(d), dims, vel, C.byref(rho))
        return d.value, tuple(int(v) for v in dims), tuple(vel), rho.value

    def types(self):
        d, dims, _, _ = self.info()
        out = np.empty(dims[0] * dims[1] * dims[2], np.uint8)
        self._L.ref_geometry_types(self._h, out)
        return out


@dataclass
class RefTileGrid:
    grid_dims: tuple
    padded_dims: tuple
    n_tn: int
    tile_map: np.ndarray
    origins: np.ndarray
    types: np.ndarray
    fluid_count: np.ndarray
    nb: np.ndarray
    stats: dict


def tile_grid(geom: RefGeometry, a: int, periodic=0) -> RefTileGrid:
    L = geom._L
    h = C.c_void_p()
    _check(L, L.ref_tile_grid(geom._h, a, per_mask(periodic), C.byref(h)))
    try:
        gd = np.zeros(3, np.int32)
        pd = np.zeros(3, np.int32)
        nt = C.c_uint64()
        ntn = C.c_int()
        L.ref_tile_grid_info(h, gd, pd, C.byref(nt), C.byref(ntn))
        T, n_tn = nt.value, ntn.value
        C_ = int(gd[0]) * int(gd[1]) * int(gd[2])
        tile_map = np.empty(C_, np.uint32)
        origins = np.empty(max(T, 1) * 3, np.int32)
        types = np.empty(max(T, 1) * n_tn, np.uint8)
        fc = np.empty(max(T, 1), np.uint32)
        L.ref_tile_grid_arrays(h, tile_map, origins, types, fc)
        nb = np.empty(max(T, 1) * 27, np.uint32)
        L.ref_tile_grid_nb(h, nb)
        st = np.zeros(8)
        L.ref_tile_stats(h, st)
        keys = ["phi_t", "eta_t", "alpha_m", "alpha_b", "ratio_tiles",
                "reduced_buffer_fraction", "n_tiles", "n_ftiles"]
        return RefTileGrid(tuple(int(v) for v in gd), tuple(int(v) for v in pd), n_tn, tile_map,
                           origins[:T * 3].reshape(T, 3), types[:T * n_tn].reshape(T, n_tn),
                           fc[:T], nb[:T * 27].reshape(T, 27), dict(zip(keys, st.tolist())))
    finally:
        L.ref_tile_grid_free(h)


def degenerate_mask(geom: RefGeometry, periodic=0) -> np.ndarray:
    d, dims, _, _ = geom.info()
    out = np.empty(dims[0] * dims[1] * dims[2], np.uint8)
    geom._L.ref_degenerate_mask(geom._h, per_mask(periodic), out)
    return out


class RefEngine:
    """The reference Engine<T> (Dense/T2C/TGB) with its own ThreadPool; T = double, or float with
    precision="f32" (the reference CLI's precision=f32, tools/splbm.cpp:278)."""

    def __init__(self, geom: RefGeometry, method="t2c", a=4, tau=0.8, incompressible=False,
                 mrt=False, periodic=0, threads=1, precision="f64"):
        self._L = geom._L
        self._geom = geom
        h = C.c_void_p()
        self.dtype = np.float32 if precision == "f32" else np.float64
        _check(self._L, self._L.ref_engine_create_p(geom._h, METHOD[method], a, tau,
                                                    int(incompressible), int(mrt),
                                                    per_mask(periodic), threads,
                                                    int(precision == "f32"), C.byref(h)))
        self._h = h
        self.dims = geom.info()[1]

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.ref_engine_free(self._h)
            self._h = None

    def initialize_uniform(self, rho=1.0, u=(0.0, 0.0, 0.0)):
        _check(self._L, self._L.ref_engine_initialize(self._h, 0, rho, np.asarray(u, np.float64)))

    def initialize_wavy(self):
        _check(self._L, self._L.ref_engine_initialize(self._h, 1, 1.0, np.zeros(3)))

    def initialize_fields(self, padded_dims, rho, ux, uy, uz):
        pd = np.asarray(padded_dims, np.int32)
        c = lambda a: np.ascontiguousarray(a, np.float64).ravel()
        _check(self._L, self._L.ref_engine_initialize_fields(self._h, pd, c(rho), c(ux), c(uy),
                                                             c(uz)))

    def step(self, n=1):
        ok = C.c_int()
        fs = C.c_long()
        sec = C.c_double()
        _check(self._L, self._L.ref_engine_step(self._h, n, C.byref(ok), C.byref(fs),
                                                C.byref(sec)))
        self.last_seconds = sec.value
        return bool(ok.value), fs.value

    def current_step(self):
        return self._L.ref_engine_current_step(self._h)

    def tile_visits(self):
        return self._L.ref_engine_tile_visits(self._h)

    def padded_dims(self):
        out = np.zeros(3, np.int32)
        self._L.ref_engine_padded_dims(self._h, out)
        return tuple(int(v) for v in out)

    def fields(self):
        n = self.dims[0] * self.dims[1] * self.dims[2]
        rho, ux, uy, uz = (np.empty(n) for _ in range(4))
        mask = np.empty(n, np.uint8)
        mass = C.c_double()
        _check(self._L, self._L.ref_engine_fields(self._h, rho, ux, uy, uz, mask,
                                                  C.byref(mass)))
        return dict(rho=rho, ux=ux, uy=uy, uz=uz, mask=mask, mass=mass.value)

    def pdf(self):
        n = self._L.ref_engine_pdf(self._h, None)
        out = np.empty(n, self.dtype)
        self._L.ref_engine_pdf(self._h, out.ctypes.data)
        return out


def run_simulation(geom: RefGeometry, method="t2c", a=4, tau=0.8, incompressible=False,
                   periodic=0, threads=1, steps=0, init="uniform", want_fields=True):
    L = geom._L
    d, dims, _, _ = geom.info()
    n = dims[0] * dims[1] * dims[2]
    out = np.zeros(6)
    arrs = [np.empty(n) for _ in range(4)] if want_fields else None
    ptrs = [a_.ctypes.data for a_ in arrs] if arrs else [None] * 4
    _check(L, L.ref_run_simulation(geom._h, METHOD[method], a, tau, int(incompressible),
                                   per_mask(periodic), threads, steps,
                                   1 if init == "wavy" else 0, out, *ptrs))
    res = dict(wall_seconds=out[0], mlups=out[1], mass_initial=out[2], mass_final=out[3],
               mass_drift_rel=out[4], tile_visits=int(out[5]))
    if arrs:
        res.update(rho=arrs[0], ux=arrs[1], uy=arrs[2], uz=arrs[3])
    return res


def overhead_t2c(d, a, phi, phi_t, alpha_m=1.0, ratio_tiles=1.0, s_d=8.0, s_t=2.0, s_ti=4.0):
    L = lib()
    out = np.zeros(8)
    _check(L, L.ref_overhead_t2c(d, a, s_d, s_t, s_ti, phi, phi_t, alpha_m, ratio_tiles, out))
    keys = ["m_node", "b_node", "delta_b", "delta_b_bt", "b_node_type", "b_addressing",
            "delta_m", "predicted_perf"]
    return dict(zip(keys, out.tolist()))


def bandwidth_utilization(d, mlups, b_peak, s_d=8.0):
    L = lib()
    out = C.c_double()
    _check(L, L.ref_bandwidth_utilization(d, s_d, mlups, b_peak, C.byref(out)))
    return out.value


def mrt_kernel(d, tau, rates=None):
    """CollisionOperator<double>::kernel_ of the reference (collision.cpp:86-113)."""
    L = lib()
    q = 9 if d == 2 else 19
    out = np.empty(q * q)
    r = None if rates is None else np.ascontiguousarray(rates, np.float64)
    _check(L, L.ref_mrt_kernel(d, tau, None if r is None else r.ctypes.data,
                               0 if r is None else r.size, out))
    return out.reshape(q, q)


def hardware_threads() -> int:
    return lib().ref_hardware_threads()
