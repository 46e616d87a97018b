"""The device T2C engine and the simulation driver (reference proj/include/splbm/engine.hpp).

`TileEngineT2C` keeps the reference `Engine<T>` surface (engine.hpp:67-92) — initialize,
initialize_uniform, step, fields, padded_dims, tile_visits, current_step — and runs every step
as the fused sm_100a kernel through the C ABI (include/splbm_b200.h). There is no CPU path:
constructing an engine without the native library or a CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _native
from .errors import ConfigError, NumericalError
from .fields import FieldData
from .geometry import Geometry
from .lattice import CollisionKind, Compressibility, FluidModel
from .tiling import Periodicity, TileGrid


class Method(enum.IntEnum):  # engine.hpp:20
    Dense = 0
    T2C = 1
    TGB = 2


# NodeInit (engine.hpp:22), vectorised: f(x, y, z) on int arrays -> (rho, ux, uy, uz) arrays
NodeInit = Callable[[np.ndarray, np.ndarray, np.ndarray], tuple]
SnapshotSink = Callable[[int, FieldData, tuple], None]


class TileEngineT2C:
    """TileEngineT2C<double> (engine.hpp:311-551) on one B200.

    Constructor mirrors `TileEngineT2C(const Geometry&, int a, const FluidModel&, Periodicity)`
    (engine.hpp:314-315); `device` selects the GPU, `slab=(z0, z1)` the owned tile planes of
    the multi-GPU slab mode, `single_copy=True` the in-place AA propagation (one PDF
    array instead of two, bit-identical results) and `precision="f32"` the
    TileEngineT2C<float> instantiation (the reference CLI's precision=f32, tools/splbm.cpp:278).
    `arithmetic="fma"` is the opt-in tolerance mode (libsplbm_b200_fma.so: contracted
    multiply-adds and a reciprocal velocity division, like the reference built with
    -march=native; within 1e-13 per step and 1e-10 after 1000 steps of the bit-exact default,
    tests/test_device_fma.py).
    """

    def __init__(self, g: Geometry, a: int, model: FluidModel, periodic=None, device: int = 0,
                 slab: tuple | None = None, single_copy: bool = False, precision: str = "f64",
                 arithmetic: str = "exact"):
        if precision not in ("f64", "f32"):
            raise ConfigError("precision must be f32 or f64")
        L = _native.lib(arithmetic)
        q = 9 if g.d == 2 else 19
        rates = None
        if model.collision == CollisionKind.MRT and model.mrt_rates:
            if len(model.mrt_rates) != q:  # collision.cpp:100-103
                raise ConfigError(f"mrt_rates must have one entry per moment ({q})")
            rates = np.ascontiguousarray(model.mrt_rates, np.float64)
        per = Periodicity.of(periodic)
        types = np.ascontiguousarray(g.types, np.uint8)
        desc = _native.DevDesc()
        desc.d = g.d
        desc.dims = (C.c_int * 3)(*[int(v) for v in g.dims])
        desc.types = types.ctypes.data_as(C.c_void_p)
        desc.bc_velocity = (C.c_double * 3)(*[float(v) for v in g.bc.velocity])
        desc.bc_density = float(g.bc.density)
        desc.tile = int(a)
        desc.tau = float(model.tau)
        desc.incompressible = int(model.compressibility == Compressibility.Incompressible)
        desc.periodic = per.mask()
        desc.device = int(device)
        desc.slab_z0, desc.slab_z1 = (int(slab[0]), int(slab[1])) if slab else (0, 0)
        desc.collision = int(model.collision)
        desc.mrt_rates = rates.ctypes.data_as(C.c_void_p) if rates is not None else None
        desc.single_copy = int(bool(single_copy))
        desc.single_precision = int(precision == "f32")
        h = C.c_void_p()
        _native.check(L.splbm_dev_create(C.byref(desc), C.byref(h)), lib_=L)
        self._h = h
        self._L = L
        self.arithmetic = arithmetic
        self.geometry_dims = tuple(int(v) for v in g.dims)
        self.d = g.d
        self.model = model
        self.periodic = per
        self.single_copy = bool(single_copy)
        self.precision = precision
        self.dtype = np.float32 if precision == "f32" else np.float64
        info = _native.DevInfo()
        _native.check(L.splbm_dev_get_info(h, C.byref(info)), lib_=L)
        self.info = info
        self.a = info.a
        self.q = info.q
        self.n_tn = info.n_tn
        self._grid = None

    def _chk(self, rc: int, step: int | None = None) -> None:
        _native.check(rc, step, lib_=self._L)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.splbm_dev_destroy(h)
            self._h = None

    # ---- tile grid --------------------------------------------------------------------------
    def tile_grid(self) -> TileGrid:
        if self._grid is None:
            gd = tuple(self.info.grid_dims)
            T = int(np.prod(gd))
            L = self._L
            tile_map = np.empty(T, np.uint32)
            self._chk(L.splbm_dev_get_tile_grid(self._h, _native.ptr(tile_map), None, None,
                                                    None, None))
            nt = int(self.info.n_tiles_global)
            origins = np.empty(max(nt, 1) * 3, np.int32)
            types = np.empty(max(nt, 1) * self.n_tn, np.uint8)
            fc = np.empty(max(nt, 1), np.uint32)
            nb = np.empty(max(nt, 1) * 27, np.uint32)
            self._chk(L.splbm_dev_get_tile_grid(self._h, None, _native.ptr(origins),
                                                    _native.ptr(types), _native.ptr(fc),
                                                    _native.ptr(nb)))
            self._grid = TileGrid(self.a, self.d, self.n_tn, self.periodic, self.geometry_dims,
                                  tuple(self.info.padded_dims), gd, tile_map,
                                  origins[:3 * nt].reshape(nt, 3),
                                  types[:nt * self.n_tn].reshape(nt, self.n_tn), fc[:nt],
                                  nb[:27 * nt].reshape(nt, 27))
        return self._grid

    def stored_tiles(self) -> np.ndarray:
        out = np.empty(max(int(self.info.n_tiles_stored), 1), np.uint64)
        self._chk(self._L.splbm_dev_stored_tiles(self._h, out))
        return out[: int(self.info.n_tiles_stored)]

    def node_coords(self):
        """node_coords(tile, p) of every stored tile node (engine.hpp:401-407), int32 arrays."""
        tg = self.tile_grid()
        o = tg.origins[self.stored_tiles().astype(np.int64)]
        a = self.a
        p = np.arange(self.n_tn)
        lx, ly, lz = p % a, (p // a) % a, p // (a * a)
        x = (o[:, 0:1] + lx[None, :]).ravel().astype(np.int32)
        y = (o[:, 1:2] + ly[None, :]).ravel().astype(np.int32)
        z = (o[:, 2:3] + lz[None, :]).ravel().astype(np.int32)
        return x, y, z

    # ---- Engine<T> ----------------------------------------------------------------------------
    def initialize(self, init: NodeInit) -> None:
        """Engine::initialize (engine.hpp:336-352): NodeInit at every stored tile node's
        coordinates (solid and padding nodes included), equilibrium computed on the device."""
        x, y, z = self.node_coords()
        rho, ux, uy, uz = init(x, y, z)
        n = x.size
        arr = [np.ascontiguousarray(np.broadcast_to(np.asarray(v, np.float64), (n,)))
               for v in (rho, ux, uy, uz)]
        self.initialize_arrays(*arr)

    def initialize_arrays(self, rho, ux, uy, uz) -> None:
        """NodeInit values at every stored tile node (node_coords() order), one array per moment;
        the C side copies n_tiles_stored * n_tn doubles from each."""
        n = int(self.info.n_tiles_stored) * self.n_tn
        c = lambda v: np.ascontiguousarray(v, np.float64).ravel()
        arrs = [c(v) for v in (rho, ux, uy, uz)]
        if any(a.size != n for a in arrs):
            raise ConfigError(f"initialize_arrays needs {n} values per moment "
                              f"(got {[a.size for a in arrs]})")
        self._chk(self._L.splbm_dev_initialize(self._h, *arrs))

    def initialize_uniform(self, rho0: float = 1.0, u0=(0.0, 0.0, 0.0)) -> None:  # engine.hpp:72-75
        self._chk(self._L.splbm_dev_initialize_uniform(self._h, float(rho0),
                                                           np.asarray(u0, np.float64)))

    def step(self) -> bool:
        """Advances one iteration; False when a non-finite moment appeared (engine.hpp:79-80)."""
        ok, _ = self.step_n(1)
        return ok

    def step_n(self, n: int) -> tuple[bool, int]:
        """n steps in one device batch; (ok, first failing step number or 0)."""
        ok = C.c_int()
        fs = C.c_long()
        self._chk(self._L.splbm_dev_step(self._h, int(n), C.byref(ok), C.byref(fs)))
        return bool(ok.value), int(fs.value)

    def step_async(self, n: int) -> None:
        self._chk(self._L.splbm_dev_step_async(self._h, int(n)))

    def sync(self) -> tuple[bool, int]:
        ok = C.c_int()
        fs = C.c_long()
        self._chk(self._L.splbm_dev_sync(self._h, C.byref(ok), C.byref(fs)))
        return bool(ok.value), int(fs.value)

    def last_batch_ms(self) -> float:
        ms = C.c_float()
        self._chk(self._L.splbm_dev_last_batch_ms(self._h, C.byref(ms)))
        return float(ms.value)

    def fields(self, with_mass: bool = False, out: FieldData | None = None):
        """Engine::fields (engine.hpp:371-390): moments of the current post-collision copy.
        `out` (optional) supplies the destination arrays, e.g. page-locked host buffers."""
        nx, ny, nz = self.geometry_dims
        n = nx * ny * nz
        if out is not None:
            rho, ux, uy, uz, mask = out.rho, out.ux, out.uy, out.uz, out.mask
            if any(a.size != n or not a.flags.c_contiguous for a in (rho, ux, uy, uz, mask)):
                raise ConfigError("fields(out=...) arrays must be contiguous raster-sized")
            if any(a.dtype != np.float64 for a in (rho, ux, uy, uz)) or mask.dtype != np.uint8:
                raise ConfigError("fields(out=...) needs float64 rho/ux/uy/uz and a uint8 mask")
        else:
            rho, ux, uy, uz = (np.empty(n) for _ in range(4))
            mask = np.empty(n, np.uint8)
        mass = C.c_double()  # the sequential host mass sum only when asked for
        self._chk(self._L.splbm_dev_fields(self._h, _native.ptr(rho), _native.ptr(ux),
                                               _native.ptr(uy), _native.ptr(uz),
                                               _native.ptr(mask), C.byref(mass) if with_mass else None))
        f = FieldData(self.d, self.geometry_dims, mask, rho, ux, uy, uz)
        return (f, mass.value) if with_mass else f

    def reduce(self) -> dict:
        out = np.zeros(3)
        self._chk(self._L.splbm_dev_reduce(self._h, out))
        return {"mass": float(out[0]), "max_speed": float(out[1]), "non_finite": int(out[2])}

    def padded_dims(self) -> tuple:
        out = np.zeros(3, np.int32)
        self._chk(self._L.splbm_dev_padded_dims(self._h, out))
        return tuple(int(v) for v in out)

    def tile_visits(self) -> int:
        return int(self._L.splbm_dev_tile_visits(self._h))

    def current_step(self) -> int:
        return int(self._L.splbm_dev_current_step(self._h))

    def launch_count(self) -> int:
        return int(self._L.splbm_dev_launch_count(self._h))

    def fluid_nodes(self) -> int:
        return int(self.info.fluid_nodes)

    # ---- parity / plumbing ------------------------------------------------------------------
    def get_pdf(self) -> np.ndarray:
        out = np.empty(int(self.info.n_tiles_stored) * self.q * self.n_tn, self.dtype)
        self._chk(self._L.splbm_dev_get_pdf(self._h, _native.ptr(out)))
        return out

    def set_pdf(self, f: np.ndarray) -> None:
        f = np.ascontiguousarray(f, self.dtype)
        if f.size != int(self.info.n_tiles_stored) * self.q * self.n_tn:
            raise ConfigError("PDF array has the wrong size")
        self._chk(self._L.splbm_dev_set_pdf(self._h, _native.ptr(f)))

    def stream_handle(self) -> int:
        return int(self._L.splbm_dev_stream(self._h) or 0)

    def halo_bytes(self) -> dict:
        a, b, c, d = (C.c_uint64() for _ in range(4))
        self._chk(self._L.splbm_dev_halo_bytes(self._h, C.byref(a), C.byref(b)))
        self._chk(self._L.splbm_dev_halo_recv_bytes(self._h, C.byref(c), C.byref(d)))
        return {"send_low": a.value, "send_high": b.value, "recv_low": c.value,
                "recv_high": d.value}

    def halo_pack(self, low_ptr: int, high_ptr: int) -> None:
        self._chk(self._L.splbm_dev_halo_pack(self._h, low_ptr or None, high_ptr or None))

    def comm_attach(self, uid: bytes, world: int, rank: int, lower: int | None,
                    upper: int | None) -> None:
        """Native NCCL halo exchange for the slab mode (splbm_dev_comm_attach)."""
        buf = C.create_string_buffer(bytes(uid), 128)
        self._chk(self._L.splbm_dev_comm_attach(self._h, buf, int(world), int(rank),
                                                    -1 if lower is None else int(lower),
                                                    -1 if upper is None else int(upper)))

    def ipc_blob(self) -> bytes:
        """What a slab neighbour needs to store faces into this engine (splbm_dev_ipc_blob)."""
        buf = C.create_string_buffer(512)
        self._chk(self._L.splbm_dev_ipc_blob(self._h, buf))
        return buf.raw

    def p2p_attach(self, lower_blob: bytes | None, upper_blob: bytes | None) -> None:
        """Fused NVLink peer-store halo exchange with the slab neighbours (splbm_dev_p2p_attach)."""
        lo = C.create_string_buffer(bytes(lower_blob), 512) if lower_blob else None
        hi = C.create_string_buffer(bytes(upper_blob), 512) if upper_blob else None
        self._chk(self._L.splbm_dev_p2p_attach(self._h, lo, hi))

    @staticmethod
    def comm_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _native.check(_native.lib().splbm_comm_unique_id(buf))
        return buf.raw

    def step_part(self, part: int) -> None:
        self._chk(self._L.splbm_dev_step_part(self._h, int(part)))

    def halo_pack_next(self, low_ptr: int, high_ptr: int) -> None:
        self._chk(self._L.splbm_dev_halo_pack_next(self._h, low_ptr or None, high_ptr or None))

    def halo_unpack(self, low_ptr: int, high_ptr: int) -> None:
        self._chk(self._L.splbm_dev_halo_unpack(self._h, low_ptr or None, high_ptr or None))

    def halo_pack_back(self, low_ptr: int, high_ptr: int) -> None:
        """Single copy, after a step from the natural layout: the halo slots the scatter wrote
        (splbm_dev_halo_pack_back)."""
        self._chk(self._L.splbm_dev_halo_pack_back(self._h, low_ptr or None, high_ptr or None))

    def halo_unpack_back(self, low_ptr: int, high_ptr: int) -> None:
        self._chk(self._L.splbm_dev_halo_unpack_back(self._h, low_ptr or None, high_ptr or None))


# ---- driver (engine.hpp:562-655) --------------------------------------------------------------
@dataclass
class SimConfig:  # engine.hpp:562-576
    method: Method = Method.T2C
    tile: int = 0  # 0 selects 16 for 2D, 4 for 3D
    steps: int = 0
    snapshot_every: int = 0
    threads: int = 1  # host threads of the reference pool; unused by the device engine
    periodic: Periodicity = field(default_factory=Periodicity)
    model: FluidModel = field(default_factory=FluidModel)
    initial_density: float = 1.0
    initial_velocity: tuple = (0.0, 0.0, 0.0)
    init: NodeInit | None = None
    snapshot_sink: SnapshotSink | None = None
    device: int = 0
    single_copy: bool = False  # device extension: in-place AA propagation
    arithmetic: str = "exact"  # device extension: "fma" = the tolerance-mode build

    def tile_edge(self, d: int) -> int:
        return self.tile if self.tile > 0 else (16 if d == 2 else 4)


@dataclass
class SimulationResult:  # engine.hpp:578-591
    steps: int = 0
    wall_seconds: float = 0.0
    mlups: float = 0.0
    mass_initial: float = 0.0
    mass_final: float = 0.0
    mass_drift_rel: float = 0.0
    tile_visits: int = 0
    fluid_nodes: int = 0
    fluid_tiles: int = 0
    snapshots_written: int = 0
    padded_dims: tuple = (0, 0, 1)
    fields: FieldData | None = None


def make_engine(g: Geometry, cfg: SimConfig, precision: str = "f64") -> TileEngineT2C:
    """make_engine<T> (engine.hpp:593-607); precision "f64"/"f32" selects T = double/float."""
    if cfg.method != Method.T2C:
        raise ConfigError("the B200 path implements Method::T2C; Dense/TGB stay on the reference")
    return TileEngineT2C(g, cfg.tile_edge(g.d), cfg.model, cfg.periodic, device=cfg.device,
                         single_copy=cfg.single_copy, precision=precision,
                         arithmetic=cfg.arithmetic)


def run_simulation(g: Geometry, cfg: SimConfig, precision: str = "f64") -> SimulationResult:
    """run_simulation<T> (engine.hpp:609-655) on the device engine; precision "f64"/"f32" is the
    template argument T = double/float (the CLI's sim.precision, tools/splbm.cpp:278).

    Steps run in device batches (one batch, or one per snapshot interval); wall time is the
    device time of the batches (CUDA events on the engine stream); a failing batch raises
    NumericalError with the first failing step number, as the reference does (engine.hpp:634).
    """
    if cfg.steps < 0:
        raise ConfigError("steps must be non-negative")
    eng = make_engine(g, cfg, precision)
    if cfg.init is not None:
        eng.initialize(cfg.init)
    else:
        eng.initialize_uniform(cfg.initial_density, cfg.initial_velocity)
    res = SimulationResult(fluid_nodes=g.fluid_count(), padded_dims=eng.padded_dims(),
                           fluid_tiles=int(eng.info.n_tiles))
    f0, m0 = eng.fields(with_mass=True)
    res.mass_initial = m0
    if cfg.steps == 0:
        res.fields = f0
    wall = 0.0
    done = 0
    every = cfg.snapshot_every if (cfg.snapshot_every > 0 and cfg.snapshot_sink) else cfg.steps
    while done < cfg.steps:
        n = min(every, cfg.steps - done) if every > 0 else cfg.steps
        eng.step_async(n)
        ok, failed = eng.sync()
        wall += eng.last_batch_ms() * 1e-3
        if not ok:
            raise NumericalError("non-finite density or velocity", failed)
        done += n
        if cfg.snapshot_sink and cfg.snapshot_every > 0 and done % cfg.snapshot_every == 0:
            cfg.snapshot_sink(done, eng.fields(), eng.padded_dims())
            res.snapshots_written += 1
    res.steps = cfg.steps
    res.wall_seconds = wall
    res.mlups = (res.fluid_nodes * cfg.steps / (wall * 1e6)) if (cfg.steps > 0 and wall > 0) else 0.0
    if cfg.steps > 0:
        res.fields, res.mass_final = eng.fields(with_mass=True)
    else:
        res.mass_final = m0
    res.mass_drift_rel = (abs(res.mass_final - res.mass_initial) / abs(res.mass_initial)
                          if res.mass_initial != 0.0 else 0.0)
    res.tile_visits = eng.tile_visits()
    return res
