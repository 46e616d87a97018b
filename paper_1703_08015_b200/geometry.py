"""Geometry raster, generators and file formats (reference proj/include/splbm/geometry.hpp:14-82).

The generators and formats run natively (csrc/geometry.cpp); the raster is a numpy uint8 array
indexed x + nx*(y + ny*z), exactly the reference layout (geometry.hpp:41-45).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConfigError


class NodeType(enum.IntEnum):  # geometry.hpp:14
    Solid = 0
    Fluid = 1
    VelocityBC = 2
    PressureBC = 3


def is_solid(t) -> bool:
    return int(t) == NodeType.Solid


@dataclass
class BcParams:  # geometry.hpp:18-21
    velocity: tuple = (0.0, 0.0, 0.0)
    density: float = 1.0


@dataclass
class Geometry:  # geometry.hpp:27-51
    d: int = 2
    dims: tuple = (0, 0, 1)
    types: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    bc: BcParams = field(default_factory=BcParams)

    @classmethod
    def filled(cls, d: int, dims, fill: int = NodeType.Fluid) -> "Geometry":
        """Geometry(d, dims): every node Fluid, like the reference constructor (geometry.hpp:32-34)."""
        dims = tuple(int(v) for v in (list(dims) + [1] * (3 - len(dims)))[:3])
        return cls(d, dims, np.full(dims[0] * dims[1] * dims[2], int(fill), np.uint8), BcParams())

    def node_count(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])

    def index(self, x, y, z=0):
        return x + self.dims[0] * (y + self.dims[1] * z)

    def at(self, x, y, z=0) -> int:
        return int(self.types[self.index(x, y, z)])

    def set(self, x, y, z=0, t: int = NodeType.Fluid) -> None:
        self.types[self.index(x, y, z)] = int(t)

    def view3d(self) -> np.ndarray:
        """The raster as a [z, y, x] array view."""
        return self.types.reshape(self.dims[2], self.dims[1], self.dims[0])

    def solid_count(self) -> int:
        return int(np.count_nonzero(self.types == 0))

    def fluid_count(self) -> int:  # non-solid (fluid and boundary) nodes
        return self.node_count() - self.solid_count()

    def copy(self) -> "Geometry":
        return Geometry(self.d, tuple(self.dims), self.types.copy(),
                        BcParams(tuple(self.bc.velocity), self.bc.density))


@dataclass
class Porosity:
    phi: float
    eta: float


def porosity(g: Geometry) -> Porosity:  # geometry.cpp:336-340
    n = float(g.node_count())
    s = float(g.solid_count())
    return Porosity((n - s) / n, s / n)


class GeometryKind(enum.IntEnum):  # geometry.hpp:68 (+ two kinds the BASELINE configs need)
    Cavity2D = 0
    Cavity3D = 1
    Channel2D = 2
    Ras3D = 3
    Channel3D = 4  # new: 3D duct
    Vessel2D = 5   # new: seeded 2D vessel tree


@dataclass
class GenerateParams:  # geometry.hpp:70-78
    dims: tuple = (0, 0, 1)
    lid_speed: float = 0.05
    inlet_speed: float = 0.05
    outlet_density: float = 1.0
    sphere_diameter: int = 40
    target_porosity: float = 0.9
    seed: int = 0


def generate(kind: GeometryKind, p: GenerateParams, device: int | None = None) -> Geometry:
    """generate() (geometry.cpp:370-382); deterministic for a fixed seed. `device` runs the RAS
    sphere loop on that CUDA device (splbm_generate_device; the same raster bit for bit)."""
    L = _native.lib()
    kind = GeometryKind(kind)
    dims = [int(v) for v in (list(p.dims) + [1, 1, 1])[:3]]
    if kind in (GeometryKind.Cavity2D, GeometryKind.Channel2D, GeometryKind.Vessel2D):
        dims[2] = 1
    if min(dims) <= 0:
        raise ConfigError("dimensions must be positive")
    cp = _native.GenerateParams((C.c_int * 3)(*dims), p.lid_speed, p.inlet_speed,
                                p.outlet_density, int(p.sphere_diameter), p.target_porosity,
                                int(p.seed))
    types = np.empty(dims[0] * dims[1] * dims[2], np.uint8)
    d = C.c_int()
    vel = np.zeros(3)
    rho = C.c_double()
    if device is None:
        _native.check(L.splbm_generate(int(kind), C.byref(cp), types, C.byref(d), vel, C.byref(rho)))
    else:
        _native.check(L.splbm_generate_device(int(kind), C.byref(cp), int(device), types,
                                              C.byref(d), vel, C.byref(rho)))
    return Geometry(d.value, tuple(dims), types, BcParams(tuple(float(v) for v in vel), rho.value))


class GeometryFormat(enum.IntEnum):  # geometry.hpp:59
    Text = 0
    Binary = 1


def load_geometry_file(path: str) -> Geometry:
    """Detects SPLB v1 binary vs text (geometry.cpp:347-355)."""
    L = _native.lib()
    d = C.c_int()
    dims = np.zeros(3, np.int32)
    vel = np.zeros(3)
    rho = C.c_double()
    _native.check(L.splbm_geometry_load(path.encode(), C.byref(d), dims, None, vel, C.byref(rho)))
    types = np.empty(int(np.prod(dims)), np.uint8)
    _native.check(L.splbm_geometry_load(path.encode(), C.byref(d), dims,
                                        types.ctypes.data_as(C.c_void_p), vel, C.byref(rho)))
    return Geometry(d.value, tuple(int(v) for v in dims), types,
                    BcParams(tuple(float(v) for v in vel), rho.value))


def save_geometry_file(g: Geometry, path: str, fmt: GeometryFormat = GeometryFormat.Binary) -> None:
    L = _native.lib()
    _native.check(L.splbm_geometry_save(path.encode(), int(fmt == GeometryFormat.Binary), g.d,
                                        np.asarray(g.dims, np.int32),
                                        np.ascontiguousarray(g.types, np.uint8),
                                        np.asarray(g.bc.velocity, np.float64), g.bc.density))
