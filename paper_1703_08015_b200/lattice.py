"""Lattice constants and fluid model (reference proj/include/splbm/lattice.hpp:16-63,
proj/src/lattice.cpp:8-90). The device kernels bake the same constants (csrc/lattice.cuh)."""
from __future__ import annotations

import enum
from dataclasses import dataclass, field


class Arrangement(enum.IntEnum):
    D2Q9 = 0
    D3Q19 = 1
    D3Q27 = 2  # cost accounting only (lattice.hpp:47-48)


_E = {
    Arrangement.D2Q9: [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (1, 1, 0),
                       (-1, -1, 0), (1, -1, 0), (-1, 1, 0)],
    Arrangement.D3Q19: [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1),
                        (0, 0, -1), (1, 1, 0), (-1, -1, 0), (1, -1, 0), (-1, 1, 0), (1, 0, 1),
                        (-1, 0, -1), (1, 0, -1), (-1, 0, 1), (0, 1, 1), (0, -1, -1), (0, 1, -1),
                        (0, -1, 1)],
}
_E[Arrangement.D3Q27] = _E[Arrangement.D3Q19] + [
    (1, 1, 1), (-1, -1, -1), (1, 1, -1), (-1, -1, 1), (1, -1, 1), (-1, 1, -1), (1, -1, -1),
    (-1, 1, 1)]


@dataclass(frozen=True)
class LatticeDescriptor:  # lattice.hpp:22-45
    arrangement: Arrangement
    d: int
    q: int
    e: tuple
    w: tuple
    opposite: tuple
    q_s: int
    q_d: int
    q_t: int
    c_s2: float = 1.0 / 3.0

    def crossings(self, i: int) -> int:
        return sum(1 for v in self.e[i] if v != 0)


def _build(arr: Arrangement) -> LatticeDescriptor:
    e = tuple(_E[arr])
    q = len(e)
    if arr == Arrangement.D2Q9:
        d, w, qs, qd, qt = 2, [4.0 / 9.0] + [1.0 / 9.0] * 4 + [1.0 / 36.0] * 4, 4, 4, 0
    elif arr == Arrangement.D3Q19:
        d, w, qs, qd, qt = 3, [1.0 / 3.0] + [1.0 / 18.0] * 6 + [1.0 / 36.0] * 12, 6, 12, 0
    else:
        d, w, qs, qd, qt = (3, [8.0 / 27.0] + [2.0 / 27.0] * 6 + [1.0 / 54.0] * 12 +
                            [1.0 / 216.0] * 8, 6, 12, 8)
    opp = tuple(next(j for j in range(q) if e[j] == tuple(-v for v in e[i])) for i in range(q))
    return LatticeDescriptor(arr, d, q, e, tuple(w), opp, qs, qd, qt)


_CACHE = {a: _build(a) for a in Arrangement}


def lattice_descriptor(arr: Arrangement) -> LatticeDescriptor:
    return _CACHE[Arrangement(arr)]


def mrt_kernel(d: int, tau: float, rates=None):
    """The MRT operator matrix K (q x q) the device applies (splbm_mrt_kernel)."""
    import numpy as np
    from . import _native
    q = 9 if d == 2 else 19
    out = np.empty(q * q)
    r = None if rates is None else np.ascontiguousarray(rates, np.float64)
    _native.check(_native.lib().splbm_mrt_kernel(d, float(tau), None if r is None else r.ctypes.data, out))
    return out.reshape(q, q)


def solver_lattice(d: int) -> LatticeDescriptor:  # engine.hpp:104-106
    return lattice_descriptor(Arrangement.D2Q9 if d == 2 else Arrangement.D3Q19)


class Compressibility(enum.IntEnum):  # lattice.hpp:53
    QuasiCompressible = 0
    Incompressible = 1


class CollisionKind(enum.IntEnum):  # lattice.hpp:54
    BGK = 0
    MRT = 1  # K = M^-1 S M (collision.cpp:86-113), SURVEY f4


@dataclass
class FluidModel:  # lattice.hpp:56-63
    compressibility: Compressibility = Compressibility.QuasiCompressible
    collision: CollisionKind = CollisionKind.BGK
    tau: float = 1.0
    mrt_rates: list = field(default_factory=list)

    def viscosity(self) -> float:
        return (self.tau - 0.5) / 3.0
