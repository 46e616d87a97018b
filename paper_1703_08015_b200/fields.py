"""Macroscopic fields (reference proj/include/splbm/fields.hpp:12-61)."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class FieldData:  # fields.hpp:12-43
    d: int = 2
    dims: tuple = (0, 0, 1)
    mask: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))  # 1 = non-solid
    rho: np.ndarray = field(default_factory=lambda: np.zeros(0))
    ux: np.ndarray = field(default_factory=lambda: np.zeros(0))
    uy: np.ndarray = field(default_factory=lambda: np.zeros(0))
    uz: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def size(self) -> int:
        return int(self.rho.size)

    def index(self, x, y, z=0):
        return x + self.dims[0] * (y + self.dims[1] * z)

    def total_mass(self) -> float:
        """Sequential sum in raster order, like fields.hpp:25-31 (ufunc.accumulate is sequential)."""
        vals = self.rho[self.mask != 0]
        return float(np.add.accumulate(vals)[-1]) if vals.size else 0.0

    def all_finite(self) -> bool:  # fields.hpp:33-42
        m = self.mask != 0
        return bool(np.all(np.isfinite(self.rho[m])) and np.all(np.isfinite(self.ux[m])) and
                    np.all(np.isfinite(self.uy[m])) and np.all(np.isfinite(self.uz[m])))


def linf_rel_diff(a: FieldData, b: FieldData) -> float:
    """Largest per-field deviation over non-solid nodes of a, relative to the field's global
    magnitude (fields.hpp:47-61)."""
    m = a.mask != 0
    worst = 0.0
    for fa, fb in ((a.rho, b.rho), (a.ux, b.ux), (a.uy, b.uy), (a.uz, b.uz)):
        xa, xb = fa[m], fb[m]
        # std::max(x, NaN) keeps x (the comparison is false), so NaN entries never raise scale or
        # diff; np.fmax skips NaN the same way.
        scale = float(np.fmax.reduce(np.abs(np.concatenate([xa, xb])), initial=0.0))
        diff = float(np.fmax.reduce(np.abs(xa - xb), initial=0.0))
        if scale > 0.0:
            worst = max(worst, diff / scale)
    return worst
