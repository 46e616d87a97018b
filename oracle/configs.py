"""TEST INFRASTRUCTURE ONLY: BASELINE.json config rasters built without the product package.

Used by tests/golden/make_golden_full.py and by bench.py's reference arm, which must run the
reference's own engine on the same geometry as the product arm without loading the product
library. The rasters are plain numpy, x-fastest (`geometry.hpp:41-45`); node types are the
reference's `NodeType` values (`geometry.hpp:14-19`: 0 Solid, 1 Fluid, 2 VelocityBC,
3 PressureBC).
"""
from __future__ import annotations

import hashlib

import numpy as np

SOLID, FLUID, VEL, PRES = 0, 1, 2, 3


def channel3d_raster(dims=(128, 128, 128)) -> np.ndarray:
    """BASELINE configs[1]: a duct with bounce-back walls at y, z in {0, n-1},
    a VelocityBC inlet at x = 0 and a PressureBC outlet at x = nx-1 on the non-wall cross-section.
    The reference has no 3D channel generator; its 2D `generate_channel2d` (geometry.cpp:226-245)
    uses the same wall / inlet / outlet rule in one dimension less."""
    nx, ny, nz = dims
    t = np.full((nz, ny, nx), FLUID, np.uint8)
    t[:, :, 0] = VEL
    t[:, :, nx - 1] = PRES
    t[:, 0, :] = SOLID
    t[:, ny - 1, :] = SOLID
    t[0, :, :] = SOLID
    t[nz - 1, :, :] = SOLID
    return t.ravel()


CHANNEL_BC = dict(bc_velocity=(0.05, 0.0, 0.0), bc_density=1.0)


def raster_sha(types: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(types, np.uint8).tobytes()).hexdigest()[:16]
