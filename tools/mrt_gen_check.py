"""Experiment check: the generated shared-product MRT collision (variants/lib_gen*.so) against the
in-tree MRT step, bitwise on every PDF slot after 50 steps (channel 48^3 and RAS 40^3, tau 0.8)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_08015_b200 as P  # noqa: E402
from paper_1703_08015_b200 import _native  # noqa: E402

geoms = {"channel": (P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(48, 40, 40))), 0),
         "ras": (P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(40, 40, 40), sphere_diameter=10,
                                                                   target_porosity=0.5, seed=3)), 7)}
base = _native.lib()
for libname in sys.argv[1:]:
    other = _native.load(os.path.join(ROOT, libname))
    for name, (g, per) in geoms.items():
        for comp in (P.Compressibility.QuasiCompressible, P.Compressibility.Incompressible):
            out = []
            for L in (base, other):
                _native._lib = L
                e = P.TileEngineT2C(g, 4, P.FluidModel(comp, collision=P.CollisionKind.MRT, tau=0.8), per)
                e.initialize(lambda x, y, z: (1.0 + 0.01 * np.sin(0.3 * x), 0.01 * np.cos(0.2 * y),
                                              0.005 * np.sin(0.1 * z), 0.0))
                assert e.step_n(50)[0]
                out.append(e.get_pdf().view(np.uint64).copy())
            _native._lib = base
            print(libname, name, comp.name, "bitwise" if np.array_equal(*out) else "MISMATCH")
