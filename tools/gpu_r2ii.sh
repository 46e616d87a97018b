#!/bin/bash
# Round 2 experiment: x-neighbour node pairs in the two-node step (SPLBM_X2=2: vector loads for
# e_x = 0 directions, vector stores) vs the (j, j + NTN/2) pairs; f32 3D and D2Q9 f64.
O=gpurun_out/r2ii
mkdir -p $O
cd "$(dirname "$0")/.."
timeout 600 python - > $O/check.txt 2>&1 <<'PY'
import numpy as np, os
import paper_1703_08015_b200 as P
for name, g, per, prec in (("channel3d", P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(64, 40, 40))), 0, "f32"),
                           ("ras3d", P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(64, 64, 64), sphere_diameter=12, target_porosity=0.4, seed=2)), 7, "f32"),
                           ("vessel", P.generate(P.GeometryKind.Vessel2D, P.GenerateParams(dims=(512, 512, 1), target_porosity=0.25, seed=3)), 0, "f64"),
                           ("cavity", P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(512, 512, 1))), 0, "f64")):
    out = []
    for v in ("1", "2"):
        os.environ["SPLBM_X2"] = v
        e = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), per, precision=prec)
        e.initialize(lambda x, y, z: (1.0 + 0.01 * np.sin(0.2 * x), 0.01 * np.cos(0.1 * y), 0.0, 0.0))
        assert e.step_n(40)[0]
        out.append(e.get_pdf().view(np.uint8).copy())
    print(name, "bitwise" if np.array_equal(*out) else "MISMATCH")
PY
cat $O/check.txt
V='{"x2": {}, "px": {"SPLBM_X2": "2"}}'
timeout 900 python tools/ab.py "$V" vessel4096 cavity2d_4096_a4 --rounds 9 --steps 192 > $O/ab2d.txt 2>&1; echo ab2d=$?; head -2 $O/ab2d.txt
V='{"x2": {"SPLBM_PRECISION": "f32"}, "px": {"SPLBM_PRECISION": "f32", "SPLBM_X2": "2"}}'
timeout 900 python tools/ab.py "$V" channel128 ras256_phi05 --rounds 9 --steps 192 > $O/abf32.txt 2>&1; echo abf32=$?; head -2 $O/abf32.txt
