"""RAS step timing at arbitrary dims (L2-reuse / traversal-order experiments):
python tools/size_probe.py NX NY NZ PHI [--single-copy] [--steps K]
SPLBM_ORDER (read at engine creation) selects the traversal order. Prints one JSON line."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_08015_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("dims", type=int, nargs=3)
ap.add_argument("phi", type=float)
ap.add_argument("--single-copy", action="store_true")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--warmup", type=int, default=4)
a = ap.parse_args()
g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=tuple(a.dims), sphere_diameter=40,
                                                      target_porosity=a.phi, seed=7), device=0)
e = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), (1, 1, 1), single_copy=a.single_copy)
e.initialize_uniform(1.0, (0.01, 0.005, 0.0))
e.step_n(a.warmup)
e.step_async(a.steps)
ok, _ = e.sync()
ms = e.last_batch_ms() / a.steps
nf = e.fluid_nodes()
mlups = nf / (ms * 1e-3) / 1e6
print(json.dumps({"dims": a.dims, "phi": a.phi, "single_copy": a.single_copy,
                  "order": os.environ.get("SPLBM_ORDER", "auto"), "ok": ok, "us_per_step": round(ms * 1e3, 2),
                  "mlups": round(mlups, 1), "frac_copy_peak": round(mlups * 1e6 * 304 / 6547.2e9, 4),
                  "tiles": int(e.info.n_tiles), "fluid_nodes": nf}))
