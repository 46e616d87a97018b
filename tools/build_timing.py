"""Time-to-first-step of the configs[4] class: GPU RAS generation, then the engine build (per-phase
host/device times via SPLBM_BUILD_TIMING=1), then one step. python tools/build_timing.py [N] [phi ...]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SPLBM_BUILD_TIMING", "1")
import paper_1703_08015_b200 as P  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    phis = [float(v) for v in sys.argv[2:]] or [0.2]
    for phi in phis:
        t0 = time.perf_counter()
        g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(n, n, n), sphere_diameter=40,
                                                              target_porosity=phi, seed=7), device=0)
        t1 = time.perf_counter()
        e = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), 7, single_copy=phi > 0.35)
        t2 = time.perf_counter()
        e.initialize_uniform(1.0, (0.0, 0.0, 0.0))
        assert e.step_n(1)[0]
        t3 = time.perf_counter()
        print(f"{n}^3 phi {phi}: generate {t2 - t2 + t1 - t0:.2f} s  engine {t2 - t1:.2f} s  "
              f"init+1 step {t3 - t2:.2f} s  tiles {e.info.n_tiles}", flush=True)
        del e


if __name__ == "__main__":
    main()
