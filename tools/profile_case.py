"""Runs one workload for a few steps (for ncu captures): python tools/profile_case.py NAME [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1703_08015_b200 as P  # noqa: E402

CASES = {
    "channel128": lambda: (P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(128, 128, 128))), 4, 0),
    "ras256_phi02": lambda: (P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(256, 256, 256), sphere_diameter=40, target_porosity=0.2, seed=7)), 4, 7),
    "ras256_phi05": lambda: (P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(256, 256, 256), sphere_diameter=40, target_porosity=0.5, seed=7)), 4, 7),
    "cavity2d_4096_a4": lambda: (P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(4096, 4096, 1))), 4, 0),
    "ras48_periodic": lambda: (P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(48, 48, 48), sphere_diameter=12, target_porosity=0.5, seed=2)), 4, 7),
    "channel3d_small": lambda: (P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(30, 18, 21))), 4, 0),
    "cavity2d_512_a4": lambda: (P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(512, 512, 1))), 4, 0),
    "cavity2d_256_a4": lambda: (P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(256, 256, 1))), 4, 0),
    "cavity2d_64_a16": lambda: (P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(64, 64, 1))), 16, 0),
    "random_a3": lambda: (__import__("cases").random_solids((23, 14, 11), seed=5, frac=0.25), 3, 0),
    "vessel4096_a4": lambda: (P.generate(P.GeometryKind.Vessel2D, P.GenerateParams(dims=(4096, 4096, 1), target_porosity=0.2, seed=1)), 4, 0),
}

if __name__ == "__main__":
    name = sys.argv[1]
    if name == "ras_device_generator":  # the RAS sphere loop on the GPU (geometry_gpu.cu)
        g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(40, 36, 32), sphere_diameter=9,
                                                              target_porosity=0.4, seed=3), device=0)
        print(name, "phi", P.porosity(g).phi)
        sys.exit(0)
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    if name.startswith("ras1024_phi"):  # BASELINE configs[4] on one GPU (device-generated raster)
        phi = float("0." + name.split("phi0")[1])
        g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(1024, 1024, 1024), sphere_diameter=40,
                                                              target_porosity=phi, seed=7), device=0)
        a, per = 4, 7
    else:
        g, a, per = CASES[name]()
    coll = P.CollisionKind.MRT if os.environ.get("SPLBM_MODEL") == "mrt" else P.CollisionKind.BGK
    e = P.TileEngineT2C(g, a, P.FluidModel(collision=coll, tau=0.8), per,
                        single_copy=os.environ.get("SPLBM_SINGLE_COPY") == "1",
                        precision=os.environ.get("SPLBM_PRECISION", "f64"))
    e.initialize_uniform(1.0, (0.01, 0.0, 0.0))
    ok, _ = e.step_n(steps)
    e.fields()
    e.reduce()
    print(name, "ok" if ok else "FAILED", "fluid nodes", e.fluid_nodes(), "tiles", e.info.n_tiles)
