"""Times the step kernel of several compile-time variants (built by `--build`) on the bench
workloads. Each variant is a separate libsplbm_b200 build loaded in its own process."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "variants")
VARIANTS = json.load(open(os.path.join(VAR, "variants.json"))) if os.path.exists(
    os.path.join(VAR, "variants.json")) else {}


def build(variants):
    from paper_1703_08015_b200 import build as B
    os.makedirs(VAR, exist_ok=True)
    for name, defs in variants.items():
        B.build(defines=defs, lib=os.path.join(VAR, f"lib_{name}.so"),
                build_dir=os.path.join(ROOT, "build", "var_" + name))
    json.dump(variants, open(os.path.join(VAR, "variants.json"), "w"))


def run_one(K=100, W=10):
    import paper_1703_08015_b200 as P
    res = {}
    cases = {
        "channel128": lambda: (P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(128, 128, 128))), 0),
        "ras256_phi05": lambda: (P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(256, 256, 256), sphere_diameter=40, target_porosity=0.5, seed=7)), 7),
        "full256": lambda: (P.Geometry.filled(3, (256, 256, 256)), 7),
        "cavity2d_4096_a4": lambda: (P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(4096, 4096, 1))), 0),
        "cavity2d_256_a4": lambda: (P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(256, 256, 1))), 0),
        "ras256_phi02": lambda: (P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(256, 256, 256), sphere_diameter=40, target_porosity=0.2, seed=7)), 7),
    }
    for name, mk in cases.items():
        g, per = mk()
        e = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), per,
                            single_copy=os.environ.get("SPLBM_SINGLE_COPY") == "1")
        e.initialize_uniform(1.0, (0.01, 0.0, 0.0))
        k = 1000 if "256_a4" in name else K
        e.step_n(max(W, 64))
        best = 1e9
        for _ in range(3):
            e.step_async(k)
            e.sync()
            best = min(best, e.last_batch_ms() / k)
        nf = e.fluid_nodes()
        bn = 304.0 if g.d == 3 else 144.0
        res[name] = {"us_per_step": round(best * 1e3, 2), "mlups": round(nf / (best * 1e-3) / 1e6, 1),
                     "gbs": round(nf * bn / (best * 1e-3) / 1e9, 1)}
        del e
    return res


if __name__ == "__main__":
    if sys.argv[1] == "--build":
        build(json.loads(sys.argv[2]))
    elif sys.argv[1] == "--run":
        out = {}
        for name in VARIANTS:
            env = dict(os.environ, SPLBM_LIB=os.path.join(VAR, f"lib_{name}.so"))
            r = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True,
                               text=True)
            out[name] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-2000:]
            print(name, out[name], flush=True)
        print(json.dumps(out))
    elif sys.argv[1] == "--run-env":  # runtime variants of the in-tree library: {name: {VAR: value}}
        out = {}
        for name, extra in json.loads(sys.argv[2]).items():
            env = dict(os.environ, **{k: str(v) for k, v in extra.items()})
            r = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True,
                               text=True)
            out[name] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-2000:]
            print(name, out[name], flush=True)
        print(json.dumps(out))
    elif sys.argv[1] == "--one":
        print(json.dumps(run_one()))
