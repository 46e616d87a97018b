"""Interleaved A/B timing of engine variants in ONE process on the same box:
python tools/ab.py '{"name": {"ENV": "value", ...}, ...}' [case ...] [--rounds R --steps K]

Every variant's engine is created with its environment settings (read at engine creation, e.g.
SPLBM_L2PF, SPLBM_SINGLE_COPY, SPLBM_PRECISION, SPLBM_MODEL=mrt; "LIB": "variants/lib_x.so" selects another build of the library)
and all engines of a case stay resident; the K-step batches are then
alternated A, B, A, B, ... for R rounds and the median per variant is reported, so box-to-box and
thermal drift cancel out of the comparison."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_08015_b200 as P  # noqa: E402

CASES = {
    "channel128": lambda: (P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(128, 128, 128))), 0),
    "ras256_phi02": lambda: (P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(256, 256, 256), sphere_diameter=40, target_porosity=0.2, seed=7)), 7),
    "ras256_phi05": lambda: (P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(256, 256, 256), sphere_diameter=40, target_porosity=0.5, seed=7)), 7),
    "full256": lambda: (P.Geometry.filled(3, (256, 256, 256)), 7),
    "channel64": lambda: (P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(64, 64, 64))), 0),  # L2-resident
    "cavity2d_4096_a4": lambda: (P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(4096, 4096, 1))), 0),
    "cavity2d_256_a4": lambda: (P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(256, 256, 1))), 0),
    "cavity2d_256_a16": lambda: (P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(256, 256, 1))), 0),
    "vessel4096": lambda: (P.generate(P.GeometryKind.Vessel2D, P.GenerateParams(dims=(4096, 4096, 1), target_porosity=0.2, seed=1)), 0),
}


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("variants")
    ap.add_argument("cases", nargs="*")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--steps", type=int, default=64)
    a = ap.parse_args()
    rounds, K = a.rounds, a.steps
    variants = json.loads(a.variants)
    cases = a.cases or list(CASES)
    out = {}
    libs = {}
    for case in cases:
        g, per = CASES[case]()
        engines = {}
        for name, env in variants.items():
            saved = {k: os.environ.get(k) for k in env if k != "LIB"}
            os.environ.update({k: str(v) for k, v in env.items() if k != "LIB"})
            single = os.environ.get("SPLBM_SINGLE_COPY") == "1"
            prec = os.environ.get("SPLBM_PRECISION", "f64")
            from paper_1703_08015_b200 import _native
            saved_lib = _native._lib
            if "LIB" in env:  # another build of the library (e.g. variants/lib_old.so)
                _native._lib = libs.setdefault(env["LIB"], _native.load(os.path.join(ROOT, env["LIB"])))
            coll = P.CollisionKind.MRT if os.environ.get("SPLBM_MODEL") == "mrt" else P.CollisionKind.BGK
            e = P.TileEngineT2C(g, 16 if case.endswith("_a16") else 4,
                                P.FluidModel(collision=coll, tau=0.8), per,
                                single_copy=single, precision=prec)
            _native._lib = saved_lib
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
            e.initialize_uniform(1.0, (0.01, 0.0, 0.0))
            e.step_n(16)
            engines[name] = e
        times = {n: [] for n in engines}
        for _ in range(rounds):
            for n, e in engines.items():
                e.step_async(K)
                ok, _ = e.sync()
                assert ok
                times[n].append(e.last_batch_ms() / K * 1e3)
        nf = next(iter(engines.values())).fluid_nodes()
        res = {}
        for n, ts in times.items():
            us = statistics.median(ts)
            res[n] = {"us_per_step": round(us, 2), "mlups": round(nf / us, 1),
                      "spread_us": round(max(ts) - min(ts), 2)}
        out[case] = res
        print(case, json.dumps(res), flush=True)
        del engines
    print(json.dumps(out))


if __name__ == "__main__":
    main()
