"""Regenerates tests/golden/fields_golden_full.json: BASELINE configs[1]-[3] at full size over the
north star's 1000 steps, run by the UNMODIFIED reference solver (oracle/_ref, built from
/root/reference by oracle/build_ref.sh, `run_simulation<double>` with Method::T2C,
engine.hpp:609-655) on all host threads. Run here, not on the GPU box (~15-25 min on 8 cores).

Geometry sources:
  * configs[1] channel 128^3: numpy raster (oracle/configs.py) — the reference has no 3D channel;
  * configs[2] RAS 256^3 d=40 seed 7: the reference's own generator (geometry.cpp:251-326);
  * configs[3] vessel tree 4096^2: the product generator (no reference equivalent),
    fed to the reference through `Geometry` from the raster; its sha256 is recorded so the GPU test
    first proves it regenerated the very same bytes.

Per case the fixture holds the bitwise FNV digest of the (rho, u, mask) fields and the final mass
(the strict bar), plus 4096 sampled non-solid node values and the per-field max |value| over the
non-solid nodes, so a tolerance-mode engine can be checked against the north star's 1e-10 bound
(`linf_rel_diff` restricted to the sample) at full size.

  python tests/golden/make_golden_full.py [case ...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import configs as CF  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fields_golden_full.json")
N_SAMPLE = 4096

CASES = [
    dict(name="configs1_channel128", source="numpy", kind="Channel3D",
         params=dict(dims=[128, 128, 128], inlet_speed=0.05, outlet_density=1.0), a=4, tau=0.8,
         periodic=0, init="uniform", steps=1000),
    dict(name="configs2_ras256_phi02", source="reference", kind="Ras3D",
         params=dict(dims=[256, 256, 256], sphere_diameter=40, target_porosity=0.2, seed=7), a=4,
         tau=0.8, periodic=7, init="wavy", steps=1000),
    dict(name="configs2_ras256_phi05", source="reference", kind="Ras3D",
         params=dict(dims=[256, 256, 256], sphere_diameter=40, target_porosity=0.5, seed=7), a=4,
         tau=0.8, periodic=7, init="wavy", steps=1000),
    dict(name="configs2_ras256_phi08", source="reference", kind="Ras3D",
         params=dict(dims=[256, 256, 256], sphere_diameter=40, target_porosity=0.8, seed=7), a=4,
         tau=0.8, periodic=7, init="wavy", steps=1000),
    dict(name="configs3_vessel4096", source="product", kind="Vessel2D",
         params=dict(dims=[4096, 4096, 1], target_porosity=0.2, seed=1), a=4, tau=0.8, periodic=0,
         init="uniform", steps=1000),
]


def geometry(c):
    p = c["params"]
    if c["source"] == "numpy":
        t = CF.channel3d_raster(tuple(p["dims"]))
        return R.RefGeometry.from_raster(3, p["dims"], t, (p["inlet_speed"], 0.0, 0.0),
                                         p["outlet_density"]), t
    if c["source"] == "reference":
        g = R.RefGeometry.generate("ras3d", p["dims"], diameter=p["sphere_diameter"],
                                   target=p["target_porosity"], seed=p["seed"])
        return g, g.types()
    import paper_1703_08015_b200 as P
    pg = P.generate(P.GeometryKind[c["kind"]], P.GenerateParams(**p))
    t = np.ascontiguousarray(pg.types, np.uint8).ravel()
    return R.RefGeometry.from_raster(pg.d, pg.dims, t, tuple(pg.bc.velocity), pg.bc.density), t


def main(names):
    old = json.load(open(OUT))["cases"] if os.path.exists(OUT) else []
    keep = {c["name"]: c for c in old}
    for c in CASES:
        if names and c["name"] not in names:
            continue
        t0 = time.time()
        g, types = geometry(c)
        r = R.run_simulation(g, "t2c", c["a"], c["tau"], periodic=c["periodic"],
                             threads=os.cpu_count(), steps=c["steps"], init=c["init"])
        mask = (types != 0).astype(np.uint8)
        f = dict(rho=r["rho"], ux=r["ux"], uy=r["uy"], uz=r["uz"], mask=mask)
        dig = O.fields_digest(f)
        fluid = np.flatnonzero(mask)
        idx = np.sort(np.random.default_rng(12345).choice(fluid, size=N_SAMPLE, replace=False))
        rec = dict(c)
        rec.update(
            raster_sha=CF.raster_sha(types), n_f=int(mask.sum()), mass0=r["mass_initial"],
            mass_final=r["mass_final"], fields_fnv=f"{dig:016x}",
            max_abs={k: float(np.abs(f[k][fluid]).max()) for k in ("rho", "ux", "uy", "uz")},
            sample_index=idx.tolist(),
            sample={k: [float(v).hex() for v in f[k][idx]] for k in ("rho", "ux", "uy", "uz")},
            ref_seconds=round(r["wall_seconds"], 1), ref_mlups=round(r["mlups"], 2),
            ref_threads=os.cpu_count())
        keep[c["name"]] = rec
        print(c["name"], rec["fields_fnv"], repr(rec["mass_final"]), f"{time.time() - t0:.0f}s",
              flush=True)
        with open(OUT, "w") as fh:
            json.dump({"source": "reference solver (oracle/_ref), T2C fp64 BGK quasi, 1000 steps, "
                                 "full BASELINE sizes; written by tests/golden/make_golden_full.py",
                       "cases": [keep[k["name"]] for k in CASES if k["name"] in keep]}, fh,
                      indent=0)


if __name__ == "__main__":
    main(sys.argv[1:])
