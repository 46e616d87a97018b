"""Regenerates tests/golden/fields_golden.json by running the UNMODIFIED reference solver
(oracle/_ref, built by oracle/build_ref.sh from /root/reference) — run here, not on the GPU box.

Each case is also checked against the digest SURVEY.md Appendix B recorded for it.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402

SURVEY = {  # SURVEY.md Appendix B "Oracle golden values"
    "cavity2d_256_a4": "7bc4ea2a6b07f185", "cavity2d_256_a16": "7bc4ea2a6b07f185",
    "ras64_d16_phi05_wavy": "09d9ff03e65af9ad", "cavity3d_128": "2e5bc22de18a71de",
    "ras256_d40_phi05_wavy": "69d5e9c481a27b3a",
}
CASES = [
    dict(name="cavity2d_256_a4", kind="Cavity2D", ref_kind="cavity2d",
         params=dict(dims=[256, 256, 1]), a=4, tau=0.8, periodic=0, init="uniform", steps=1000),
    dict(name="cavity2d_256_a16", kind="Cavity2D", ref_kind="cavity2d",
         params=dict(dims=[256, 256, 1]), a=16, tau=0.8, periodic=0, init="uniform", steps=1000),
    dict(name="ras64_d16_phi05_wavy", kind="Ras3D", ref_kind="ras3d",
         params=dict(dims=[64, 64, 64], sphere_diameter=16, target_porosity=0.5, seed=7), a=4,
         tau=0.8, periodic=7, init="wavy", steps=1000),
    dict(name="cavity3d_128", kind="Cavity3D", ref_kind="cavity3d",
         params=dict(dims=[128, 128, 128]), a=4, tau=0.8, periodic=0, init="uniform", steps=100),
    dict(name="ras256_d40_phi05_wavy", kind="Ras3D", ref_kind="ras3d",
         params=dict(dims=[256, 256, 256], sphere_diameter=40, target_porosity=0.5, seed=7), a=4,
         tau=0.8, periodic=7, init="wavy", steps=20),
]


def main():
    out = []
    for c in CASES:
        p = c["params"]
        g = R.RefGeometry.generate(c["ref_kind"], p["dims"], diameter=p.get("sphere_diameter", 40),
                                   target=p.get("target_porosity", 0.9), seed=p.get("seed", 0))
        r = R.run_simulation(g, "t2c", c["a"], c["tau"], periodic=c["periodic"], threads=os.cpu_count(),
                             steps=c["steps"], init=c["init"])
        types = g.types()
        mask = (types != 0).astype("uint8")
        dig = O.fields_digest(dict(rho=r["rho"], ux=r["ux"], uy=r["uy"], uz=r["uz"], mask=mask))
        rec = dict(c)
        rec.update(n_f=int(mask.sum()), mass0=r["mass_initial"], mass_final=r["mass_final"],
                   fields_fnv=f"{dig:016x}")
        assert rec["fields_fnv"] == SURVEY[c["name"]], (c["name"], rec["fields_fnv"])
        print(c["name"], rec["fields_fnv"], repr(rec["mass_final"]), flush=True)
        out.append(rec)
    with open(os.path.join(os.path.dirname(__file__), "fields_golden.json"), "w") as f:
        json.dump({"source": "reference solver (oracle/_ref), T2C fp64 BGK quasi", "cases": out}, f,
                  indent=1)


if __name__ == "__main__":
    main()
