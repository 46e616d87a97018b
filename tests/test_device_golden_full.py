"""BASELINE configs[1]-[3] at full size over the north star's 1000 steps, against fields recorded
from the UNMODIFIED reference solver (tests/golden/fields_golden_full.json, written by
tests/golden/make_golden_full.py from oracle/_ref: `run_simulation<double>`, Method::T2C,
/root/reference/proj/include/splbm/engine.hpp:609-655).

The bar is bitwise: the FNV digest of the (rho, u, mask) raster fields and the final mass. The
north star's own bound (rho/u within 1e-10 after 1000 steps, `linf_rel_diff`,
/root/reference/proj/include/splbm/fields.hpp:47-61) is also evaluated on the recorded sample so
a failure reports how far off it is.
"""
import json
import os

import numpy as np
import pytest

import paper_1703_08015_b200 as P
from oracle import configs as CF

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "fields_golden_full.json")))
NAMES = [c["name"] for c in GOLD["cases"]]


def case(name):
    return next(c for c in GOLD["cases"] if c["name"] == name)


def geometry(c):
    return P.generate(P.GeometryKind[c["kind"]], P.GenerateParams(**c["params"]))


def sampled_linf(c, f):
    """linf_rel_diff restricted to the recorded sample nodes, scaled by the reference's per-field
    max |value| over all non-solid nodes (fields.hpp:47-61)."""
    idx = np.asarray(c["sample_index"], np.int64)
    worst = 0.0
    for k in ("rho", "ux", "uy", "uz"):
        ref = np.array([float.fromhex(v) for v in c["sample"][k]])
        got = getattr(f, k)[idx]
        scale = max(c["max_abs"][k], float(np.max(np.abs(got))))
        if scale > 0:
            worst = max(worst, float(np.max(np.abs(got - ref))) / scale)
    return worst


@pytest.mark.parametrize("name", NAMES)
def test_golden_rasters(name):
    """The product generators rebuild exactly the rasters the reference was run on (CPU)."""
    c = case(name)
    g = geometry(c)
    assert CF.raster_sha(g.types) == c["raster_sha"]
    assert int(np.count_nonzero(np.asarray(g.types))) == c["n_f"]
    if c["kind"] == "Channel3D":
        assert np.array_equal(np.asarray(g.types).ravel(), CF.channel3d_raster(tuple(c["params"]["dims"])))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_golden_full_1000_steps(name, oracle):
    c = case(name)
    g = geometry(c)
    assert CF.raster_sha(g.types) == c["raster_sha"]
    cfg = P.SimConfig(tile=c["a"], steps=c["steps"], model=P.FluidModel(tau=c["tau"]),
                      periodic=P.Periodicity.of(c["periodic"]),
                      init=oracle.wavy if c["init"] == "wavy" else None)
    r = P.run_simulation(g, cfg)
    f = r.fields
    assert r.fluid_nodes == c["n_f"] and r.steps == c["steps"]
    err = sampled_linf(c, f)
    assert err <= 1e-10, f"north-star bound violated: sampled linf_rel_diff {err:.3e}"
    assert r.mass_initial == c["mass0"]
    assert r.mass_final == c["mass_final"]
    d = oracle.fields_digest(dict(rho=f.rho, ux=f.ux, uy=f.uy, uz=f.uz, mask=f.mask))
    assert f"{d:016x}" == c["fields_fnv"], f"not bitwise (sampled linf {err:.3e})"
