"""GPU runs reproduce the reference's golden field digests bit for bit.

The digests were recorded from the reference solver itself (T2C, fp64, BGK quasi, tau 0.8); see
tests/golden/fields_golden.json and tests/golden/make_golden.py.
"""
import json
import os

import numpy as np
import pytest

import paper_1703_08015_b200 as P

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fields_golden.json")))


@pytest.mark.parametrize("case", [c["name"] for c in GOLD["cases"]])
def test_golden_fields(case, oracle):
    c = next(c for c in GOLD["cases"] if c["name"] == case)
    g = P.generate(P.GeometryKind[c["kind"]], P.GenerateParams(**c["params"]))
    cfg = P.SimConfig(tile=c["a"], steps=c["steps"], model=P.FluidModel(tau=c["tau"]),
                      periodic=P.Periodicity.of(c["periodic"]),
                      init=oracle.wavy if c["init"] == "wavy" else None)
    r = P.run_simulation(g, cfg)
    f = r.fields
    assert r.fluid_nodes == c["n_f"]
    assert r.mass_initial == c["mass0"]
    assert r.mass_final == c["mass_final"]
    d = oracle.fields_digest(dict(rho=f.rho, ux=f.ux, uy=f.uy, uz=f.uz, mask=f.mask))
    assert f"{d:016x}" == c["fields_fnv"]
