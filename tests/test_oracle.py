"""Pins the C oracle (oracle/splbm_oracle.c) to the reference solver itself (oracle/_ref, built in
place from /root/reference) and to the golden digests recorded from it (tests/golden/)."""
import json
import os

import numpy as np
import pytest

import paper_1703_08015_b200 as P

from cases import CASES, make_oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fields_golden.json")))
FAST = ["cavity2d_64_a4", "plug_channel_quasi", "plug_channel_incompr", "plug_channel_a8_odd",
        "ras24_periodic", "ras24_periodic_incompr", "corner_contact", "periodic_single_tile_2d",
        "periodic_single_tile_3d", "random_solids_a2", "random_solids_a3", "cavity3d_odd_incompr",
        "channel3d_32", "vessel_256"]


@pytest.mark.parametrize("name", FAST)
def test_oracle_matches_reference_bitwise(name, ref, oracle):
    factory, a, tau, inc, per, init = CASES[name]
    g = factory()
    rg = ref.RefGeometry.from_raster(g.d, g.dims, g.types, g.bc.velocity, g.bc.density)
    re = ref.RefEngine(rg, "t2c", a, tau, incompressible=inc, periodic=per, threads=2)
    oe = make_oracle(oracle, g, a, tau, inc, per)
    if init == "uniform":
        re.initialize_uniform()
        oe.initialize_uniform()
    else:
        re.initialize_wavy()
        oe.initialize_wavy()
    assert np.array_equal(re.pdf(), oe.current_pdf())
    for n in (1, 9, 20):
        ok_r, _ = re.step(n)
        ok_o, _ = oe.step(n)
        assert ok_r and ok_o
        assert np.array_equal(re.pdf().view(np.uint64), oe.current_pdf().view(np.uint64))
    fr, fo = re.fields(), oe.fields()
    for k in ("rho", "ux", "uy", "uz", "mask"):
        assert np.array_equal(fr[k], fo[k]), k
    assert fr["mass"] == fo["mass"]
    assert re.tile_visits() == 30 * oe.T


F32 = ["cavity2d_64_a4", "plug_channel_quasi", "plug_channel_incompr", "ras24_periodic",
       "ras24_periodic_incompr", "random_solids_a3", "cavity3d_odd_incompr", "channel3d_32"]


@pytest.mark.parametrize("mrt", [False, True])
@pytest.mark.parametrize("name", F32)
def test_oracle_f32_matches_reference_float_engine(name, mrt, ref, oracle):
    """The float instance of the restatement (oracle/t2c_real.inc) against the reference's own
    TileEngineT2C<float> (the CLI's precision=f32): every PDF slot and (rho, u) bit for bit."""
    factory, a, tau, inc, per, init = CASES[name]
    g = factory()
    rg = ref.RefGeometry.from_raster(g.d, g.dims, g.types, g.bc.velocity, g.bc.density)
    re = ref.RefEngine(rg, "t2c", a, tau, incompressible=inc, mrt=mrt, periodic=per, threads=2,
                       precision="f32")
    oe = make_oracle(oracle, g, a, tau, inc, per, precision="f32", mrt=mrt)
    if init == "uniform":
        re.initialize_uniform()
        oe.initialize_uniform()
    else:
        re.initialize_wavy()
        oe.initialize_wavy()
    assert re.pdf().dtype == np.float32
    assert np.array_equal(re.pdf().view(np.uint32), oe.current_pdf().view(np.uint32))
    for n in (1, 9, 20):
        ok_r, _ = re.step(n)
        ok_o, _ = oe.step(n)
        assert ok_r and ok_o
        assert np.array_equal(re.pdf().view(np.uint32), oe.current_pdf().view(np.uint32))
    fr, fo = re.fields(), oe.fields()
    for k in ("rho", "ux", "uy", "uz", "mask"):
        assert np.array_equal(fr[k], fo[k]), k
    assert fr["mass"] == fo["mass"]


def test_oracle_matches_dense_engine(ref, oracle):
    """Dense == T2C in the reference; the oracle agrees with the Dense engine too."""
    g = CASES["plug_channel_quasi"][0]()
    rg = ref.RefGeometry.from_raster(g.d, g.dims, g.types, g.bc.velocity, g.bc.density)
    rd = ref.RefEngine(rg, "dense", 16, 0.8)
    rd.initialize_uniform()
    rd.step(60)
    oe = make_oracle(oracle, g, 16, 0.8, False, 0)
    oe.initialize_uniform()
    oe.step(60)
    fd, fo = rd.fields(), oe.fields()
    for k in ("rho", "ux", "uy"):
        assert np.array_equal(fd[k], fo[k])


@pytest.mark.parametrize("case", ["cavity2d_256_a4", "cavity2d_256_a16", "ras64_d16_phi05_wavy"])
def test_oracle_golden_digest(case, oracle):
    """The oracle alone reproduces the reference's recorded field digests (no _ref needed)."""
    c = next(c for c in GOLD["cases"] if c["name"] == case)
    g = P.generate(P.GeometryKind[c["kind"]], P.GenerateParams(**c["params"]))
    oe = oracle.OracleT2C(g.types, g.d, g.dims, c["a"], c["tau"], periodic=c["periodic"],
                          bc_velocity=g.bc.velocity, bc_density=g.bc.density,
                          threads=os.cpu_count() or 1)
    if c["init"] == "wavy":
        oe.initialize_wavy()
    else:
        oe.initialize_uniform()
    assert oe.fields()["mass"] == c["mass0"]
    ok, _ = oe.step(c["steps"])
    assert ok
    f = oe.fields()
    assert f["mass"] == c["mass_final"]
    assert f"{oracle.fields_digest(f):016x}" == c["fields_fnv"]


def test_oracle_failure_detection(oracle):
    g = P.Geometry.filled(2, (16, 16, 1))
    oe = oracle.OracleT2C(g.types, 2, g.dims, 4, 0.8, periodic=3)
    oe.initialize_uniform()
    oe.pdf[oe.read][3] = np.nan
    ok, step = oe.step(2)
    assert not ok and step == 1
