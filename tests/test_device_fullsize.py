"""Parity at BASELINE.json's full sizes (the driver's GPU suite).

configs[1]-[3] are small enough for the C oracle to follow for a few steps at full size, so they
are compared bit for bit; configs[4] (RAS 1024^3) is beyond the oracle (two-copy PDFs
>= 106 GB), so it is checked through size-independent properties: the single-copy engine equals
the two-copy engine (device checksums of every non-solid node: mass and max |u|, bitwise), and a
periodic domain conserves mass.
"""
import numpy as np
import pytest

import paper_1703_08015_b200 as P

from cases import make_oracle
from test_device_parity import assert_fields_equal, fluid_slot_mask

pytestmark = pytest.mark.gpu


def run_both(oracle, g, a, per, steps, init="uniform", u0=(0.0, 0.0, 0.0), tau=0.8, inc=False):
    model = P.FluidModel(P.Compressibility.Incompressible if inc else P.Compressibility.QuasiCompressible,
                         tau=tau)
    de = P.TileEngineT2C(g, a, model, per)
    oe = make_oracle(oracle, g, a, tau, inc, per)
    oe.threads = 16
    if init == "wavy":
        de.initialize(lambda x, y, z: oracle.wavy(x, y, z))
        oe.initialize_wavy()
    else:
        de.initialize_uniform(1.0, u0)
        oe.initialize_uniform(1.0, u0)
    assert de.step_n(steps)[0] and oe.step(steps)[0]
    return de, oe


def test_config1_channel_128_full_size(oracle):
    """configs[1]: D3Q19 channel 128^3, V inlet / P outlet, bounce-back walls."""
    g = P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(128, 128, 128)))
    de, oe = run_both(oracle, g, 4, 0, 40)
    mask = fluid_slot_mask(oe.tiles["types"], oe.q)
    assert np.array_equal(de.get_pdf()[mask].view(np.uint64), oe.current_pdf()[mask].view(np.uint64))
    fd, md = de.fields(with_mass=True)
    fo = oe.fields()
    assert_fields_equal(fo, fd)
    assert md == fo["mass"]


@pytest.mark.parametrize("phi", [0.2, 0.8])
def test_config2_ras_256_full_size(oracle, phi):
    """configs[2]: RAS 256^3, d 40, seed 7, periodic, wavy init (phi 0.5 is a golden digest)."""
    g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(256, 256, 256), sphere_diameter=40,
                                                          target_porosity=phi, seed=7))
    de, oe = run_both(oracle, g, 4, 7, 4, init="wavy")
    fd, md = de.fields(with_mass=True)
    fo = oe.fields()
    assert_fields_equal(fo, fd)
    assert md == fo["mass"]


def test_config3_vessel_4096_full_size(oracle):
    """configs[3]: D2Q9 seeded vessel tree 4096^2, a = 4, V inlet / P outlets."""
    g = P.generate(P.GeometryKind.Vessel2D, P.GenerateParams(dims=(4096, 4096, 1), target_porosity=0.2,
                                                            seed=1))
    de, oe = run_both(oracle, g, 4, 0, 12)
    mask = fluid_slot_mask(oe.tiles["types"], oe.q)
    assert np.array_equal(de.get_pdf()[mask].view(np.uint64), oe.current_pdf()[mask].view(np.uint64))
    assert_fields_equal(oe.fields(), de.fields())


@pytest.mark.slow
def test_config4_ras_1024_properties():
    """configs[4]: RAS 1024^3 phi 0.2 on one B200 (GPU generator). Two copies (107 GB) and then the
    single copy (53 GB) run the same 21 steps; their device checksums agree bit for bit, and the
    periodic domain conserves mass to round-off."""
    g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(1024, 1024, 1024), sphere_diameter=40,
                                                          target_porosity=0.2, seed=7), device=0)
    out = {}
    for single in (False, True):
        e = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), 7, single_copy=single)
        e.initialize_uniform(1.0, (0.01, 0.005, 0.0))
        m0 = e.reduce()
        assert e.step_n(21)[0]  # odd: the single-copy state ends swapped
        out[single] = (m0, e.reduce(), e.current_step(), e.tile_visits())
        del e
    (a0, a1, sa, va), (b0, b1, sb, vb) = out[False], out[True]
    assert a0 == b0 and a1 == b1 and sa == sb and va == vb
    assert a1["non_finite"] == 0
    assert abs(a1["mass"] - a0["mass"]) <= 1e-12 * a0["mass"]


@pytest.mark.parametrize("variant", ["mrt", "f32", "f32_incompressible", "single_copy"])
def test_config1_channel_128_model_variants(oracle, variant):
    """configs[1] at full size for the paper's Table 2 model rows and the single-copy storage:
    MRT, the f32 engine (quasi-compressible and incompressible) and the in-place AA pair, each
    bit for bit against the oracle after 12 steps from rest (the bench's workload)."""
    g = P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(128, 128, 128)))
    inc = variant == "f32_incompressible"
    prec = "f32" if variant.startswith("f32") else "f64"
    mrt = variant == "mrt"
    model = P.FluidModel(P.Compressibility.Incompressible if inc else P.Compressibility.QuasiCompressible,
                         collision=P.CollisionKind.MRT if mrt else P.CollisionKind.BGK, tau=0.8)
    de = P.TileEngineT2C(g, 4, model, 0, precision=prec, single_copy=variant == "single_copy")
    oe = make_oracle(oracle, g, 4, 0.8, inc, 0, precision=prec, mrt=mrt)
    oe.threads = 16
    de.initialize_uniform()
    oe.initialize_uniform()
    assert de.step_n(12)[0] and oe.step(12)[0]
    mask = fluid_slot_mask(oe.tiles["types"], oe.q)
    width = np.uint32 if prec == "f32" else np.uint64
    assert np.array_equal(de.get_pdf()[mask].view(width), oe.current_pdf()[mask].view(width))
    assert_fields_equal(oe.fields(), de.fields())
