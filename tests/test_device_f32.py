"""GPU parity of the f32 engine (TileEngineT2C<float>, the reference's precision=f32, paper
Table 2 f32 rows) against the float instance of the C oracle, which tests/test_oracle.py
pins bit for bit to the reference's own float engine. Every comparison is bitwise: the kernel's
float arithmetic is the reference's operation order with __fadd_rn/__fmul_rn/__fdiv_rn.
"""
import numpy as np
import pytest

import paper_1703_08015_b200 as P

from cases import CASES, init_both, make_oracle
from test_device_parity import fluid_slot_mask

pytestmark = pytest.mark.gpu

NAMES = sorted(CASES)


def model_of(tau, inc, mrt=False):
    return P.FluidModel(P.Compressibility.Incompressible if inc else P.Compressibility.QuasiCompressible,
                        tau=tau, collision=P.CollisionKind.MRT if mrt else P.CollisionKind.BGK)


def assert_fields(fo, fd):
    assert np.array_equal(fo["mask"], fd.mask)
    for k in ("rho", "ux", "uy", "uz"):
        assert np.array_equal(fo[k].view(np.uint64), getattr(fd, k).view(np.uint64)), k


@pytest.mark.parametrize("name", NAMES)
def test_f32_step_bitwise(name, oracle):
    factory, a, tau, inc, per, init = CASES[name]
    g = factory()
    de = P.TileEngineT2C(g, a, model_of(tau, inc), per, precision="f32")
    oe = make_oracle(oracle, g, a, tau, inc, per, precision="f32")
    init_both(oracle, oe, de, init)
    mask = fluid_slot_mask(oe.tiles["types"], oe.q)
    assert de.get_pdf().dtype == np.float32
    assert np.array_equal(de.get_pdf()[mask].view(np.uint32), oe.current_pdf()[mask].view(np.uint32))
    done = 0
    for n in (1, 1, 5, 33):
        ok_d, _ = de.step_n(n)
        ok_o, _ = oe.step(n)
        done += n
        assert ok_d and ok_o
        assert np.array_equal(de.get_pdf()[mask].view(np.uint32), oe.current_pdf()[mask].view(np.uint32)), \
            f"PDF mismatch after {done} steps"
    fd, mass = de.fields(with_mass=True)
    fo = oe.fields()
    assert_fields(fo, fd)
    assert mass == fo["mass"]
    assert de.tile_visits() == done * oe.T


@pytest.mark.parametrize("name", ["ras24_periodic", "channel3d_32_incompr", "plug_channel_quasi",
                                  "cavity2d_64_a4", "random_solids_a2"])
def test_f32_single_copy_and_mrt_bitwise(name, oracle):
    factory, a, tau, inc, per, init = CASES[name]
    g = factory()
    for mrt in (False, True):
        de = P.TileEngineT2C(g, a, model_of(tau, inc, mrt), per, precision="f32", single_copy=True)
        oe = make_oracle(oracle, g, a, tau, inc, per, precision="f32", mrt=mrt)
        init_both(oracle, oe, de, init)
        mask = fluid_slot_mask(oe.tiles["types"], oe.q)
        for n in (1, 2, 7):  # totals 1, 3, 10: swapped, swapped, natural layouts
            assert de.step_n(n)[0] and oe.step(n)[0]
            assert np.array_equal(de.get_pdf()[mask].view(np.uint32),
                                  oe.current_pdf()[mask].view(np.uint32))
            assert_fields(oe.fields(), de.fields())


def test_f32_halves_pdf_memory():
    g = P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(32, 20, 20)))
    e64 = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8))
    e32 = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), precision="f32")
    pdf64 = 2 * int(e64.info.n_tiles_stored) * 19 * 64 * 8
    assert int(e64.info.device_bytes) - int(e32.info.device_bytes) == pdf64 // 2


def test_f32_rejects_slab():
    g = P.Geometry.filled(3, (8, 8, 16))
    with pytest.raises(P.ConfigError):
        P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), 7, slab=(0, 2), precision="f32")
