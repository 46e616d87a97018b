"""GPU parity of the single-copy (AA) propagation mode against the C oracle.

The in-place mode stores one PDF array; after an odd number of steps it is in the swapped layout.
get_pdf() and fields() return the natural state, so every comparison below is the same bitwise
check as tests/test_device_parity.py: per-step non-solid PDF slots, (rho, u), mass, visits.
"""
import numpy as np
import pytest

import paper_1703_08015_b200 as P

from cases import CASES, init_both, make_oracle
from test_device_parity import assert_fields_equal, fluid_slot_mask

pytestmark = pytest.mark.gpu

POW2 = sorted(n for n, c in CASES.items() if c[1] in (2, 4) or (c[1] in (8, 16) and "3d" not in n
                                                               and "ras" not in n and "random" not in n))


def model_of(tau, inc, mrt=False):
    return P.FluidModel(P.Compressibility.Incompressible if inc else P.Compressibility.QuasiCompressible,
                        tau=tau, collision=P.CollisionKind.MRT if mrt else P.CollisionKind.BGK)


@pytest.mark.parametrize("name", POW2)
def test_single_copy_bitwise(name, oracle):
    factory, a, tau, inc, per, init = CASES[name]
    g = factory()
    de = P.TileEngineT2C(g, a, model_of(tau, inc), per, single_copy=True)
    oe = make_oracle(oracle, g, a, tau, inc, per)
    init_both(oracle, oe, de, init)
    mask = fluid_slot_mask(oe.tiles["types"], oe.q)
    done = 0
    for n in (1, 1, 1, 4, 33):  # odd totals end in the swapped layout
        ok_d, _ = de.step_n(n)
        ok_o, _ = oe.step(n)
        done += n
        assert ok_d and ok_o
        assert np.array_equal(de.get_pdf()[mask].view(np.uint64), oe.current_pdf()[mask].view(np.uint64)), \
            f"PDF mismatch after {done} steps"
        assert_fields_equal(oe.fields(), de.fields())
    assert de.current_step() == done
    assert de.tile_visits() == done * oe.T


def test_single_copy_halves_memory():
    g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(48, 48, 48), sphere_diameter=10,
                                                          target_porosity=0.5, seed=4))
    two = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), 7)
    one = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), 7, single_copy=True)
    pdf_bytes = int(two.info.n_tiles_stored) * 19 * 64 * 8
    assert int(two.info.device_bytes) - int(one.info.device_bytes) == pdf_bytes


@pytest.mark.parametrize("inc", [False, True])
def test_single_copy_mrt_equals_two_copy(inc):
    g = P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(32, 20, 20)))
    ref = P.TileEngineT2C(g, 4, model_of(0.8, inc, mrt=True))
    aa = P.TileEngineT2C(g, 4, model_of(0.8, inc, mrt=True), single_copy=True)
    for e in (ref, aa):
        e.initialize_uniform(1.0, (0.02, 0.0, 0.0))
    for n in (1, 6, 31):
        assert ref.step_n(n)[0] and aa.step_n(n)[0]
        assert np.array_equal(ref.get_pdf().view(np.uint64)[fluid_slot_mask(ref.tile_grid().types, 19)],
                              aa.get_pdf().view(np.uint64)[fluid_slot_mask(aa.tile_grid().types, 19)])
        assert ref.reduce() == aa.reduce()


def test_single_copy_long_run_matches_two_copy_large():
    """A multi-wave domain (graph batches, PDL, L2 prefetch all active): 101 steps, bitwise."""
    g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(96, 96, 96), sphere_diameter=20,
                                                          target_porosity=0.4, seed=9))
    ref = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.7), 7)
    aa = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.7), 7, single_copy=True)
    from oracle import oracle as O
    for e in (ref, aa):
        e.initialize(lambda x, y, z: O.wavy(x, y, z))
        assert e.step_n(101)[0]
    fr, mr = ref.fields(with_mass=True)
    fa, ma = aa.fields(with_mass=True)
    for k in ("rho", "ux", "uy", "uz"):
        assert np.array_equal(getattr(fr, k).view(np.uint64), getattr(fa, k).view(np.uint64)), k
    assert mr == ma
    assert ref.reduce() == aa.reduce()


def test_single_copy_failure_step_and_set_pdf():
    g = P.Geometry.filled(3, (8, 8, 8))
    e = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), 7, single_copy=True)
    e.initialize_uniform(1.0)
    assert e.step_n(3) == (True, 0)  # leaves the swapped layout
    f = e.get_pdf()
    e.set_pdf(f)                      # natural layout again
    assert np.array_equal(e.get_pdf(), f)
    bad = f.copy()
    bad[5 * 64 + 3] = np.nan          # tile 0, direction 5, node 3
    e.set_pdf(bad)
    ok, step = e.step_n(4)
    assert not ok and step == 4       # the NaN is streamed and collided in the first batch step


def test_single_copy_rejects_unsupported():
    g = P.Geometry.filled(3, (12, 12, 12))
    with pytest.raises(P.ConfigError):
        P.TileEngineT2C(g, 3, P.FluidModel(tau=0.8), 7, single_copy=True)
    with pytest.raises(P.ConfigError):
        P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), 7, slab=(0, 2), single_copy=True)
