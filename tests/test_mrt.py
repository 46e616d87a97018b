"""MRT collision (reference collision.hpp:54-63, collision.cpp:86-113)."""
import numpy as np
import pytest

import paper_1703_08015_b200 as P
from paper_1703_08015_b200.lattice import mrt_kernel

from cases import CASES, make_oracle


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("rates", [None, "custom"])
def test_operator_matrix_bit_identical(d, rates, ref, oracle):
    q = 9 if d == 2 else 19
    r = None if rates is None else np.linspace(0.2, 1.7, q)
    K = mrt_kernel(d, 0.9, r)
    assert np.array_equal(K.view(np.uint64), ref.mrt_kernel(d, 0.9, r).view(np.uint64))
    assert np.array_equal(K.view(np.uint64), oracle.mrt_kernel(d, 0.9, r).view(np.uint64))


@pytest.mark.parametrize("name", ["plug_channel_a8_odd", "ras24_periodic", "cavity3d_odd_incompr",
                                  "random_solids_a3"])
def test_oracle_mrt_matches_reference(name, ref, oracle):
    factory, a, tau, inc, per, init = CASES[name]
    g = factory()
    rg = ref.RefGeometry.from_raster(g.d, g.dims, g.types, g.bc.velocity, g.bc.density)
    re = ref.RefEngine(rg, "t2c", a, tau, incompressible=inc, mrt=True, periodic=per)
    oe = oracle.OracleT2C(g.types, g.d, g.dims, a, tau, incompressible=inc, periodic=per,
                          bc_velocity=g.bc.velocity, bc_density=g.bc.density, mrt=True)
    if init == "uniform":
        re.initialize_uniform()
        oe.initialize_uniform()
    else:
        re.initialize_wavy()
        oe.initialize_wavy()
    re.step(15)
    oe.step(15)
    assert np.array_equal(re.pdf().view(np.uint64), oe.current_pdf().view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["plug_channel_a8_odd", "ras24_periodic", "cavity3d_odd_incompr",
                                  "random_solids_a3", "channel3d_32", "cavity2d_64_a4"])
def test_device_mrt_bitwise(name, oracle):
    factory, a, tau, inc, per, init = CASES[name]
    g = factory()
    model = P.FluidModel(P.Compressibility.Incompressible if inc else P.Compressibility.QuasiCompressible,
                         P.CollisionKind.MRT, tau=tau)
    de = P.TileEngineT2C(g, a, model, per)
    oe = oracle.OracleT2C(g.types, g.d, g.dims, a, tau, incompressible=inc, periodic=per,
                          bc_velocity=g.bc.velocity, bc_density=g.bc.density, mrt=True)
    if init == "uniform":
        de.initialize_uniform()
        oe.initialize_uniform()
    else:
        de.initialize(oracle.wavy)
        oe.initialize_wavy()
    assert de.step_n(40)[0] and oe.step(40)[0]
    fluid = np.broadcast_to((oe.tiles["types"] != 0)[:, None, :], (oe.T, oe.q, oe.n_tn)).ravel()
    assert np.array_equal(de.get_pdf()[fluid].view(np.uint64), oe.current_pdf()[fluid].view(np.uint64))


@pytest.mark.gpu
def test_mrt_uniform_rates_reproduce_bgk():  # acceptance.cpp:237-252: <= 1e-12
    g = P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(32, 32, 1), lid_speed=0.05))
    bgk = P.run_simulation(g, P.SimConfig(tile=16, steps=100, model=P.FluidModel(tau=0.8)))
    mrt = P.run_simulation(g, P.SimConfig(tile=16, steps=100, model=P.FluidModel(
        collision=P.CollisionKind.MRT, tau=0.8, mrt_rates=[1 / 0.8] * 9)))
    assert P.linf_rel_diff(bgk.fields, mrt.fields) <= 1e-12
