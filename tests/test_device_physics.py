"""The reference's physics acceptance criteria (acceptance.cpp:257-311, test_engine.cpp:193-271)
run on the B200 engine."""
import numpy as np
import pytest

import paper_1703_08015_b200 as P
from cases import closed_box

pytestmark = pytest.mark.gpu


def test_poiseuille_profile():  # acceptance.cpp:257-294: L2 <= 2 %
    g = P.generate(P.GeometryKind.Channel2D, P.GenerateParams(dims=(192, 66, 1), inlet_speed=0.02))
    cfg = P.SimConfig(tile=16, steps=10000, model=P.FluidModel(tau=0.8),
                      initial_velocity=(0.02, 0.0, 0.0))
    res = P.run_simulation(g, cfg)
    yc = 0.5 + 32.0
    u = np.array([res.fields.ux[res.fields.index(96, y)] for y in range(1, 65)])
    shape = np.array([1.0 - ((y - yc) / 32.0) ** 2 for y in range(1, 65)])
    amp = u.sum() / shape.sum()
    l2 = np.sqrt(((u - amp * shape) ** 2).sum() / ((amp * shape) ** 2).sum())
    assert l2 <= 0.02, l2


@pytest.mark.parametrize("d,dims,a", [(2, (64, 64, 1), 16), (3, (24, 20, 18), 4)])
def test_closed_box_conserves_mass(d, dims, a):  # test_engine.cpp:193-205, acceptance.cpp:296-311
    from oracle import oracle as O
    cfg = P.SimConfig(tile=a, steps=1000, model=P.FluidModel(tau=0.8), init=O.wavy)
    res = P.run_simulation(closed_box(d, dims), cfg)
    assert res.mass_drift_rel <= 1e-12


def test_lid_driven_cavity_mirror_symmetry():  # test_engine.cpp:233-271
    g = P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(64, 64, 1), lid_speed=0.05))
    cfg = P.SimConfig(tile=16, steps=2000, model=P.FluidModel(tau=0.8))
    res = P.run_simulation(g, cfg)
    f = res.fields
    m = f.mask != 0
    assert np.max(np.hypot(f.ux[m], f.uy[m])) <= 0.05 * 1.1
    gm = g.copy()
    gm.bc.velocity = (-0.05, 0.0, 0.0)
    fm = P.run_simulation(gm, cfg).fields
    a = f.ux.reshape(64, 64)
    b = fm.ux.reshape(64, 64)[:, ::-1]
    mask = m.reshape(64, 64)
    worst = max(np.max(np.abs(a + b)[mask]),
                np.max(np.abs(f.uy.reshape(64, 64) - fm.uy.reshape(64, 64)[:, ::-1])[mask]),
                np.max(np.abs(f.rho.reshape(64, 64) - fm.rho.reshape(64, 64)[:, ::-1])[mask]))
    assert worst <= 1e-3


def test_cavity3d_stays_bounded():  # test_engine.cpp:367-383
    g = P.generate(P.GeometryKind.Cavity3D, P.GenerateParams(dims=(24, 24, 24), lid_speed=0.05))
    res = P.run_simulation(g, P.SimConfig(tile=4, steps=100, model=P.FluidModel(tau=0.8)))
    f = res.fields
    m = f.mask != 0
    assert f.all_finite()
    assert np.max(np.sqrt(f.ux[m] ** 2 + f.uy[m] ** 2 + f.uz[m] ** 2)) <= 0.05 * 1.1


def test_channel3d_develops_flow():
    """BASELINE configs[1] geometry (scaled down): the inlet drives a finite, bounded duct flow."""
    g = P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(64, 24, 24), inlet_speed=0.05))
    res = P.run_simulation(g, P.SimConfig(tile=4, steps=2000, model=P.FluidModel(tau=0.8)))
    f = res.fields
    assert f.all_finite()
    mid = f.ux.reshape(24, 24, 64)[12, 12, 32]
    assert 0.0 < mid < 0.2
