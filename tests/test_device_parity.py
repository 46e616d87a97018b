"""GPU parity: the sm_100a T2C path against the C oracle (bitwise) — the parity tests proper.

Every comparison is bit-exact on the non-solid PDF slots and on (rho, u): the kernel follows the
reference's operation order with round-to-nearest intrinsics. Solid slots are
never read by any step or by fields() (engine.hpp:485-500, 371-390); the device may write 0.0 there
to keep store sectors whole, so they are excluded from the slot comparison.
"""
import numpy as np
import pytest

import paper_1703_08015_b200 as P

from cases import CASES, init_both, make_oracle

pytestmark = pytest.mark.gpu


def fluid_slot_mask(tiles_types, q):
    T, n_tn = tiles_types.shape
    return np.broadcast_to((tiles_types != 0)[:, None, :], (T, q, n_tn)).ravel()


def assert_fields_equal(fo, fd):
    assert np.array_equal(fo["mask"], fd.mask)
    for k in ("rho", "ux", "uy", "uz"):
        a, b = fo[k], getattr(fd, k)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), k


@pytest.mark.parametrize("path", ["resident", "streamed"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_step_bitwise(name, path, oracle, monkeypatch):
    """`resident`: the default engine (small domains run whole batches in the resident multi-step
    kernel); `streamed`: SPLBM_RESIDENT=0, one step-kernel launch per step."""
    factory, a, tau, inc, per, init = CASES[name]
    g = factory()
    model = P.FluidModel(P.Compressibility.Incompressible if inc else P.Compressibility.QuasiCompressible,
                         tau=tau)
    monkeypatch.setenv("SPLBM_RESIDENT", "1" if path == "resident" else "0")
    de = P.TileEngineT2C(g, a, model, per)
    if path == "streamed":
        assert de.info.resident_ctas == 0
    oe = make_oracle(oracle, g, a, tau, inc, per)
    tg = de.tile_grid()
    assert np.array_equal(tg.tile_map, oe.tiles["tile_map"])
    assert np.array_equal(tg.types, oe.tiles["types"])
    init_both(oracle, oe, de, init)
    mask = fluid_slot_mask(oe.tiles["types"], oe.q)
    assert np.array_equal(de.get_pdf()[mask], oe.current_pdf()[mask])
    done = 0
    for n in (1, 1, 5, 33):
        ok_d, _ = de.step_n(n)
        ok_o, _ = oe.step(n)
        done += n
        assert ok_d and ok_o
        assert np.array_equal(de.get_pdf()[mask].view(np.uint64), oe.current_pdf()[mask].view(np.uint64)), \
            f"PDF mismatch after {done} steps"
    assert de.current_step() == done
    assert de.tile_visits() == done * oe.T  # engine.hpp:505-507
    fd, mass_d = de.fields(with_mass=True)
    fo = oe.fields()
    assert_fields_equal(fo, fd)
    assert mass_d == fo["mass"]
    assert fd.total_mass() == fo["mass"]


def test_uniform_equilibrium_is_fixed_point():  # test_engine.cpp:49-70
    g = P.Geometry.filled(2, (32, 32, 1))
    e = P.TileEngineT2C(g, 16, P.FluidModel(tau=0.8), (1, 1, 0))
    e.initialize_uniform(1.0)
    assert e.step_n(5)[0]
    f = e.fields()
    assert np.max(np.abs(f.rho - 1.0)) < 1e-15
    assert np.max(np.abs(f.ux)) < 1e-15 and np.max(np.abs(f.uy)) < 1e-15


def test_single_link_locality():  # test_engine.cpp:72-111
    g = P.Geometry.filled(2, (16, 16, 1))
    e = P.TileEngineT2C(g, 4, P.FluidModel(tau=1.0), (1, 1, 0))

    def init(x, y, z):
        hit = (x == 8) & (y == 8)
        return (np.where(hit, 1.1, 1.0), np.where(hit, 0.02, 0.0), np.where(hit, -0.01, 0.0),
                np.zeros(x.shape))
    e.initialize(init)
    assert e.step()
    f = e.fields()
    lat = P.solver_lattice(2)
    moved = (np.abs(f.rho - 1) > 1e-13) | (np.abs(f.ux) > 1e-13) | (np.abs(f.uy) > 1e-13)
    idx = np.flatnonzero(moved)
    allowed = {f.index(8 + ex, 8 + ey) for ex, ey, _ in lat.e}
    assert set(idx.tolist()) <= allowed and len(idx) == lat.q


def test_failure_reports_first_failing_step(oracle):
    """A broken density fails step() like the reference (collision.hpp:44-47, engine.hpp:634)."""
    g = P.Geometry.filled(2, (32, 32, 1))
    e = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), (1, 1, 0))
    e.initialize_uniform(1.0)
    assert e.step_n(3) == (True, 0)
    f = e.get_pdf()
    f[5] = np.nan
    e.set_pdf(f)
    ok, failed = e.step_n(4)
    assert not ok and failed == 4
    cfg = P.SimConfig(tile=4, steps=10, model=P.FluidModel(tau=0.8),
                      init=lambda x, y, z: (np.where((x == 3) & (y == 3), -5.0, 1.0), 0.0, 0.0, 0.0))
    with pytest.raises(P.DomainError):  # equilibrium(rho <= 0) under quasi (lattice.hpp:76-78)
        P.run_simulation(g, cfg)


def test_run_simulation_contract():
    g = P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(64, 64, 1)))
    cfg = P.SimConfig(tile=16, steps=0, model=P.FluidModel(tau=0.8))
    r0 = P.run_simulation(g, cfg)  # test_engine.cpp:422-434
    assert r0.mlups == 0.0 and r0.steps == 0
    assert np.allclose(r0.fields.rho[r0.fields.mask != 0], 1.0)
    calls = []
    cfg = P.SimConfig(tile=16, steps=10, snapshot_every=5, model=P.FluidModel(tau=0.8),
                      snapshot_sink=lambda s, f, pd: calls.append((s, pd)))
    r = P.run_simulation(g, cfg)
    assert [c[0] for c in calls] == [5, 10] and r.snapshots_written == 2
    assert r.padded_dims == (64, 64, 1) and r.mlups > 0
    assert r.tile_visits == 10 * 16
    box = P.Geometry.filled(2, (20, 12, 1))
    e = P.TileEngineT2C(box, 8, P.FluidModel(tau=0.8))
    assert e.padded_dims() == (24, 16, 1)  # test_io.cpp:14-22


def test_empty_tiles_do_no_work():  # test_engine.cpp:297-330
    from cases import closed_box
    small = closed_box(2, (64, 32, 1))
    emb = P.Geometry.filled(2, (64, 64, 1), 0)
    emb.types[: 64 * 32] = small.types
    from oracle import oracle as O
    cfg = P.SimConfig(tile=16, steps=40, model=P.FluidModel(tau=0.8), init=O.wavy)
    a = P.run_simulation(small, cfg)
    b = P.run_simulation(emb, cfg)
    assert a.tile_visits == b.tile_visits == 40 * (64 // 16) * (32 // 16)
    m = a.fields.mask != 0
    assert np.array_equal(a.fields.rho[m], b.fields.rho[: 64 * 32][m])
    assert np.array_equal(a.fields.ux[m], b.fields.ux[: 64 * 32][m])


def test_errors_match_reference():
    g = P.Geometry.filled(2, (16, 16, 1))
    with pytest.raises(P.ConfigError):
        P.TileEngineT2C(g, 4, P.FluidModel(tau=0.5))
    with pytest.raises(P.ConfigError):
        P.TileEngineT2C(g, 1, P.FluidModel(tau=0.8))
    with pytest.raises(P.ConfigError):
        P.TileEngineT2C(P.Geometry.filled(2, (30, 32, 1)), 16, P.FluidModel(tau=0.8), (1, 0, 0))


def test_all_solid_geometry_has_no_tiles():
    g = P.Geometry.filled(3, (16, 16, 16), 0)
    e = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8))
    assert e.info.n_tiles == 0
    e.initialize_uniform()
    assert e.step_n(5) == (True, 0)
    f, mass = e.fields(with_mass=True)
    assert mass == 0.0 and not f.mask.any() and e.tile_visits() == 0
