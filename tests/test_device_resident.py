"""The resident multi-step kernel (small whole-domain engines: a batch of steps inside one
cooperative grid with grid barriers, `t2c_resident_kernel`) against the one-launch-per-step path
(SPLBM_RESIDENT=0): every PDF slot bit-identical, same failure step, same counters. The oracle
parity of both paths is `tests/test_device_parity.py::test_step_bitwise[...-resident/streamed]`."""
import numpy as np
import pytest

import paper_1703_08015_b200 as P

from cases import CASES

pytestmark = pytest.mark.gpu


def _engine(monkeypatch, on, g, a, model, per, **kw):
    monkeypatch.setenv("SPLBM_RESIDENT", "1" if on else "0")
    e = P.TileEngineT2C(g, a, model, per, **kw)
    assert (e.info.resident_ctas > 0) == on
    return e


def _wavy(x, y, z):
    return (1.0 + 0.01 * np.sin(0.3 * x + 0.2 * y), 0.02 * np.cos(0.1 * y), 0.01 * np.sin(0.2 * x),
            0.005 * np.cos(0.15 * z))


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("name", ["cavity2d_64_a4", "vessel_256", "cavity3d_24", "ras24_periodic",
                                  "random_solids_a3", "plug_channel_incompr"])
def test_resident_equals_streamed(name, precision, monkeypatch):
    factory, a, tau, inc, per, _ = CASES[name]
    g = factory()
    model = P.FluidModel(P.Compressibility.Incompressible if inc else P.Compressibility.QuasiCompressible,
                         tau=tau)
    r = _engine(monkeypatch, True, g, a, model, per, precision=precision)
    s = _engine(monkeypatch, False, g, a, model, per, precision=precision)
    for e in (r, s):
        e.initialize(_wavy)
    for n in (1, 2, 31, 64, 1200):  # odd / even batches, a batch above one resident launch
        assert r.step_n(n) == s.step_n(n)
        assert np.array_equal(r.get_pdf().view(np.uint8), s.get_pdf().view(np.uint8)), n
    assert r.current_step() == s.current_step() and r.tile_visits() == s.tile_visits()
    fr, fs = r.fields(), s.fields()
    for k in ("rho", "ux", "uy", "uz"):
        assert np.array_equal(getattr(fr, k).view(np.uint64), getattr(fs, k).view(np.uint64))


def test_resident_failure_step(monkeypatch):
    """A NaN planted after 3 steps: both paths report step 4 (engine.hpp:634), also when the
    failing step is deep inside one resident batch."""
    g = P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(64, 64, 1)))
    out = []
    for on in (True, False):
        e = _engine(monkeypatch, on, g, 4, P.FluidModel(tau=0.8), 0)
        e.initialize_uniform()
        assert e.step_n(3) == (True, 0)
        f = e.get_pdf()
        f[5] = np.nan
        e.set_pdf(f)
        out.append(e.step_n(50))
        assert e.current_step() == 53
    assert out[0] == out[1] == (False, 4)


def test_resident_engines_concurrently(monkeypatch):
    """Two small engines stepping at once on their own streams (resident grids are serialised per
    device, so their barriers cannot starve each other) give the sequential results."""
    g = P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(256, 256, 1)))
    engines = [_engine(monkeypatch, True, g, 4, P.FluidModel(tau=0.8), 0) for _ in range(3)]
    for e in engines:
        e.initialize_uniform()
    for e in engines:  # enqueued back to back: three streams with resident batches in flight
        e.step_async(2000)
    res = [e.sync() for e in engines]
    assert all(r == (True, 0) for r in res)
    ref = _engine(monkeypatch, False, g, 4, P.FluidModel(tau=0.8), 0)
    ref.initialize_uniform()
    assert ref.step_n(2000) == (True, 0)
    for e in engines:
        assert np.array_equal(e.get_pdf().view(np.uint64), ref.get_pdf().view(np.uint64))


def test_configs0_is_resident():
    """BASELINE configs[0] (D2Q9 cavity 256^2, a = 4 and 16) takes the resident path by default."""
    g = P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(256, 256, 1)))
    for a in (4, 16):
        e = P.TileEngineT2C(g, a, P.FluidModel(tau=0.8))
        assert 0 < e.info.resident_ctas <= 2 * 148 and e.info.resident_threads <= 1024
    big = P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(128, 128, 128)))
    assert P.TileEngineT2C(big, 4, P.FluidModel(tau=0.8)).info.resident_ctas == 0
