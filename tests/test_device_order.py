"""Column traversal order (SPLBM_ORDER, tiling_gpu.h build_column_order): only the CTA -> tile
mapping changes, so every engine flavour steps bit-identically to the compact order and to the
oracle, including ragged column edges and empty columns."""
import numpy as np
import pytest

import paper_1703_08015_b200 as P

pytestmark = pytest.mark.gpu


def _engine(monkeypatch, B, g, per, **kw):
    monkeypatch.setenv("SPLBM_ORDER", str(B))
    from oracle import oracle as O
    e = P.TileEngineT2C(g, 4, kw.pop("model", P.FluidModel(tau=0.8)), per, **kw)
    e.initialize(O.wavy)
    return e


@pytest.mark.parametrize("B", ["1", "3", "5", "16", "2x3", "3x1"])
@pytest.mark.parametrize("flavour", ["two_copy", "single_copy", "mrt", "incompressible"])
def test_column_order_bitwise(monkeypatch, B, flavour):
    from oracle import oracle as O
    g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(44, 36, 40), sphere_diameter=12,
                                                          target_porosity=0.4, seed=11))
    per = (1, 0, 1)
    kw = {}
    if flavour == "single_copy":
        kw["single_copy"] = True
    elif flavour == "mrt":
        kw["model"] = P.FluidModel(collision=P.CollisionKind.MRT, tau=0.8)
    elif flavour == "incompressible":
        kw["model"] = P.FluidModel(P.Compressibility.Incompressible, tau=0.8)
    ref = _engine(monkeypatch, 0, g, per, **dict(kw))
    col = _engine(monkeypatch, B, g, per, **dict(kw))
    for e in (ref, col):
        assert e.step_n(9) == (True, 0)
    assert np.array_equal(ref.get_pdf().view(np.uint64), col.get_pdf().view(np.uint64))
    if flavour == "two_copy":
        ora = O.OracleT2C(g.types, g.d, g.dims, 4, 0.8, periodic=per)
        ora.initialize_wavy()
        ora.step(9)
        f = col.fields()
        fo = ora.fields()
        for k in ("rho", "ux", "uy", "uz"):
            assert np.array_equal(getattr(f, k), fo[k])
