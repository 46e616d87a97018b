"""Software-pipelined persistent step (SPLBM_PIPE=1, t2c_step_pipe_kernel): same addresses, slots
and arithmetic as the one-shot kernel, so PDFs are bit-identical — BGK (both compressibilities),
MRT, velocity/pressure boundaries, periodic and walled domains, and full-size goldens."""
import numpy as np
import pytest

import paper_1703_08015_b200 as P

pytestmark = pytest.mark.gpu

GEOMS = {
    "ras_mixed_periodic": (lambda: P.generate(P.GeometryKind.Ras3D, P.GenerateParams(
        dims=(44, 36, 40), sphere_diameter=12, target_porosity=0.4, seed=11)), (1, 0, 1)),
    "channel3d_bc": (lambda: P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(37, 22, 26))), 0),
    "cavity3d": (lambda: P.generate(P.GeometryKind.Cavity3D, P.GenerateParams(dims=(24, 24, 24))), 0),
}
MODELS = {
    "bgk": P.FluidModel(tau=0.8),
    "bgk_inc": P.FluidModel(P.Compressibility.Incompressible, tau=0.8),
    "mrt": P.FluidModel(collision=P.CollisionKind.MRT, tau=0.8),
}


@pytest.mark.parametrize("model", sorted(MODELS))
@pytest.mark.parametrize("geom", sorted(GEOMS))
def test_pipe_bitwise(monkeypatch, geom, model):
    from oracle import oracle as O
    g = GEOMS[geom][0]()
    per = GEOMS[geom][1]
    engines = []
    for pipe in ("0", "1"):
        monkeypatch.setenv("SPLBM_PIPE", pipe)
        e = P.TileEngineT2C(g, 4, MODELS[model], per)
        e.initialize(O.wavy)
        engines.append(e)
    for e in engines:
        assert e.step_n(13) == (True, 0)  # odd: both copies exercised, plus a partial graph
    a, b = (e.get_pdf() for e in engines)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("name", ["configs1_channel128", "configs2_ras256_phi02"])
def test_pipe_full_size_golden(monkeypatch, name, oracle):
    from test_device_golden_full import case, geometry
    monkeypatch.setenv("SPLBM_PIPE", "1")
    c = case(name)
    g = geometry(c)
    cfg = P.SimConfig(tile=c["a"], steps=c["steps"], model=P.FluidModel(tau=c["tau"]),
                      periodic=P.Periodicity.of(c["periodic"]),
                      init=oracle.wavy if c["init"] == "wavy" else None)
    r = P.run_simulation(g, cfg)
    f = r.fields
    assert r.mass_final == c["mass_final"]
    d = oracle.fields_digest(dict(rho=f.rho, ux=f.ux, uy=f.uy, uz=f.uz, mask=f.mask))
    assert f"{d:016x}" == c["fields_fnv"]
