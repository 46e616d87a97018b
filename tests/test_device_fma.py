"""Tolerance mode (`arithmetic="fma"`, libsplbm_b200_fma.so): the same kernels with contracted
multiply-adds and a reciprocal velocity division. Not bit-exact by design; checked against the
north star's bounds (BASELINE.json): per-step PDFs within 1e-13 relative of the oracle, rho/u
within 1e-10 (`linf_rel_diff`, /root/reference/proj/include/splbm/fields.hpp:47-61) after 1000
steps — at small sizes against the C oracle and at BASELINE configs[1]/[2] full size against the
reference-recorded samples (tests/golden/fields_golden_full.json)."""
import json
import os

import numpy as np
import pytest

import paper_1703_08015_b200 as P

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _pair(kind, dims, per, model, **gp):
    from oracle import oracle as O
    g = P.generate(kind, P.GenerateParams(dims=dims, **gp))
    e = P.TileEngineT2C(g, 4, model, per, arithmetic="fma")
    ora = O.OracleT2C(g.types, g.d, g.dims, 4, model.tau, periodic=per,
                      incompressible=model.compressibility == P.Compressibility.Incompressible,
                      bc_velocity=g.bc.velocity, bc_density=g.bc.density,
                      mrt=model.collision == P.CollisionKind.MRT)
    return g, e, ora


MODELS = {
    "bgk": P.FluidModel(tau=0.8),
    "bgk_inc": P.FluidModel(P.Compressibility.Incompressible, tau=0.8),
    "mrt": P.FluidModel(collision=P.CollisionKind.MRT, tau=0.8),
}
GEOMS = {
    "ras40": (P.GeometryKind.Ras3D, (40, 40, 40), 7, dict(sphere_diameter=12, target_porosity=0.5, seed=3)),
    "channel3d": (P.GeometryKind.Channel3D, (40, 24, 28), 0, {}),
    "cavity2d": (P.GeometryKind.Cavity2D, (64, 64, 1), 0, {}),
}


@pytest.mark.parametrize("model", sorted(MODELS))
@pytest.mark.parametrize("geom", sorted(GEOMS))
def test_fma_one_step_within_1e13(geom, model):
    from oracle import oracle as O
    kind, dims, per, gp = GEOMS[geom]
    g, e, ora = _pair(kind, dims, per, MODELS[model], **gp)
    e.initialize(O.wavy)
    ora.initialize_wavy()
    assert e.step_n(1)[0] and ora.step(1)[0]
    fluid = np.broadcast_to((ora.tiles["types"] != 0)[:, None, :], (ora.T, ora.q, ora.n_tn)).ravel()
    a, b = e.get_pdf()[fluid], ora.current_pdf()[fluid]
    rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
    assert rel.max() <= 1e-13, rel.max()
    assert e.arithmetic == "fma"


@pytest.mark.parametrize("model", ["bgk", "mrt"])
@pytest.mark.parametrize("geom", sorted(GEOMS))
def test_fma_1000_steps_within_1e10(geom, model):
    from oracle import oracle as O
    kind, dims, per, gp = GEOMS[geom]
    g, e, ora = _pair(kind, dims, per, MODELS[model], **gp)
    e.initialize(O.wavy)
    ora.initialize_wavy()
    assert e.step_n(1000)[0] and ora.step(1000)[0]
    fo = ora.fields()
    ref = P.FieldData(g.d, g.dims, fo["mask"], fo["rho"], fo["ux"], fo["uy"], fo["uz"])
    err = P.linf_rel_diff(e.fields(), ref)
    assert err <= 1e-10, err


@pytest.mark.parametrize("name", ["configs1_channel128", "configs2_ras256_phi02"])
def test_fma_full_size_goldens_within_1e10(name, oracle):
    """1000 steps at BASELINE size in tolerance mode against the reference solver's recorded
    sample (sampled linf_rel_diff, scaled by the reference's per-field max)."""
    from test_device_golden_full import case, geometry, sampled_linf
    c = case(name)
    g = geometry(c)
    cfg = P.SimConfig(tile=c["a"], steps=c["steps"], model=P.FluidModel(tau=c["tau"]),
                      periodic=P.Periodicity.of(c["periodic"]),
                      init=oracle.wavy if c["init"] == "wavy" else None, arithmetic="fma")
    r = P.run_simulation(g, cfg)
    err = sampled_linf(c, r.fields)
    assert err <= 1e-10, err
    assert abs(r.mass_final - c["mass_final"]) <= 1e-10 * abs(c["mass_final"])
