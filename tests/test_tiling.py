"""Tile map (reference tiling.cpp:85-141, engine.hpp:446-463): product builder vs reference,
bit-exact, plus the reference's own known answers (test_tiling.cpp) and SURVEY App. B digests."""
import numpy as np
import pytest

import paper_1703_08015_b200 as P

from cases import CASES


def ref_geom(ref, g):
    return ref.RefGeometry.from_raster(g.d, g.dims, g.types, g.bc.velocity, g.bc.density)


@pytest.mark.parametrize("name,a,per", [(n, a, p) for n in sorted(CASES) for a, p in
                                        [(2, 0), (4, 0), (16, 0), (4, -1)]])
def test_tile_map_matches_reference(name, a, per, ref):
    g = CASES[name][0]()
    if per == -1:
        per = CASES[name][4]
    if g.d == 3 and a == 16:
        a = 8
    dims = g.dims
    if any(((per >> k) & 1) and dims[k] % a for k in range(3)):
        pytest.skip("periodic extent not divisible")
    tg = P.build_tile_grid(g, a, per)
    rt = ref.tile_grid(ref_geom(ref, g), a, per)
    assert tg.grid_dims == rt.grid_dims and tg.padded_dims == rt.padded_dims
    assert np.array_equal(tg.tile_map, rt.tile_map)
    assert np.array_equal(tg.origins, rt.origins)
    assert np.array_equal(tg.types, rt.types)
    assert np.array_equal(tg.fluid_count, rt.fluid_count)
    assert np.array_equal(tg.nb, rt.nb)
    st = P.tile_stats(tg)
    assert st.phi_t == rt.stats["phi_t"] and st.ratio_tiles == rt.stats["ratio_tiles"]


def test_known_answers():  # test_tiling.cpp:65-97
    g = P.Geometry.filled(2, (32, 32, 1), 0)
    tg = P.build_tile_grid(g, 16)
    assert tg.tile_count() == 4 and tg.fluid_tile_count() == 0 and P.tile_stats(tg).phi_t == 0.0
    tg = P.build_tile_grid(P.Geometry.filled(2, (32, 32, 1)), 16)
    assert tg.fluid_tile_count() == 4 and P.tile_stats(tg).phi_t == 1.0
    tg = P.build_tile_grid(P.Geometry.filled(2, (33, 32, 1)), 16)
    assert tg.padded_dims[:2] == (48, 32) and tg.tile_count() == 6 and tg.fluid_tile_count() == 6
    assert P.tile_stats(tg).phi_t == 1056.0 / 1536.0


def test_tiling_errors():  # test_tiling.cpp:99-106
    g = P.Geometry.filled(2, (16, 16, 1))
    with pytest.raises(P.ConfigError):
        P.build_tile_grid(g, 1)
    with pytest.raises(P.ConfigError):
        P.build_tile_grid(P.Geometry.filled(2, (30, 32, 1)), 16, (1, 0, 0))


def test_node_conservation_and_origins():  # test_tiling.cpp:108-148
    g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(48, 48, 48), sphere_diameter=12,
                                                          target_porosity=0.75, seed=9))
    tg = P.build_tile_grid(g, 4)
    assert int(tg.fluid_count.sum()) == g.fluid_count()
    cells = np.flatnonzero(tg.tile_map != P.kEmptyTile)
    gd = tg.grid_dims
    cx, cy, cz = cells % gd[0], (cells // gd[0]) % gd[1], cells // (gd[0] * gd[1])
    t = tg.tile_map[cells]
    assert np.array_equal(tg.origins[t], np.stack([cx * 4, cy * 4, cz * 4], 1))
    assert np.array_equal(t, np.arange(t.size))  # compact index in cz->cy->cx order
    assert P.porosity(g).phi <= P.tile_stats(tg).phi_t


@pytest.mark.parametrize("n,phi,digest", [
    (128, 0.8, "25487ba4550b11b5"), (256, 0.2, "6e54a0b7aff33a27"),
    (256, 0.5, "8cb2f86372710d8f"), (256, 0.8, "d0f5f866c3a4638e")])
def test_tile_map_digest_survey(n, phi, digest, oracle):
    """SURVEY.md Appendix B tile-map digests (RAS d=40 seed 7, a=4, periodic xyz)."""
    g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(n, n, n), sphere_diameter=40,
                                                          target_porosity=phi, seed=7))
    tg = P.build_tile_grid(g, 4, (1, 1, 1), with_neighbours=False)
    d = oracle.tilemap_digest(dict(tile_map=tg.tile_map, origins=tg.origins, types=tg.types,
                                   n_tn=tg.n_tn))
    assert f"{d:016x}" == digest


@pytest.mark.parametrize("name", ["cavity2d_64_a4", "plug_channel_quasi", "channel3d_32",
                                  "cavity3d_24", "vessel_256"])
def test_degenerate_mask_matches_reference(name, ref, oracle):
    g = CASES[name][0]()
    m = P.degenerate_bc_mask(g)
    assert np.array_equal(m, ref.degenerate_mask(ref_geom(ref, g)))
    assert np.array_equal(m, oracle.degenerate_mask(g.types, g.d, g.dims))


def test_oracle_tile_builder_matches_product(oracle):
    for name in ("random_solids_a3", "ras48_periodic_a4", "vessel_256"):
        factory, a, _, _, per, _ = CASES[name]
        g = factory()
        tg = P.build_tile_grid(g, a, per)
        ot = oracle.build_tiles(g.types, g.d, g.dims, a, per)
        assert np.array_equal(tg.tile_map, ot["tile_map"])
        assert np.array_equal(tg.types, ot["types"])
        nb = oracle.nb_table(ot["grid_dims"], per, ot["tile_map"], ot["origins"].shape[0])
        assert np.array_equal(tg.nb, nb)
