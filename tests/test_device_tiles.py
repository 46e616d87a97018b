"""The GPU tile builder (csrc/tiling_gpu.cu) against the host builder (SPLBM_HOST_TILES=1, the
restatement of tiling.cpp:85-141 / engine.hpp:110-140 / 446-463 that tests/test_tiling.py pins):
identical tile cover, neighbour ids, node types, fluid counts and bc_degenerate flags (checked
through the steps, which read them), on geometries with ragged padding, scattered BC nodes next to
solids and periodic edges, a mixed periodicity mask, and the degenerate cases (one tile, all solid
but one node)."""
import numpy as np
import pytest

import paper_1703_08015_b200 as P

pytestmark = pytest.mark.gpu


def random_geometry(d, dims, seed, solid=0.3, bc=0.05):
    rng = np.random.default_rng(seed)
    n = dims[0] * dims[1] * dims[2]
    u = rng.random(n)
    t = np.ones(n, np.uint8)
    t[u < solid] = 0
    t[(u >= solid) & (u < solid + bc / 2)] = 2
    t[(u >= solid + bc / 2) & (u < solid + bc)] = 3
    g = P.Geometry(d, tuple(dims), t, P.BcParams(velocity=(0.01, -0.005, 0.002), density=1.0))
    return g


CASES = {
    "3d_ragged_open": (lambda: random_geometry(3, (37, 29, 23), 1), 4, 0),
    "3d_periodic_xz": (lambda: random_geometry(3, (32, 21, 24), 2), 4, 0b101),
    "3d_periodic_all": (lambda: random_geometry(3, (24, 24, 24), 3, solid=0.6), 4, 7),
    "3d_a2": (lambda: random_geometry(3, (15, 16, 9), 4), 2, 0b010),
    "3d_a5_generic": (lambda: random_geometry(3, (23, 14, 11), 5), 5, 0),
    "2d_ragged_a16": (lambda: random_geometry(2, (250, 130, 1), 6), 16, 0),
    "2d_periodic_y_a4": (lambda: random_geometry(2, (61, 64, 1), 7), 4, 0b010),
    "2d_a3": (lambda: random_geometry(2, (40, 31, 1), 8, solid=0.7), 3, 0),
    "ras64": (lambda: P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(64, 64, 64), sphere_diameter=12,
                                                                       target_porosity=0.3, seed=9)), 4, 7),
    "channel3d": (lambda: P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(40, 24, 20))), 4, 0),
    "one_tile": (lambda: P.Geometry.filled(3, (4, 4, 4)), 4, 7),
    "single_fluid_node": (lambda: single_node(), 4, 0),
}


def single_node():
    g = P.Geometry.filled(3, (13, 9, 7), fill=0)
    g.set(6, 4, 3, 1)
    return g


def engines(monkeypatch, g, a, per):
    dev = P.TileEngineT2C(g, a, P.FluidModel(tau=0.8), per)
    monkeypatch.setenv("SPLBM_HOST_TILES", "1")
    host = P.TileEngineT2C(g, a, P.FluidModel(tau=0.8), per)
    monkeypatch.delenv("SPLBM_HOST_TILES")
    return dev, host


@pytest.mark.parametrize("name", sorted(CASES))
def test_gpu_tile_builder_matches_host(name, monkeypatch):
    factory, a, per = CASES[name]
    g = factory()
    dev, host = engines(monkeypatch, g, a, per)
    td, th = dev.tile_grid(), host.tile_grid()
    for k in ("tile_map", "origins", "types", "fluid_count", "nb"):
        assert np.array_equal(getattr(td, k), getattr(th, k)), k
    assert dev.info.n_tiles == host.info.n_tiles
    assert dev.info.fluid_nodes == host.info.fluid_nodes == int(np.count_nonzero(g.types))
    assert tuple(dev.info.padded_dims) == tuple(host.info.padded_dims)
    for e in (dev, host):
        e.initialize(lambda x, y, z: (1.0 + 0.01 * np.sin(0.3 * x + 0.2 * y + 0.1 * z), 0.01 * np.cos(0.2 * y),
                                      0.005 * np.sin(0.1 * x), 0.002 * np.cos(0.3 * z)))
        e.step_n(3)
    # identical node-info words (blocked masks from nb, bc_degenerate) => identical PDFs, bitwise
    assert np.array_equal(dev.get_pdf().view(np.uint64), host.get_pdf().view(np.uint64))
    fd, fh = dev.fields(), host.fields()
    assert np.array_equal(fd.mask, fh.mask)
    assert np.array_equal(fd.rho.view(np.uint64), fh.rho.view(np.uint64))
