"""Parity cases shared by the CPU oracle tests and the GPU parity tests.

Each case mirrors a reference test geometry (test_engine.cpp / acceptance.cpp / SURVEY §8c)."""
from __future__ import annotations

import numpy as np

import paper_1703_08015_b200 as P


def channel_with_plug(nx, ny, cx, cy, r, inlet=0.04):  # test_engine.cpp:22-32
    g = P.generate(P.GeometryKind.Channel2D, P.GenerateParams(dims=(nx, ny, 1), inlet_speed=inlet))
    v = g.view3d()[0]
    yy, xx = np.mgrid[0:ny, 0:nx]
    v[(xx - cx) ** 2 + (yy - cy) ** 2 <= r * r] = 0
    return g


def closed_box(d, dims):  # test_util.hpp:24-36
    g = P.Geometry.filled(d, dims)
    v = g.view3d()
    v[:, :, 0] = 0
    v[:, :, -1] = 0
    v[:, 0, :] = 0
    v[:, -1, :] = 0
    if d == 3:
        v[0] = 0
        v[-1] = 0
    return g


def random_solids(dims=(21, 18, 13), seed=99, frac=0.3):  # test_engine.cpp:385-405 (numpy RNG)
    rng = np.random.default_rng(seed)
    g = P.Geometry.filled(3, dims)
    g.types[:] = np.where(rng.random(g.node_count()) < frac, 0, 1).astype(np.uint8)
    return g


def corner_contact():  # test_engine.cpp:166-191
    g = P.Geometry.filled(2, (8, 8, 1), 0)
    v = g.view3d()[0]
    v[0:4, 0:4] = 1
    v[4:8, 4:8] = 1
    return g


# name -> (geometry factory, a, tau, incompressible, periodic mask, init)
CASES = {
    "cavity2d_64_a4": (lambda: P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(64, 64, 1))), 4, 0.8, False, 0, "uniform"),
    "cavity2d_64_a16": (lambda: P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(64, 64, 1))), 16, 0.8, False, 0, "uniform"),
    "plug_channel_quasi": (lambda: channel_with_plug(96, 48, 24, 24, 7), 16, 0.8, False, 0, "uniform"),
    "plug_channel_incompr": (lambda: channel_with_plug(96, 48, 24, 24, 7), 16, 0.8, True, 0, "uniform"),
    "plug_channel_a8_odd": (lambda: channel_with_plug(50, 30, 14, 15, 5), 8, 0.9, False, 0, "uniform"),
    "plug_channel_a4": (lambda: channel_with_plug(50, 30, 14, 15, 5), 4, 0.9, False, 0, "wavy"),
    "ras24_periodic": (lambda: P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(24, 24, 24), sphere_diameter=8, target_porosity=0.8, seed=13)), 4, 0.7, False, 7, "wavy"),
    "ras24_periodic_incompr": (lambda: P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(24, 24, 24), sphere_diameter=8, target_porosity=0.8, seed=13)), 4, 0.7, True, 7, "wavy"),
    "corner_contact": (corner_contact, 4, 0.8, False, 0, "wavy"),
    "periodic_single_tile_2d": (lambda: P.Geometry.filled(2, (16, 16, 1)), 16, 0.8, False, 3, "wavy"),
    "periodic_single_tile_3d": (lambda: P.Geometry.filled(3, (4, 4, 4)), 4, 0.8, False, 7, "wavy"),
    "random_solids_a2": (random_solids, 2, 0.8, False, 0, "wavy"),
    "random_solids_a4": (random_solids, 4, 0.8, False, 0, "wavy"),
    "random_solids_a3": (random_solids, 3, 0.8, False, 0, "wavy"),
    "closed_box_2d": (lambda: closed_box(2, (48, 48, 1)), 16, 0.8, False, 0, "wavy"),
    "cavity3d_24": (lambda: P.generate(P.GeometryKind.Cavity3D, P.GenerateParams(dims=(24, 24, 24))), 4, 0.8, False, 0, "uniform"),
    "cavity3d_odd_incompr": (lambda: P.generate(P.GeometryKind.Cavity3D, P.GenerateParams(dims=(24, 20, 18))), 4, 0.8, True, 0, "uniform"),
    "channel3d_32": (lambda: P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(32, 20, 20))), 4, 0.8, False, 0, "uniform"),
    "channel3d_32_incompr": (lambda: P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(30, 18, 21))), 4, 0.8, True, 0, "uniform"),
    "ras48_periodic_a4": (lambda: P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(48, 48, 48), sphere_diameter=10, target_porosity=0.8, seed=42)), 4, 0.7, False, 7, "wavy"),
    "cavity3d_a8_generic": (lambda: P.generate(P.GeometryKind.Cavity3D, P.GenerateParams(dims=(20, 17, 19))), 8, 0.8, False, 0, "uniform"),
    "random_solids_a5_generic": (lambda: random_solids((23, 14, 11), seed=5, frac=0.25), 5, 0.9, True, 0, "wavy"),
    "full2d_periodic_a8": (lambda: P.Geometry.filled(2, (40, 24, 1)), 8, 0.7, False, 3, "wavy"),
    "vessel_256": (lambda: P.generate(P.GeometryKind.Vessel2D, P.GenerateParams(dims=(256, 256, 1), target_porosity=0.3, seed=3)), 4, 0.8, False, 0, "uniform"),
}


def make_oracle(O, g, a, tau, inc, per, precision="f64", mrt=False):
    return O.OracleT2C(g.types, g.d, g.dims, a, tau, incompressible=inc, periodic=per,
                       bc_velocity=g.bc.velocity, bc_density=g.bc.density, threads=4,
                       precision=precision, mrt=mrt)


def init_both(O, oe, de, init):
    """Initialise the oracle and the device engine identically (NodeInit at tile-node coords)."""
    if init == "uniform":
        oe.initialize_uniform()
        if de is not None:
            de.initialize_uniform()
    else:
        oe.initialize_wavy()
        if de is not None:
            de.initialize(lambda x, y, z: O.wavy(x, y, z))
