"""The RAS generator on the device (splbm_generate_device) against the host
restatement, which tests/test_geometry.py pins to the reference's generate_ras: bit-identical
rasters, including the accept/skip/retry endgame and boxes wider than the domain."""
import time

import numpy as np
import pytest

import paper_1703_08015_b200 as P

pytestmark = pytest.mark.gpu

CASES = [((32, 32, 32), 10, 0.5, 1), ((48, 40, 36), 12, 0.3, 3), ((64, 64, 64), 16, 0.8, 7),
         ((24, 24, 24), 23, 0.5, 5), ((30, 20, 25), 19, 0.6, 11), ((40, 40, 40), 4, 0.2, 2),
         ((256, 256, 256), 40, 0.2, 7), ((128, 96, 160), 40, 0.5, 9),
         # one sphere moves phi by several percent: the batch path hands over to the sequential
         # loop at the first skip
         ((20, 20, 20), 10, 0.5, 4), ((28, 28, 28), 12, 0.7, 6), ((36, 36, 36), 14, 0.4, 8),
         ((22, 26, 24), 11, 0.25, 12)]


@pytest.mark.parametrize("dims,d,phi,seed", CASES)
def test_device_ras_equals_host(dims, d, phi, seed):
    p = P.GenerateParams(dims=dims, sphere_diameter=d, target_porosity=phi, seed=seed)
    host = P.generate(P.GeometryKind.Ras3D, p)
    dev = P.generate(P.GeometryKind.Ras3D, p, device=0)
    assert dev.d == 3 and dev.dims == host.dims
    assert np.array_equal(dev.types, host.types)
    assert dev.bc.velocity == host.bc.velocity and dev.bc.density == host.bc.density


def test_device_ras_rejects_like_reference():
    for p in (P.GenerateParams(dims=(16, 16, 16), sphere_diameter=16, target_porosity=0.5),
              P.GenerateParams(dims=(16, 16, 16), sphere_diameter=1, target_porosity=0.5),
              P.GenerateParams(dims=(16, 16, 16), sphere_diameter=4, target_porosity=1.0)):
        with pytest.raises(P.ConfigError):
            P.generate(P.GeometryKind.Ras3D, p, device=0)


def test_device_generator_other_kinds_delegate():
    p = P.GenerateParams(dims=(40, 30, 1))
    assert np.array_equal(P.generate(P.GeometryKind.Cavity2D, p, device=0).types,
                          P.generate(P.GeometryKind.Cavity2D, p).types)


def test_device_ras_is_fast_at_512():
    p = P.GenerateParams(dims=(512, 512, 512), sphere_diameter=40, target_porosity=0.5, seed=7)
    P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(64, 64, 64), sphere_diameter=10,
                                                      target_porosity=0.5), device=0)  # warm
    t0 = time.time()
    g = P.generate(P.GeometryKind.Ras3D, p, device=0)
    dt = time.time() - t0
    phi = P.porosity(g).phi
    assert 0.49 <= phi <= 0.51
    assert dt < 5.0, dt
