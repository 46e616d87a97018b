"""The step kernel's shared-reciprocal velocity division equals IEEE m/rho bit for bit (f64 and the
f32 engine's binary32 version)."""
import numpy as np
import pytest

from paper_1703_08015_b200 import _native

pytestmark = pytest.mark.gpu


def test_divide_matches_ieee():
    rng = np.random.default_rng(0)
    n = 2_000_000
    rho = np.concatenate([1 + 0.1 * rng.standard_normal(n // 2), np.exp(rng.uniform(-700, 700, n // 2))])
    m = np.concatenate([0.05 * rng.standard_normal((n // 2, 3)),
                        np.exp(rng.uniform(-700, 700, (n // 2, 3))) * rng.choice([-1, 1], (n // 2, 3))])
    edge_r = np.array([1.0, 1.0, 1.0, 1e-310, 3.0, 1e300, 0.7, 2.0 ** -480, 2.0 ** 480])
    edge_m = np.array([[0.0, -0.0, 1e-320], [1e-300, -1e-300, 5e-324], [np.inf, -np.inf, np.nan],
                       [1.0, 1e-10, -0.0], [1.0, 2.0, 3.0], [1e308, -1e300, 1e-10],
                       [0.1, 0.2, 0.3], [2.0 ** -470, 1.0, 0.0], [2.0 ** 479, -1.0, 0.0]])
    rho = np.concatenate([rho, edge_r])
    m = np.ascontiguousarray(np.concatenate([m, edge_m]))
    out = np.empty_like(m)
    _native.check(_native.lib().splbm_selftest_divide(rho.size, m.ravel(), rho, out.ravel()))
    with np.errstate(all="ignore"):
        ref = m / rho[:, None]
    same = (out.view(np.uint64) == ref.view(np.uint64)) | (np.isnan(out) & np.isnan(ref))
    assert same.all(), (m[~same.all(1)][:5], rho[~same.all(1)][:5])


def test_divide_f32_matches_ieee():
    rng = np.random.default_rng(1)
    n = 4_000_000
    # velocity-like tuples, then wide exponents (guard edges at 2^+-50), then significands near
    # 2 (the largest relative rounding error of RN(m * RN(1/rho)))
    rho = np.concatenate([1 + 0.1 * rng.standard_normal(n // 4), np.exp2(rng.uniform(-120, 120, n // 4)),
                          np.exp2(rng.integers(-60, 60, n // 4)) * rng.uniform(1.9, 2.0, n // 4),
                          rng.uniform(0.5, 2.0, n // 4)]).astype(np.float32)
    m = np.concatenate([0.05 * rng.standard_normal((n // 4, 3)),
                        np.exp2(rng.uniform(-120, 120, (n // 4, 3))) * rng.choice([-1, 1], (n // 4, 3)),
                        np.exp2(rng.integers(-60, 60, (n // 4, 3))) * rng.uniform(1.9, 2.0, (n // 4, 3)),
                        rng.uniform(-2.0, 2.0, (n // 4, 3))]).astype(np.float32)
    edge_r = np.array([1.0, 1.0, 1.0, 1e-40, 3.0, 1e38, 0.7, 2.0 ** -50, 2.0 ** 50, 2.0 ** -51],
                      np.float32)
    edge_m = np.array([[0.0, -0.0, 1e-45], [1e-38, -1e-38, 1e-45], [np.inf, -np.inf, np.nan],
                       [1.0, 1e-10, -0.0], [1.0, 2.0, 3.0], [3e38, -1e30, 1e-10],
                       [0.1, 0.2, 0.3], [2.0 ** -50, 1.0, 0.0], [2.0 ** 50, -1.0, 0.0],
                       [1.0, 2.0 ** -50, 2.0 ** 50]], np.float32)
    rho = np.concatenate([rho, edge_r])
    m = np.ascontiguousarray(np.concatenate([m, edge_m]))
    out = np.empty_like(m)
    _native.check(_native.lib().splbm_selftest_divide_f32(rho.size, m.ctypes.data, rho.ctypes.data,
                                                          out.ctypes.data))
    with np.errstate(all="ignore"):
        ref = m / rho[:, None]
    same = (out.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(out) & np.isnan(ref))
    assert same.all(), (m[~same.all(1)][:5], rho[~same.all(1)][:5])
