import numpy as np
import pytest

import paper_1703_08015_b200 as P


def test_linf_rel_diff_semantics():  # fields.hpp:47-61
    n = 6
    mask = np.array([1, 1, 0, 1, 1, 1], np.uint8)
    a = P.FieldData(2, (6, 1, 1), mask, np.ones(n), np.zeros(n), np.zeros(n), np.zeros(n))
    b = P.FieldData(2, (6, 1, 1), mask, np.ones(n), np.zeros(n), np.zeros(n), np.zeros(n))
    assert P.linf_rel_diff(a, b) == 0.0
    b.ux[1] = 0.01
    a.ux[3] = 0.02
    assert P.linf_rel_diff(a, b) == 1.0  # |0.02-0|/0.02
    b.rho[2] = 5.0  # masked node ignored
    assert P.linf_rel_diff(a, b) == 1.0


def test_linf_rel_diff_skips_nan_like_std_max():
    """std::max(x, NaN) keeps x (fields.hpp:55-56): a NaN node must not hide the finite deviation
    of the same field."""
    n = 4
    mask = np.ones(n, np.uint8)
    z = lambda: np.zeros(n)
    a = P.FieldData(2, (4, 1, 1), mask, np.ones(n), z(), z(), z())
    b = P.FieldData(2, (4, 1, 1), mask, np.ones(n), z(), z(), z())
    a.ux[:] = [0.1, 0.2, np.nan, 0.4]
    b.ux[:] = [0.1, 0.1, 0.3, 0.4]
    assert P.linf_rel_diff(a, b) == pytest.approx(0.1 / 0.4)
    b.rho[0] = np.nan
    assert P.linf_rel_diff(a, b) == pytest.approx(0.1 / 0.4)


def test_total_mass_is_sequential(oracle):
    rng = np.random.default_rng(1)
    rho = 1 + rng.standard_normal(100000) * 1e-3
    mask = (rng.random(100000) > 0.3).astype(np.uint8)
    f = P.FieldData(3, (100000, 1, 1), mask, rho, rho, rho, rho)
    assert f.total_mass() == oracle.lib().oracle_total_mass(rho.size, rho, mask)
