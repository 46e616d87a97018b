"""Ancillary-transfer accounting (overhead.cpp) against the reference and the paper's values."""
import pytest

import paper_1703_08015_b200 as P


def params(d, a=None):
    lat = P.solver_lattice(d)
    return P.CostParams(lat=lat, a=a if a else (16 if d == 2 else 4))


def test_paper_constants():  # acceptance.cpp:63-85, 175-182; test_overhead.cpp:157-164
    dense = P.GeometryStats.manual(1.0, 1.0, 1.0, 1.0)
    assert abs(P.overhead_t2c(params(3), dense).delta_b - 0.0259) <= 1e-3
    assert abs(P.overhead_t2c(params(2), dense).delta_b - 0.0184) <= 1e-3
    assert abs(P.bandwidth_utilization(682.0, params(3), 288.4e9) - 0.719) <= 1e-3
    assert abs(P.bandwidth_utilization(1060.0, params(2), 288.4e9) - 0.529) <= 1e-3
    assert P.node_costs(params(3)).b_node == 304.0 and P.node_costs(params(2)).b_node == 144.0


@pytest.mark.parametrize("d,a,phi,phi_t,ratio", [(3, 4, 0.2, 0.64, 3.1), (3, 4, 0.8, 0.94, 1.16),
                                                 (2, 4, 0.2, 0.7, 4.0), (2, 16, 1.0, 1.0, 1.0)])
def test_overhead_t2c_matches_reference(d, a, phi, phi_t, ratio, ref):
    r = ref.overhead_t2c(d, a, phi, phi_t, 1.0, ratio)
    o = P.overhead_t2c(params(d, a), P.GeometryStats.manual(phi, phi_t, 1.0, ratio))
    assert o.delta_b == r["delta_b"] and o.delta_b_bt == r["delta_b_bt"]
    assert o.b_node_type == r["b_node_type"] and o.b_addressing == r["b_addressing"]
    assert o.delta_m == r["delta_m"] and o.predicted_perf == r["predicted_perf"]
    assert P.bandwidth_utilization(1234.5, params(d, a), 8e12) == ref.bandwidth_utilization(
        d, 1234.5, 8e12)


def test_overhead_errors():
    with pytest.raises(P.ConfigError):
        P.overhead_t2c(P.CostParams(), P.GeometryStats())
    with pytest.raises(P.DomainError):
        P.overhead_t2c(params(3), P.GeometryStats(phi_t=0.0))
    with pytest.raises(P.DomainError):
        P.bandwidth_utilization(1.0, params(3), 0.0)
