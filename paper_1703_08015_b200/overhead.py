"""Ancillary-transfer accounting of the T2C scheme (reference overhead.hpp:14-96, overhead.cpp).

Only the T2C subset is on this path: node costs (Eq. 9/10), the T2C overheads (Eq. 24/35/41)
and the bandwidth utilisation (Eq. 43). The TGB / CM / FIA formulas and report rendering are
pure analytics outside the hot path.
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError, DomainError
from .lattice import LatticeDescriptor


@dataclass
class CostParams:  # overhead.hpp:14-28
    lat: LatticeDescriptor | None = None
    s_d: float = 8
    s_t: float = 2
    s_ti: float = 4
    s_gbi: float = 4
    s_idx_cm: float = 4
    s_idx_fia: float = 4
    s_b: float = 32
    a: int = 4

    def validate(self) -> None:  # overhead.cpp:26-37
        if self.lat is None:
            raise ConfigError("cost parameters need a lattice")
        if self.s_d not in (4, 8):
            raise ConfigError("s_d must be 4 or 8 bytes")
        for v in (self.s_t, self.s_ti, self.s_gbi, self.s_b):
            if not v > 0:
                raise ConfigError("size parameters must be positive")
        for v in (self.s_idx_cm, self.s_idx_fia):
            if v < 0:
                raise ConfigError("index sizes must be non-negative")
        if self.a < 2:
            raise ConfigError("tile edge must be at least 2")


@dataclass
class GeometryStats:  # overhead.hpp:32-46
    phi: float = 1.0
    phi_t: float = 1.0
    alpha_m: float = 1.0
    alpha_b: float = 1.0
    ratio_tiles: float = 1.0
    alpha_b_estimated: bool = False

    @classmethod
    def manual(cls, phi, phi_t, alpha_m, ratio_tiles=4.0):  # overhead.cpp:47-57
        return cls(phi, phi_t, alpha_m, 0.95 * alpha_m, ratio_tiles, True)


@dataclass
class NodeCosts:
    m_node: float
    b_node: float


def node_costs(p: CostParams) -> NodeCosts:  # overhead.cpp:59-62
    q = p.lat.q
    return NodeCosts(q * p.s_d, 2.0 * q * p.s_d)


@dataclass
class TileOverhead:  # overhead.hpp:67-84
    delta_m: float
    m_solid_fill: float
    m_node_type: float
    m_sync: float
    m_addressing: float
    delta_b: float
    b_node_type: float
    b_addressing: float
    delta_b_bt: float
    predicted_perf: float


def overhead_t2c(p: CostParams, s: GeometryStats) -> TileOverhead:  # overhead.cpp:99-118
    p.validate()
    if not s.phi_t > 0.0:
        raise DomainError("tile porosity must be positive")
    nc = node_costs(p)
    n_tn = float(p.a) ** p.lat.d
    solid_fill = 1.0 / s.phi_t - 1.0
    m_node_type = p.s_t / (nc.m_node * s.phi_t)
    m_sync = 1.0 / s.phi_t
    m_addr = s.ratio_tiles * p.s_ti / (s.phi_t * n_tn * nc.m_node)
    bt = n_tn * s.phi_t * nc.b_node
    b_node_type = (p.a + 2.0) ** p.lat.d * p.s_t / bt
    b_addr = (p.lat.q - 1) * p.s_ti / bt
    delta_b = b_node_type + b_addr
    return TileOverhead(solid_fill + m_node_type + m_sync + m_addr, solid_fill, m_node_type, m_sync,
                        m_addr, delta_b, b_node_type, b_addr, delta_b + (1.0 / s.phi_t - 1.0),
                        1.0 / (1.0 + delta_b))


def bandwidth_utilization(p_mlups: float, p: CostParams, b_peak: float) -> float:
    """BU = P * 1e6 * B_node / B_peak (Eq. 43, overhead.cpp:148-152)."""
    if not b_peak > 0.0:
        raise DomainError("peak bandwidth must be positive")
    if p_mlups < 0.0:
        raise DomainError("performance must be non-negative")
    return p_mlups * 1e6 * node_costs(p).b_node / b_peak
