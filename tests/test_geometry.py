"""Geometry generators and formats (reference geometry.cpp) — product vs reference, bytewise."""
import os

import numpy as np
import pytest

import paper_1703_08015_b200 as P


@pytest.mark.parametrize("kind,dims,kw", [
    ("cavity2d", (64, 48, 1), dict(lid=0.05)),
    ("cavity2d", (256, 256, 1), dict(lid=0.07)),
    ("cavity3d", (24, 20, 18), dict(lid=0.05)),
    ("channel2d", (96, 48, 1), dict(inlet=0.04)),
    ("channel2d", (33, 17, 5), dict(inlet=0.02, outlet=1.01)),  # 3D dims reduce to 2D
    ("ras3d", (48, 48, 48), dict(diameter=12, target=0.75, seed=9)),
    ("ras3d", (96, 64, 48), dict(diameter=20, target=0.3, seed=3)),
    ("ras3d", (64, 64, 64), dict(diameter=16, target=0.5, seed=7)),
])
def test_generators_match_reference(kind, dims, kw, ref):
    rg = ref.RefGeometry.generate(kind, dims, **kw)
    kinds = {"cavity2d": P.GeometryKind.Cavity2D, "cavity3d": P.GeometryKind.Cavity3D,
             "channel2d": P.GeometryKind.Channel2D, "ras3d": P.GeometryKind.Ras3D}
    p = P.GenerateParams(dims=dims, lid_speed=kw.get("lid", 0.05), inlet_speed=kw.get("inlet", 0.05),
                         outlet_density=kw.get("outlet", 1.0), sphere_diameter=kw.get("diameter", 40),
                         target_porosity=kw.get("target", 0.9), seed=kw.get("seed", 0))
    g = P.generate(kinds[kind], p)
    d, rdims, vel, rho = rg.info()
    assert g.d == d and tuple(g.dims) == rdims
    assert np.array_equal(g.types, rg.types())
    assert tuple(g.bc.velocity) == vel and g.bc.density == rho


def test_generator_errors():
    with pytest.raises(P.ConfigError):
        P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(2, 8, 1)))
    with pytest.raises(P.ConfigError):
        P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(16, 16, 16), sphere_diameter=16))
    with pytest.raises(P.ConfigError):
        P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(16, 16, 16), sphere_diameter=4,
                                                          target_porosity=1.0))


def test_channel3d_config1_counts():
    """BASELINE configs[1]: 128^3 channel, N_f = 128*126*126 = 2,032,128."""
    g = P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(128, 128, 128)))
    assert g.fluid_count() == 2032128
    v = g.view3d()
    assert (v[1:-1, 1:-1, 0] == P.NodeType.VelocityBC).all()
    assert (v[1:-1, 1:-1, -1] == P.NodeType.PressureBC).all()
    assert (v[0] == 0).all() and (v[:, 0] == 0).all()
    assert g.bc.velocity == (0.05, 0.0, 0.0) and g.bc.density == 1.0


def test_vessel_tree_deterministic():
    p = P.GenerateParams(dims=(512, 512, 1), target_porosity=0.2, seed=11)
    a = P.generate(P.GeometryKind.Vessel2D, p)
    b = P.generate(P.GeometryKind.Vessel2D, p)
    assert np.array_equal(a.types, b.types)
    phi = P.porosity(a).phi
    assert 0.2 <= phi < 0.35
    v = a.view3d()[0]
    assert (v[:, 0] != P.NodeType.Fluid).all() and (v[:, 0] == P.NodeType.VelocityBC).any()
    assert (v[:, -1] == P.NodeType.PressureBC).any()


@pytest.mark.parametrize("fmt", [P.GeometryFormat.Binary, P.GeometryFormat.Text])
def test_format_roundtrip_and_reference_interop(fmt, tmp_path, ref):
    g = P.generate(P.GeometryKind.Channel2D, P.GenerateParams(dims=(40, 12, 1), inlet_speed=0.03,
                                                              outlet_density=1.02))
    path = str(tmp_path / "g.splb")
    P.save_geometry_file(g, path, fmt)
    h = P.load_geometry_file(path)
    assert h.d == g.d and h.dims == g.dims and np.array_equal(h.types, g.types)
    if fmt == P.GeometryFormat.Text:
        assert h.bc.velocity == g.bc.velocity and h.bc.density == g.bc.density
    # the reference loads what we wrote and we load what it writes
    rg = ref.RefGeometry.load(path)
    assert np.array_equal(rg.types(), g.types)
    path2 = str(tmp_path / "r.splb")
    rg.save(path2, binary=fmt == P.GeometryFormat.Binary)
    assert open(path2, "rb").read() == open(path, "rb").read()


def test_format_errors(tmp_path):
    with pytest.raises(P.IoError):
        P.load_geometry_file(str(tmp_path / "missing.splb"))
    bad = tmp_path / "bad.splb"
    bad.write_bytes(b"SPLB\x02\x02" + b"\x00" * 12)
    with pytest.raises(P.ParseError):
        P.load_geometry_file(str(bad))
    txt = tmp_path / "bad.txt"
    txt.write_text("D2 3 2\n...\n.x.\n")
    with pytest.raises(P.ParseError):
        P.load_geometry_file(str(txt))
