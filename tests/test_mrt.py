"""MRT collision (reference collision.hpp:54-63, collision.cpp:86-113)."""
import numpy as np
import pytest

import paper_1703_08015_b200 as P
from paper_1703_08015_b200.lattice import mrt_kernel

from cases import CASES, make_oracle


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("rates", [None, "custom"])
def test_operator_matrix_bit_identical(d, rates, ref, oracle):
    q = 9 if d == 2 else 19
    r = None if rates is None else np.linspace(0.2, 1.7, q)
    K = mrt_kernel(d, 0.9, r)
    assert np.array_equal(K.view(np.uint64), ref.mrt_kernel(d, 0.9, r).view(np.uint64))
    assert np.array_equal(K.view(np.uint64), oracle.mrt_kernel(d, 0.9, r).view(np.uint64))


@pytest.mark.parametrize("name", ["plug_channel_a8_odd", "ras24_periodic", "cavity3d_odd_incompr",
                                  "random_solids_a3"])
def test_oracle_mrt_matches_reference(name, ref, oracle):
    factory, a, tau, inc, per, init = CASES[name]
    g = factory()
    rg = ref.RefGeometry.from_raster(g.d, g.dims, g.types, g.bc.velocity, g.bc.density)
    re = ref.RefEngine(rg, "t2c", a, tau, incompressible=inc, mrt=True, periodic=per)
    oe = oracle.OracleT2C(g.types, g.d, g.dims, a, tau, incompressible=inc, periodic=per,
                          bc_velocity=g.bc.velocity, bc_density=g.bc.density, mrt=True)
    if init == "uniform":
        re.initialize_uniform()
        oe.initialize_uniform()
    else:
        re.initialize_wavy()
        oe.initialize_wavy()
    re.step(15)
    oe.step(15)
    assert np.array_equal(re.pdf().view(np.uint64), oe.current_pdf().view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["specialised", "generic"])
@pytest.mark.parametrize("name", ["plug_channel_a8_odd", "ras24_periodic", "cavity3d_odd_incompr",
                                  "random_solids_a3", "channel3d_32", "cavity2d_64_a4"])
def test_device_mrt_bitwise(name, path, oracle, monkeypatch):
    """`specialised`: the default engine (power-of-two tiles run the step compiled for this
    operator, csrc/mrt_jit.cpp); `generic`: SPLBM_MRT_JIT=0."""
    factory, a, tau, inc, per, init = CASES[name]
    g = factory()
    model = P.FluidModel(P.Compressibility.Incompressible if inc else P.Compressibility.QuasiCompressible,
                         P.CollisionKind.MRT, tau=tau)
    monkeypatch.setenv("SPLBM_MRT_JIT", "1" if path == "specialised" else "0")
    de = P.TileEngineT2C(g, a, model, per)
    assert de.info.mrt_specialised == (path == "specialised" and a in (2, 4, 8, 16))
    oe = oracle.OracleT2C(g.types, g.d, g.dims, a, tau, incompressible=inc, periodic=per,
                          bc_velocity=g.bc.velocity, bc_density=g.bc.density, mrt=True)
    if init == "uniform":
        de.initialize_uniform()
        oe.initialize_uniform()
    else:
        de.initialize(oracle.wavy)
        oe.initialize_wavy()
    assert de.step_n(40)[0] and oe.step(40)[0]
    fluid = np.broadcast_to((oe.tiles["types"] != 0)[:, None, :], (oe.T, oe.q, oe.n_tn)).ravel()
    assert np.array_equal(de.get_pdf()[fluid].view(np.uint64), oe.current_pdf()[fluid].view(np.uint64))


@pytest.mark.gpu
def test_mrt_uniform_rates_reproduce_bgk():  # acceptance.cpp:237-252: <= 1e-12
    g = P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(32, 32, 1), lid_speed=0.05))
    bgk = P.run_simulation(g, P.SimConfig(tile=16, steps=100, model=P.FluidModel(tau=0.8)))
    mrt = P.run_simulation(g, P.SimConfig(tile=16, steps=100, model=P.FluidModel(
        collision=P.CollisionKind.MRT, tau=0.8, mrt_rates=[1 / 0.8] * 9)))
    assert P.linf_rel_diff(bgk.fields, mrt.fields) <= 1e-12


def _specialise(d, inc, f32, tau, rates, tile):
    import ctypes as C
    from paper_1703_08015_b200 import _native
    L = _native.lib()
    n = C.c_int()
    r = None if rates is None else np.ascontiguousarray(rates, np.float64)
    rc = L.splbm_mrt_specialise(d, int(inc), int(f32), C.c_double(tau),
                                None if r is None else r.ctypes.data_as(C.c_void_p), tile, C.byref(n))
    return rc, n.value, L.splbm_last_error().decode(errors="replace")


def test_specialised_operator_shares_products():
    """Default rates at tau 0.8: the rows of K share 139 of the 361 D3Q19 products (46 of 81 in
    D2Q9); a generic operator (custom rates) shares fewer but never more than q*q."""
    assert _specialise(3, False, False, 0.8, None, 0)[:2] == (0, 139)
    assert _specialise(2, False, False, 0.8, None, 0)[:2] == (0, 46)
    rc, n, _ = _specialise(3, False, False, 0.9, np.linspace(0.2, 1.7, 19), 0)
    assert rc == 0 and 19 <= n <= 361
    assert _specialise(3, False, False, 0.4, None, 0)[0] == 1  # ConfigError, tau <= 0.5


@pytest.mark.parametrize("d,tile", [(3, 2), (3, 4), (2, 2), (2, 4), (2, 8), (2, 16)])
@pytest.mark.parametrize("f32", [False, True])
def test_specialised_step_compiles(d, tile, f32):
    """The specialised step compiles with NVRTC for every power-of-two tile edge (no GPU needed)."""
    for inc in (False, True):
        rc, _, err = _specialise(d, inc, f32, 0.7, None, tile)
        assert rc == 0, err
    assert _specialise(3, False, f32, 0.7, None, 8)[0] == 1  # 3D a = 8: generic kernel only


@pytest.mark.gpu
@pytest.mark.parametrize("tau,rates", [(0.8, None), (0.6, None), (1.3, None), (0.9, "custom")])
@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("kind", ["ras3d", "cavity2d", "ras3d_a2", "cavity2d_a16"])
@pytest.mark.parametrize("single_copy", [False, True])
def test_specialised_equals_generic(kind, precision, tau, rates, single_copy, monkeypatch):
    """Every PDF slot of the specialised MRT step (two copies, or both single-copy phases) equals
    the generic one bit for bit."""
    if kind.startswith("ras3d"):
        g, a, per = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(
            dims=(32, 32, 32), sphere_diameter=10, target_porosity=0.6, seed=4)), 2 if kind.endswith("a2") else 4, 7
    else:
        g, a, per = P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(96, 64, 1))), \
            16 if kind.endswith("a16") else 8, 0
    q = 19 if g.d == 3 else 9
    r = list(np.linspace(0.3, 1.6, q)) if rates else []
    for inc in (P.Compressibility.QuasiCompressible, P.Compressibility.Incompressible):
        out = []
        for jit in ("1", "0"):
            monkeypatch.setenv("SPLBM_MRT_JIT", jit)
            e = P.TileEngineT2C(g, a, P.FluidModel(inc, P.CollisionKind.MRT, tau=tau, mrt_rates=r), per,
                                precision=precision, single_copy=single_copy)
            assert e.info.mrt_specialised == (jit == "1")
            e.initialize(lambda x, y, z: (1.0 + 0.01 * np.sin(0.3 * x + 0.1 * z), 0.01 * np.cos(0.2 * y),
                                          0.005 * np.sin(0.1 * x), 0.002 * np.cos(0.3 * z)))
            assert e.step_n(30)[0]
            out.append(e.get_pdf().view(np.uint8).copy())
        assert np.array_equal(out[0], out[1]), (inc, precision, tau, rates)


@pytest.mark.gpu
def test_mrt_without_nvrtc_runs_the_generic_kernel(tmp_path):
    """Without libnvrtc (SPLBM_NVRTC pointing nowhere) an MRT engine falls back to the generic
    ahead-of-time MRT kernel and produces the same bits."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, paper_1703_08015_b200 as P\n"
        "g = P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(64, 64, 1)))\n"
        "e = P.TileEngineT2C(g, 4, P.FluidModel(collision=P.CollisionKind.MRT, tau=0.7))\n"
        "e.initialize_uniform(); assert e.step_n(20)[0]\n"
        "np.save(%r, e.get_pdf()); print(e.info.mrt_specialised)\n")
    outs = []
    for k, nvrtc in enumerate(("/nonexistent/libnvrtc.so", None)):
        env = dict(os.environ)
        env.pop("SPLBM_NVRTC", None)
        if nvrtc:
            env["SPLBM_NVRTC"] = nvrtc
        f = str(tmp_path / f"pdf{k}.npy")
        r = subprocess.run([sys.executable, "-c", code % f], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr
        outs.append((r.stdout.strip().splitlines()[-1], np.load(f)))
    assert outs[0][0] == "0" and outs[1][0] == "1"
    assert np.array_equal(outs[0][1].view(np.uint64), outs[1][1].view(np.uint64))
