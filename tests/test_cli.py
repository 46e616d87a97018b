"""CLI subcommands in the reference's key=value format and exit codes (test_cli.cpp analogue)."""
import io
import subprocess
import sys

import pytest

import paper_1703_08015_b200 as P
from paper_1703_08015_b200 import cli


def run(argv):
    out = io.StringIO()
    rc = cli.main(argv, out=out)
    kv = dict(line.split("=", 1) for line in out.getvalue().splitlines() if "=" in line)
    return rc, kv


def test_generate_and_reload(tmp_path):
    path = str(tmp_path / "ras.splb")
    rc, kv = run(["generate", path, "--set", "geometry.kind=ras3d", "--set", "geometry.dims=32 32 32",
                  "--set", "geometry.diameter=8", "--set", "geometry.porosity=0.7",
                  "--set", "geometry.seed=3"])
    assert rc == 0 and kv["nodes"] == "32768" and kv["output"] == path
    g = P.load_geometry_file(path)
    assert abs(float(kv["phi"]) - P.porosity(g).phi) < 1e-12


def test_stats_matches_library(tmp_path):
    cfgf = tmp_path / "c.cfg"
    cfgf.write_text("geometry.kind = cavity2d\ngeometry.dims = 33 32\nsim.tile = 16  # reference default\n")
    rc, kv = run(["stats", "-c", str(cfgf)])
    assert rc == 0
    g = P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(33, 32, 1)))
    assert float(kv["phi_t"]) == pytest.approx(P.tile_stats(P.build_tile_grid(g, 16)).phi_t, abs=1e-12)
    assert kv["n_tiles"] == "6" and "t2c.delta_b" in kv and "t2c.delta_b_bt" in kv


def test_exit_codes():
    assert run(["stats"])[0] == cli.EXIT_CONFIG  # no geometry
    assert run(["stats", "--set", "geometry.kind=nope"])[0] == cli.EXIT_CONFIG
    assert run(["run", "--set", "geometry.kind=cavity2d", "--set", "geometry.dims=16 16",
                "--set", "sim.collision=trt"])[0] == cli.EXIT_CONFIG


def test_module_entry_point():
    r = subprocess.run([sys.executable, "-m", "paper_1703_08015_b200", "stats", "--set",
                        "geometry.kind=channel3d", "--set", "geometry.dims=16 12 12"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "phi_t=" in r.stdout


@pytest.mark.gpu
def test_run_and_bench_on_device():
    rc, kv = run(["run", "--set", "geometry.kind=cavity2d", "--set", "geometry.dims=64 64",
                  "--set", "sim.steps=100", "--set", "sim.tile=16"])
    assert rc == 0 and kv["steps"] == "100" and float(kv["mlups"]) > 0
    assert int(kv["tile_visits"]) == 100 * 16
    rc, kv = run(["bench", "--set", "geometry.kind=channel3d", "--set", "geometry.dims=64 32 32",
                  "--set", "bench.steps=40", "--set", "bench.mem_bandwidth=6.537e12",
                  "--set", "bench.models=bgk-quasi bgk-incompressible"])
    assert rc == 0 and float(kv["bench.t2c-b200.bgk-quasi.mlups"]) > 0
    mlups = float(kv["bench.t2c-b200.bgk-incompressible.mlups"])
    assert float(kv["bench.t2c-b200.bgk-incompressible.bu"]) == pytest.approx(mlups * 1e6 * 304 / 6.537e12, rel=1e-5)


def test_precision_and_storage_keys():
    """sim.precision (f32|f64, the reference's parse_precision, splbm.cpp:36-40) sets the stats
    model's s_d; sim.storage selects the single-copy engine; bad values are configuration errors."""
    c = cli.Config({"sim.storage": "single-copy"})
    assert cli.build_sim(c).single_copy
    assert not cli.build_sim(cli.Config()).single_copy
    assert cli.parse_precision(cli.Config({"sim.precision": "f32"})) == "f32"
    with pytest.raises(P.ConfigError):
        cli.parse_precision(cli.Config({"sim.precision": "f16"}))
    with pytest.raises(P.ConfigError):
        cli.build_sim(cli.Config({"sim.storage": "triple"}))
    base = ["stats", "--set", "geometry.kind=channel3d", "--set", "geometry.dims=16 12 12"]
    rc64, kv64 = run(base)
    rc32, kv32 = run(base + ["--set", "sim.precision=f32"])
    assert rc64 == rc32 == 0
    # delta_b = ((a+2)^d s_t + (q-1) s_ti) / (n_tn phi_t B_node) doubles when s_d halves
    assert float(kv32["t2c.delta_b"]) == pytest.approx(2 * float(kv64["t2c.delta_b"]), rel=1e-12)
    assert run(base + ["--set", "sim.precision=f16"])[0] == cli.EXIT_CONFIG


@pytest.mark.gpu
def test_run_f32_and_single_copy_on_device():
    base = ["run", "--set", "geometry.kind=cavity2d", "--set", "geometry.dims=64 64",
            "--set", "sim.steps=50", "--set", "sim.tile=16"]
    rc, kv = run(base)
    rc1, kv1 = run(base + ["--set", "sim.storage=single-copy"])
    rc2, kv2 = run(base + ["--set", "sim.precision=f32"])
    assert rc == rc1 == rc2 == 0
    assert kv1["mass_final"] == kv["mass_final"]  # bit-identical engines
    assert float(kv2["mass_final"]) == pytest.approx(float(kv["mass_final"]), rel=1e-5)


@pytest.mark.gpu
def test_bench_failure_step_is_absolute(capsys):
    """A blow-up after the warm-up reports warmup + s + 1 like the reference (splbm.cpp:250): the
    device failure stamp already counts from initialize, so the CLI must not add the warm-up."""
    g = cli.build_geometry(cli.Config({"geometry.kind": "cavity2d", "geometry.dims": "32 32"}))
    for u in (0.7, 0.5, 0.4, 0.3, 0.25, 0.2, 0.15, 0.1):  # an unstable start failing after step 3
        e = P.TileEngineT2C(g, 16, P.FluidModel(tau=0.5001))
        e.initialize_uniform(1.0, (u, 0.8 * u, 0.0))
        ok, first = e.step_n(5000)
        if not ok and first > 3:
            break
    else:
        pytest.skip("no unstable configuration failing after step 3")
    base = ["--set", "geometry.kind=cavity2d", "--set", "geometry.dims=32 32", "--set",
            "sim.tile=16", "--set", "sim.tau=0.5001", "--set", f"sim.initial_velocity={u} {0.8 * u}"]
    warm = first - 2
    rc, _ = run(["bench", *base, "--set", f"bench.warmup={warm}", "--set", "bench.steps=50"])
    assert rc == cli.EXIT_NUMERICAL
    err = capsys.readouterr().err
    assert f"non-finite state at step {first}" in err, err
