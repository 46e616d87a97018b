"""`python -m paper_1703_08015_b200 generate|stats|run|bench` — the reference CLI's subcommands
(proj/tools/splbm.cpp:370-485) for the B200 engine, with its configuration keys, key=value output
and exit codes (0 ok, 2 configuration error, 3 numerical error; splbm.cpp:18-20).

Configuration is layered like the reference: an optional `key = value` file (dotted keys, later
keys win; config.cpp:20-41), then `--set key=value` overrides. Method name: `t2c-b200`
(the name INTEGRATION.md adds to parse_method, splbm.cpp:29-34).
"""
from __future__ import annotations

import argparse
import sys

from . import engine as E
from . import geometry as G
from . import overhead as O
from .errors import ConfigError, Error, NumericalError
from .lattice import CollisionKind, Compressibility, FluidModel, solver_lattice
from .tiling import Periodicity, build_tile_grid, tile_stats

EXIT_OK, EXIT_CONFIG, EXIT_NUMERICAL = 0, 2, 3
KINDS = {"cavity2d": G.GeometryKind.Cavity2D, "cavity3d": G.GeometryKind.Cavity3D,
         "channel2d": G.GeometryKind.Channel2D, "ras3d": G.GeometryKind.Ras3D,
         "channel3d": G.GeometryKind.Channel3D, "vessel2d": G.GeometryKind.Vessel2D}


class Config(dict):
    """key = value configuration with dotted keys (reference config.cpp)."""

    @classmethod
    def parse(cls, text: str) -> "Config":
        c = cls()
        for n, raw in enumerate(text.splitlines(), 1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise ConfigError(f"expected 'key = value' on line {n}")
            k, v = line.split("=", 1)
            c[k.strip()] = v.strip()
        return c

    def get_str(self, k, default=None):
        return self.get(k, default)

    def get_float(self, k, default):
        try:
            return float(self[k]) if k in self else default
        except ValueError as ex:
            raise ConfigError(f"{k} must be a number") from ex

    def get_int(self, k, default):
        try:
            return int(self[k]) if k in self else default
        except ValueError as ex:
            raise ConfigError(f"{k} must be an integer") from ex

    def get_list(self, k):
        v = self.get(k, "")
        return [x.strip() for x in v.replace(",", " ").split() if x.strip()]


def parse_dims(spec: str):
    parts = [int(x) for x in spec.replace("x", " ").replace(",", " ").split()]
    if len(parts) not in (2, 3):
        raise ConfigError("geometry.dims must have 2 or 3 entries")
    return tuple(parts + [1] * (3 - len(parts)))


def parse_periodic(spec: str) -> Periodicity:  # splbm.cpp:42-57
    per = Periodicity()
    if spec in ("", "none", None):
        return per
    for ch in spec:
        if ch in "xyz":
            setattr(per, ch, True)
        elif ch not in ", ":
            raise ConfigError("periodic axes must be drawn from x,y,z")
    return per


def build_geometry(cfg: Config) -> G.Geometry:  # splbm.cpp:91-116
    if "geometry.path" in cfg:
        g = G.load_geometry_file(cfg["geometry.path"])
    elif "geometry.kind" in cfg:
        kind = cfg["geometry.kind"]
        if kind not in KINDS:
            raise ConfigError(f"unknown geometry kind: {kind}")
        p = G.GenerateParams(dims=parse_dims(cfg.get("geometry.dims", "")))
        p.lid_speed = cfg.get_float("geometry.lid_velocity", p.lid_speed)
        p.inlet_speed = cfg.get_float("geometry.inlet_velocity", p.inlet_speed)
        p.outlet_density = cfg.get_float("geometry.outlet_density", p.outlet_density)
        p.sphere_diameter = cfg.get_int("geometry.diameter", p.sphere_diameter)
        p.target_porosity = cfg.get_float("geometry.porosity", p.target_porosity)
        p.seed = cfg.get_int("geometry.seed", 0)
        g = G.generate(KINDS[kind], p)
    else:
        raise ConfigError("set geometry.path or geometry.kind")
    if "bc.velocity" in cfg:
        v = [float(x) for x in cfg["bc.velocity"].replace(",", " ").split()]
        g.bc.velocity = tuple((v + [0.0, 0.0, 0.0])[:3])
    g.bc.density = cfg.get_float("bc.density", g.bc.density)
    return g


def build_model(cfg: Config) -> FluidModel:  # splbm.cpp:118-134
    coll = cfg.get("sim.collision", "bgk")
    if coll not in ("bgk", "mrt"):
        raise ConfigError("sim.collision must be bgk or mrt")
    comp = cfg.get("sim.compressibility", "quasi")
    if comp in ("quasi", "quasi-compressible"):
        c = Compressibility.QuasiCompressible
    elif comp == "incompressible":
        c = Compressibility.Incompressible
    else:
        raise ConfigError("sim.compressibility must be quasi or incompressible")
    return FluidModel(c, CollisionKind.MRT if coll == "mrt" else CollisionKind.BGK,
                      tau=cfg.get_float("sim.tau", 0.8))


def parse_precision(cfg: Config) -> str:  # splbm.cpp:36-40
    name = cfg.get("sim.precision", "f64")
    if name not in ("f32", "f64"):
        raise ConfigError("precision must be f32 or f64")
    return name


def build_sim(cfg: Config) -> E.SimConfig:  # splbm.cpp:136-150
    method = cfg.get("sim.method", "t2c-b200")
    if method not in ("t2c-b200", "t2c"):
        raise ConfigError(f"unknown method: {method} (the B200 engine is t2c-b200)")
    sim = E.SimConfig(tile=cfg.get_int("sim.tile", 0), steps=cfg.get_int("sim.steps", 0),
                      periodic=parse_periodic(cfg.get("sim.periodic", "")),
                      model=build_model(cfg), device=cfg.get_int("sim.device", 0),
                      single_copy=cfg.get("sim.storage", "two-copy") == "single-copy")
    if cfg.get("sim.storage", "two-copy") not in ("two-copy", "single-copy"):
        raise ConfigError("sim.storage must be two-copy or single-copy")
    sim.arithmetic = cfg.get("sim.arithmetic", "exact")
    if sim.arithmetic not in ("exact", "fma"):
        raise ConfigError("sim.arithmetic must be exact or fma")
    sim.initial_density = cfg.get_float("sim.initial_density", 1.0)
    if "sim.initial_velocity" in cfg:
        v = [float(x) for x in cfg["sim.initial_velocity"].replace(",", " ").split()]
        sim.initial_velocity = tuple((v + [0.0, 0.0, 0.0])[:3])
    return sim


def kv(key, value, out):
    out.write(f"{key}={value:.12g}\n" if isinstance(value, float) else f"{key}={value}\n")


def cmd_generate(cfg, output, out):  # splbm.cpp:156-170
    g = build_geometry(cfg)
    fmt = (G.GeometryFormat.Text if output.endswith((".txt", ".geo", ".text"))
           else G.GeometryFormat.Binary)
    G.save_geometry_file(g, output, fmt)
    p = G.porosity(g)
    kv("nodes", g.node_count(), out)
    kv("phi", p.phi, out)
    kv("eta", p.eta, out)
    kv("output", output, out)


def cmd_stats(cfg, out):  # splbm.cpp:172-225, T2C subset of the overhead report
    g = build_geometry(cfg)
    lat = solver_lattice(g.d)
    a = cfg.get_int("sim.tile", 16 if g.d == 2 else 4)
    tg = build_tile_grid(g, a, parse_periodic(cfg.get("sim.periodic", "")), with_neighbours=False)
    ts = tile_stats(tg)
    p = G.porosity(g)
    params = O.CostParams(lat=lat, a=a, s_d=4.0 if parse_precision(cfg) == "f32" else 8.0,
                          s_t=cfg.get_float("cost.s_t", 2.0), s_ti=cfg.get_float("cost.s_ti", 4.0))
    gs = O.GeometryStats(phi=p.phi, phi_t=ts.phi_t, ratio_tiles=ts.ratio_tiles)
    kv("n_nodes", g.node_count(), out)
    for k, v in (("phi", p.phi), ("eta", p.eta), ("phi_t", ts.phi_t), ("eta_t", ts.eta_t),
                 ("ratio_tiles", ts.ratio_tiles)):
        kv(k, v, out)
    kv("n_tiles", ts.n_tiles, out)
    kv("n_ftiles", ts.n_ftiles, out)
    if ts.n_ftiles:
        o = O.overhead_t2c(params, gs)
        for k, v in (("delta_m", o.delta_m), ("delta_m.solid_fill", o.m_solid_fill),
                     ("delta_m.node_type", o.m_node_type), ("delta_m.sync", o.m_sync),
                     ("delta_m.addressing", o.m_addressing), ("delta_b", o.delta_b),
                     ("delta_b.node_type", o.b_node_type), ("delta_b.addressing", o.b_addressing),
                     ("delta_b_bt", o.delta_b_bt), ("predicted_perf", o.predicted_perf)):
            kv("t2c." + k, v, out)


def cmd_run(cfg, out):  # splbm.cpp:265-293 (VTK/CSV output stays on the reference)
    g = build_geometry(cfg)
    res = E.run_simulation(g, build_sim(cfg), parse_precision(cfg))
    kv("steps", res.steps, out)
    for k in ("wall_seconds", "mlups", "mass_initial", "mass_final", "mass_drift_rel"):
        kv(k, float(getattr(res, k)), out)
    kv("fluid_nodes", res.fluid_nodes, out)
    kv("tile_visits", res.tile_visits, out)
    kv("snapshots", res.snapshots_written, out)


def cmd_bench(cfg, out):  # splbm.cpp:295-366 for method t2c-b200
    g = build_geometry(cfg)
    sim = build_sim(cfg)
    warmup = cfg.get_int("bench.warmup", 10)
    steps = cfg.get_int("bench.steps", max(sim.steps, 50))
    bandwidth = cfg.get_float("bench.mem_bandwidth", 0.0)
    models = cfg.get_list("bench.models") or ["current"]
    precision = parse_precision(cfg)
    rows = []
    for model in models:
        c = Config(cfg)
        if model != "current":
            if "-" not in model:
                raise ConfigError(f"model spec must look like bgk-quasi: {model}")
            coll, comp = model.split("-", 1)
            c["sim.collision"], c["sim.compressibility"] = coll, comp
        s = build_sim(c)
        eng = E.make_engine(g, s, precision)
        eng.initialize_uniform(s.initial_density, s.initial_velocity)
        ok, failed = eng.step_n(warmup)
        if not ok:
            raise NumericalError("non-finite state in warmup", failed)
        eng.step_async(steps)
        ok, failed = eng.sync()
        if not ok:
            raise NumericalError("non-finite state", failed)  # already absolute (splbm.cpp:250)
        wall = eng.last_batch_ms() * 1e-3
        mlups = g.fluid_count() * steps / (wall * 1e6) if wall > 0 else 0.0
        cost = O.CostParams(lat=solver_lattice(g.d), s_d=4.0 if precision == "f32" else 8.0)
        bu = O.bandwidth_utilization(mlups, cost, bandwidth) if bandwidth > 0 else None
        rows.append((model, mlups, bu))
    kv("warmup", warmup, out)
    kv("steps", steps, out)
    for model, mlups, bu in rows:
        out.write(f"bench.t2c-b200.{model}.mlups={mlups:.6g}\n")
        if bu is not None:
            out.write(f"bench.t2c-b200.{model}.bu={bu:.6g}\n")


def main(argv=None, out=sys.stdout) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1703_08015_b200")
    ap.add_argument("command", choices=["generate", "stats", "run", "bench"])
    ap.add_argument("output", nargs="?", help="geometry file written by `generate`")
    ap.add_argument("-c", "--config", help="key = value configuration file")
    ap.add_argument("--set", action="append", default=[], metavar="KEY=VALUE")
    args = ap.parse_args(argv)
    try:
        cfg = Config.parse(open(args.config).read()) if args.config else Config()
        for item in args.set:
            if "=" not in item:
                raise ConfigError(f"--set expects key=value, got {item}")
            k, v = item.split("=", 1)
            cfg[k.strip()] = v.strip()
        if args.command == "generate":
            if not args.output:
                raise ConfigError("generate needs an output path")
            cmd_generate(cfg, args.output, out)
        elif args.command == "stats":
            cmd_stats(cfg, out)
        elif args.command == "run":
            cmd_run(cfg, out)
        else:
            cmd_bench(cfg, out)
        return EXIT_OK
    except NumericalError as ex:  # splbm.cpp:477-479
        sys.stderr.write(f"error: {ex}\n")
        return EXIT_NUMERICAL
    except (Error, OSError) as ex:
        sys.stderr.write(f"error: {ex}\n")
        return EXIT_CONFIG
