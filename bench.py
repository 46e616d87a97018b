#!/usr/bin/env python3
"""Benchmark of the T2C time-step path on B200 (BASELINE.json metric: MLUPS (D3Q19 fp64 BGK) vs
porosity; % of HBM peak GB/s; at 1/2/4/8 B200).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload at N=1: BASELINE configs[1], the D3Q19 BGK fp64 128^3 channel with bounce-back walls
(velocity inlet / pressure outlet), tiles 4^3, synthetic geometry. A "step" is one LBM time step
(one launch of the fused step kernel over all tiles). value = N_f * K / device time of the K
timed steps (CUDA events on the engine stream, max over ranks). The two PDF copies (319 MB each) are
larger than L2, so no flush is needed between steps. Also reported: the MLUPS-vs-porosity sweep
(configs[2]: RAS 256^3, d=40, seed 7, periodic), the roofline of the step kernel against the
measured HBM copy peak, the CPU reference baseline, and an end-to-end number through the public
API with host buffers.

N>1 (torchrun, one process per GPU): weak scaling of the z-slab mode — every rank
owns a 128^3-node channel slab of one (128 x 128 x 128*N) duct and exchanges tile-face halos with
its neighbours over NCCL each step.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B_NODE = {2: 144.0, 3: 304.0}  # algorithmic bytes per node update, 2*q*8 (overhead.cpp:59-62)
METRIC = "MLUPS (D3Q19 fp64 BGK) vs porosity; % of HBM peak GB/s; at 1/2/4/8 B200"
WORKLOAD_1 = ("D3Q19 BGK fp64 channel 128^3 (BASELINE configs[1]), bounce-back walls, V inlet / "
              "P outlet, tiles 4^3, quasi-compressible, tau 0.8")


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clock and throttle reasons sampled every ~2 ms through NVML during the timed region
    (nvidia-smi as a fallback)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.samples = []
        self.error = None
        self._stop = threading.Event()
        self._first = threading.Event()
        self.index = index

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._first.wait(5.0)  # the first sample precedes the timed region's start
        return self

    def _run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            reasons = (getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None)
                       or N.nvmlDeviceGetCurrentClocksThrottleReasons)
            while True:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                self.samples.append((sm, mx, reasons(h)))
                self._first.set()
                if self._stop.wait(0.002):
                    return
        except Exception as ex:  # noqa: BLE001 - fall back to nvidia-smi
            self.error = repr(ex)
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                sm, mx, rs = [v.strip() for v in out.split(",")]
                self.samples.append((float(sm), float(mx), int(rs, 16)))
            except Exception:
                self._first.set()
                return
            self._first.set()
            self._stop.wait(0.02)

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0,
                    "error": self.error}
        reasons = sorted({n for _, _, rs in self.samples for n, bit in self.REASONS.items()
                          if rs & bit})
        return {"sm_mhz": float(np.median([s[0] for s in self.samples])),
                "sm_max_mhz": float(max(s[1] for s in self.samples)), "reasons": reasons,
                "samples": len(self.samples)}


def load_ncu_traffic(workload):
    """dram bytes per launch of the step kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_step_kernel.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    rec = d.get(workload)
    return rec.get("dram_bytes_per_launch") if rec else None


# ---------------------------------------------------------------------------------------------
def channel_geometry(P, dims):
    return P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=dims, inlet_speed=0.05,
                                                                  outlet_density=1.0))


def time_steps(eng, K, W, sampler_index=0):
    """W warm-up steps, then exactly K timed steps in one device batch (events on the engine
    stream, synchronised on both sides)."""
    if W > 0:
        ok, _ = eng.step_n(W)
        assert ok, "non-finite state during warm-up"
    eng.sync()
    l0 = eng.launch_count()
    with ClockSampler(sampler_index) as cs:
        eng.step_async(K)
        ok, failed = eng.sync()
    assert ok, f"non-finite state at step {failed}"
    ms = eng.last_batch_ms()
    return ms, eng.launch_count() - l0, cs.summary()


NCU_CASE = {0.2094: "ras256_phi02", 0.509: "ras256_phi05"}  # sweep points with a committed ncu capture


def accounting(P, eng, nf, bnode, workload=None):
    """The paper's ancillary-transfer accounting for one run: the T2C overhead model
    (overhead_t2c with the measured phi_t and tile ratio, Eqs. 35/41), the geometric lower bounds
    of the per-tile SoA layout at 32-B sector and 128-B line granularity (B200 loads fetch lines,
    tools/gran_probe.cu), and the measured overhead = ncu DRAM bytes / algorithmic bytes - 1 where
    a committed capture of the same workload exists (Table 5 analogue)."""
    lat = P.solver_lattice(eng.d)
    g = P.GeometryStats(phi=nf / max(1, int(np.prod(eng.geometry_dims))), phi_t=eng.info.phi_t,
                        ratio_tiles=eng.info.ratio_tiles)
    o = P.overhead_t2c(P.CostParams(lat=lat, a=eng.a), g)
    types = eng.tile_grid().types
    fl = types != 0
    T, n = fl.shape
    es = 8
    out = {"model_delta_b": round(o.delta_b, 4), "model_delta_b_bt": round(o.delta_b_bt, 4)}
    for name, nodes in (("sector_bound", 32 // es), ("line_bound", 128 // es)):
        if n % nodes == 0:
            out[name] = round(float(fl.reshape(T, n // nodes, nodes).any(axis=2).sum() * nodes / fl.sum()) - 1.0, 4)
    tr = load_ncu_traffic(workload) if workload else None
    if tr:
        out["measured"] = round(tr / (nf * bnode) - 1.0, 4)
        out["measured_source"] = f"profiles/ncu_step_kernel.json[{workload}]"
    return out


def porosity_sweep(P, K, W, peak):
    out = []
    for phi in (0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 1.0):
        if phi < 1.0:
            g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(
                dims=(256, 256, 256), sphere_diameter=40, target_porosity=phi, seed=7))
        else:
            g = P.Geometry.filled(3, (256, 256, 256))
        eng = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), (1, 1, 1))
        eng.initialize_uniform(1.0, (0.01, 0.005, 0.0))
        ms, _, _ = time_steps(eng, K, W)
        nf = eng.fluid_nodes()
        mlups = nf * K / (ms * 1e-3) / 1e6
        gbs = mlups * 1e6 * B_NODE[3] / 1e9
        ph = round(P.porosity(g).phi, 4)
        out.append({"phi": ph, "phi_t": round(eng.info.phi_t, 4),
                    "tiles": int(eng.info.n_tiles), "fluid_nodes": nf, "mlups": round(mlups, 1),
                    "achieved_gbs": round(gbs, 1), "frac_of_measured_peak": round(gbs / peak, 4),
                    "bu_of_8tbs": round(gbs / 8000.0, 4),
                    "overhead": accounting(P, eng, nf, B_NODE[3], NCU_CASE.get(ph))})
        del eng
    return out


def other_configs(P, K, W, peak):
    """The other BASELINE configs on one GPU: configs[0] (D2Q9 cavity 256^2, 1000 steps, a=4 and
    the reference 2D default a=16), configs[3] (D2Q9 4096^2 seeded vessel tree, a=4), and the
    paper's Table 2 collision variants on the configs[1] channel (BGK incompressible, MRT)."""
    rows = []
    inc = P.FluidModel(P.Compressibility.Incompressible, tau=0.8)
    mrt = P.FluidModel(collision=P.CollisionKind.MRT, tau=0.8)
    mrt_inc = P.FluidModel(P.Compressibility.Incompressible, P.CollisionKind.MRT, tau=0.8)
    chan = lambda: channel_geometry(P, (128, 128, 128))
    cases = [("configs[1] channel 128^3, BGK incompressible (paper Table 2 headline model)",
              chan, 4, K, inc),
             ("configs[1] channel 128^3, MRT quasi-compressible", chan, 4, K, mrt),
             ("configs[1] channel 128^3, MRT incompressible", chan, 4, K, mrt_inc),
             ("configs[1] channel 128^3, single-copy (AA) propagation, half the HBM", chan, 4, K,
              "single_copy"),
             ("configs[1] channel 128^3, f32 BGK quasi (TileEngineT2C<float>, paper Table 2 f32)",
              chan, 4, K, "f32"),
             ("configs[1] channel 128^3, f32 BGK incompressible (paper Table 2 f32 headline model)",
              chan, 4, K, ("f32", inc)),
             ("configs[0] D2Q9 cavity 256^2 a=4, 1000 steps",
              lambda: P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(256, 256, 1))), 4, 1000,
              None),
             ("configs[0] D2Q9 cavity 256^2 a=16, 1000 steps",
              lambda: P.generate(P.GeometryKind.Cavity2D, P.GenerateParams(dims=(256, 256, 1))), 16,
              1000, None),
             ("configs[3] D2Q9 vessel tree 4096^2 a=4 (seed 1, phi~0.23)",
              lambda: P.generate(P.GeometryKind.Vessel2D, P.GenerateParams(
                  dims=(4096, 4096, 1), target_porosity=0.2, seed=1)), 4, K, None)]
    for name, mk, a, steps, model in cases:
        g = mk()
        single = model == "single_copy"
        prec = "f32" if model == "f32" or (isinstance(model, tuple) and model[0] == "f32") else "f64"
        fm = model[1] if isinstance(model, tuple) else model
        if not isinstance(fm, P.FluidModel):
            fm = P.FluidModel(tau=0.8)
        eng = P.TileEngineT2C(g, a, fm, single_copy=single, precision=prec)
        eng.initialize_uniform()
        ms, _, _ = time_steps(eng, steps, W)
        nf = eng.fluid_nodes()
        mlups = nf * steps / (ms * 1e-3) / 1e6
        gbs = mlups * 1e6 * B_NODE[g.d] * (0.5 if prec == "f32" else 1.0) / 1e9
        rows.append({"config": name, "steps": steps, "fluid_nodes": nf,
                     "phi_t": round(eng.info.phi_t, 4), "us_per_step": round(ms / steps * 1e3, 2),
                     "mlups": round(mlups, 1), "achieved_gbs": round(gbs, 1),
                     "frac_of_measured_peak": round(gbs / peak, 4),
                     "step_path": ("resident multi-step kernel" if eng.info.resident_ctas else
                                   "MRT step specialised for the operator (NVRTC)" if eng.info.mrt_specialised
                                   else "one step launch per step (CUDA-graph batches)")})
        del eng
    return rows


def e2e_public_api(P, g, steps, bench_steps=None, samples=5):
    """End to end through the public API with host buffers: NodeInit fields H2D from pinned host
    memory, `steps` LBM steps (first-failure check), the final (rho, u) FieldData D2H; wall clock,
    median of `samples` runs. `steps` is the workload's run length (BASELINE configs[1]: 1000
    steps); the same measurement at the bench's own --steps is reported beside it."""
    import torch
    eng = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8))
    n = int(eng.info.n_tiles_stored) * eng.n_tn
    pinned = [torch.empty(n, dtype=torch.float64, pin_memory=True).numpy() for _ in range(4)]
    pinned[0][:] = 1.0
    for a in pinned[1:]:
        a[:] = 0.0
    nr = g.node_count()
    out = P.FieldData(g.d, g.dims, torch.empty(nr, dtype=torch.uint8, pin_memory=True).numpy(),
                      *[torch.empty(nr, dtype=torch.float64, pin_memory=True).numpy()
                        for _ in range(4)])
    eng.initialize_arrays(*pinned)  # warm: the 32-step CUDA graph of this parity is built here
    eng.step_n(64)
    eng.fields(out=out)
    nf = eng.fluid_nodes()

    def run(k):
        t0 = time.perf_counter()
        eng.initialize_arrays(*pinned)
        ok, failed = eng.step_n(k)
        f = eng.fields(out=out)  # Engine::fields() (the caller sums mass separately, engine.hpp:640)
        wall = time.perf_counter() - t0
        assert ok and np.isfinite(f.rho).all()
        return wall

    walls = sorted(run(steps) for _ in range(samples))
    wall = walls[len(walls) // 2]
    h2d = 4 * n * 8  # NodeInit (rho, u) at every stored tile node
    d2h = 4 * nr * 8 + nr + 8  # the raster FieldData (rho, u, mask; assembled on the device) + the failure stamp
    out_d = {"value": round(nf * steps / wall / 1e6, 1), "unit": "MLUPS",
             "h2d_bytes_per_step": round(h2d / steps, 1), "d2h_bytes_per_step": round(d2h / steps, 1),
             "steps": steps, "wall_s": round(wall, 4), "samples": samples,
             "wall_s_all": [round(w, 4) for w in walls]}
    if bench_steps and bench_steps != steps:
        wk = sorted(run(bench_steps) for _ in range(samples))[samples // 2]
        out_d["at_bench_steps"] = {"steps": bench_steps, "value": round(nf * bench_steps / wk / 1e6, 1),
                                   "wall_s": round(wk, 4),
                                   "h2d_bytes_per_step": round(h2d / bench_steps, 1),
                                   "d2h_bytes_per_step": round(d2h / bench_steps, 1)}
    return out_d


def _ref_build():
    """(fast-variant key, description) of the reference timing build this host runs best."""
    from oracle import ref as R
    v = R.best_timing_build()
    if v is None:
        return False, "-O3 (CMake Release flags, baseline x86-64)"
    return v, f"-O3 -march=x86-64-{v}"


def cpu_baseline(dims, budget_s=15.0, samples=3):
    """The reference's own T2C engine (oracle/_ref, built from /root/reference) on all host cores,
    on a bounded sample of the same workload (same geometry, fewer steps): best of `samples`
    timed batches, plus the 1-thread figure."""
    from oracle import configs as CF
    from oracle import ref as R
    fast, build = _ref_build()
    if not R.available(fast=fast):
        return None
    threads = os.cpu_count() or 1
    types = CF.channel3d_raster(dims)
    rg = R.RefGeometry.from_raster(3, dims, types, fast=fast, **CF.CHANNEL_BC)
    e = R.RefEngine(rg, "t2c", 4, 0.8, threads=threads)
    e.initialize_uniform()
    e.step(1)
    probe = max(e.last_seconds, 1e-3)
    steps = int(max(2, min(100, budget_s / samples / probe)))
    secs = []
    for _ in range(samples):
        e.step(steps)
        secs.append(e.last_seconds)
    sec = min(secs)
    nf = int(np.count_nonzero(types))
    e1 = R.RefEngine(rg, "t2c", 4, 0.8, threads=1)  # the 1-thread figure
    e1.initialize_uniform()
    e1.step(2)
    single = nf * 2 / e1.last_seconds / 1e6
    return {"value": round(nf * steps / sec / 1e6, 2), "unit": "MLUPS", "cores": threads,
            "single_thread_mlups": round(single, 2),
            "kind": "reference",
            "sample": f"best of {samples} x {steps} T2C steps of the {dims[0]}x{dims[1]}x{dims[2]} "
                      f"channel ({build} build of /root/reference sources, ThreadPool({threads}))",
            "samples_mlups": [round(nf * steps / s / 1e6, 2) for s in secs],
            "seconds": round(sec, 3)}


# ---------------------------------------------------------------------------------------------
def workload_config(n, nf):
    """The `config` object of the JSON line, identical for both arms (the driver compares them):
    N=1 is BASELINE configs[1]; N>1 is the weak-scaled duct, one 128^3-node z-slab per GPU."""
    if n == 1:
        return {"workload": WORKLOAD_1, "fluid_nodes": int(nf),
                "l2": "inputs > L2 (two PDF copies of 319 MB each); no flush", "parallelism": "single GPU"}
    return {"workload": f"D3Q19 BGK fp64 channel 128x128x{128 * n}, z-slab per GPU (128^3 nodes each)",
            "fluid_nodes": int(nf),
            "l2": "inputs > L2 (two PDF copies of 319 MB each per rank); no flush",
            "parallelism": f"zslab{n}"}


def run_reference_arm(args):
    """--impl reference: the reference's own CPU T2C implementation (oracle/_ref, the unmodified
    /root/reference sources) on the host cores, same metric/config; rank 0 only. The geometry is
    built in numpy (oracle/configs.py): nothing of the product package is loaded on this arm."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import configs as CF
    from oracle import ref as R
    world = int(os.environ.get("WORLD_SIZE", "1"))
    n = max(world, args.gpus)
    dims = (128, 128, 128 * n)  # our arm's workload at this N (one 128^3 slab per GPU)
    fast, build = _ref_build()
    if not R.available(fast=fast):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    threads = os.cpu_count() or 1
    types = CF.channel3d_raster(dims)
    rg = R.RefGeometry.from_raster(3, dims, types, fast=fast, **CF.CHANNEL_BC)
    e = R.RefEngine(rg, "t2c", 4, 0.8, threads=threads)
    e.initialize_uniform()
    e.step(max(args.warmup, 1))
    times = []
    for _ in range(args.steps):
        e.step(1)
        times.append(e.last_seconds)
    sec = float(np.sum(times))
    nf = int(np.count_nonzero(types))
    mlups = nf * args.steps / sec / 1e6
    line = {"metric": METRIC,
            "value": round(mlups, 2), "unit": "MLUPS", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(sec / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": workload_config(n, nf),
            "reference_engine": f"TileEngineT2C<double> + ThreadPool({threads}), {build} build of "
                                "/root/reference/proj/src (oracle/_ref)",
            "cpu_baseline": {"value": round(mlups, 2), "unit": "MLUPS", "cores": threads,
                             "kind": "reference",
                             "sample": f"{args.steps} steps of the full {dims[0]}x{dims[1]}x{dims[2]} "
                                       f"channel, TileEngineT2C<double> + ThreadPool({threads})"},
            "e2e": {"value": round(mlups, 2), "unit": "MLUPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_ours(args):
    import paper_1703_08015_b200 as P
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_1703_08015_b200 import slab
        return slab.bench_main(args, P, clock_sampler=ClockSampler, peak=measured_peaks(),
                               config_fn=workload_config)
    peak, peak_kind = measured_peaks()
    K, W = args.steps, args.warmup
    dims = (128, 128, 128)
    g = channel_geometry(P, dims)
    eng = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8))
    eng.initialize_uniform()
    ms, launches, clocks = time_steps(eng, K, W)
    nf = eng.fluid_nodes()
    mlups = nf * K / (ms * 1e-3) / 1e6
    step_ms = ms / K
    alg_bytes = nf * B_NODE[3]
    achieved = alg_bytes / (step_ms * 1e-3) / 1e9
    workload = "channel3d_128"
    line = {
        "metric": METRIC,
        "value": round(mlups, 1), "unit": "MLUPS", "n_gpus": 1, "steps": K, "warmup": W,
        "ms_per_step": round(step_ms, 5), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(1, nf),
        "geometry_stats": {"tiles": int(eng.info.n_tiles), "phi_t": round(eng.info.phi_t, 4)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_source": peak_kind,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "traffic": load_ncu_traffic(workload),
                     "traffic_source": "committed ncu --set full capture (profiles/ncu_step_kernel.json), "
                                       "dram__bytes_read.sum + dram__bytes_write.sum per launch"},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "overhead": accounting(P, eng, nf, B_NODE[3], workload),
    }
    del eng
    if not args.no_sweep:
        line["porosity_sweep"] = porosity_sweep(P, min(K, 64), max(W, 3), peak)  # whole 32-step graphs
    if not args.no_other:
        line["other_configs"] = other_configs(P, min(K, 64), max(W, 3), peak)
    line["e2e"] = e2e_public_api(P, g, 1000, bench_steps=K)  # configs[1] is a 1000-step run
    if not args.no_configs4:  # the north-star 1024^3 point (BASELINE configs[4], N=1)
        line["configs4"] = configs4_point(P, args.c4_size, args.c4_phi, K, W, args.c4_single_copy,
                                          (peak, peak_kind))
        # ... and the rest of its porosity range on the same GPU: phi 0.5 / 0.8 only fit 180 GB
        # with the single-copy (AA) propagation (106 / 147 GB)
        line["configs4_porosity"] = [configs4_point(P, args.c4_size, phi, min(K, 100), W, True,
                                                    (peak, peak_kind)) for phi in (0.5, 0.8)]
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(dims)
    print(json.dumps(line))
    return 0


def configs4_point(P, size, phi, steps, warmup, single_copy=False, peak=(6547.2, "measured")):
    """BASELINE configs[4] on ONE B200 (the N=1 point of the 1024^3 curve): RAS size^3, d=40,
    seed 7, periodic, tiles 4^3, porosity target `phi`, the raster generated on the GPU (same bytes
    as the host generator). Two PDF copies fit phi <~ 0.35 in 180 GB; single copy (AA) up to ~0.8."""
    t0 = time.time()
    g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(size, size, size), sphere_diameter=40,
                                                          target_porosity=phi, seed=7), device=0)
    t_gen = time.time() - t0
    t0 = time.time()
    eng = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), (1, 1, 1), single_copy=single_copy)
    t_build = time.time() - t0
    eng.initialize_uniform(1.0, (0.01, 0.005, 0.0))
    ms, launches, clocks = time_steps(eng, steps, warmup)
    nf = eng.fluid_nodes()
    mlups = nf * steps / (ms * 1e-3) / 1e6
    gbs = mlups * 1e6 * B_NODE[3] / 1e9
    red = eng.reduce()
    out = {"workload": f"configs[4] RAS {size}^3 d=40 seed 7 periodic, phi target {phi}, tiles 4^3, "
                       + ("single-copy (AA) propagation" if single_copy else "two PDF copies"),
           "value": round(mlups, 1), "unit": "MLUPS", "steps": steps, "warmup": warmup,
           "ms_per_step": round(ms / steps, 4),
           "phi": round(P.porosity(g).phi, 4), "phi_t": round(eng.info.phi_t, 4),
           "tiles": int(eng.info.n_tiles), "fluid_nodes": nf,
           "device_gb": round(eng.info.device_bytes / 1e9, 1),
           "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak[0], "unit": "GB/s",
                        "frac": round(gbs / peak[0], 4), "peak_source": peak[1],
                        "bu_of_8tbs": round(gbs / 8000.0, 4)},
           "gpu_launches": int(launches), "clocks": clocks, "mass": red["mass"],
           "non_finite": red["non_finite"],
           "host_seconds": {"generate": round(t_gen, 2), "engine_build": round(t_build, 2)}}
    del eng
    return out


def run_big(args):
    """--config ras1024: BASELINE configs[4] on ONE B200 (see configs4_point); under torchrun
    the slab strong-scaling run of the same domain."""
    import paper_1703_08015_b200 as P
    peak = measured_peaks()
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:  # strong scaling across ranks (z-slabs)
        from paper_1703_08015_b200 import slab
        return slab.bench_main(args, P, clock_sampler=ClockSampler, peak=peak, ras1024=True)
    c = configs4_point(P, args.c4_size, args.phi, args.steps, args.warmup, args.single_copy, peak)
    line = {"metric": METRIC, "value": c.pop("value"), "unit": c.pop("unit"), "n_gpus": 1,
            "steps": c.pop("steps"), "warmup": c.pop("warmup"), "ms_per_step": c.pop("ms_per_step"),
            "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": {"workload": c.pop("workload"), "phi": c.pop("phi"), "phi_t": c.pop("phi_t"),
                       "tiles": c.pop("tiles"), "fluid_nodes": c.pop("fluid_nodes"),
                       "device_gb": c.pop("device_gb")}}
    line.update(c)
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-other", action="store_true")
    ap.add_argument("--config", default="default", choices=["default", "ras1024"])
    ap.add_argument("--phi", type=float, default=0.2)
    ap.add_argument("--single-copy", action="store_true",
                    help="ras1024: in-place AA propagation (one PDF array)")
    ap.add_argument("--no-configs4", action="store_true",
                    help="skip the BASELINE configs[4] point (N=1) / strong-scaling key (N>1)")
    ap.add_argument("--c4-size", type=int, default=1024, help="configs[4] RAS edge (validation runs)")
    ap.add_argument("--c4-phi", type=float, default=0.2, help="configs[4] porosity target")
    ap.add_argument("--c4-single-copy", action="store_true",
                    help="configs[4] key with the single-copy (AA) engines (phi 0.5/0.8 fit)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.config == "ras1024":
        return run_big(args)  # N>1 under torchrun: the slab strong-scaling run
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
