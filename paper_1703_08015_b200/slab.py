"""Multi-GPU z-slab mode of the T2C path (the reference has no counterpart —
multi-GPU is the paper's future work).

The compact tile index is z-major, so a slab of tile planes is a contiguous tile range. Each rank
(one process per GPU) owns a slab balanced by non-empty tiles, stores one halo plane on each side,
and after every step exchanges the tile-face PDFs that cross its two slab faces:

  upward:   my top plane, layer a-1, directions with e_axis = +1  -> upper rank's low halo plane
  downward: my bottom plane, layer 0, directions with e_axis = -1 -> lower rank's high halo plane

Transports (SlabRun): "p2p" (default) — the boundary-plane step kernel stores the faces straight
into the neighbours' halo tiles over NVLink (CUDA IPC), ordered by GPU-side 64-bit flags, on a side
stream beside the interior planes; "nccl" — native NCCL send/recv from the engine; "torch" — this
module's HaloExchange over torch.distributed (gloo CPU tests). Everything is stream-ordered with no
host sync per step. The per-node arithmetic is unchanged, so N-GPU results are bitwise equal to the
1-GPU run.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from . import _native
from .geometry import Geometry
from .tiling import Periodicity


def plane_tile_counts(g: Geometry, a: int, periodic=None) -> np.ndarray:
    """Non-empty tiles per tile plane along the slab axis (z in 3D, y in 2D)."""
    from .tiling import tile_dims
    gd, _ = tile_dims(g.d, g.dims, a)
    L = gd[2] if g.d == 3 else gd[1]
    out = np.zeros(L, np.uint64)
    _native.check(_native.lib().splbm_plane_tile_counts(
        np.ascontiguousarray(g.types, np.uint8), g.d, np.asarray(g.dims, np.int32), a,
        Periodicity.of(periodic).mask(), out))
    return out


def min_planes(world: int, periodic, d: int) -> int:
    """Fewest tile planes a rank may own. Two ranks on a periodic slab axis are each other's lower
    AND upper neighbour: a one-plane slab would make the other rank's low and high halo the same
    plane, which the slab layout does not store twice (splbm_slab_layout rejects it)."""
    axis = 2 if d == 3 else 1
    return 2 if world == 2 and Periodicity.of(periodic).axis(axis) else 1


def plan_slabs(counts, world: int, min_planes: int = 1) -> list[tuple[int, int]]:
    """Contiguous plane ranges [z0, z1), one per rank, minimising the largest per-rank count of
    non-empty tiles (equal z-extents would be load-imbalanced on sparse media), each at least
    `min_planes` planes thick. Linear partition: binary search on the capacity with a greedy
    sweep, then split groups until every rank owns a range."""
    counts = [int(c) for c in np.asarray(counts).ravel()]
    L = len(counts)
    m = max(1, int(min_planes))
    if world < 1 or world * m > L:
        raise ValueError(f"cannot split {L} tile planes over {world} ranks "
                         f"(at least {m} plane(s) each)")

    def greedy(cap):
        cuts, load = [0], 0
        for z, c in enumerate(counts):
            if load + c > cap and z - cuts[-1] >= m and L - z >= m:
                cuts.append(z)
                load = 0
            load += c
        return cuts + [L]

    lo, hi = max(counts + [0]), sum(counts)
    while lo < hi:
        mid = (lo + hi) // 2
        if len(greedy(mid)) - 1 <= world:
            hi = mid
        else:
            lo = mid + 1
    cuts = greedy(lo)
    while len(cuts) - 1 < world:  # split the heaviest splittable group at its balance point
        groups = [(sum(counts[cuts[i]:cuts[i + 1]]), i) for i in range(len(cuts) - 1)
                  if cuts[i + 1] - cuts[i] >= 2 * m]
        _, i = max(groups)
        a, b = cuts[i], cuts[i + 1]
        half, acc, z = sum(counts[a:b]) / 2.0, 0, a + m
        for zz in range(a, b - m):
            acc += counts[zz]
            z = max(a + m, zz + 1)
            if acc >= half:
                break
        cuts.insert(i + 1, min(z, b - m))
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def slab_layout(g: Geometry, a: int, periodic, z0: int, z1: int, tables: bool = False):
    """The stored-tile layout a slab engine builds (splbm_slab_layout)."""
    L = _native.lib()
    per = Periodicity.of(periodic)
    lay = _native.SlabLayout()
    types = np.ascontiguousarray(g.types, np.uint8)
    dims = np.asarray(g.dims, np.int32)
    _native.check(L.splbm_slab_layout(types, g.d, dims, a, per.mask(), z0, z1, C.byref(lay), None,
                                      None))
    out = {k: getattr(lay, k) for k, _ in _native.SlabLayout._fields_}
    if tables:
        S = lay.n_low + lay.n_own + lay.n_high
        n_tn = a * a * (a if g.d == 3 else 1)
        nb = np.empty(max(S, 1) * 27, np.uint32)
        tt = np.empty(max(S, 1) * n_tn, np.uint8)
        _native.check(L.splbm_slab_layout(types, g.d, dims, a, per.mask(), z0, z1, C.byref(lay),
                                          _native.ptr(nb), _native.ptr(tt)))
        out["nb_local"] = nb[:S * 27]
        out["types_local"] = tt[:S * n_tn]
    return out


def neighbours(rank: int, world: int, periodic_axis: bool) -> tuple[int | None, int | None]:
    """(lower, upper) ranks along the slab axis; None at a non-periodic domain edge."""
    if world == 1:
        return None, None
    lower = rank - 1 if rank > 0 else (world - 1 if periodic_axis else None)
    upper = rank + 1 if rank < world - 1 else (0 if periodic_axis else None)
    return lower, upper


class HaloExchange:
    """Per-step face exchange between slab neighbours. `begin(pack)` packs the outgoing faces and
    starts the transfers, `end(unpack)` completes them and stores the incoming faces; work issued
    in between (the interior tiles) overlaps the transfers. All four transfers form one batch in
    the fixed order [send up, recv from below, send down, recv from above]: point-to-point
    operations between a pair of ranks match in issue order, so even when the lower and upper
    neighbour are the same rank (two ranks, periodic axis) send-up meets recv-from-below and
    send-down meets recv-from-above."""

    def __init__(self, rank, world, periodic_axis, sizes, alloc, comm):
        self.lower, self.upper = neighbours(rank, world, periodic_axis)
        self.comm = comm
        n = {k: int(v) // 8 for k, v in sizes.items()}
        self.send_low = alloc(n["send_low"])
        self.send_high = alloc(n["send_high"])
        self.recv_low = alloc(n["recv_low"])
        self.recv_high = alloc(n["recv_high"])
        self._pending = []

    def begin(self, pack):
        pack(self.send_low, self.send_high)
        ops = []
        if self.upper is not None and self.send_high.numel():
            ops.append(("send", self.send_high, self.upper))
        if self.lower is not None and self.recv_low.numel():
            ops.append(("recv", self.recv_low, self.lower))
        if self.lower is not None and self.send_low.numel():
            ops.append(("send", self.send_low, self.lower))
        if self.upper is not None and self.recv_high.numel():
            ops.append(("recv", self.recv_high, self.upper))
        self._pending = [self.comm.start(ops)] if ops else []

    def end(self, unpack):
        for h in self._pending:
            self.comm.finish(h)
        self._pending = []
        unpack(self.recv_low if self.lower is not None else None,
               self.recv_high if self.upper is not None else None)

    def exchange(self, pack, unpack):
        self.begin(pack)
        self.end(unpack)


class TorchComm:
    """torch.distributed point-to-point: NCCL on device buffers, ordered on `stream` (the engine
    stream), or gloo on CPU tensors. host_staged=True moves device buffers through host memory so
    the same schedule runs over gloo (multi-process tests on a single GPU)."""

    def __init__(self, stream=None, host_staged=False):
        import torch.distributed as dist
        self.dist = dist
        self.stream = stream
        self.host_staged = host_staged

    def start(self, ops):
        import torch
        dist = self.dist
        if self.host_staged:
            if self.stream is not None:
                self.stream.synchronize()
            else:
                torch.cuda.synchronize()
            staged = [(op, t.cpu() if op == "send" else torch.empty(t.shape, dtype=t.dtype), t, peer)
                      for op, t, peer in ops]
            works = dist.batch_isend_irecv([
                dist.P2POp(dist.isend if op == "send" else dist.irecv, h, peer)
                for op, h, _, peer in staged])
            return works, staged
        p2p = [dist.P2POp(dist.isend if op == "send" else dist.irecv, t, peer) for op, t, peer in ops]
        if self.stream is not None:
            with torch.cuda.stream(self.stream):  # NCCL waits for the pack on the engine stream
                return dist.batch_isend_irecv(p2p), None
        return dist.batch_isend_irecv(p2p), None

    def finish(self, handle):
        import torch
        works, staged = handle
        if self.stream is not None and not self.host_staged:
            with torch.cuda.stream(self.stream):
                for w in works:
                    w.wait()  # the engine stream waits for the transfer (no host sync)
            return
        for w in works:
            w.wait()
        if staged:
            with torch.cuda.stream(self.stream):
                for op, h, t, _ in staged:
                    if op == "recv":
                        t.copy_(h, non_blocking=False)

    def exchange(self, ops):
        self.finish(self.start(ops))


class SlabRun:
    """One rank of the multi-GPU slab mode: a slab TileEngineT2C + its NCCL halo exchange,
    overlapped with the interior tiles of every step."""

    def __init__(self, g: Geometry, a: int, model, periodic, rank: int, world: int, device: int,
                 slabs=None, host_staged: bool = False, native: bool = False,
                 transport: str | None = None, single_copy: bool = False):
        import torch
        from .engine import TileEngineT2C
        per = Periodicity.of(periodic)
        self.rank, self.world = rank, world
        self.slabs = slabs or plan_slabs(plane_tile_counts(g, a, per), world,
                                         min_planes(world, per, g.d))
        z0, z1 = self.slabs[rank]
        self.engine = TileEngineT2C(g, a, model, per, device=device,
                                    slab=None if world == 1 else (z0, z1), single_copy=single_copy)
        self.single_copy = bool(single_copy)
        axis_periodic = per.axis(2 if g.d == 3 else 1)
        self.stream = torch.cuda.ExternalStream(self.engine.stream_handle(), device=device)
        dev = torch.device("cuda", device)
        # transport: "p2p" (fused NVLink peer stores), "nccl" (native NCCL), "torch" (HaloExchange)
        transport = transport or ("nccl" if native else "torch")
        self.transport = transport if world > 1 else "none"
        self.native = self.transport in ("nccl", "p2p")
        lower, upper = neighbours(rank, world, axis_periodic)
        self.xchg = None
        if self.transport == "p2p":
            import torch.distributed as dist
            blobs = [None] * world
            dist.all_gather_object(blobs, self.engine.ipc_blob())
            self.engine.p2p_attach(blobs[lower] if lower is not None else None,
                                   blobs[upper] if upper is not None else None)
        elif self.transport == "nccl":
            # the engine runs the whole step sequence itself: NCCL send/recv from C++ on a side
            # stream, no per-step Python; rank 0's unique id reaches the others via torch.distributed
            import torch.distributed as dist
            uid = [TileEngineT2C.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            self.engine.comm_attach(uid[0], world, rank, lower, upper)
        elif self.transport == "torch":
            alloc = lambda n: torch.empty(n, dtype=torch.float64, device=dev)
            sizes = self.engine.halo_bytes()
            self.xchg = HaloExchange(rank, world, axis_periodic, sizes, alloc,
                                     TorchComm(self.stream, host_staged=host_staged))
            if single_copy:  # the backward exchange after steps from the natural layout
                back = {"send_low": sizes["recv_low"], "send_high": sizes["recv_high"],
                        "recv_low": sizes["send_low"], "recv_high": sizes["send_high"]}
                self.xback = HaloExchange(rank, world, axis_periodic, back, alloc,
                                          TorchComm(self.stream, host_staged=host_staged))

    def _pack(self, lo, hi):
        self.engine.halo_pack_next(lo.data_ptr() if lo.numel() else 0,
                                   hi.data_ptr() if hi.numel() else 0)

    def _unpack(self, lo, hi):
        self.engine.halo_unpack(lo.data_ptr() if lo is not None and lo.numel() else 0,
                                hi.data_ptr() if hi is not None and hi.numel() else 0)

    def _pack_cur(self, lo, hi):
        self.engine.halo_pack(lo.data_ptr() if lo.numel() else 0, hi.data_ptr() if hi.numel() else 0)

    def _pack_back(self, lo, hi):
        self.engine.halo_pack_back(lo.data_ptr() if lo.numel() else 0,
                                   hi.data_ptr() if hi.numel() else 0)

    def _unpack_back(self, lo, hi):
        self.engine.halo_unpack_back(lo.data_ptr() if lo is not None and lo.numel() else 0,
                                     hi.data_ptr() if hi is not None and hi.numel() else 0)

    def initialize(self, init=None) -> None:
        """Initialise every rank, then a barrier: a neighbour's first step may already store its
        faces into this rank's halo tiles, which initialisation must not overwrite afterwards."""
        import torch.distributed as dist
        if init is None:
            self.engine.initialize_uniform()
        else:
            self.engine.initialize(init)
        if self.world > 1:
            dist.barrier()

    def step_async(self, n: int) -> None:
        """n steps: boundary planes -> pack -> start exchange -> interior planes (overlapping the
        transfers) -> complete exchange -> unpack; all ordered on the engine stream."""
        if self.world == 1 or self.native:
            self.engine.step_async(n)
            return
        if self.single_copy:  # AA: forward faces before, backward slots after natural-layout steps
            for _ in range(n):
                if self.engine.current_step() % 2 == 0:
                    self.xchg.exchange(self._pack_cur, self._unpack)
                    self.engine.step_async(1)
                    self.xback.exchange(self._pack_back, self._unpack_back)
                else:
                    self.engine.step_async(1)
            return
        for _ in range(n):
            self.engine.step_part(1)
            self.xchg.begin(self._pack)
            self.engine.step_part(2)
            self.xchg.end(self._unpack)

    def sync(self):
        return self.engine.sync()


def configs4_strong(P, rank, world, device, size=1024, phi=0.2, steps=20, warmup=5,
                    transport="p2p", single_copy=False):
    """BASELINE configs[4] strong scaling inside a torchrun job: the RAS size^3 (d 40, seed 7,
    periodic, phi target `phi`) split into z-slabs balanced by non-empty tiles, `steps` timed steps
    (CUDA events on the engine stream, max over ranks), then rank 0 alone steps the whole domain
    on its GPU (the N=1 point of the same job) so the efficiency is against a same-box N=1.
    Returns the dict rank 0 attaches as `configs4_strong` (None on the other ranks)."""
    import torch
    import torch.distributed as dist
    red = torch.device("cuda", device) if dist.get_backend() == "nccl" else torch.device("cpu")

    def allred(v, op):
        t = torch.tensor([float(v)], dtype=torch.float64, device=red)
        dist.all_reduce(t, op=op)
        return float(t.item())

    per = (1, 1, 1)
    params = P.GenerateParams(dims=(size, size, size), sphere_diameter=40, target_porosity=phi,
                              seed=7)
    g = P.generate(P.GeometryKind.Ras3D, params, device=device)
    slabs = plan_slabs(plane_tile_counts(g, 4, Periodicity.of(per)), world,
                       min_planes(world, per, g.d))
    run = SlabRun(g, 4, P.FluidModel(tau=0.8), per, rank, world, device, slabs=slabs,
                  transport=transport, single_copy=single_copy)
    eng = run.engine
    eng.initialize_uniform(1.0, (0.01, 0.005, 0.0))
    dist.barrier()
    run.step_async(warmup)
    ok_w, _ = run.sync()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(run.stream):
        start.record()
    run.step_async(steps)
    with torch.cuda.stream(run.stream):
        stop.record()
    ok, _ = run.sync()
    torch.cuda.synchronize()
    dist.barrier()
    t = allred(start.elapsed_time(stop), dist.ReduceOp.MAX) * 1e-3
    nf_local = eng.fluid_nodes()
    nf = allred(nf_local, dist.ReduceOp.SUM)
    tiles = allred(eng.info.n_tiles, dist.ReduceOp.SUM)
    all_ok = allred(1.0 if (ok and ok_w) else 0.0, dist.ReduceOp.MIN) == 1.0
    loads = [None] * world
    dist.all_gather_object(loads, (int(nf_local), int(eng.info.n_tiles)))
    del run, eng
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    dist.barrier()
    out = None
    if rank == 0:
        whole = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8), per, device=device,
                                single_copy=single_copy)
        whole.initialize_uniform(1.0, (0.01, 0.005, 0.0))
        ok1, _ = whole.step_n(warmup)
        whole.step_async(steps)
        ok2, _ = whole.sync()
        t1 = whole.last_batch_ms() * 1e-3
        v1 = nf * steps / t1 / 1e6
        vN = nf * steps / t / 1e6
        out = {"workload": f"configs[4] RAS {size}^3 d=40 seed 7 periodic, phi target {phi}, "
                           f"tiles 4^3, {'single-copy (AA)' if single_copy else 'two PDF copies'}, "
                           f"z-slabs balanced by non-empty tiles",
               "scaling": "strong", "n_gpus": world, "steps": steps, "warmup": warmup,
               "value": round(vN, 1), "unit": "MLUPS", "ms_per_step": round(t / steps * 1e3, 4),
               "n1_value": round(v1, 1), "n1_ms_per_step": round(t1 / steps * 1e3, 4),
               "efficiency": round(vN / (world * v1), 4), "ok": bool(all_ok and ok1 and ok2),
               "phi": round(P.porosity(g).phi, 4), "fluid_nodes": int(nf), "tiles": int(tiles),
               "per_rank": [{"slab": list(slabs[r]), "fluid_nodes": loads[r][0],
                             "tiles": loads[r][1]} for r in range(world)],
               "transport": transport, "devices": torch.cuda.device_count(),
               "achieved_gbs_per_gpu": round(vN * 1e6 * 304 / world / 1e9, 1)}
        del whole
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    dist.barrier()
    return out


def bench_main(args, P, clock_sampler=None, peak=(6547.2, "measured"), ras1024=False,
               config_fn=None) -> int:
    """bench.py at N>1 (torchrun). Default: weak scaling — each rank owns a 128^3-node slab of one
    (128 x 128 x 128*N) D3Q19 channel. `ras1024` (bench.py --config ras1024): strong scaling of
    BASELINE configs[4], the RAS 1024^3 (phi --phi, d 40, seed 7, periodic) split into z-slabs
    balanced by non-empty tiles. Tile-face halos go through the fused NVLink peer stores
    (SPLBM_SLAB_TRANSPORT=nccl|torch selects the others); value = N_f*K summed over ranks / the
    max-over-ranks device time. e2e: the same through the public API with host buffers (NodeInit
    fields H2D, the steps, fields D2H), max-over-ranks wall clock. With fewer GPUs than ranks
    (validation on a one-GPU box) the ranks share the devices round-robin."""
    import time

    import numpy as np
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    device = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(device)
    dist.init_process_group("nccl" if torch.cuda.device_count() >= world else "gloo",
                            **({"device_id": torch.device("cuda", device)}
                               if torch.cuda.device_count() >= world else {}))
    transport = os.environ.get("SPLBM_SLAB_TRANSPORT", "p2p")
    single_copy = bool(ras1024 and getattr(args, "single_copy", False))
    if single_copy and transport == "nccl":
        transport = "p2p"  # the native NCCL schedule is the two-copy one
    if ras1024:
        per = (1, 1, 1)
        g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(
            dims=(1024, 1024, 1024), sphere_diameter=40, target_porosity=args.phi, seed=7), device=device)
        slabs = plan_slabs(plane_tile_counts(g, 4, Periodicity.of(per)), world,
                           min_planes(world, per, g.d))
        workload = (f"configs[4] RAS 1024^3 d=40 seed 7 periodic, phi target {args.phi}, z-slabs "
                    f"balanced by non-empty tiles"
                    + (", single-copy (AA) propagation" if single_copy else ""))
    else:
        per = None
        g = P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(128, 128, 128 * world)))
        L = g.dims[2] // 4
        slabs = [(r * L // world, (r + 1) * L // world) for r in range(world)]
        workload = f"D3Q19 BGK fp64 channel 128x128x{128 * world}, z-slab per GPU (128^3 nodes each)"
    try:
        run = SlabRun(g, 4, P.FluidModel(tau=0.8), per, rank, world, device, slabs=slabs,
                      transport=transport, single_copy=single_copy)
        ok_setup = 1.0
    except Exception:  # noqa: BLE001 - e.g. no peer access between these GPUs
        ok_setup = 0.0
    flag = torch.tensor([ok_setup], device=torch.device("cuda", device)
                        if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if flag.item() < 1.0:  # every rank falls back together: native NCCL send/recv halos
        transport = "nccl"
        run = SlabRun(g, 4, P.FluidModel(tau=0.8), per, rank, world, device, slabs=slabs,
                      transport=transport, single_copy=single_copy)
    dist.barrier()  # transports up before the first step
    eng = run.engine
    if ras1024:
        eng.initialize_uniform(1.0, (0.01, 0.005, 0.0))
        dist.barrier()
    else:
        run.initialize()
    run.step_async(args.warmup)
    run.sync()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = eng.launch_count()
    sampler = clock_sampler(device) if (clock_sampler and rank == 0) else None
    if sampler:
        sampler.__enter__()
    with torch.cuda.stream(run.stream):
        start.record()
    run.step_async(args.steps)
    with torch.cuda.stream(run.stream):
        stop.record()
    ok, failed = run.sync()
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__(None, None, None)
    dist.barrier()
    launches = eng.launch_count() - launches0

    red_dev = torch.device("cuda", device) if dist.get_backend() == "nccl" else torch.device("cpu")

    def max_over_ranks(v):
        t = torch.tensor([float(v)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        t = torch.tensor([float(v)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t)
        return float(t.item())

    t = max_over_ranks(start.elapsed_time(stop)) * 1e-3
    nf_local = float(eng.fluid_nodes())
    nf = sum_over_ranks(nf_local)
    all_ok = sum_over_ranks(1.0 if ok else 0.0) == world
    # e2e through the public API with host buffers: pinned NodeInit arrays H2D, the steps, the
    # (rho, u) fields D2H into pinned rasters; wall clock, max over ranks
    n_nodes = int(eng.info.n_tiles_stored) * eng.n_tn
    wall, ok2 = None, True
    if not ras1024:  # (configs[4]: tens of GB of host fields per rank — no e2e leg)
        pinned = [torch.empty(n_nodes, dtype=torch.float64, pin_memory=True).numpy() for _ in range(4)]
        pinned[0][:] = 1.0
        for a in pinned[1:]:
            a[:] = 0.0
        nr = g.node_count()
        out = P.FieldData(g.d, g.dims, torch.empty(nr, dtype=torch.uint8, pin_memory=True).numpy(),
                          *[torch.empty(nr, dtype=torch.float64, pin_memory=True).numpy() for _ in range(4)])
        dist.barrier()
        t0 = time.perf_counter()
        eng.initialize_arrays(*pinned)
        if world > 1:
            dist.barrier()  # neighbours store faces into my halos from their first step on
        run.step_async(args.steps)
        ok2, _ = run.sync()
        eng.fields(out=out)
        wall = max_over_ranks(time.perf_counter() - t0)
    if rank == 0:
        alg = nf_local * 304.0 / (t / args.steps) / 1e9  # one rank's step kernel traffic, GB/s
        line = {
            "metric": "MLUPS (D3Q19 fp64 BGK) vs porosity; % of HBM peak GB/s; at 1/2/4/8 B200",
            "value": round(nf * args.steps / t / 1e6, 1), "unit": "MLUPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t / args.steps * 1e3, 5),
            "higher_is_better": True, "scaling": "strong" if ras1024 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "ok": bool(all_ok and ok2),
            "config": (config_fn(world, nf) if config_fn else
                       {"workload": workload, "fluid_nodes": int(nf),
                        "l2": "inputs > L2 (PDF copies of several GB per rank); no flush",
                        "parallelism": f"zslab{world}"}),
            "transport": f"tile-face halos via {transport}", "devices": torch.cuda.device_count(),
            "roofline": {"bound": "hbm", "achieved": round(alg, 1), "peak": peak[0], "unit": "GB/s",
                         "frac": round(alg / peak[0], 4), "peak_source": peak[1],
                         "per": "one rank (the slowest rank's time)"},
            "gpu_launches": int(launches),
            "e2e": None if wall is None else {
                "value": round(nf * args.steps / wall / 1e6, 1), "unit": "MLUPS",
                "h2d_bytes_per_step": round(4 * n_nodes * 8 / args.steps, 1),
                "d2h_bytes_per_step": round((4 * g.node_count() * 8 + g.node_count() + 8) / args.steps, 1),
                "steps": args.steps, "wall_s": round(wall, 4), "per": "rank 0's buffers"},
        }
        if sampler:
            line["clocks"] = sampler.summary()
    if not ras1024 and not getattr(args, "no_configs4", False):
        # the north-star curve (BASELINE configs[4]) beside the weak-scaled headline value
        c4 = configs4_strong(P, rank, world, device, size=getattr(args, "c4_size", 1024),
                             phi=getattr(args, "c4_phi", 0.2), steps=args.steps,
                             warmup=args.warmup, transport=transport,
                             single_copy=getattr(args, "c4_single_copy", False))
        if rank == 0:
            line["configs4_strong"] = c4
    if rank == 0:
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0
