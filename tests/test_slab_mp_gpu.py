"""Multi-process slab mode on one B200: 2-3 ranks (processes) share cuda:0 and run SlabRun with
(a) the fused peer-store exchange across processes (CUDA IPC handles, GPU-side flag waits), and
(b) the torch HaloExchange schedule with faces over gloo through host memory (NCCL refuses two
ranks on one GPU; the native NCCL path shares that schedule). Owned PDFs after K steps equal the
single-engine run bit for bit."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
STEPS = 7


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _geom(name):
    import paper_1703_08015_b200 as P
    if name == "ras40_periodic":
        return P.generate(P.GeometryKind.Ras3D, P.GenerateParams(
            dims=(40, 40, 40), sphere_diameter=12, target_porosity=0.55, seed=5)), 4, 7
    return P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(24, 20, 48))), 4, 0


def _worker(rank, world, port, name, transport, q, spread=False, single_copy=False):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_1703_08015_b200 as P
        from oracle import oracle as O
        from paper_1703_08015_b200 import slab
        g, a, per = _geom(name)
        m = P.FluidModel(tau=0.8)
        import torch
        dev = rank % torch.cuda.device_count() if spread else 0
        if transport == "p2p":  # CUDA IPC peer stores between the processes
            run = slab.SlabRun(g, a, m, per, rank, world, dev, transport="p2p",
                               single_copy=single_copy)
        else:  # torch HaloExchange over gloo through host memory
            run = slab.SlabRun(g, a, m, per, rank, world, dev, host_staged=True,
                               single_copy=single_copy)
        steps = STEPS + (STEPS % 2 if single_copy else 0)  # single copy: compare a natural layout
        run.initialize(O.wavy)
        run.step_async(steps)
        ok, _ = run.sync()
        whole = P.TileEngineT2C(g, a, m, per)
        whole.initialize(O.wavy)
        whole.step_n(steps)
        z0, z1 = run.slabs[rank]
        lay = slab.slab_layout(g, a, per, z0, z1)
        st = whole.q * whole.n_tn
        g0, n = lay["g_own0"], lay["n_own"]
        mine = run.engine.get_pdf()[lay["n_low"] * st:(lay["n_low"] + n) * st]
        ref = whole.get_pdf()[g0 * st:(g0 + n) * st]
        types = whole.tile_grid().types[g0:g0 + n]
        fluid = np.broadcast_to((types != 0)[:, None, :], (n, whole.q, whole.n_tn)).ravel()
        same = np.array_equal(mine[fluid].view(np.uint64), ref[fluid].view(np.uint64))
        dist.destroy_process_group()
        q.put((rank, bool(ok and same), run.engine.current_step() - (steps - STEPS)))
    except Exception as ex:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))


def _run(name, world, transport, spread=False, single_copy=False):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, name, transport, q, spread, single_copy))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(r[1] for r in res), res
    assert all(r[2] == STEPS for r in res)


@pytest.mark.parametrize("transport", ["torch", "p2p"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["ras40_periodic", "channel3d"])
def test_slabrun_processes_match_whole(name, world, transport):
    _run(name, world, transport)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", ["ras40_periodic", "channel3d"])
def test_slabrun_processes_on_distinct_devices(name, world):
    """One process per physical GPU (rank r on device r mod N), faces stored across processes
    and devices over CUDA IPC + NVLink. Skips on a one-GPU box."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two or more GPUs")
    _run(name, world, "p2p", spread=True)


@pytest.mark.parametrize("transport", ["torch", "p2p"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["ras40_periodic", "channel3d"])
def test_single_copy_slabrun_processes_match_whole(name, world, transport):
    """Single-copy (AA) slab ranks as processes: forward/backward face exchanges over gloo (torch)
    or in-place neighbour slots over CUDA IPC (p2p); bitwise equal to the single engine."""
    _run(name, world, transport, single_copy=True)
