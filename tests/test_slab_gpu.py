"""Slab mode on one B200: several slab engines (the ranks) in one process exchange their face
halos through device buffers; owned PDFs and fields stay bitwise equal to the single-engine run.
This exercises the device halo pack/unpack kernels and the slab layout; the NCCL schedule itself
is covered by tests/test_slab_cpu.py (gloo, world 2 and 3)."""
import numpy as np
import pytest

import paper_1703_08015_b200 as P
from paper_1703_08015_b200 import slab

pytestmark = pytest.mark.gpu

CASES = {
    "ras48_periodic": (lambda: P.generate(P.GeometryKind.Ras3D, P.GenerateParams(
        dims=(48, 48, 48), sphere_diameter=12, target_porosity=0.5, seed=2)), 4, 7),
    "channel3d": (lambda: P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(32, 24, 64))), 4, 0),
    "channel2d": (lambda: P.generate(P.GeometryKind.Channel2D, P.GenerateParams(dims=(64, 128, 1))), 4, 0),
    "full2d_periodic_a16": (lambda: P.Geometry.filled(2, (64, 128, 1)), 16, 3),
}


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("name", sorted(CASES))
def test_slab_engines_match_whole(name, world):
    import torch
    from oracle import oracle as O
    factory, a, per = CASES[name]
    g = factory()
    m = P.FluidModel(tau=0.8)
    whole = P.TileEngineT2C(g, a, m, per)
    whole.initialize(O.wavy)
    slabs = slab.plan_slabs(slab.plane_tile_counts(g, a, per), world)
    ranks = [P.TileEngineT2C(g, a, m, per, slab=s) for s in slabs]
    for e in ranks:
        e.initialize(O.wavy)
    ax_per = P.Periodicity.of(per).axis(2 if g.d == 3 else 1)
    buf = []
    for e in ranks:
        hb = e.halo_bytes()
        buf.append({k: torch.zeros(max(v // 8, 1), dtype=torch.float64, device="cuda")
                    for k, v in hb.items()})
    K = 9
    assert whole.step_n(K)[0]
    for _ in range(K):
        for r, e in enumerate(ranks):
            e.step_async(1)
            e.halo_pack(buf[r]["send_low"].data_ptr(), buf[r]["send_high"].data_ptr())
        for e in ranks:
            assert e.sync()[0]
        for r, e in enumerate(ranks):
            lo, hi = slab.neighbours(r, world, ax_per)
            if lo is not None:
                n = buf[r]["recv_low"].numel()
                buf[r]["recv_low"][:n].copy_(buf[lo]["send_high"][:n])
            if hi is not None:
                n = buf[r]["recv_high"].numel()
                buf[r]["recv_high"][:n].copy_(buf[hi]["send_low"][:n])
        torch.cuda.synchronize()
        for r, e in enumerate(ranks):
            lo, hi = slab.neighbours(r, world, ax_per)
            e.halo_unpack(buf[r]["recv_low"].data_ptr() if lo is not None else 0,
                          buf[r]["recv_high"].data_ptr() if hi is not None else 0)
    wf = whole.fields()
    tg = whole.tile_grid()
    st = whole.q * whole.n_tn
    wp = whole.get_pdf()
    rho = np.zeros_like(wf.rho)
    for e in ranks:
        lay = slab.slab_layout(g, a, per, e.info.n_tiles and slabs[ranks.index(e)][0],
                               slabs[ranks.index(e)][1])
        g0, n = lay["g_own0"], lay["n_own"]
        mine = e.get_pdf()[lay["n_low"] * st:(lay["n_low"] + n) * st]
        ref = wp[g0 * st:(g0 + n) * st]
        fluid = np.broadcast_to((tg.types[g0:g0 + n] != 0)[:, None, :], (n, whole.q, whole.n_tn)).ravel()
        assert np.array_equal(mine[fluid].view(np.uint64), ref[fluid].view(np.uint64))
        f = e.fields()
        rho += f.rho
    assert np.array_equal(rho, wf.rho)


def test_native_comm_attach_single_rank():
    """The native exchange path (splbm_dev_comm_attach: NCCL communicator, side stream, split
    boundary/interior step) on a one-rank communicator steps exactly like the plain engine."""
    from oracle import oracle as O
    g, a, per = CASES["channel3d"][0](), 4, 0
    m = P.FluidModel(tau=0.8)
    e1 = P.TileEngineT2C(g, a, m, per)
    e2 = P.TileEngineT2C(g, a, m, per)
    e2.comm_attach(P.TileEngineT2C.comm_unique_id(), 1, 0, None, None)
    for e in (e1, e2):
        e.initialize(O.wavy)
        assert e.step_n(33) == (True, 0)
    assert np.array_equal(e1.get_pdf(), e2.get_pdf())
    assert e2.current_step() == 33 and e2.tile_visits() == e1.tile_visits()


def _p2p_slabs_vs_whole(name, world, devices, monkeypatch, wait=None, single_copy=False, K=11):
    from oracle import oracle as O
    if wait:
        monkeypatch.setenv("SPLBM_P2P_WAIT", wait)
    factory, a, per = CASES[name]
    g = factory()
    m = P.FluidModel(tau=0.8)
    whole = P.TileEngineT2C(g, a, m, per)
    whole.initialize(O.wavy)
    slabs = slab.plan_slabs(slab.plane_tile_counts(g, a, per), world,
                            min_planes=slab.min_planes(world, P.Periodicity.of(per), g.d))
    ranks = [P.TileEngineT2C(g, a, m, per, slab=s, device=devices[r % len(devices)],
                             single_copy=single_copy) for r, s in enumerate(slabs)]
    blobs = [e.ipc_blob() for e in ranks]
    ax_per = P.Periodicity.of(per).axis(2 if g.d == 3 else 1)
    for r, e in enumerate(ranks):
        lo, hi = slab.neighbours(r, world, ax_per)
        e.p2p_attach(blobs[lo] if lo is not None else None, blobs[hi] if hi is not None else None)
        e.initialize(O.wavy)
    # GPU-side flags order the ranks. Several engines share ONE device here, so their streams can
    # share hardware work queues: a rank's halo wait queued ahead of a neighbour's boundary planes
    # in a shared queue would never be satisfied. Enqueue step by step across the ranks (as one
    # process per GPU never has to); every wait then sits behind the work it waits for.
    for _ in range(K):
        for e in ranks:
            e.step_async(1)
    for e in ranks:
        assert e.sync() == (True, 0)
    assert whole.step_n(K)[0]
    tg = whole.tile_grid()
    st = whole.q * whole.n_tn
    wp = whole.get_pdf()
    for r, e in enumerate(ranks):
        lay = slab.slab_layout(g, a, per, *slabs[r])
        g0, n = lay["g_own0"], lay["n_own"]
        mine = e.get_pdf()[lay["n_low"] * st:(lay["n_low"] + n) * st]
        fluid = np.broadcast_to((tg.types[g0:g0 + n] != 0)[:, None, :], (n, whole.q, whole.n_tn)).ravel()
        assert np.array_equal(mine[fluid].view(np.uint64), wp[g0 * st:(g0 + n) * st][fluid].view(np.uint64))


@pytest.mark.parametrize("wait", ["auto", "kernel"])
@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("name", sorted(CASES))
def test_p2p_peer_store_slabs_match_whole(name, world, wait, monkeypatch):
    """Fused exchange: the boundary-plane kernel stores its faces straight into the neighbours'
    halo tiles, ordered by GPU-side flag waits/writes (same-process peers on one GPU; across
    processes the blob carries CUDA IPC handles). Bitwise equal to the single engine. `wait`:
    the halo-arrival wait the device supports (stream wait + remote-write flush, else the
    acquire-polling kernel) or the polling kernel forced."""
    _p2p_slabs_vs_whole(name, world, [0], monkeypatch, None if wait == "auto" else wait)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", sorted(CASES))
def test_p2p_slabs_on_distinct_devices(name, world, monkeypatch):
    """One process driving two or more physical GPUs: slab engines on distinct devices store their
    faces into each other's halos over NVLink (peer access enabled by p2p_attach). Skips on a
    one-GPU box."""
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs two or more GPUs")
    _p2p_slabs_vs_whole(name, world, list(range(n)), monkeypatch)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("name", sorted(CASES))
def test_p2p_single_copy_slabs_match_whole(name, world, monkeypatch):
    """Single-copy (AA) slabs over the fused p2p transport: the boundary planes' steps from the
    natural layout read and write the halo nodes' slots in place in the neighbours' memory.
    After an even step count the owned PDFs equal the two-copy single engine bit for bit."""
    _p2p_slabs_vs_whole(name, world, [0], monkeypatch, single_copy=True, K=12)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", sorted(CASES))
def test_single_copy_slab_engines_exchange_buffers(name, world):
    """Single-copy slab engines with the forward (before natural-layout steps) and backward
    (after them: the scatter's halo slots back to their owners, masked to the slots whose
    downstream node is non-solid) exchanges through device buffers: bitwise equal to the whole
    domain after an even step count; the swapped layout of a slab engine is not readable."""
    import torch
    from oracle import oracle as O
    factory, a, per = CASES[name]
    g = factory()
    m = P.FluidModel(tau=0.8)
    whole = P.TileEngineT2C(g, a, m, per)
    whole.initialize(O.wavy)
    slabs = slab.plan_slabs(slab.plane_tile_counts(g, a, per), world,
                            min_planes=slab.min_planes(world, P.Periodicity.of(per), g.d))
    ranks = [P.TileEngineT2C(g, a, m, per, slab=s, single_copy=True) for s in slabs]
    for e in ranks:
        e.initialize(O.wavy)
    ax_per = P.Periodicity.of(per).axis(2 if g.d == 3 else 1)
    fwd, back = [], []
    for e in ranks:
        hb = e.halo_bytes()
        mk = lambda n: torch.zeros(max(n // 8, 1), dtype=torch.float64, device="cuda")
        fwd.append({k: mk(v) for k, v in hb.items()})
        back.append({"send_low": mk(hb["recv_low"]), "send_high": mk(hb["recv_high"]),
                     "recv_low": mk(hb["send_low"]), "recv_high": mk(hb["send_high"])})

    def exchange(buf, pack, unpack):
        for r, e in enumerate(ranks):
            getattr(e, pack)(buf[r]["send_low"].data_ptr(), buf[r]["send_high"].data_ptr())
        for e in ranks:
            e.sync()
        for r in range(world):
            lo, hi = slab.neighbours(r, world, ax_per)
            if lo is not None:
                n = min(buf[r]["recv_low"].numel(), buf[lo]["send_high"].numel())
                buf[r]["recv_low"][:n].copy_(buf[lo]["send_high"][:n])
            if hi is not None:
                n = min(buf[r]["recv_high"].numel(), buf[hi]["send_low"].numel())
                buf[r]["recv_high"][:n].copy_(buf[hi]["send_low"][:n])
        torch.cuda.synchronize()
        for r, e in enumerate(ranks):
            lo, hi = slab.neighbours(r, world, ax_per)
            getattr(e, unpack)(buf[r]["recv_low"].data_ptr() if lo is not None else 0,
                               buf[r]["recv_high"].data_ptr() if hi is not None else 0)

    K = 10
    assert whole.step_n(K)[0]
    for s in range(K):
        if s % 2 == 0:
            exchange(fwd, "halo_pack", "halo_unpack")
            for e in ranks:
                assert e.step_n(1)[0]
            if s == 0:
                with pytest.raises(P.ConfigError):
                    ranks[0].get_pdf()  # swapped layout of a slab engine
            exchange(back, "halo_pack_back", "halo_unpack_back")
        else:
            for e in ranks:
                assert e.step_n(1)[0]
    tg = whole.tile_grid()
    st = whole.q * whole.n_tn
    wp = whole.get_pdf()
    for r, e in enumerate(ranks):
        lay = slab.slab_layout(g, a, per, *slabs[r])
        g0, n = lay["g_own0"], lay["n_own"]
        mine = e.get_pdf()[lay["n_low"] * st:(lay["n_low"] + n) * st]
        fluid = np.broadcast_to((tg.types[g0:g0 + n] != 0)[:, None, :], (n, whole.q, whole.n_tn)).ravel()
        assert np.array_equal(mine[fluid].view(np.uint64), wp[g0 * st:(g0 + n) * st][fluid].view(np.uint64))
