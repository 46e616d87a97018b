"""Multi-GPU slab mode, host side, on CPU: world_size 2 and 3 with the gloo backend. Every rank runs
its slab (native layout + C oracle physics + the product's HaloExchange over torch.distributed);
the owned PDFs after K steps equal the single-domain oracle run bit for bit."""
import os
import socket

import numpy as np
import pytest

import paper_1703_08015_b200 as P
from paper_1703_08015_b200 import slab

CASES = {
    "ras32_periodic": (lambda: P.generate(P.GeometryKind.Ras3D, P.GenerateParams(
        dims=(32, 32, 32), sphere_diameter=10, target_porosity=0.6, seed=4)), 4, 7),
    "channel3d": (lambda: P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(24, 20, 36))), 4, 0),
    "channel2d_a4": (lambda: P.generate(P.GeometryKind.Channel2D, P.GenerateParams(dims=(40, 64, 1))), 4, 0),
    "cavity2d_periodic_y": (lambda: P.Geometry.filled(2, (32, 48, 1)), 4, 2),
}
STEPS = 12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q, single_copy=False):
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import oracle as O
        from slab_host_model import HostSlabRank
        factory, a, per = CASES[name]
        g = factory()
        slabs = slab.plan_slabs(slab.plane_tile_counts(g, a, per), world)
        z0, z1 = slabs[rank]
        m = HostSlabRank(O, g, a, 0.8, per, z0, z1, single_copy=single_copy)
        ax_per = P.Periodicity.of(per).axis(2 if g.d == 3 else 1)
        alloc = lambda n: torch.zeros(n, dtype=torch.float64)
        xchg = slab.HaloExchange(rank, world, ax_per, m.sizes(), alloc, slab.TorchComm())
        if single_copy:
            xback = slab.HaloExchange(rank, world, ax_per, m.sizes_back(), alloc, slab.TorchComm())
            for _ in range(STEPS):  # STEPS is even: the final state is in the natural layout
                if m.state == 0:
                    xchg.exchange(m.pack, m.unpack)
                    assert m.step()
                    xback.exchange(m.pack_back, m.unpack_back)
                else:
                    assert m.step()
        else:
            for _ in range(STEPS):
                assert m.step()
                xchg.exchange(m.pack, m.unpack)
        # full-domain oracle
        full = O.OracleT2C(g.types, g.d, g.dims, a, 0.8, periodic=per, bc_velocity=g.bc.velocity,
                           bc_density=g.bc.density)
        full.initialize_wavy()
        full.step(STEPS)
        st = full.q * full.n_tn
        L = m.lay
        ref = full.current_pdf()[L["g_own0"] * st:(L["g_own0"] + L["n_own"]) * st]
        mine = m.owned_pdf()
        fluid = np.broadcast_to((full.tiles["types"][L["g_own0"]:L["g_own0"] + L["n_own"]] != 0)[:, None, :],
                                (L["n_own"], full.q, full.n_tn)).ravel()
        ok = np.array_equal(mine[fluid].view(np.uint64), ref[fluid].view(np.uint64))
        dist.destroy_process_group()
        q.put((rank, ok, (z0, z1), int(L["n_own"])))
    except Exception as ex:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, False, repr(ex), traceback.format_exc()))


@pytest.mark.parametrize("single_copy", [False, True], ids=["two_copy", "single_copy"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", sorted(CASES))
def test_slab_exchange_matches_single_domain(name, world, single_copy, oracle):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q, single_copy))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), res
    assert sum(r[3] for r in res) == P.build_tile_grid(CASES[name][0](), CASES[name][1],
                                                       CASES[name][2]).fluid_tile_count()


def test_plan_slabs_balances_tiles():
    counts = np.array([10, 0, 5, 5, 30, 10, 10, 10, 10, 10])
    sl = slab.plan_slabs(counts, 3)
    assert sl[0][0] == 0 and sl[-1][1] == 10
    assert all(a < b for a, b in sl) and all(sl[i][1] == sl[i + 1][0] for i in range(2))
    loads = [counts[a:b].sum() for a, b in sl]
    assert max(loads) <= 40
    with pytest.raises(ValueError):
        slab.plan_slabs(counts, 11)


def test_neighbours():
    assert slab.neighbours(0, 1, True) == (None, None)
    assert slab.neighbours(0, 3, False) == (None, 1)
    assert slab.neighbours(2, 3, False) == (1, None)
    assert slab.neighbours(0, 2, True) == (1, 1)
    assert slab.neighbours(2, 3, True) == (1, 0)


def test_slab_layout_partitions_tiles():
    g = CASES["ras32_periodic"][0]()
    counts = slab.plane_tile_counts(g, 4, 7)
    T = int(counts.sum())
    owned = 0
    for z0, z1 in slab.plan_slabs(counts, 4):
        lay = slab.slab_layout(g, 4, 7, z0, z1)
        assert lay["zl"] == (z0 - 1) % 8 and lay["zh"] == z1 % 8
        owned += lay["n_own"]
    assert owned == T
    with pytest.raises(P.ConfigError):
        slab.slab_layout(g, 4, 7, 0, 7)  # halo planes would overlap the slab


def test_plan_slabs_two_ranks_periodic_skewed():
    """Two ranks on a periodic axis never get a one-plane slab (the other rank's low and high halo
    would be the same plane); every such plan builds a valid layout."""
    g = P.generate(P.GeometryKind.Ras3D, P.GenerateParams(dims=(16, 16, 24), sphere_diameter=6,
                                                          target_porosity=0.6, seed=3))
    counts = slab.plane_tile_counts(g, 4, 7)
    skew = np.array(counts, dtype=np.int64)
    skew[-1] *= 50  # one very heavy plane: the unconstrained plan isolates it
    assert slab.plan_slabs(skew, 2)[1] == (5, 6)
    m = slab.min_planes(2, 7, 3)
    assert m == 2 and slab.min_planes(3, 7, 3) == 1 and slab.min_planes(2, 3, 3) == 1
    for c in (counts, skew):
        sl = slab.plan_slabs(c, 2, m)
        assert all(b - a >= 2 for a, b in sl) and sl[0][0] == 0 and sl[-1][1] == 6
        for z0, z1 in sl:
            slab.slab_layout(g, 4, 7, z0, z1)
    with pytest.raises(ValueError):
        slab.plan_slabs([1, 1, 1], 2, 2)
    for world in range(1, 7):
        for mm in (1, 2, 3):
            if world * mm > 6:
                continue
            sl = slab.plan_slabs(skew, world, mm)
            assert len(sl) == world and all(b - a >= mm for a, b in sl)
            assert all(sl[i][1] == sl[i + 1][0] for i in range(world - 1))
