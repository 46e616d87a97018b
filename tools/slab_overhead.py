"""Cost of the multi-GPU slab step on ONE B200: the whole 128x128x(128*W) channel in one engine vs
W slab engines in one process exchanging faces with the fused peer stores (p2p). Both run the same
total work on the same GPU, so the wall-time ratio is the slab mode's own overhead (the boundary
plane launch, flag waits/writes), an upper bound for the per-GPU overhead of the N-GPU run.
With `asym` the split is (all but one tile plane | one plane): the big engine's time then stands for
one GPU of an N-GPU run, and the overhead is measured against its share of the whole-engine time.
The slab engines' steps are enqueued interleaved one step at a time (every rank of a real run
enqueues its own steps concurrently; enqueueing one engine's K steps before the next would stall
the first on its neighbour's flags for the whole enqueue time).
usage: python tools/slab_overhead.py [W] [K] [asym]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1703_08015_b200 as P  # noqa: E402
from paper_1703_08015_b200 import slab  # noqa: E402


def main():
    import torch
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    g = P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(128, 128, 128 * W)))
    m = P.FluidModel(tau=0.8)
    whole = P.TileEngineT2C(g, 4, m)
    whole.initialize_uniform()
    whole.step_n(8)
    L = g.dims[2] // 4
    asym = len(sys.argv) > 3 and sys.argv[3] == "asym"
    slabs = [(0, L - 1), (L - 1, L)] if asym else [(r * L // W, (r + 1) * L // W) for r in range(W)]
    W = len(slabs)
    ranks = [P.TileEngineT2C(g, 4, m, slab=s) for s in slabs]
    blobs = [e.ipc_blob() for e in ranks]
    for r, e in enumerate(ranks):
        lo, hi = slab.neighbours(r, W, False)
        e.p2p_attach(blobs[lo] if lo is not None else None, blobs[hi] if hi is not None else None)
    for e in ranks:
        e.initialize_uniform()
    for _ in range(8):  # interleaved: the engines share one GPU's work queues
        for e in ranks:
            e.step_async(1)
    for e in ranks:
        e.sync()
    out = {}
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        whole.step_async(K)
        whole.sync()
        t1 = time.perf_counter()
        for _ in range(K):  # interleaved, as each rank of a real run enqueues its own steps
            for e in ranks:
                e.step_async(1)
        for e in ranks:
            assert e.sync()[0]
        t2 = time.perf_counter()
        out.setdefault("whole_us", []).append((t1 - t0) / K * 1e6)
        out.setdefault("slabs_us", []).append((t2 - t1) / K * 1e6)
    w = min(out["whole_us"])
    s = min(out["slabs_us"])
    share = (L - 1) / L if asym else 1.0
    print(f"W={W}{' asym' if asym else ''} whole {w:.1f} us/step, slab engines {s:.1f} us/step, "
          f"overhead {100 * (s / (w * share) - 1):.1f} %")


if __name__ == "__main__":
    main()
