"""Where the end-to-end time goes (bench.py's e2e leg): NodeInit H2D + init, the steps, fields D2H
+ scatter + mass, on the configs[1] channel."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import paper_1703_08015_b200 as P  # noqa: E402


def main():
    import torch
    g = P.generate(P.GeometryKind.Channel3D, P.GenerateParams(dims=(128, 128, 128)))
    eng = P.TileEngineT2C(g, 4, P.FluidModel(tau=0.8))
    n = int(eng.info.n_tiles_stored) * eng.n_tn
    pinned = [torch.empty(n, dtype=torch.float64, pin_memory=True).numpy() for _ in range(4)]
    pinned[0][:] = 1.0
    for a in pinned[1:]:
        a[:] = 0.0
    nr = g.node_count()
    out = P.FieldData(g.d, g.dims, torch.empty(nr, dtype=torch.uint8, pin_memory=True).numpy(),
                      *[torch.empty(nr, dtype=torch.float64, pin_memory=True).numpy() for _ in range(4)])
    eng.initialize_arrays(*pinned)
    eng.step_n(64)  # builds the 32-step graph
    eng.fields(out=out)
    for _ in range(3):
        t0 = time.perf_counter()
        eng.initialize_arrays(*pinned)
        t1 = time.perf_counter()
        eng.step_n(1000)
        t2 = time.perf_counter()
        eng.fields(out=out)
        t3 = time.perf_counter()
        print(f"init {1e3 * (t1 - t0):.2f} ms  steps {1e3 * (t2 - t1):.2f} ms  fields {1e3 * (t3 - t2):.2f} ms  total {1e3 * (t3 - t0):.2f} ms")


if __name__ == "__main__":
    main()
