"""Wall time of repeated GMRES solves in one context (graph capture on the first solve, replay
afterwards) vs the eager path (timing instrumentation on forces eager)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bipb_inputs as g  # noqa: E402
import paper_1301_5885_b200 as bp  # noqa: E402

for cfg in sys.argv[1:] or ["C1", "C2"]:
    p = g.config(cfg)
    ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
    bp.bipb_source(ctx)
    for mode in ("eager", "graph"):
        ctx.timing_enable(mode == "eager")
        ts = []
        for rep in range(4):
            x = np.zeros(2 * p.n)
            t = time.perf_counter()
            st, r = bp.bipb_gmres_solve(ctx, x, None, 20, 1e-10, 500)
            ts.append((time.perf_counter() - t) * 1e3)
        print(cfg, mode, r["iterations"], " ".join(f"{v:.2f}" for v in ts), "ms", flush=True)
    ctx.close()
