"""Single-GPU estimate of the multi-GPU matvec scaling: time rank r's share of the product
(BIPB_DIST_NO_COMM: the rank's I-blocks / rows, no communicator) for P = 1, 2, 4, 8 and compare
with the P = 1 time / P.  The exchange (one 2N-double all-reduce / all-gather) is not included."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bipb_inputs as g  # noqa: E402
import paper_1301_5885_b200 as bp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
p = g.config(cfg)
u = torch.from_numpy(g.random_vector(2 * p.n, 1)).cuda()
y = torch.empty_like(u)
base = None
for kind in (1, 0):
    for P in (1, 2, 4, 8):
        worst = 0.0
        for r in sorted({0, P - 1}):
            dist = None if P == 1 else (r, P, None, -1, bp.DIST_NO_COMM)
            ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa, dist=dist)
            ctx.set_matvec_kernel(kind)
            bp.bipb_matvec(ctx, u, y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(2):
                bp.bipb_matvec(ctx, u, y)
            e1.record()
            e1.synchronize()
            worst = max(worst, e0.elapsed_time(e1) / 2)
            ctx.close()
        if P == 1:
            base = worst
        print(json.dumps({"kind": kind, "P": P, "ms_per_matvec_slowest_rank": worst,
                          "efficiency_vs_P1": base / (P * worst)}), flush=True)
