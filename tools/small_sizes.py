"""Small-problem products: row kernel vs the symmetric kernel (which picks its block shape by size:
B = 128 / 384 / 640) at N from 640 to 20,480, with CUDA-event times per product, and the default
kernel the library picks (bipb.cu SYM_MIN_TASKS).  Usage: python tools/small_sizes.py"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bipb_inputs as g  # noqa: E402
import paper_1301_5885_b200 as bp  # noqa: E402


def problem(n_keep):
    level = 3 if n_keep <= 1280 else (4 if n_keep <= 5120 else 5)
    p = g.sphere_problem(level, 4.0, g.charges_in_ball(10, 3.0, 1))
    idx = np.sort(np.random.default_rng(n_keep).choice(p.n, n_keep, replace=False))
    return g.Problem(f"n{n_keep}", np.ascontiguousarray(p.centroids[idx]), np.ascontiguousarray(p.normals[idx]),
                     np.ascontiguousarray(p.areas[idx]), p.charges, p.eps1, p.eps2, p.kappa)


for n in (640, 1280, 1920, 2560, 3840, 5120, 7680, 10240, 20480):
    p = problem(n)
    ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
    rec = {"n": n, "default_kind": ctx.matvec_kernel}
    u = g.random_vector(2 * p.n, 1)
    ys = []
    for kind in (0, 1):
        ctx.set_matvec_kernel(kind)
        bp.bipb_matvec(ctx, u)
        ctx.timing_enable(True)
        ctx.timing_reset()
        reps = 50
        for _ in range(reps):
            y = bp.bipb_matvec(ctx, u)
        ms, cnt = ctx.timing_get(0)
        ctx.timing_enable(False)
        rec[f"us_kind{kind}"] = 1e3 * ms / cnt  # pair / sym kernel only (CUDA events)
        ud = torch.from_numpy(u).cuda()
        yd = torch.empty_like(ud)
        bp.bipb_matvec(ctx, ud, yd)
        t = time.perf_counter()
        for _ in range(reps):
            bp.bipb_matvec(ctx, ud, yd)
        rec[f"us_call_kind{kind}"] = 1e6 * (time.perf_counter() - t) / reps  # whole synchronous call
        ys.append(y)
    rec["rel_diff"] = float(np.linalg.norm(ys[0] - ys[1]) / np.linalg.norm(ys[0]))
    ctx.close()
    print(json.dumps(rec), flush=True)
