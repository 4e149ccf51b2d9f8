"""Small end-to-end run for compute-sanitizer: row + symmetric (R = 1, 2, 4) matvecs, source,
GMRES (plain and preconditioned; fused cluster Arnoldi step), energy, kappa > 0 and kappa = 0,
ragged sizes."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bipb_inputs as g  # noqa: E402
import paper_1301_5885_b200 as bp  # noqa: E402

for kappa in (g.KAPPA, 0.0):
    p = g.sphere_problem(3, 4.0, g.charges_in_ball(11, 3.0, 1), kappa=kappa)
    keep = np.arange(0, p.n - 37)
    q = g.Problem("rag", np.ascontiguousarray(p.centroids[keep]), np.ascontiguousarray(p.normals[keep]),
                  np.ascontiguousarray(p.areas[keep]), p.charges, p.eps1, p.eps2, kappa)
    for prob in (p, q):
        ctx = bp.bipb_setup(prob.centroids, prob.normals, prob.areas, prob.charges, prob.eps1, prob.eps2, prob.kappa)
        for kind in (0, 1):
            ctx.set_matvec_kernel(kind)
            u = g.random_vector(2 * prob.n, 1)
            bp.bipb_matvec(ctx, u)
            bp.bipb_matvec_batch(ctx, np.stack([u, 2 * u, 3 * u, u, u]))
            sol = bp.solve(ctx, restart_m=10, tol=1e-8)
            sol = bp.solve(ctx, restart_m=10, tol=1e-8, precond=1)
        ctx.close()
# r02: an eps1 != 1, large-kappa case (edge parameters) and the exact-sum symmetric product
pe = g.sphere_problem(3, 4.0, g.charges_in_ball(11, 3.0, 1), eps1=2.0, eps2=80.0, kappa=2.0)
ctx = bp.bipb_setup(pe.centroids, pe.normals, pe.areas, pe.charges, pe.eps1, pe.eps2, pe.kappa)
ctx.set_matvec_kernel(1)
ctx.set_sum_mode(1)
bp.solve(ctx, restart_m=20, tol=1e-10)
ctx.close()
print("sanitize driver done")
