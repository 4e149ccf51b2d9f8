"""Device-side GMRES cycles (BIPB_GRAPHS=2: one CUDA graph per Arnoldi cycle, each step in an IF
node cleared by cycle_check_kernel when the host loop would leave the cycle) against the eager
host loop (forced by the timing instrumentation) in the same process: bitwise the same x,
iterations, restarts and residual history -- for both matvec kernels, the fused cluster Arnoldi
step (2N <= 32768) and the multi-launch MGS (larger N), m = 10 / 20, the opt-in preconditioner,
convergence inside a cycle, a cap at max_iters (NOT_CONVERGED) -- and the
energy against the oracle."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %(root)r)
import bipb_inputs as g
import oracle
import paper_1301_5885_b200 as bp

out = []
cases = [
    ("L4", g.sphere_problem(4, 4.0, g.charges_in_ball(20, 3.0, 9)), True),
    ("L6", g.sphere_problem(6, 20.0, g.charges_in_ball(30, 15.0, 4)), False),
]
for name, p, with_oracle in cases:
    ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
    bp.bipb_source(ctx)
    ref_e = oracle.solve(p, restart=10, tol=1e-10)["energy"] if with_oracle else None
    for kind in (0, 1):
        ctx.set_matvec_kernel(kind)
        for m, tol, maxit, pre in ((10, 1e-10, 500, 0), (20, 1e-10, 500, 0), (10, 1e-10, 500, 1),
                                    (10, 1e-10, 13, 0)):
            ctx.set_precond(pre)
            res = []
            for timing in (True, False, False):  # eager (warms the product), then two graph solves
                ctx.timing_enable(timing)
                x = np.zeros(2 * p.n)
                st, rep = bp.bipb_gmres_solve(ctx, x, None, m, tol, maxit)
                res.append((st, rep, x, rep["history"]))
            (s0, r0, x0, h0) = res[0]
            rec = {"case": name, "kind": kind, "m": m, "maxit": maxit, "pre": pre, "its": r0["iterations"],
                   "status": s0, "arnoldi": ctx.arnoldi, "graph_cycles": ctx.graph_cycles}
            rec["bitwise"] = all(s == s0 and r["iterations"] == r0["iterations"] and r["restarts"] == r0["restarts"]
                                 and np.array_equal(x, x0) and np.array_equal(h, h0) for (s, r, x, h) in res[1:])
            if ref_e is not None and maxit == 500 and pre == 0 and m == 10:
                rec["e_rel"] = abs(bp.bipb_energy(ctx, res[2][2]) - ref_e) / abs(ref_e)
            out.append(rec)
        ctx.set_precond(0)
    ctx.close()
print(json.dumps(out))
"""


def test_cycle_graphs_bitwise_equal_eager():
    env = dict(os.environ, BIPB_GRAPHS="2")
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    recs = json.loads(r.stdout.strip().splitlines()[-1])
    assert len(recs) == 16
    assert recs[-1]["graph_cycles"] > 0 and recs[7]["graph_cycles"] > 0  # the graph path ran (L6, L4)
    for rec in recs:
        assert rec["bitwise"], rec
        if rec["maxit"] == 13:
            assert rec["status"] == 2 and rec["its"] == 13, rec  # NOT_CONVERGED exactly at the cap
        else:
            assert rec["status"] == 0, rec
        if "e_rel" in rec:
            assert rec["e_rel"] <= 1e-8, rec
    assert {rec["arnoldi"] > 0 for rec in recs if rec["case"] == "L4"} == {True}  # fused cluster step
    assert {rec["arnoldi"] for rec in recs if rec["case"] == "L6"} == {0}  # multi-launch MGS
