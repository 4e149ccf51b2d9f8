"""Command line for one solve on the GPU path (SURVEY.md §5 "config / flags" and "metrics / logging"):
Table 1 of the paper -- setup, source (Eq. (11)), GMRES(m), energy
(Eq. (14)) -- through the C ABI, printing ONE JSON line: config, input SHA-256, N, N_c, m, tol,
status, iterations, restarts, residual history, E_sol, per-phase wall times, pair-interactions/s.

  python -m paper_1301_5885_b200 --config C2 [--m 20 --tol 1e-10 --maxit 500]
  python -m paper_1301_5885_b200 --msms mol.vert mol.face --pqr mol.pqr [--eps1 1 --eps2 80 --kappa 0.1257]

Argument marshalling only: every step runs in libbipb.so's kernels (no CPU fallback)."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def parse(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_1301_5885_b200",
                                 description=" ".join(__doc__.split("\n\n")[0].split()))
    src = ap.add_mutually_exclusive_group(required=True)
    src.add_argument("--config", choices=["C1", "C2", "C3", "C4", "C5"], help="a BASELINE config (seeded, synthetic)")
    src.add_argument("--msms", nargs=2, metavar=("VERT", "FACE"), help="an MSMS triangulation (.vert, .face)")
    ap.add_argument("--pqr", help="charges (PQR) for --msms")
    ap.add_argument("--eps1", type=float, default=1.0, help="solute dielectric (--msms; configs fix 1)")
    ap.add_argument("--eps2", type=float, default=80.0, help="solvent dielectric (--msms; configs fix 80)")
    ap.add_argument("--kappa", type=float, default=0.1257, help="Debye-Hueckel parameter, 1/A (--msms)")
    ap.add_argument("--m", type=int, default=20, help="GMRES restart length (default 20, R7)")
    ap.add_argument("--tol", type=float, default=1e-10, help="relative residual tolerance (default 1e-10)")
    ap.add_argument("--maxit", type=int, default=500, help="iteration cap (status 2 when reached)")
    ap.add_argument("--precond", type=int, default=0, choices=[0, 1],
                    help="1: the opt-in jump-term diagonal right preconditioner (not in the paper)")
    ap.add_argument("--kernel", choices=["auto", "row", "sym"], default="auto", help="matvec kernel")
    ap.add_argument("--check-true", action="store_true", help="also report the true relative residual")
    args = ap.parse_args(argv)
    if args.msms and not args.pqr:
        ap.error("--msms needs --pqr")
    return args


def problem(args):
    import numpy as np

    import bipb_inputs as g
    if args.config:
        return g.config(args.config), {"workload": args.config}
    vt, ft = (open(p).read() for p in args.msms)
    V, VN, F = g.parse_msms(vt, ft)
    c, nrm, a, dropped = g.elements_from_msms(V, VN, F)
    q = g.parse_pqr(open(args.pqr).read())
    p = g.Problem(os.path.basename(args.msms[0]), c, nrm, a, np.ascontiguousarray(q), args.eps1, args.eps2,
                  args.kappa)
    return p, {"workload": "msms", "vert": args.msms[0], "face": args.msms[1], "pqr": args.pqr,
               "dropped_faces": int(dropped)}


def main(argv=None) -> int:
    args = parse(argv)
    import paper_1301_5885_b200 as bp
    p, cfg = problem(args)
    t = [time.perf_counter()]
    ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
    if args.kernel != "auto":
        ctx.set_matvec_kernel(1 if args.kernel == "sym" else 0)
    ctx.set_precond(args.precond)
    t.append(time.perf_counter())
    import numpy as np
    bp.bipb_source(ctx)
    t.append(time.perf_counter())
    x = np.zeros(2 * p.n)
    st, rep = bp.bipb_gmres_solve(ctx, x, None, args.m, args.tol, args.maxit, check_true=args.check_true)
    t.append(time.perf_counter())
    e = bp.bipb_energy(ctx, x)
    t.append(time.perf_counter())
    kernel = ctx.matvec_kernel
    ctx.close()
    solve_s = t[4] - t[1]
    pairs = rep["matvecs"] * p.n * (p.n - 1) + 2 * p.n * p.nc
    line = {"config": dict(cfg, n_elements=p.n, n_charges=p.nc, eps1=p.eps1, eps2=p.eps2, kappa=p.kappa,
                           restart_m=args.m, tol=args.tol, max_iters=args.maxit, precond=args.precond,
                           matvec_kernel="symmetric" if kernel == 1 else "row"),
            "input_sha256": p.sha256(), "status": {0: "converged", 2: "not_converged"}.get(st, st),
            "iterations": rep["iterations"], "restarts": rep["restarts"], "matvecs": rep["matvecs"],
            "rel_res_est": rep["rel_res_est"], "residual_history": [float(h) for h in rep["history"]],
            "energy_kcal_mol": e,
            "seconds": {"setup": t[1] - t[0], "source": t[2] - t[1], "gmres": t[3] - t[2], "energy": t[4] - t[3]},
            "pair_interactions_per_s": pairs / solve_s}
    if args.check_true:
        line["rel_res_true"] = rep["rel_res_true"]
    print(json.dumps(line), flush=True)
    return 0 if st == bp.OK else 2


if __name__ == "__main__":
    sys.exit(main())
