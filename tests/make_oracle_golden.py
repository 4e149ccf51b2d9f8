"""Write tests/golden/oracle_<cfg>.json: full oracle solves (source -> GMRES -> energy) of
BASELINE configs, keyed by the input SHA-256.  Calls ONLY oracle/ and bipb_inputs/
(never the CUDA path).  Usage: python tests/make_oracle_golden.py C1 C2 [C3 ...] [--out=DIR] [--store=DIR]
(--store: GMRES products kept on disk, oracle.gmres_checkpointed; used for C4, whose solve takes
longer than one GPU-box call, tools/c4_golden_box.sh)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("OMP_PROC_BIND", "close")
os.environ.setdefault("OMP_PLACES", "cores")

import bipb_inputs as g  # noqa: E402
import oracle  # noqa: E402


def _host():
    """CPU model and thread count the oracle ran on (recorded beside the golden values)."""
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "omp_num_threads": os.environ.get("OMP_NUM_THREADS")}


def main(names, restarts=(20,), outdir=None, store=None):
    for name in names:
        p = g.config(name)
        out = {"config": name, "sha256": p.sha256(), "n": p.n, "nc": p.nc, "eps1": p.eps1, "eps2": p.eps2,
               "kappa": p.kappa, "tol": 1e-10, "solves": {}, "host": _host()}
        rows = np.unique(np.linspace(0, p.n - 1, 64).astype(np.int64))
        for m in restarts:
            t = time.time()
            if store:  # products kept on disk: the solve can span several time-limited runs
                b = oracle.source(p)
                x, st, rep = oracle.gmres_checkpointed(p, b, os.path.join(store, f"{name}_m{m}"), restart=m,
                                                       tol=1e-10, max_iters=500, check_true=True,
                                                       log=lambda s: print(name, s, flush=True))
                r = {"b": b, "x": x, "status": st, "report": rep, "energy": oracle.energy(p, x)}
            else:
                r = oracle.solve(p, restart=m, tol=1e-10, max_iters=500, check_true=True)
            out["solves"][str(m)] = {
                "energy": r["energy"], "status": r["status"], "iterations": r["report"]["iterations"],
                "restarts": r["report"]["restarts"], "matvecs": r["report"]["matvecs"],
                "rel_res_true": r["report"]["rel_res_true"], "seconds": time.time() - t,
                "rows": rows.tolist(), "x_phi": r["x"][rows].tolist(), "x_dphi": r["x"][rows + p.n].tolist(),
                "b_phi": r["b"][rows].tolist(), "b_dphi": r["b"][rows + p.n].tolist(),
                "b_norm": float(np.linalg.norm(r["b"])), "x_norm": float(np.linalg.norm(r["x"]))}
            print(name, m, out["solves"][str(m)]["energy"], out["solves"][str(m)]["iterations"],
                  f"{time.time() - t:.1f}s", flush=True)
        with open(os.path.join(outdir or os.path.join(ROOT, "tests", "golden"), f"oracle_{name}.json"), "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")] or ["C1", "C2"]
    opt = dict(a[2:].split("=", 1) for a in sys.argv[1:] if a.startswith("--"))
    ms = (10, 20) if all(a in ("C1", "C2") for a in args) else (20,)
    main(args, ms, opt.get("out"), opt.get("store"))
