"""Time the symmetric product at one config for several run lengths W (offsets per CTA;
BIPB_SYM_W) and both sum modes, each in a fresh process.  Usage (GPU):
  python tools/sweep_runs.py [C4] [W ...]   -> one JSON line per (W, mode)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, json, numpy as np
sys.path.insert(0, %r)
import bipb_inputs as g, paper_1301_5885_b200 as bp
p = g.config(%r)
c = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
c.set_matvec_kernel(1)
u = g.random_vector(2 * p.n, 1)
bp.bipb_matvec(c, u)
c.timing_enable(True); c.timing_reset()
for _ in range(%d):
    y = bp.bipb_matvec(c, u)
ms, k = c.timing_get(0)
print(json.dumps({"ms_per_product": ms / %d, "sum_mode": c.sum_mode, "ynorm": float(np.linalg.norm(y))}))
"""

if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    ws = [int(a) for a in sys.argv[2:]] or [16, 12, 8, 6, 4]
    reps = 4
    for w in ws:
        for mode in ("exact", "fixed"):
            env = dict(os.environ, BIPB_SYM_W=str(w), BIPB_SUM=mode)
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg, reps, reps)], env=env,
                                 capture_output=True, text=True, timeout=600)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(json.dumps({"config": cfg, "W": w, "mode": mode, "result": line}), flush=True)
