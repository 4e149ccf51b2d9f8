"""Wall-clock breakdown of one end-to-end solve through the C ABI with host buffers
(bench.py's e2e step): setup / source / gmres / energy / destroy."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bipb_inputs as g  # noqa: E402
import paper_1301_5885_b200 as bp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
p = g.config(cfg)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
hc, hn, ha, hq = pin(p.centroids), pin(p.normals), pin(p.areas), pin(p.charges)
hx = torch.zeros(2 * p.n, dtype=torch.float64).pin_memory()
torch.cuda.init()
for rep in range(3):
    t = [time.perf_counter()]
    c = bp.bipb_setup(hc, hn, ha, hq, p.eps1, p.eps2, p.kappa)
    t.append(time.perf_counter())
    bp.bipb_source(c)
    t.append(time.perf_counter())
    hx.zero_()
    st, r = bp.bipb_gmres_solve(c, hx, None, 20, 1e-10, 500)
    t.append(time.perf_counter())
    e = bp.bipb_energy(c, hx)
    t.append(time.perf_counter())
    c.close()
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: setup {d[0]:.1f} ms, source {d[1]:.1f}, gmres {d[2]:.1f} ({r['matvecs']} matvecs), "
          f"energy {d[3]:.1f}, destroy {d[4]:.1f}, total {sum(d):.1f} ms", flush=True)
