"""Minimal driver for ncu captures: setup a BASELINE config and run `reps` matvecs (and
optionally one source + energy) through the C ABI.  Usage:
  python tools/profile_driver.py C4 [reps] [--all]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bipb_inputs as g  # noqa: E402
import paper_1301_5885_b200 as bp  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2
p = g.config(cfg)
ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
u = g.random_vector(2 * p.n, 1)
y = u
for _ in range(reps):
    y = bp.bipb_matvec(ctx, u)
if "--all" in sys.argv:
    bp.bipb_source(ctx)
    bp.bipb_energy(ctx, u)
print(cfg, p.n, float(np.linalg.norm(y)))
ctx.close()
