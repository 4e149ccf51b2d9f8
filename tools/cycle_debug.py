import sys, numpy as np
sys.path.insert(0, '/root/repo')
import os
os.environ["BIPB_CYCLE_VERBOSE"] = "1"
import bipb_inputs as g, paper_1301_5885_b200 as bp
p = g.config("C1")
ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
bp.bipb_source(ctx)
for kind in (0, 1):
    ctx.set_matvec_kernel(kind)
    for i in range(3):
        x = np.zeros(2 * p.n)
        try:
            st, r = bp.bipb_gmres_solve(ctx, x, None, 20, 1e-10, 500)
            print(kind, i, st, r["iterations"], ctx.graph_cycles)
        except Exception as e:
            print(kind, i, "ERR", e)
