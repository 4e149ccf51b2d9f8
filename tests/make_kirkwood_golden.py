"""Write tests/golden/kirkwood.json: the Kirkwood-series E_sol (oracle/kirkwood.py, SURVEY.md
App. A.3) of the sphere configs C1, C2, C4, C5.  Calls only oracle/ and bipb_inputs/."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bipb_inputs as g  # noqa: E402
from oracle.kirkwood import kirkwood_energy  # noqa: E402

out = {}
for name, radius in (("C1", 2.0), ("C2", 4.0), ("C4", 20.0), ("C5", 20.0)):
    p = g.config(name)
    e, nterms = kirkwood_energy(p.charges, radius, p.eps1, p.eps2, p.kappa)
    out[name] = {"energy": e, "terms": nterms, "radius": radius, "sha256": p.sha256()}
    print(name, e, nterms, flush=True)
with open(os.path.join(ROOT, "tests", "golden", "kirkwood.json"), "w") as f:
    json.dump(out, f, indent=1)
