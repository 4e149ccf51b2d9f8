"""Compile tools/fref_probe.cu for sm_100a (default nvcc contraction, libdevice exp) and
count the FP64 instructions of its pair-loop body -> F_ref (ncu FLOP convention)."""
import os
import re
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
with tempfile.TemporaryDirectory() as d:
    cub = os.path.join(d, "p.cubin")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-cubin", "-o", cub,
                           os.path.join(HERE, "fref_probe.cu")])
    sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
lines = [l for l in sass.splitlines() if re.search(r"/\*[0-9a-f]{4}\*/", l)]
# the loop body: between the backward branch target and the backward branch
addr = lambda l: int(re.search(r"/\*([0-9a-f]{4,})\*/", l).group(1), 16)
back = [l for l in lines if "BRA" in l and re.search(r"BRA[^;]*0x([0-9a-f]+)", l) and
        int(re.search(r"BRA[^;]*0x([0-9a-f]+)", l).group(1), 16) < addr(l)]
best = None
for b in back:
    tgt = int(re.search(r"BRA[^;]*0x([0-9a-f]+)", b).group(1), 16)
    body = [l for l in lines if tgt <= addr(l) <= addr(b)]
    cnt = {op: sum(1 for l in body if re.search(rf"\b{op}\b", l)) for op in ("DFMA", "DMUL", "DADD")}
    if best is None or sum(cnt.values()) > sum(best[1].values()):
        best = (len(body), cnt)
n, c = best
flops = 2 * c["DFMA"] + c["DMUL"] + c["DADD"]
print({"body_instructions": n, **c, "fp64_instructions": sum(c.values()), "ncu_flops_per_pair": flops,
       "mufu": "main path without the exp/rcp slow-path calls"})
