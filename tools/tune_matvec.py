"""Build (here) or time (on the GPU) launch-configuration variants of the matvec pair kernel.
  python tools/tune_matvec.py build            # nvcc all variants into build/variants/
  python tools/tune_matvec.py run [C4] [reps]  # time each variant in a subprocess
"""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "variants")

VARIANTS = []
# symmetric-kernel variants: launch shape (TPB * T a multiple of the 128-source smem tile) plus
# extra -D macros ("defs")
# (session 2: {"BIPB_RSQ_INT": 1}, {"BIPB_EXP_F32K": 1} and both measured slower at C4 —
# profiles/r01/tune_int_variants_C4.jsonl; now: block-shape sweep for mid-size problems)
# (block-shape sweep for R = 1: profiles/r01/tune_shape_C*.jsonl); multi-RHS shapes (`batch` mode,
# profiles/r01/tune_batch_shapes_C4.jsonl).
# r02: R = 1 issue-efficiency set at C4: unrolling the 32-step source rotation
# (overlap of one step's reverse-accumulator chain with the next step) at T = 5 / 4, and occupancy.
# 3 CTAs per SM (12 warps, 3 per scheduler) at T = 4 / 5: 166 registers without spills; T = 5 needs
# the per-stage combine of the reverse sums (BIPB_SYM_RS_STAGE) to fit 3 x 49 KB of shared memory;
# 4 CTAs per SM: T = 3 at 128 registers (no spills), T = 4 (small spills).  All slower (session 1,
# profiles/r02/tune_sym_C4.jsonl).  Session 3: the non-FP64 instructions of a step (the prefetched
# record's register moves: ping-pong buffers, PREFETCH = 2; the exp exponent clamp: NOCLAMP is a
# speed probe only, exact at C4 which has no padded rows), and the baseline twice for the noise.
# The multi-RHS kernels (R = 2, 4) spend ~16 register moves per pair on the prefetched record copy
# (40 IMAD.MOV per R = 4 step): PREFETCH = 0 / 2 are timed for them too (`runbatch`).
# (session-3 set, measured in r02 session 4: profiles/r02/session4/tune_sym_C4.jsonl -- all slower
# than or equal to the default.)  Session 4: CTA size at 8 warps per SM -- one 256-thread CTA
# (B = 1280, per-stage reverse combine to fit the shared memory) or four 64-thread CTAs (B = 256, T = 4).
# (measured: profiles/r02/session4/tune_sym_cta_C4.jsonl, both slower.)  Then a register-cap sweep
# (__maxnreg__, BIPB_SYM_MAXNREG: the same code, ptxas schedules the five pair chains under a tighter budget).
# (measured: tune_sym_maxnreg_C4.jsonl, all slower; T = 6: tune_sym_t6_C4.jsonl, slower.)
# Small problems (C1, C2): the symmetric kernel with small blocks (the mid-size shape, chosen below
# 2,048 block pairs at B = 640, at T = 1 / 2 / 3, i.e. B = 128 / 256 / 384) against the row kernel.
# (measured: profiles/r02/session4/small/tune_small_C*.jsonl -> the B = 128 small shape.)
# Exact sums: forward partials per offset (rank-count invariant at any size) vs per run of W offsets.
# (measured: tune_fpo_C4.jsonl; the rank invariance came from a global W instead.)  ptxas options
# (the same source scheduled differently): -O2, -O1, --allow-expensive-optimizations.
for px in ([], ["-Xptxas", "-O2"], ["-Xptxas", "-O1"], ["-Xptxas", "--allow-expensive-optimizations=true"], []):
    VARIANTS.append({"kind": "sym", "tpb": 128, "t": 5, "minb": 1, "exp_bits": 11, "pf": 1, "un": 1,
                     "tile": 128, "stages": 3, "ptxas": px,
                     "defs": {"BIPB_SYM_STUNROLL": 1, "BIPB_SYM_RS_STAGE": 0}})


def name(v):
    extra = "".join(f"_{k.replace('BIPB_', '').lower()}{val}" for k, val in sorted(v.get("defs", {}).items()))
    return (f"{v.get('kind', 'row')}_tpb{v['tpb']}_t{v['t']}_minb{v['minb']}_eb{v['exp_bits']}_pf{v.get('pf', 0)}"
            f"_un{v.get('un', 1)}_tile{v.get('tile', 128)}_st{v.get('stages', 3)}{extra}"
            + (f"_mr{v['maxrreg']}" if v.get("maxrreg") else "")
            + "".join("_" + a.strip("-").split("=")[0] for a in v.get("ptxas", []) if a != "-Xptxas"))


def build():
    import importlib.util
    spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_1301_5885_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    os.makedirs(OUT, exist_ok=True)
    procs = []
    for v in VARIANTS:
        if v.get("kind") == "sym":
            extra = [f"-DBIPB_SYM_TPB={v['tpb']}", f"-DBIPB_SYM_T={v['t']}", f"-DBIPB_SYM_MINB={v['minb']}",
                     f"-DBIPB_EXP_BITS={v['exp_bits']}", f"-DBIPB_SYM_PREFETCH={v.get('pf', 0)}",
                     f"-DBIPB_SYM_UNROLL={v.get('un', 1)}", f"-DBIPB_TILE={v.get('tile', 128)}",
                     f"-DBIPB_STAGES={v.get('stages', 3)}"]
            extra += [f"-D{k}={val}" for k, val in v.get("defs", {}).items()]
            if v.get("maxrreg"):
                extra += [f"-DBIPB_SYM_MAXNREG={v['maxrreg']}"]
            extra += v.get("ptxas", [])
        else:
            extra = [f"-DBIPB_MV_TPB={v['tpb']}", f"-DBIPB_MV_T={v['t']}", f"-DBIPB_MV_MINB={v['minb']}",
                     f"-DBIPB_EXP_BITS={v['exp_bits']}"]
        out = os.path.join(OUT, f"libbipb_{name(v)}.so")
        cmd = [b.NVCC, *b.FLAGS, *extra, "-o", out, *b.SRC, "-ldl"]
        procs.append(subprocess.Popen(cmd))
    for p in procs:
        assert p.wait() == 0


def one(cfg, reps):
    import numpy as np
    import torch
    import bipb_inputs as g
    import paper_1301_5885_b200 as bp
    p = g.config(cfg)
    ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
    dev = torch.device("cuda:0")
    u = torch.from_numpy(g.random_vector(2 * p.n, 1)).to(dev)
    y = torch.empty_like(u)
    bp.bipb_matvec(ctx, u, y)
    ctx.timing_enable(True)
    ctx.timing_reset()
    for _ in range(reps):
        bp.bipb_matvec(ctx, u, y)
    ms, cnt = ctx.timing_get(0)
    ctx.close()
    per = ms / cnt
    return {"ms": per, "pairs_per_s": p.n * (p.n - 1) / (per / 1e3), "checksum": float(y.norm().item()),
            "y0": float(y[0].item())}


def run(cfg, reps):
    res = []
    for v in VARIANTS:
        lib = os.path.join(OUT, f"libbipb_{name(v)}.so")
        env = dict(os.environ, BIPB_LIB=lib, BIPB_MATVEC=v.get("kind", "row"))
        out = subprocess.run([sys.executable, __file__, "one", cfg, str(reps)], env=env, capture_output=True,
                             text=True, timeout=600)
        try:
            r = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            r = {"error": out.stderr[-500:]}
        r.update(v)
        res.append(r)
        print(json.dumps(r), flush=True)
    return res


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "kinds":  # time the default library's two matvec kernels
        cfg = sys.argv[2] if len(sys.argv) > 2 else "C4"
        for kind in ("row", "sym"):
            env = dict(os.environ, BIPB_MATVEC=kind)
            out = subprocess.run([sys.executable, __file__, "one", cfg, "3"], env=env, capture_output=True, text=True)
            print(kind, out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-800:], flush=True)
    elif cmd == "batch":  # multi-RHS throughput of the default library: R operands per product
        import numpy as np
        import torch
        import bipb_inputs as g
        import paper_1301_5885_b200 as bp
        cfg = sys.argv[2] if len(sys.argv) > 2 else "C4"
        p = g.config(cfg)
        ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
        ctx.set_matvec_kernel(1)
        for R in (1, 2, 4, 8):
            U = torch.from_numpy(np.stack([g.random_vector(2 * p.n, r) for r in range(R)])).cuda()
            Y = torch.empty_like(U)
            bp.bipb_matvec_batch(ctx, U, Y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(2):
                bp.bipb_matvec_batch(ctx, U, Y)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / 2
            print(json.dumps({"R": R, "ms_per_batch": ms, "pairs_per_s_all_rhs": R * p.n * (p.n - 1) / (ms / 1e3),
                              "ms_per_rhs": ms / R}), flush=True)
        ctx.close()
    elif cmd == "runbatch":  # the batch measurement for every variant library
        cfg = sys.argv[2] if len(sys.argv) > 2 else "C4"
        for v in VARIANTS:
            env = dict(os.environ, BIPB_LIB=os.path.join(OUT, f"libbipb_{name(v)}.so"))
            out = subprocess.run([sys.executable, __file__, "batch", cfg], env=env, capture_output=True, text=True,
                                 timeout=900)
            for line in out.stdout.strip().splitlines():
                d = json.loads(line)
                d.update({"pf": v.get("pf"), **v["defs"]})
                print(json.dumps(d), flush=True)
            if out.returncode:
                print(json.dumps({"error": out.stderr[-400:], **v["defs"]}), flush=True)
    elif cmd == "build":
        build()
    elif cmd == "one":
        print(json.dumps(one(sys.argv[2], int(sys.argv[3]))))
    else:
        run(sys.argv[2] if len(sys.argv) > 2 else "C4", int(sys.argv[3]) if len(sys.argv) > 3 else 3)
