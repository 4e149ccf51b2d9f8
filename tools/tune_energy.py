"""A/B of the source and energy pair launches: energy targets per thread
(BIPB_EN_T) x the whole-wave chunk rule (BIPB_EN_WAVES), timed with the library's CUDA events.
  python tools/tune_energy.py build           # nvcc the variants into build/variants/ (here)
  python tools/tune_energy.py run [C4] [reps] # on the GPU: one subprocess per (variant, waves)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "variants")
VARIANTS = [{"en_t": 2, "en_minb": 4}, {"en_t": 3, "en_minb": 3}, {"en_t": 4, "en_minb": 2}]


def name(v):
    return f"en_t{v['en_t']}_minb{v['en_minb']}"


def build():
    import importlib.util
    spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_1301_5885_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    os.makedirs(OUT, exist_ok=True)
    procs = [subprocess.Popen([b.NVCC, *b.FLAGS, f"-DBIPB_EN_T={v['en_t']}", f"-DBIPB_EN_MINB={v['en_minb']}", "-o",
                               os.path.join(OUT, f"libbipb_{name(v)}.so"), *b.SRC, "-ldl"]) for v in VARIANTS]
    for p in procs:
        assert p.wait() == 0


def one(cfg, reps):
    import torch
    import bipb_inputs as g
    import paper_1301_5885_b200 as bp
    p = g.config(cfg)
    ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
    x = torch.from_numpy(g.random_vector(2 * p.n, 3)).cuda()
    b = torch.empty_like(x)
    bp.bipb_source(ctx, b)
    e = bp.bipb_energy(ctx, x)
    ctx.timing_enable(True)
    ctx.timing_reset()
    for _ in range(reps):
        bp.bipb_source(ctx, b)
        e = bp.bipb_energy(ctx, x)
    src_ms, src_n = ctx.timing_get(1)
    en_ms, en_n = ctx.timing_get(2)
    ctx.close()
    return {"cfg": cfg, "source_ms": src_ms / src_n, "energy_ms": en_ms / en_n, "energy": e,
            "energy_pairs_per_s": p.n * p.nc / (en_ms / en_n / 1e3), "b_norm": float(b.norm().item())}


def run(cfg, reps):
    for v in VARIANTS:
        for waves in ("0", "1"):
            env = dict(os.environ, BIPB_LIB=os.path.join(OUT, f"libbipb_{name(v)}.so"), BIPB_EN_WAVES=waves)
            out = subprocess.run([sys.executable, __file__, "one", cfg, str(reps)], env=env, capture_output=True,
                                 text=True, timeout=600)
            try:
                r = json.loads(out.stdout.strip().splitlines()[-1])
            except Exception:
                r = {"error": out.stderr[-500:]}
            r.update(v, en_waves=int(waves))
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "build":
        build()
    elif cmd == "one":
        print(json.dumps(one(sys.argv[2], int(sys.argv[3]))))
    else:
        run(sys.argv[2] if len(sys.argv) > 2 else "C4", int(sys.argv[3]) if len(sys.argv) > 3 else 20)
