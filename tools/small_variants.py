"""Build (here) / time (GPU) compile-time variants of the small-problem kernels (fused Arnoldi
reduction, chunk-partial reduce unrolling) on a BASELINE config through bench.py.
  python tools/small_variants.py build
  python tools/small_variants.py run C1
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "build", "small_variants")
# (session 2 also timed two fused-Arnoldi reduction variants and a one-wave chunk rule for the row
# kernel, since removed: profiles/r01/small_variants_C1.jsonl / _C2.jsonl)
VARIANTS = {"default": [], "red_unroll1": ["-DBIPB_RED_UNROLL=1"], "diag_branch": ["-DBIPB_DIAG_SELECT=0"]}


def build():
    import importlib.util
    spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_1301_5885_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    os.makedirs(OUT, exist_ok=True)
    procs = [subprocess.Popen([b.NVCC, *b.FLAGS, *extra, "-o", os.path.join(OUT, f"libbipb_{k}.so"), *b.SRC, "-ldl"])
             for k, extra in VARIANTS.items()]
    assert all(p.wait() == 0 for p in procs)


def run(cfg):
    runs = [(k, {"BIPB_LIB": os.path.join(OUT, f"libbipb_{k}.so")}) for k in VARIANTS]
    runs.append(("arnoldi_launches", {"BIPB_LIB": os.path.join(OUT, "libbipb_default.so"), "BIPB_ARNOLDI": "launches"}))
    for rep in range(2):
        for name, env in runs:
            out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "10",
                                  "--warmup", "3", "--e2e-steps", "0", "--no-cpu-baseline"],
                                 env=dict(os.environ, **env), capture_output=True, text=True, timeout=600)
            try:
                d = json.loads(out.stdout.strip().splitlines()[-1])
                r = {"variant": name, "rep": rep, "ms_per_step": d["ms_per_step"], "iterations": d["iterations"][0],
                     "energy": d["energy_kcal_mol"], "kernel_ms_per_step": {k: v / 10 for k, v in d["kernel_ms"].items()}}
            except Exception:
                r = {"variant": name, "error": out.stderr[-400:]}
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    build() if sys.argv[1] == "build" else run(sys.argv[2] if len(sys.argv) > 2 else "C1")
