"""bench.py contract: the JSON line carries the keys the driver reads (reference arm on CPU;
native arm on the GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_reference_arm_json():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0"], 300)
    assert REQUIRED <= set(d) and d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0 and d["gpu_launches"] == 0
    cb = d["cpu_baseline"]  # all host cores and one core (the paper's "one CPU"), with the CPU model
    assert cb["value_1core"] > 0 and cb["nproc"] >= 1 and "cpu_model" in cb
    # identical config keys in both arms (the driver compares them)
    sys.path.insert(0, ROOT)
    import bench
    import bipb_inputs as g
    assert d["config"] == json.loads(json.dumps(bench.bench_config(g.config("C1"), 1)))


def test_golden_check_logic():
    """bench.golden_check: matched by input SHA-256, tolerance north_star's (1e-8, +-1 iteration);
    a config without a stored solve (C5) or another input gives no entry."""
    sys.path.insert(0, ROOT)
    import bench
    import bipb_inputs as g
    p = g.config("C2")
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_C2.json")))["solves"]["20"]
    ok = bench.golden_check(p, gold["energy"] * (1 + 5e-9), gold["iterations"] + 1)
    assert ok["pass"] and ok["file"].endswith("oracle_C2.json") and ok["iterations_diff"] == 1
    assert not bench.golden_check(p, gold["energy"] * (1 + 2e-8), gold["iterations"])["pass"]
    assert not bench.golden_check(p, gold["energy"], gold["iterations"] + 2)["pass"]
    q = g.Problem(p.name, p.centroids, p.normals, p.areas, p.charges, 2.0, p.eps2, p.kappa)  # another input
    assert bench.golden_check(q, gold["energy"], gold["iterations"]) is None


@pytest.mark.gpu
def test_native_arm_json():
    d = _run(["--config", "C2", "--steps", "1", "--warmup", "3", "--e2e-steps", "1", "--cpu-seconds", "2",
              "--precond-steps", "1"], 900)
    assert REQUIRED <= set(d) and d["metric"] == "fp64_pair_interactions_per_sec"
    r = d["roofline"]
    assert r["bound"] == "alu" and 0 < r["frac"] < 1.5 and r["peak"] > 30
    assert {"fref_frac", "ncu_fp64_flop_frac", "executed_fp64_flops_per_unit", "peak_measured",
            "unordered_pair_evaluations_per_s"} <= set(r)
    assert d["paper_tol"]["tol"] == 1e-4 and max(d["paper_tol"]["iterations"]) < min(d["iterations"])
    assert len(d["input_sha256"]) == 64 and len(d["residual_history"]) == d["iterations"][-1]
    assert d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert d["cpu_baseline"]["kind"] == "oracle"
    pc = d["precond"]  # the opt-in preconditioned solve, beside the headline
    assert pc["energy_rel_diff_vs_plain"] <= 1e-8 and max(pc["iterations"]) < min(d["iterations"])
    og = d["oracle_golden"]  # the timed solve against tests/golden/oracle_C2.json
    assert og["pass"] and og["energy_rel_diff"] <= 1e-8 and abs(og["iterations_diff"]) <= 1


@pytest.mark.gpu
def test_native_arm_two_ranks_one_gpu():
    """The torchrun launch the driver uses for N > 1, with two ranks sharing this GPU (gloo for
    torch.distributed, the NCCL stand-in for the library's collectives)."""
    fake = os.path.join(ROOT, "tests", "fakenccl", "libfakenccl.so")
    env = dict(os.environ, BIPB_BENCH_PG="gloo", BIPB_NCCL_LIB=fake, BIPB_GRAPHS="0")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--steps", "1", "--warmup", "1", "--config", "C2", "--e2e-steps", "1"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert REQUIRED <= set(d) and d["n_gpus"] == 2 and d["scaling"] == "strong" and "cpu_baseline" not in d
    assert d["exchange"] == "p2p"  # default: peer stores (both ranks map each other's mailbox)
    assert d["oracle_golden"]["pass"]  # the 2-rank solve against the stored oracle solve
