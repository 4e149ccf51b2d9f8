"""The command line (python -m paper_1301_5885_b200; SURVEY.md §5 "config / flags", "metrics /
logging"): argument handling on CPU, one solve per input kind on the GPU against the oracle."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import bipb_inputs as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cli(*args, timeout=600):
    return subprocess.run([sys.executable, "-m", "paper_1301_5885_b200", *args], capture_output=True, text=True,
                          cwd=ROOT, timeout=timeout)


def test_cli_arguments():
    r = _cli("--help")
    assert r.returncode == 0 and "--config" in r.stdout and "--msms" in r.stdout
    assert _cli().returncode == 2  # an input is required
    r = _cli("--msms", "a.vert", "a.face")
    assert r.returncode == 2 and "--pqr" in r.stderr


@pytest.mark.gpu
def test_cli_config_c1_against_golden():
    r = _cli("--config", "C1", "--check-true")
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_C1.json")))
    ref = gold["solves"]["20"]
    assert d["input_sha256"] == gold["sha256"] and d["status"] == "converged"
    assert abs(d["iterations"] - ref["iterations"]) <= 1
    assert d["energy_kcal_mol"] == pytest.approx(ref["energy"], rel=1e-8)
    assert d["rel_res_true"] <= 1e-9 and len(d["residual_history"]) == d["iterations"]


@pytest.mark.gpu
def test_cli_msms_pqr_against_oracle(tmp_path):
    """An icosphere written as MSMS .vert/.face plus a PQR of helix charges: the CLI's E_sol equals
    the oracle's solve of the same ingested elements."""
    import oracle
    v, f = g.icosphere(3, 4.0)
    vn = v / np.linalg.norm(v, axis=1, keepdims=True)
    vt, ft = g.write_msms(v, vn, f)
    (tmp_path / "s.vert").write_text(vt)
    (tmp_path / "s.face").write_text(ft)
    q = g.helix_charges()
    (tmp_path / "s.pqr").write_text("".join(f"ATOM {i + 1} C HEL A 1 {x:.6f} {y:.6f} {z:.6f} {c:.4f} 1.5000\n"
                                            for i, (x, y, z, c) in enumerate(q)))
    r = _cli("--msms", str(tmp_path / "s.vert"), str(tmp_path / "s.face"), "--pqr", str(tmp_path / "s.pqr"))
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    V, VN, F = g.parse_msms(vt, ft)
    c, nrm, a, _ = g.elements_from_msms(V, VN, F)
    qq = g.parse_pqr((tmp_path / "s.pqr").read_text())
    p = g.Problem("s", c, nrm, a, qq)
    ref = oracle.solve(p, restart=20, tol=1e-10)
    assert d["config"]["n_elements"] == p.n and d["config"]["n_charges"] == p.nc
    assert abs(d["iterations"] - ref["report"]["iterations"]) <= 1
    assert d["energy_kcal_mol"] == pytest.approx(ref["energy"], rel=1e-8)
