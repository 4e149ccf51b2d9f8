"""Pins for the oracle's GMRES and for the whole Table 1 pipeline
(source -> GMRES -> energy) against textbook cases, LAPACK, and the Born / Kirkwood
closed forms the paper cites."""
import json
import os

import numpy as np
import pytest

import bipb_inputs as g
import oracle
from oracle.kirkwood import born_energy, kirkwood_energy

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_gmres_identity_one_iteration():
    b = np.random.default_rng(0).normal(size=17)
    x, st, rep = oracle.gmres_dense(np.eye(17), b, restart=10, tol=1e-12)
    assert st == 0 and rep["iterations"] == 1
    np.testing.assert_allclose(x, b, rtol=1e-14)


def test_gmres_2x2_spec_example():
    gd = GOLD["gmres_2x2"]
    x, st, rep = oracle.gmres_dense(np.array(gd["A"]), np.array(gd["b"]), restart=10, tol=1e-10)
    assert st == 0 and rep["iterations"] <= gd["max_iters"]
    np.testing.assert_allclose(x, gd["x"], rtol=1e-12)


def test_gmres_zero_rhs_and_max_iters():
    x, st, rep = oracle.gmres_dense(np.eye(3), np.zeros(3), x0=np.ones(3))
    assert st == 0 and np.all(x == 0) and rep["iterations"] == 0
    A = np.diag(np.arange(1.0, 51.0))
    x, st, rep = oracle.gmres_dense(A, np.ones(50), restart=5, tol=1e-14, max_iters=7)
    assert st == 2 and rep["iterations"] == 7 and not rep["converged"]


@pytest.mark.parametrize("m", [10, 20])
def test_gmres_bem_vs_lapack(m):
    p = g.sphere_problem(2, 4.0, g.helix_charges())
    A = oracle.dense_assemble(p)
    b = oracle.source(p)
    x_lu = np.linalg.solve(A, b)
    x, st, rep = oracle.gmres(p, b, restart=m, tol=1e-12)
    assert st == 0
    assert np.linalg.norm(x - x_lu) / np.linalg.norm(x_lu) < 1e-9
    assert rep["rel_res_true"] < 1e-11
    h = rep["history"]
    # residual estimate monotone non-increasing within each cycle (GMRES minimisation)
    for c0 in range(0, len(h), m):
        seg = h[c0:c0 + m]
        assert np.all(np.diff(seg) <= 1e-15 * seg[0])
    assert oracle.energy(p, x) == pytest.approx(oracle.energy(p, x_lu), rel=1e-10)


def test_born_converges_to_closed_form():
    """Born ion a = 4, kappa = 0 (-40.99): error decreases under refinement."""
    exact = born_energy(1.0, 4.0, 1.0, 80.0, 0.0)
    assert exact == pytest.approx(GOLD["born_a4_k0"]["value"], abs=GOLD["born_a4_k0"]["tol_abs"])
    errs, its = [], []
    for L in (2, 3, 4):
        p = g.sphere_problem(L, 4.0, np.array([[0.0, 0, 0, 1.0]]), kappa=0.0)
        r = oracle.solve(p, restart=10, tol=1e-10)
        assert r["status"] == 0
        errs.append(abs(r["energy"] / exact - 1))
        its.append(r["report"]["iterations"])
    assert errs[0] > errs[1] > errs[2] and errs[2] < 0.01
    assert max(its) <= 2 * min(its)  # iteration count flat under refinement


def test_born_with_salt_and_eps1():
    # eps1 = 2 exercises the 1/eps1 of reading R2; kappa > 0 the screened parts.
    for eps1, kappa, L, tolrel in ((1.0, 0.1257, 3, 0.025), (2.0, 0.0, 3, 0.025)):
        p = g.sphere_problem(L, 2.0 if kappa else 4.0, np.array([[0.0, 0, 0, 1.0]]), eps1=eps1, kappa=kappa)
        exact = born_energy(1.0, 2.0 if kappa else 4.0, eps1, 80.0, kappa)
        r = oracle.solve(p, restart=20, tol=1e-10)
        assert r["energy"] == pytest.approx(exact, rel=tolrel)
        assert r["energy"] < 0


def test_kirkwood_series_pins():
    # n = 0 term == Born with salt (independent closed form), kappa -> 0 continuity
    for a, k in ((4.0, 0.0), (2.0, 0.1257), (4.0, 0.5)):
        e, _ = kirkwood_energy(np.array([[0.0, 0, 0, 1.0]]), a, 1.0, 80.0, k)
        assert e == pytest.approx(born_energy(1.0, a, 1.0, 80.0, k), rel=1e-14)
    h = g.helix_charges()
    e0, _ = kirkwood_energy(h, 4.0, 1.0, 80.0, 0.0)
    e1, _ = kirkwood_energy(h, 4.0, 1.0, 80.0, 1e-9)
    assert e1 == pytest.approx(e0, rel=1e-8)
    # eps1 == eps2 and kappa == 0 => no reaction field
    e, _ = kirkwood_energy(h, 4.0, 2.0, 2.0, 0.0)
    assert abs(e) < 1e-12
    # g_n ratio recurrence vs scipy's modified Bessel K (library routine)
    from scipy.special import kv
    from oracle.kirkwood import g_ratio
    x = 0.5028
    kn = lambda n, t: kv(n + 0.5, t) / np.sqrt(t)
    hh = 1e-6
    ref = [x * (kn(n, x + hh) - kn(n, x - hh)) / (2 * hh) / kn(n, x) for n in range(12)]
    np.testing.assert_allclose(g_ratio(11, x), ref, rtol=1e-7)
    # rotation invariance of the series
    R = np.linalg.qr(np.random.default_rng(3).normal(size=(3, 3)))[0]
    hr = np.concatenate([h[:, :3] @ R.T, h[:, 3:]], 1)
    assert kirkwood_energy(hr, 4.0, 1.0, 80.0, 0.1257)[0] == pytest.approx(
        kirkwood_energy(h, 4.0, 1.0, 80.0, 0.1257)[0], rel=1e-12)


def test_bem_converges_to_kirkwood_random_charges():
    """C2-like (50 random charges in r <= 3, sphere a = 4): BEM -> Kirkwood, error ratio < 0.5/level."""
    ch = g.charges_in_ball(50, 3.0, 2)
    exact, _ = kirkwood_energy(ch, 4.0, 1.0, 80.0, 0.1257)
    errs = []
    for L in (2, 3, 4):
        p = g.sphere_problem(L, 4.0, ch)
        r = oracle.solve(p, restart=20, tol=1e-10)
        assert r["status"] == 0
        errs.append(abs(r["energy"] / exact - 1))
    assert errs[1] < 0.5 * errs[0] and errs[2] < 0.5 * errs[1] and errs[2] < 0.02


def test_energy_charge_scaling_quadratic():
    ch = g.helix_charges()
    p = g.sphere_problem(2, 4.0, ch)
    e1 = oracle.solve(p, tol=1e-12)["energy"]
    p2 = g.sphere_problem(2, 4.0, np.concatenate([ch[:, :3], 2 * ch[:, 3:]], 1))
    e2 = oracle.solve(p2, tol=1e-12)["energy"]
    assert e2 == pytest.approx(4 * e1, rel=1e-8)


def test_table2_trend_helix():
    """Table 2 trend: E_sol decreases in magnitude monotonically toward the
    exact value under refinement.  Parity with the printed numbers is unpinned (R9)."""
    ch = g.helix_charges()
    exact, _ = kirkwood_energy(ch, 4.0, 1.0, 80.0, 0.1257)
    es = [oracle.solve(g.sphere_problem(L, 4.0, ch), tol=1e-8)["energy"] for L in (2, 3, 4)]
    assert es[0] < es[1] < es[2] < exact < 0
    paper = GOLD["table2_sphere"]["E_sol"]
    assert all(a < b for a, b in zip(paper, paper[1:]))  # same monotone approach in the paper


# ---- right-preconditioned GMRES (jump-term diagonal; the library's opt-in bipb_set_precond) ----

@pytest.mark.parametrize("m", [10, 20])
def test_gmres_jacobi_vs_lapack_and_scaled_matrix(m):
    """Right preconditioning M = diag(1/2 (1 + eps), 1/2 (1 + 1/eps)) (Saad Alg. 9.5): the solution is
    LAPACK's; the iteration is plain GMRES on the explicitly scaled matrix A M^-1 (a different loop:
    dense scaled matrix, plain core, x = M^-1 y), same iteration count; the estimate stays monotone
    per cycle, the true residual meets the tolerance."""
    p = g.sphere_problem(2, 4.0, g.helix_charges())
    A = oracle.dense_assemble(p)
    b = oracle.source(p)
    eps = p.eps2 / p.eps1
    minv = np.concatenate([np.full(p.n, 1.0 / (0.5 * (1 + eps))), np.full(p.n, 1.0 / (0.5 * (1 + 1 / eps)))])
    x_lu = np.linalg.solve(A, b)
    x, st, rep = oracle.gmres(p, b, restart=m, tol=1e-12, precond=True)
    assert st == 0 and rep["rel_res_true"] < 1e-11
    assert np.linalg.norm(x - x_lu) / np.linalg.norm(x_lu) < 1e-9
    y, st2, rep2 = oracle.gmres_dense(A * minv[None, :], b, restart=m, tol=1e-12)
    assert st2 == 0 and rep2["iterations"] == rep["iterations"]
    assert np.linalg.norm(minv * y - x) / np.linalg.norm(x) < 1e-10
    xd, _, rep3 = oracle.gmres_dense(A, b, restart=m, tol=1e-12, minv=minv)
    assert rep3["iterations"] == rep["iterations"] and np.linalg.norm(xd - x) / np.linalg.norm(x) < 1e-10
    h = rep["history"]
    for c0 in range(0, len(h), m):
        seg = h[c0:c0 + m]
        assert np.all(np.diff(seg) <= 1e-15 * seg[0])


def test_gmres_jacobi_identity_when_eps_is_one():
    """eps1 = eps2 => M = I: the preconditioned iteration is the plain one, bit for bit."""
    p = g.sphere_problem(2, 4.0, g.helix_charges(), eps2=1.0)
    b = oracle.source(p)
    x0, _, r0 = oracle.gmres(p, b, restart=10, tol=1e-12)
    x1, _, r1 = oracle.gmres(p, b, restart=10, tol=1e-12, precond=True)
    assert r0["iterations"] == r1["iterations"]
    assert np.array_equal(x0, x1) and np.array_equal(r0["history"], r1["history"])


def test_gmres_jacobi_same_energy_fewer_iterations():
    """Same linear system => same solvation energy; the scaling of the 2x2 jump structure
    (1/2 (1 + eps) = 40.5 vs 1/2 (1 + 1/eps) = 0.506) cuts the iteration count (L3: 27 -> 10)."""
    p = g.sphere_problem(3, 4.0, g.charges_in_ball(20, 3.0, 7))
    a = oracle.solve(p, restart=20, tol=1e-10)
    j = oracle.solve(p, restart=20, tol=1e-10, precond=True)
    assert j["report"]["rel_res_true"] <= 1e-9
    assert j["energy"] == pytest.approx(a["energy"], rel=1e-8)
    assert j["report"]["iterations"] <= 0.6 * a["report"]["iterations"]


def test_gmres_checkpointed_replays_bitwise(tmp_path):
    """The product store used for the full-size C4 golden (tests/make_oracle_golden.py --store):
    same x, history and counts as the plain oracle GMRES, also when resumed from a partial store,
    and a stored product made from another x is detected."""
    p = g.sphere_problem(2, 4.0, g.helix_charges())
    b = oracle.source(p)
    x0, st0, r0 = oracle.gmres(p, b, restart=10, tol=1e-12)
    store = str(tmp_path / "store")
    x1, st1, r1 = oracle.gmres_checkpointed(p, b, store, restart=10, tol=1e-12)
    assert st1 == st0 and np.array_equal(x0, x1) and np.array_equal(r0["history"], r1["history"])
    assert r1["matvecs"] == r0["matvecs"] == len(os.listdir(store))
    files = sorted(os.listdir(store))
    for f in files[len(files) // 2:]:  # a run cut off half way
        os.remove(os.path.join(store, f))
    x2, _, r2 = oracle.gmres_checkpointed(p, b, store, restart=10, tol=1e-12)
    assert np.array_equal(x0, x2) and r2["iterations"] == r0["iterations"]
    os.rename(os.path.join(store, files[1]), os.path.join(store, files[1][:4] + "0000000000000000.npy"))
    with pytest.raises(RuntimeError):
        oracle.gmres_checkpointed(p, b, store, restart=10, tol=1e-12)
