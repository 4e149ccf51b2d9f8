"""GPU checks of the exact fixed-point sums of the symmetric product (bipb_set_sum_mode(ctx, 1);
csrc/bipb_exact.cuh): parity with the oracle (north_star tolerances), agreement with the
fixed-order double partials to rounding, bitwise independence of the launch schedule and of the
rank count (integer sums are associative), and the out-of-range fallback."""
import os

import numpy as np
import pytest

import bipb_inputs as g
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bp():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1301_5885_b200 as bp
    return bp


def _ctx(bp, p, mode):
    ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
    ctx.set_matvec_kernel(1)
    ctx.set_sum_mode(mode)
    assert ctx.sum_mode == mode
    return ctx


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _ragged(keep, seed=1, kappa=g.KAPPA, level=5, radius=4.0):
    p = g.sphere_problem(level, radius, g.charges_in_ball(37, 0.75 * radius, 8), kappa=kappa)
    idx = np.sort(np.random.default_rng(seed).choice(p.n, keep, replace=False))
    return g.Problem(f"ragged{keep}", np.ascontiguousarray(p.centroids[idx]), np.ascontiguousarray(p.normals[idx]),
                     np.ascontiguousarray(p.areas[idx]), p.charges, p.eps1, p.eps2, kappa)


CASES = [
    ("L3", lambda k: g.sphere_problem(3, 4.0, g.charges_in_ball(20, 3.0, 7), kappa=k)),
    ("ragged4999", lambda k: _ragged(4999, kappa=k)),
    ("ellipsoidL4", lambda k: g.Problem("ell", *g.elements(*g.ellipsoid(4, (24.0, 18.0, 14.0))),
                                       g.charges_in_ball(300, 1.0, 3, axes=(21.0, 15.0, 11.0)), kappa=k)),
    ("mid20000", lambda k: _ragged(20000, 2, kappa=k)),       # B = 384 block shape
    ("L6", lambda k: g.sphere_problem(6, 20.0, g.charges_in_ball(50, 18.0, 4), kappa=k)),  # B = 640
    ("ragged45001", lambda k: _ragged(45001, 11, kappa=k, level=6, radius=20.0)),  # B = 640, partial block
]


@pytest.mark.parametrize("kappa", [g.KAPPA, 0.0])
@pytest.mark.parametrize("name,make", CASES)
def test_exact_matvec_parity(bp, name, make, kappa):
    p = make(kappa)
    u = g.random_vector(2 * p.n, 11)
    c1 = _ctx(bp, p, 1)
    y1 = bp.bipb_matvec(c1, u)
    y1b = bp.bipb_matvec(c1, u)
    assert c1.sum_mode == 1  # no out-of-range partial on these inputs
    c0 = _ctx(bp, p, 0)
    y0 = bp.bipb_matvec(c0, u)
    assert np.array_equal(y1, y1b)
    assert _rel(y1, y0) <= 1e-14
    # the whole vector against the oracle, also for the bench's configuration (B = 640 blocks with
    # exact limb sums: L6 and the ragged 45,001): overall, per block and
    # element-wise against the block's scale
    ref = oracle.matvec(p, u)
    assert _rel(y1, ref) <= 1e-11
    for h in (slice(0, p.n), slice(p.n, 2 * p.n)):
        assert _rel(y1[h], ref[h]) <= 1e-11
        assert np.max(np.abs(y1[h] - ref[h])) <= 1e-11 * np.max(np.abs(ref[h]))
    c0.close()
    c1.close()


def test_exact_schedule_independent_bitwise(bp, monkeypatch):
    """The same product launched as one grid and as many I-block groups (different CTA sets and
    completion orders): bitwise identical with exact sums."""
    p = g.sphere_problem(6, 20.0, g.charges_in_ball(50, 18.0, 4))
    u = g.random_vector(2 * p.n, 3)
    c = _ctx(bp, p, 1)
    y_one = bp.bipb_matvec(c, u)
    c.close()
    monkeypatch.setenv("BIPB_SYM_MEM_GB", "0.01")
    c = _ctx(bp, p, 1)
    y_groups = bp.bipb_matvec(c, u)
    c.close()
    assert np.array_equal(y_one, y_groups)


@pytest.mark.parametrize("name,make", CASES[:3])
def test_exact_solve_parity(bp, name, make):
    p = make(g.KAPPA)
    ref = oracle.solve(p, restart=20, tol=1e-10)
    c = _ctx(bp, p, 1)
    x = np.zeros(2 * p.n)
    bp.bipb_source(c)
    st, rep = bp.bipb_gmres_solve(c, x, None, 20, 1e-10, 500, check_true=True)
    e = bp.bipb_energy(c, x)
    assert st == bp.OK and rep["converged"] and c.sum_mode == 1
    assert abs(rep["iterations"] - ref["report"]["iterations"]) <= 1
    assert e == pytest.approx(ref["energy"], rel=1e-8)
    assert _rel(x, ref["x"]) <= 1e-8
    c.close()


def test_exact_out_of_range_falls_back(bp, monkeypatch):
    """A shift far too large (test hook) puts every partial out of range: the product and the
    solve are recomputed with the double partials (bitwise the mode-0 results) and the context
    stays in mode 0."""
    p = g.sphere_problem(4, 4.0, g.charges_in_ball(20, 3.0, 7))
    u = g.random_vector(2 * p.n, 5)
    c0 = _ctx(bp, p, 0)
    y0 = bp.bipb_matvec(c0, u)
    x0 = np.zeros(2 * p.n)
    bp.bipb_source(c0)
    st0, rep0 = bp.bipb_gmres_solve(c0, x0, None, 20, 1e-10, 500)
    c0.close()
    monkeypatch.setenv("BIPB_EXACT_BIAS", "90")
    c = _ctx(bp, p, 1)
    y = bp.bipb_matvec(c, u)
    assert c.sum_mode == 0 and np.array_equal(y, y0)
    c.set_sum_mode(1)
    assert c.sum_mode == 1
    x = np.zeros(2 * p.n)
    bp.bipb_source(c)
    st, rep = bp.bipb_gmres_solve(c, x, None, 20, 1e-10, 500)
    assert st == st0 and rep["iterations"] == rep0["iterations"] and np.array_equal(x, x0)
    assert c.sum_mode == 0
    c.close()


def test_exact_zero_operand_and_errors(bp):
    p = g.sphere_problem(4, 4.0, g.charges_in_ball(20, 3.0, 7))
    c = _ctx(bp, p, 1)
    assert np.array_equal(bp.bipb_matvec(c, np.zeros(2 * p.n)), np.zeros(2 * p.n))
    with pytest.raises(bp.BipbError):
        c.set_sum_mode(2)
    c.close()
