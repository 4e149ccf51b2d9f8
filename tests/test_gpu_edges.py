"""GPU parity at the method's parameter edges: the CUDA path against the
oracle for (eps1, eps2, kappa) away from the generator defaults (1, 80, 0.1257), both matvec
kernels, element-wise and per block.

  (2, 80, 0.1257)  eps1 != 1: the 1/eps1 of the sources (reading R2, Eq. (11)) and
                   eps = eps2/eps1 = 40 (reading R1, Eqs. (8)-(10)) differ from
                   eps2 -- a path that confused them is exact only at eps1 = 1;
  (4, 4, 0)        eps = 1 and kappa = 0: K1..K4 vanish identically (Eq. (10)), A = I, x = b,
                   E_sol = 0 (the jump terms 1/2(1+eps) = 1/2(1+1/eps) = 1);
  (1, 2, 0.5)      kappa r up to 4 on the R = 4 sphere (the table exp well past t = 1);
  (1, 80, 2.0)     kappa r up to 16 (t > 10 on the table exp, where only an absolute bound holds);
tolerances are north_star's (BASELINE.json): matvec rel-L2 <= 1e-11 overall, per block and
element-wise against the block's scale; source <= 1e-12; E_sol 1e-8; iterations +-1."""
import numpy as np
import pytest

import bipb_inputs as g
import oracle

pytestmark = pytest.mark.gpu

PARAMS = [(2.0, 80.0, 0.1257), (4.0, 4.0, 0.0), (1.0, 2.0, 0.5), (1.0, 80.0, 2.0)]


@pytest.fixture(scope="module")
def bp():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1301_5885_b200 as bp
    return bp


def _with(p, eps1, eps2, kappa):
    return g.Problem(p.name, p.centroids, p.normals, p.areas, p.charges, eps1, eps2, kappa)


def _ragged(keep, seed=1):
    p = g.sphere_problem(4, 4.0, g.charges_in_ball(37, 3.0, 8))
    idx = np.sort(np.random.default_rng(seed).choice(p.n, keep, replace=False))
    return g.Problem(f"ragged{keep}", np.ascontiguousarray(p.centroids[idx]), np.ascontiguousarray(p.normals[idx]),
                     np.ascontiguousarray(p.areas[idx]), p.charges)


SHAPES = {
    "L3": lambda: g.sphere_problem(3, 4.0, g.charges_in_ball(20, 3.0, 7)),
    "ragged4999": lambda: _ragged(4999),
}


def _ctx(bp, p, kind):
    c = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
    c.set_matvec_kernel(kind)
    return c


def _close(y, ref, n):
    """rel-L2 overall and per block, and element-wise against each block's scale."""
    tol = 1e-11
    assert np.linalg.norm(y - ref) <= tol * np.linalg.norm(ref)
    for h in (slice(0, n), slice(n, 2 * n)):
        scale = np.max(np.abs(ref[h]))
        assert np.linalg.norm(y[h] - ref[h]) <= tol * np.linalg.norm(ref[h]) + 1e-300
        assert np.max(np.abs(y[h] - ref[h])) <= tol * scale + 1e-300


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("shape", list(SHAPES))
@pytest.mark.parametrize("eps1,eps2,kappa", PARAMS)
def test_edge_matvec_source_energy(bp, eps1, eps2, kappa, shape, kind):
    p = _with(SHAPES[shape](), eps1, eps2, kappa)
    c = _ctx(bp, p, kind)
    for u in (g.random_vector(2 * p.n, 11), g.random_vector(2 * p.n, 0, smooth_centroids=p.centroids)):
        y = bp.bipb_matvec(c, u)
        ref = oracle.matvec(p, u)
        _close(y, ref, p.n)
        if eps1 == eps2 and kappa == 0.0:  # A = I exactly (K1..K4 = 0, jump terms 1)
            assert np.array_equal(y, u)
    b = bp.bipb_source(c)
    bo = oracle.source(p)
    for h in (slice(0, p.n), slice(p.n, 2 * p.n)):
        assert np.linalg.norm(b[h] - bo[h]) <= 1e-12 * np.linalg.norm(bo[h])
    x = g.random_vector(2 * p.n, 5)
    phi = np.zeros(p.nc)
    e = bp.bipb_energy(c, x, phi)
    phio = oracle.reaction_potential(p, x)
    eo = oracle.energy(p, x)
    if eps1 == eps2 and kappa == 0.0:
        assert e == 0.0 and eo == 0.0 and not np.any(phi)
    else:
        assert np.linalg.norm(phi - phio) <= 1e-12 * np.linalg.norm(phio)
        assert e == pytest.approx(eo, rel=1e-11)
    c.close()


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("shape", list(SHAPES))
@pytest.mark.parametrize("eps1,eps2,kappa", PARAMS)
def test_edge_solve(bp, eps1, eps2, kappa, shape, kind):
    p = _with(SHAPES[shape](), eps1, eps2, kappa)
    ref = oracle.solve(p, restart=20, tol=1e-10)
    c = _ctx(bp, p, kind)
    out = bp.solve(c, restart_m=20, tol=1e-10, check_true=True)
    c.close()
    assert out["status"] == bp.OK
    assert abs(out["report"]["iterations"] - ref["report"]["iterations"]) <= 1
    if eps1 == eps2 and kappa == 0.0:  # A = I: one Arnoldi step, x = b, no reaction field
        assert out["report"]["iterations"] == ref["report"]["iterations"] == 1
        assert out["energy"] == 0.0 and ref["energy"] == 0.0
        np.testing.assert_allclose(out["x"], ref["b"], rtol=1e-14, atol=1e-14 * np.abs(ref["b"]).max())
    else:
        assert out["energy"] == pytest.approx(ref["energy"], rel=1e-8)
    assert np.linalg.norm(out["x"] - ref["x"]) <= 1e-8 * np.linalg.norm(ref["x"])
    assert out["report"]["rel_res_true"] <= 1e-9
