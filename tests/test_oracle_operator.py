"""Pins for the oracle's direct sums: source (Eq. (11)), matvec (Eqs. (12)-(13)),
reaction potential / energy (Eq. (14)), against closed forms, dense assembly, Gauss's
law, symmetry and invariance properties -- never against a retyped copy of itself."""
import math

import numpy as np
import pytest

import bipb_inputs as g
import oracle
from oracle.kirkwood import born_energy

EPS = 80.0


def _rot(angle=0.7, axis=(1.0, 2.0, 3.0)):
    a = np.asarray(axis) / np.linalg.norm(axis)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(angle) * K + (1 - math.cos(angle)) * K @ K


def test_source_single_central_charge_closed_form():
    # one charge Q at the centre: b_i = Q/(4 pi eps1 |x_i|), b_{i+N} = -Q (x_i.nu_i)/(4 pi eps1 |x_i|^3)
    for eps1 in (1.0, 2.0):
        p = g.sphere_problem(3, 4.0, np.array([[0.0, 0.0, 0.0, 0.7]]), eps1=eps1)
        b = oracle.source(p)
        r = np.linalg.norm(p.centroids, axis=1)
        xn = np.einsum("ij,ij->i", p.centroids, p.normals)
        np.testing.assert_allclose(b[:p.n], 0.7 / (4 * np.pi * eps1 * r), rtol=1e-14)
        np.testing.assert_allclose(b[p.n:], -0.7 * xn / (4 * np.pi * eps1 * r ** 3), rtol=1e-13)


def test_source_zero_charges():
    p = g.sphere_problem(2, 4.0, np.zeros((0, 4)))
    assert np.all(oracle.source(p) == 0.0)


def test_matvec_n1_diagonal_only():
    p = g.Problem("n1", np.array([[1.0, 0, 0]]), np.array([[1.0, 0, 0]]), np.array([0.3]),
                  np.zeros((0, 4)))
    y = oracle.matvec(p, np.array([2.0, 3.0]))
    assert y[0] == 0.5 * (1 + EPS) * 2.0 and y[1] == 0.5 * (1 + 1 / EPS) * 3.0


@pytest.mark.parametrize("kappa", [0.0, 0.1257])
def test_matvec_equals_dense(kappa):
    p = g.sphere_problem(2, 4.0, np.zeros((0, 4)), kappa=kappa)
    A = oracle.dense_assemble(p)
    for seed in (1, 2):
        u = g.random_vector(2 * p.n, seed)
        y = oracle.matvec(p, u)
        ref = A @ u
        assert np.max(np.abs(y - ref)) / np.max(np.abs(ref)) < 1e-13
    rows = np.array([0, 5, 77, p.n - 1])
    yi, yin = oracle.matvec_rows(p, u, rows)
    assert np.array_equal(yi, y[rows]) and np.array_equal(yin, y[rows + p.n])


def test_matvec_linearity():
    p = g.sphere_problem(2, 4.0, np.zeros((0, 4)))
    u, v = g.random_vector(2 * p.n, 3), g.random_vector(2 * p.n, 4)
    lhs = oracle.matvec(p, 2.5 * u - 0.75 * v)
    rhs = 2.5 * oracle.matvec(p, u) - 0.75 * oracle.matvec(p, v)
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs) < 1e-13


def test_dense_block_symmetry():
    """W-scaled K1 block symmetric (to the rounding of the W multiply/divide); K4 block symmetric to rounding (K1, K4 of Eq. (10)
    are symmetric in (x, nu_x) <-> (y, nu_y))."""
    p = g.sphere_problem(2, 4.0, np.zeros((0, 4)))
    A = oracle.dense_assemble(p)
    n = p.n
    B1 = A[:n, n:] / -p.areas[None, :]
    np.fill_diagonal(B1, 0.0)
    assert np.max(np.abs(B1 - B1.T)) / np.max(np.abs(B1)) < 1e-15
    B4 = A[n:, :n] / -p.areas[None, :]
    np.fill_diagonal(B4, 0.0)
    assert np.max(np.abs(B4 - B4.T)) / np.max(np.abs(B4)) < 1e-12


def test_gauss_law_double_layer():
    """kappa = 0: K2 = (eps - 1) dG0/dnu_y.  Gauss: sum_j W_j dG0/dnu_y(p, x_j) -> -1 for p
    inside (O(h^2)), and -> -1/2 at a centroid (principal value, O(h)).  So for
    u = [1; 0]:  phi_reac(p) = (eps-1) sum -> -(eps - 1)  and  (A u)_i -> eps."""
    errs_in, errs_on = [], []
    for L in (2, 3, 4):
        p = g.sphere_problem(L, 4.0, np.array([[0.0, 0, 0, 1.0], [1.0, 2.0, -1.5, 1.0]]), kappa=0.0)
        u = np.concatenate([np.ones(p.n), np.zeros(p.n)])
        phi = oracle.reaction_potential(p, u)
        errs_in.append(np.max(np.abs(phi / (EPS - 1) + 1.0)))
        y = oracle.matvec(p, u)
        errs_on.append(abs(np.mean(y[:p.n]) / EPS - 1.0))
    assert errs_in[-1] < 2e-3 and errs_in[0] / errs_in[1] > 3.5 and errs_in[1] / errs_in[2] > 3.5
    assert errs_on[-1] < 0.01 and errs_on[0] > errs_on[1] > errs_on[2]


def test_rotation_invariance():
    R = _rot()
    p = g.sphere_problem(2, 4.0, g.charges_in_ball(7, 3.0, 11))
    q = g.Problem("rot", p.centroids @ R.T, p.normals @ R.T, p.areas,
                  np.concatenate([p.charges[:, :3] @ R.T, p.charges[:, 3:]], 1))
    u = g.random_vector(2 * p.n, 5)
    y1, y2 = oracle.matvec(p, u), oracle.matvec(q, u)
    assert np.linalg.norm(y1 - y2) / np.linalg.norm(y1) < 1e-13
    b1, b2 = oracle.source(p), oracle.source(q)
    assert np.linalg.norm(b1 - b2) / np.linalg.norm(b1) < 1e-13
    e1, e2 = oracle.energy(p, u), oracle.energy(q, u)
    assert abs(e1 - e2) / abs(e1) < 1e-12


def test_energy_linearity_zero():
    p = g.sphere_problem(2, 4.0, g.charges_in_ball(5, 3.0, 9))
    x = g.random_vector(2 * p.n, 6)
    assert np.all(oracle.reaction_potential(p, np.zeros(2 * p.n)) == 0.0)
    phi = oracle.reaction_potential(p, x)
    np.testing.assert_allclose(oracle.reaction_potential(p, 2 * x), 2 * phi, rtol=1e-14)
    # E = 1/2 * 4 pi * 332.0716 * sum_k Q_k phi_reac(x_k)   (Eq. (14), reading R3)
    e = oracle.energy(p, x)
    assert e == pytest.approx(0.5 * 4 * np.pi * 332.0716 * float(np.dot(p.charges[:, 3], phi)), rel=1e-14)
    p0 = g.sphere_problem(2, 4.0, np.zeros((0, 4)))
    assert oracle.energy(p0, x) == 0.0
