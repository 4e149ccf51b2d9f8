"""Pins for the Kirkwood surface field (oracle/kirkwood.py), the phi^exa of the paper's
e_phi (Eq. (15)): closed forms, interface conditions Eq. (3), and the oracle BEM's
surface potential converging to it (Table 2 behaviour)."""
import numpy as np
import pytest

import bipb_inputs as g
import oracle
from oracle.kirkwood import kirkwood_exterior, kirkwood_surface


def _sphere_points(m, a, seed=1):
    u = np.random.default_rng(seed).normal(size=(m, 3))
    return a * u / np.linalg.norm(u, axis=1)[:, None]


@pytest.mark.parametrize("kappa", [0.0, 0.1257, 0.5])
def test_interface_conditions(kappa):
    """phi1 = phi2 and eps1 dphi1/dr = eps2 dphi2/dr on r = a (Eq. (3))."""
    ch, a = g.helix_charges(), 4.0
    pts = _sphere_points(40, a)
    p1, d1 = kirkwood_surface(pts, ch, a, 1.0, 80.0, kappa)
    p2, d2, _ = kirkwood_exterior(pts, ch, a, 1.0, 80.0, kappa)
    assert np.max(np.abs(p1 - p2)) <= 1e-12 * np.max(np.abs(p1))
    assert np.max(np.abs(1.0 * d1 - 80.0 * d2)) <= 1e-8 * np.max(np.abs(d1))


def test_central_charge_is_born():
    a, k = 2.0, 0.1257
    pts = _sphere_points(10, a)
    p, d = kirkwood_surface(pts, np.array([[0.0, 0, 0, 1.0]]), a, 1.0, 80.0, k)
    np.testing.assert_allclose(p, 1.0 / (4 * np.pi * a * 80.0 * (1 + k * a)), rtol=1e-12)
    np.testing.assert_allclose(d, -1.0 / (4 * np.pi * a * a), rtol=1e-14)  # Gauss: eps1 dphi/dr = -Q/(4 pi a^2)


def test_bem_surface_potential_converges():
    """e_phi = max|phi_num - phi_exa| / max|phi_exa| (Eq. (15)) decreases under refinement with
    an order near the paper's 0.5-0.6 per element count (Table 2)."""
    ch, a = g.helix_charges(), 4.0
    errs, ns = [], []
    for L in (2, 3, 4):
        p = g.sphere_problem(L, a, ch)
        x = oracle.solve(p, tol=1e-10)["x"]
        proj = a * p.centroids / np.linalg.norm(p.centroids, axis=1)[:, None]
        pe, _ = kirkwood_surface(proj, ch, a, p.eps1, p.eps2, p.kappa)
        errs.append(np.max(np.abs(x[:p.n] - pe)) / np.max(np.abs(pe)))
        ns.append(p.n)
    orders = [np.log(errs[i] / errs[i + 1]) / np.log(ns[i + 1] / ns[i]) for i in range(2)]
    assert errs[0] > errs[1] > errs[2]
    assert all(0.3 < o < 1.2 for o in orders), orders
