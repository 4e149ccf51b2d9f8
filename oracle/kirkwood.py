"""ORACLE — TEST INFRASTRUCTURE ONLY.  Closed-form solvation energies for a dielectric
sphere, the analytic references of PAPER.md §3.1-3.2 (P:104-106, 371-372, 420-422:
"analytical solutions in terms of spherical harmonics are available [Kirkwood34]").

The paper cites Kirkwood (1934) without printing coefficients; they are re-derived in
SURVEY.md Appendix A.3 by matching phi and eps*dphi/dr on r = a order by order
(interface conditions Eq. (3)):

  E_sol = 1/2 C_E sum_k sum_l Q_k Q_l sum_n (|y_k||y_l|)^n / (eps1 a^(2n+1)) f_n P_n(cos g_kl)
  f_n   = (eps2 g_n + (n+1) eps1) / (n eps1 - eps2 g_n),   g_n = x k_n'(x)/k_n(x), x = kappa a

with k_n the modified spherical Bessel function of the second kind.  Units follow
reading R3 (q = Q in e_c, C_E = 332.0716 kcal A / mol).
"""
from __future__ import annotations

import numpy as np

C_E = 332.0716


def born_energy(Q: float, a: float, eps1: float, eps2: float, kappa: float) -> float:
    """Born ion with salt: 1/2 C_E Q^2/a [1/(eps2 (1+kappa a)) - 1/eps1]."""
    return 0.5 * C_E * Q * Q / a * (1.0 / (eps2 * (1.0 + kappa * a)) - 1.0 / eps1)


def g_ratio(nmax: int, x: float) -> np.ndarray:
    """g_n = x k_n'(x)/k_n(x) for n = 0..nmax via the ratio R_n = k_{n-1}/k_n:
    R_0 = 1 (k_{-1} = k_0), 1/R_{n+1} = R_n + (2n+1)/x, and g_n = -x R_n - (n+1)
    (from k_n' = -k_{n-1} - (n+1) k_n / x).  For x = 0: g_n = -(n+1)."""
    g = np.empty(nmax + 1)
    if x == 0.0:
        return -(np.arange(nmax + 1) + 1.0)
    R = 1.0
    for n in range(nmax + 1):
        g[n] = -x * R - (n + 1.0)
        R = 1.0 / (R + (2.0 * n + 1.0) / x)
    return g


def f_coeff(nmax: int, eps1: float, eps2: float, kappa: float, a: float) -> np.ndarray:
    g = g_ratio(nmax, kappa * a)
    n = np.arange(nmax + 1, dtype=np.float64)
    return (eps2 * g + (n + 1.0) * eps1) / (n * eps1 - eps2 * g)


def kirkwood_energy(charges: np.ndarray, a: float, eps1: float, eps2: float, kappa: float,
                    center=(0.0, 0.0, 0.0), rtol: float = 1e-13, nmax: int = 400) -> tuple[float, int]:
    """Kirkwood-series E_sol [kcal/mol] for charges (x,y,z,Q) strictly inside the sphere
    |y - center| < a.  Terms are added until the last three are below rtol*|E|.
    Returns (E, number of terms used)."""
    ch = np.asarray(charges, dtype=np.float64)
    if ch.shape[0] == 0:
        return 0.0, 0
    pos = ch[:, :3] - np.asarray(center)[None, :]
    Q = ch[:, 3]
    s = np.linalg.norm(pos, axis=1)
    if np.any(s >= a):
        raise ValueError("charges must lie strictly inside the sphere")
    with np.errstate(invalid="ignore", divide="ignore"):
        u = np.where(s[:, None] > 0, pos / np.where(s > 0, s, 1.0)[:, None], 0.0)
    cosg = np.clip(u @ u.T, -1.0, 1.0)
    f = f_coeff(nmax, eps1, eps2, kappa, a)
    ss = np.outer(s, s) / (a * a)
    QQ = np.outer(Q, Q)
    total = 0.0
    small = 0
    p_prev, p_cur = None, np.ones_like(cosg)  # P_0; Bonnet recurrence carried along
    w = QQ.copy()                              # Q_k Q_l (s_k s_l / a^2)^n
    for n in range(nmax + 1):
        if n == 1:
            p_prev, p_cur = p_cur, cosg.copy()
        elif n > 1:
            p_prev, p_cur = p_cur, ((2 * n - 1) * cosg * p_cur - (n - 1) * p_prev) / n
        if n > 0:
            w *= ss
        term = float(np.sum(w * p_cur)) * f[n] / (eps1 * a)
        total += term
        if n > 2 and abs(term) <= rtol * max(abs(total), 1e-300):
            small += 1
            if small >= 3:
                return 0.5 * C_E * total, n + 1
        else:
            small = 0
    raise RuntimeError("Kirkwood series did not converge within nmax terms")


def _charge_sums(points, charges, a, center, nmax):
    """For each point x (|x - center| = r) and order n: S_n(x) = sum_k Q_k s_k^n P_n(cos g_k),
    yielded as (n, S_n) with s_k = |y_k| / a scaled out (returns sums of Q_k (s_k/a)^n P_n)."""
    ch = np.asarray(charges, dtype=np.float64)
    pos = ch[:, :3] - np.asarray(center)[None, :]
    Q = ch[:, 3]
    s = np.linalg.norm(pos, axis=1)
    x = np.asarray(points, dtype=np.float64) - np.asarray(center)[None, :]
    r = np.linalg.norm(x, axis=1)
    with np.errstate(invalid="ignore", divide="ignore"):
        uy = np.where(s[:, None] > 0, pos / np.where(s > 0, s, 1.0)[:, None], 0.0)
        ux = x / np.where(r > 0, r, 1.0)[:, None]
    cosg = np.clip(ux @ uy.T, -1.0, 1.0)  # [M, K]
    w = np.broadcast_to(Q, cosg.shape).copy()
    sa = s / a
    p_prev, p_cur = None, np.ones_like(cosg)
    for n in range(nmax + 1):
        if n == 1:
            p_prev, p_cur = p_cur, cosg.copy()
        elif n > 1:
            p_prev, p_cur = p_cur, ((2 * n - 1) * cosg * p_cur - (n - 1) * p_prev) / n
        if n > 0:
            w *= sa[None, :]
        yield n, (w * p_cur).sum(axis=1), r


def kirkwood_surface(points, charges, a, eps1, eps2, kappa, center=(0.0, 0.0, 0.0), nmax=None):
    """Interior-limit potential phi1 and normal derivative d(phi1)/dr at points with
    |x - center| <= a (the quantities the BEM unknowns approximate; Eq. (15) uses
    phi^exa "by Kirkwood's spherical harmonic expansion").  Internal units of
    reading R3 (q/(4 pi eps1 r) Coulomb).  SURVEY.md App. A.3:
      phi1(x) = sum_k Q_k / (4 pi eps1 |x - y_k|)
              + sum_n r^n f_n / (4 pi eps1 a^(2n+1)) sum_k Q_k s_k^n P_n(cos g_k).
    Returns (phi1, dphi1_dr) arrays."""
    ch = np.asarray(charges, dtype=np.float64)
    x = np.asarray(points, dtype=np.float64)
    if nmax is None:
        smax = np.max(np.linalg.norm(ch[:, :3] - np.asarray(center)[None, :], axis=1)) / a
        nmax = int(min(400, max(10, np.ceil(np.log(1e-17) / np.log(max(smax, 1e-3))) + 5)))
    f = f_coeff(nmax, eps1, eps2, kappa, a)
    d = x[:, None, :] - ch[None, :, :3]
    dist = np.linalg.norm(d, axis=2)
    xc = x - np.asarray(center)[None, :]
    r = np.linalg.norm(xc, axis=1)
    rhat = xc / np.where(r > 0, r, 1.0)[:, None]
    phi = (ch[None, :, 3] / (4 * np.pi * eps1 * dist)).sum(axis=1)
    dphi = (-ch[None, :, 3] * np.einsum("mkc,mc->mk", d, rhat) / (4 * np.pi * eps1 * dist ** 3)).sum(axis=1)
    for n, S, rr in _charge_sums(x, ch, a, center, nmax):
        # S = sum_k Q_k (s_k/a)^n P_n ; reaction term r^n f_n/(4 pi eps1 a^(2n+1)) sum Q s^n P_n
        #   = f_n/(4 pi eps1 a) (r/a)^n S
        ra = rr / a
        phi = phi + f[n] / (4 * np.pi * eps1 * a) * ra ** n * S
        if n > 0:
            dphi = dphi + f[n] / (4 * np.pi * eps1 * a) * n * ra ** (n - 1) / a * S
    return phi, dphi


def kirkwood_exterior(points, charges, a, eps1, eps2, kappa, center=(0.0, 0.0, 0.0), nmax=60):
    """Exterior potential phi2 and d(phi2)/dr at |x - center| = r >= a (same expansion, matched
    at r = a: C_n k_n(kappa a) = A_n (1 + f_n)); used to pin the interface conditions Eq. (3)."""
    ch = np.asarray(charges, dtype=np.float64)
    f = f_coeff(nmax, eps1, eps2, kappa, a)
    g = g_ratio(nmax, kappa * a)
    phi = 0.0
    dphi = 0.0
    for n, S, rr in _charge_sums(points, ch, a, center, nmax):
        An = S / (4 * np.pi * eps1 * a)  # sum_k Q_k s_k^n P_n / (4 pi eps1 a^(n+1)) in units of a^n
        if kappa == 0.0:
            rad, drad = (a / rr) ** (n + 1), -(n + 1) / rr * (a / rr) ** (n + 1)
        else:
            from scipy.special import kv
            kn = lambda z: kv(n + 0.5, z) / np.sqrt(z)
            rad = kn(kappa * rr) / kn(kappa * a)
            # d/dr k_n(kappa r) / k_n(kappa a) at r: central difference of the library Bessel
            h = 1e-6 * rr
            drad = (kn(kappa * (rr + h)) - kn(kappa * (rr - h))) / (2 * h) / kn(kappa * a)
        phi = phi + An * (1 + f[n]) * rad
        dphi = dphi + An * (1 + f[n]) * drad
    return phi, dphi, g
