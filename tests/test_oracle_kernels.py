"""Pins for the oracle's pair functions (Eq. (5), Eq. (10), Eq. (11) of arXiv 1301.5885)
against things other than themselves: printed values, finite differences, exact
structural cancellations and symmetries of the definitions."""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
RNG = np.random.default_rng(12345)


def _unit(v):
    return v / np.linalg.norm(v)


def _configs(n=100):
    out = []
    for _ in range(n):
        x = RNG.uniform(-5, 5, 3)
        r = RNG.uniform(0.5, 10.0)
        y = x + r * _unit(RNG.normal(size=3))
        out.append((x, _unit(RNG.normal(size=3)), y, _unit(RNG.normal(size=3))))
    return out


def test_green_printed_values():
    # Eq. (5)
    o = np.zeros(3)
    assert oracle.G0(np.array([1.0, 0, 0]), o) == pytest.approx(GOLD["G0_r1"]["value"], rel=1e-15)
    assert oracle.G0(np.array([0, 4.0, 0]), o) == pytest.approx(GOLD["G0_r4"]["value"], rel=1e-15)
    gk = oracle.Gk(np.array([0, 0, 1.0]), o, 1.0)
    assert gk == pytest.approx(GOLD["Gk_k1_r1"]["value"], rel=1e-15)
    assert gk == pytest.approx(GOLD["Gk_k1_r1"]["printed"], rel=GOLD["Gk_k1_r1"]["printed_rtol"])


def test_gk_limits():
    for x, _, y, _ in _configs(20):
        assert oracle.Gk(x, y, 0.0) == oracle.G0(x, y)  # kappa = 0 limit, exact
        for k in (0.1257, 0.5, 2.0):
            assert 0 < oracle.Gk(x, y, k) <= oracle.G0(x, y)
        assert oracle.G0(x, y) == oracle.G0(y, x)


@pytest.mark.parametrize("kappa", [0.0, 0.1257, 0.5])
def test_first_derivatives_fd(kappa):
    """d/dnu_y and d/dnu_x against central FD (h = 1e-5 r), error normalised by G/r
    (expected max ~1e-10)."""
    worst = 0.0
    for x, nx, y, ny in _configs():
        r = np.linalg.norm(x - y)
        h = 1e-5 * r
        G = (lambda a, b: oracle.Gk(a, b, kappa))
        fd_y = (G(x, y + h * ny) - G(x, y - h * ny)) / (2 * h)
        fd_x = (G(x + h * nx, y) - G(x - h * nx, y)) / (2 * h)
        scale = G(x, y) / r
        worst = max(worst, abs(oracle.dGk_dny(x, y, ny, kappa) - fd_y) / scale,
                    abs(oracle.dGk_dnx(x, nx, y, kappa) - fd_x) / scale)
        if kappa == 0.0:
            assert oracle.dG0_dny(x, y, ny) == oracle.dGk_dny(x, y, ny, 0.0)
            assert oracle.dG0_dnx(x, nx, y) == oracle.dGk_dnx(x, nx, y, 0.0)
    assert worst < 1e-8


@pytest.mark.parametrize("kappa", [0.0, 0.1257, 0.5])
def test_mixed_derivative_fd(kappa):
    """d2G/dnu_x dnu_y against the 4-point mixed stencil (H = 1e-3 r), normalised by G/r^2."""
    worst = 0.0
    for x, nx, y, ny in _configs():
        r = np.linalg.norm(x - y)
        H = 1e-3 * r
        G = (lambda a, b: oracle.Gk(a, b, kappa))
        fd = (G(x + H * nx, y + H * ny) - G(x + H * nx, y - H * ny)
              - G(x - H * nx, y + H * ny) + G(x - H * nx, y - H * ny)) / (4 * H * H)
        worst = max(worst, abs(oracle.d2Gk_dnxdny(x, nx, y, ny, kappa) - fd) / (G(x, y) / r ** 2))
        if kappa == 0.0:
            assert oracle.d2G0_dnxdny(x, nx, y, ny) == oracle.d2Gk_dnxdny(x, nx, y, ny, 0.0)
    assert worst < 1e-4


def test_derivative_signs_hand_case():
    # target at origin with normal +x, charge/source one unit along +x:
    # dG0/dnu_x = -(x-y).nu_x/(4 pi r^3) = +1/(4 pi)
    x, n = np.zeros(3), np.array([1.0, 0, 0])
    y = np.array([1.0, 0, 0])
    assert oracle.dG0_dnx(x, n, y) == pytest.approx(1 / (4 * math.pi), rel=1e-15)
    assert oracle.dG0_dny(x, y, n) == pytest.approx(-1 / (4 * math.pi), rel=1e-15)
    # swap identity: dG/dnu_y(x, y) with normal n == dG/dnu_x(y, x) with the same normal
    for a, na, b, nb in _configs(20):
        assert oracle.dGk_dny(a, b, nb, 0.3) == pytest.approx(oracle.dGk_dnx(b, nb, a, 0.3), rel=1e-14)


def test_kernel_structural_zero():
    # kappa = 0 and eps = 1 => K1..K4 = 0 exactly
    for x, nx, y, ny in _configs(50):
        K = oracle.kernels(x, nx, y, ny, 1.0, 0.0)
        assert np.all(K == 0.0)
        K = oracle.kernels(x, nx, y, ny, 80.0, 0.0)
        assert K[0] == 0.0 and K[3] == 0.0


def test_kernel_symmetries():
    for x, nx, y, ny in _configs(50):
        Kxy = oracle.kernels(x, nx, y, ny, 80.0, 0.1257)
        Kyx = oracle.kernels(y, ny, x, nx, 80.0, 0.1257)
        assert Kxy[0] == Kyx[0]  # K1 symmetric (bitwise: |x-y| is exact under swap)
        assert Kxy[3] == pytest.approx(Kyx[3], rel=1e-12, abs=1e-15)  # K4 symmetric
        # K2(x,y) = eps dGk/dny - dG0/dny and K3(y,x) = dG0/dnx - dGk/dnx/eps with nu = ny:
        # eps*K3(y,x)|... relation: K2 uses +eps*Gk', K3 uses -Gk'/eps on the same derivative
        dk = oracle.dGk_dny(x, y, ny, 0.1257)
        d0 = oracle.dG0_dny(x, y, ny)
        assert Kxy[1] == pytest.approx(80.0 * dk - d0, rel=1e-15)


def test_kernel_values_vs_definition_fd():
    """x=(1,0,0), y=0, nx=ny=(1,0,0), kappa=0.5, eps -> K via FD of G0/Gk."""
    x, y, n = np.array([1.0, 0, 0]), np.zeros(3), np.array([1.0, 0, 0])
    eps, k, h = 80.0, 0.5, 1e-5
    G0 = oracle.G0
    Gk = (lambda a, b: oracle.Gk(a, b, k))
    K = oracle.kernels(x, n, y, n, eps, k)
    K1 = G0(x, y) - Gk(x, y)
    K2 = eps * (Gk(x, y + h * n) - Gk(x, y - h * n)) / (2 * h) - (G0(x, y + h * n) - G0(x, y - h * n)) / (2 * h)
    K3 = (G0(x + h * n, y) - G0(x - h * n, y)) / (2 * h) - (Gk(x + h * n, y) - Gk(x - h * n, y)) / (2 * h) / eps
    H = 1e-3

    def mixed(G):
        return (G(x + H * n, y + H * n) - G(x + H * n, y - H * n) - G(x - H * n, y + H * n)
                + G(x - H * n, y - H * n)) / (4 * H * H)
    K4 = mixed(Gk) - mixed(G0)
    assert K[0] == pytest.approx(K1, rel=1e-14)
    assert K[1] == pytest.approx(K2, rel=1e-6)
    assert K[2] == pytest.approx(K3, rel=1e-6)
    assert K[3] == pytest.approx(K4, rel=1e-4)
