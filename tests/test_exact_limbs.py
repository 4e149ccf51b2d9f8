"""Host checks of the exact fixed-point accumulation arithmetic (csrc/bipb_exact.cuh, used by
the symmetric kernel's `bipb_set_sum_mode(ctx, 1)`): the header's __host__ __device__ functions
compiled for the host with g++ and compared with Python's arbitrary-precision integers and
fractions (an independent exact model of the same definitions)."""
import ctypes
import os
import random
import subprocess
from fractions import Fraction

import numpy as np
import pytest

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1301_5885_b200", "csrc",
                   "bipb_exact.cuh")
SHIM = r"""
#include "%s"
extern "C" int split(double v, int S, long long* o) {
  bipb::ExactLimbs l; bool ok = bipb::exact_split(v, std::ldexp(1.0, S), l);
  o[0] = l.l0; o[1] = l.l1; o[2] = l.l2; return ok ? 1 : 0; }
extern "C" double value(long long a, long long b, long long c, int S) {
  return bipb::exact_value(a, b, c, std::ldexp(1.0, -S)); }
extern "C" int shift(int eb) { return bipb::exact_shift(eb); }
extern "C" int expf_(double v) { return bipb::exact_exp_field(v); }
"""


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    d = tmp_path_factory.mktemp("exact")
    src = d / "shim.cpp"
    src.write_text(SHIM % HDR)
    so = d / "shim.so"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC", "-o", str(so),
                           str(src)])
    L = ctypes.CDLL(str(so))
    L.split.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong)]
    L.value.argtypes = [ctypes.c_longlong] * 3 + [ctypes.c_int]
    L.value.restype = ctypes.c_double
    L.expf_.argtypes = [ctypes.c_double]
    return L


def _split(L, v, S):
    o = (ctypes.c_longlong * 3)()
    ok = L.split(v, S, o)
    return ok, (o[0], o[1], o[2])


def _int(l):
    return l[0] + (l[1] << 40) + (l[2] << 80)


def _round_half_even(fr):
    f = fr.numerator // fr.denominator
    rem = fr - f
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and f % 2 == 1):
        f += 1
    return f


def test_split_is_the_rounded_scaled_value(lib):
    """limbs(v) represent round_half_even(v 2^S) exactly, with 0 <= |l|, |m| < 2^40 (+1 for l)."""
    rng = random.Random(1)
    for _ in range(4000):
        S = rng.randint(-60, 200)
        e = rng.randint(-120, 117) - S
        v = rng.choice((-1, 1)) * rng.random() * 2.0 ** e
        ok, l = _split(lib, v, S)
        assert ok
        assert _int(l) == _round_half_even(Fraction(v) * Fraction(2) ** S) * 1, (v, S)
        assert abs(l[0]) <= 2 ** 40 and abs(l[1]) < 2 ** 40 and abs(l[2]) < 2 ** 38


def test_split_range_and_nonfinite(lib):
    S = 80
    assert _split(lib, 2.0 ** (117 - S) * 1.999, S)[0] == 1
    for bad in (2.0 ** (118 - S), -2.0 ** (119 - S), float("inf"), float("nan"), -float("inf")):
        assert _split(lib, bad, S)[0] == 0


def test_sum_exact_and_order_independent(lib):
    """Accumulated limbs (wrapping int64 adds, any order) equal the exact sum of the rounded
    terms; the converted double is within 1 ulp of that exact sum and identical for every order."""
    rng = np.random.default_rng(2)
    for trial in range(30):
        S = int(rng.integers(40, 120))
        K = int(rng.integers(1, 3000))
        mags = 2.0 ** rng.uniform(-70, 30, K) * 2.0 ** (80 - S)
        vals = (rng.choice([-1.0, 1.0], K) * mags).tolist()
        if trial % 3 == 0:  # heavy cancellation
            vals += [-v for v in vals[: K // 2]]
        exact = 0
        sums = []
        for perm in range(3):
            order = list(range(len(vals)))
            if perm:
                random.Random(perm).shuffle(order)
            acc = [0, 0, 0]
            for i in order:
                ok, l = _split(lib, vals[i], S)
                assert ok
                acc = [(acc[k] + l[k] + 2 ** 63) % 2 ** 64 - 2 ** 63 for k in range(3)]  # int64 wrap
            sums.append(lib.value(acc[0], acc[1], acc[2], S))
            if perm == 0:
                exact = sum(_round_half_even(Fraction(v) * Fraction(2) ** S) for v in vals)
                assert _int(acc) == exact
        assert sums[0] == sums[1] == sums[2]
        ref = float(Fraction(exact) / Fraction(2) ** S)
        assert abs(sums[0] - ref) <= 2 * np.spacing(abs(ref)) + 2.0 ** -S, (sums[0], ref)


def test_value_carry_normalisation(lib):
    """Unnormalised limbs (negative low limbs, carries) convert to the same double as the
    normalised representation of the same integer."""
    rng = random.Random(3)
    for _ in range(2000):
        x = rng.randint(-(2 ** 110), 2 ** 110)
        S = rng.randint(0, 150)
        a = rng.randint(-(2 ** 62), 2 ** 62)
        b = rng.randint(-(2 ** 21), 2 ** 21)
        # x = l0 + l1 2^40 + l2 2^80 with l0 = a (arbitrary), l1 chosen, l2 fitted
        l1 = b * 2 ** 20 + rng.randint(0, 2 ** 20)
        rest = x - a - (l1 << 40)
        l2, r = divmod(rest, 2 ** 80)
        l1 += r >> 40
        a += r & (2 ** 40 - 1)
        assert a + (l1 << 40) + (l2 << 80) == x
        if not (-(2 ** 63) <= a < 2 ** 63 and -(2 ** 63) <= l1 < 2 ** 63 and -(2 ** 63) <= l2 < 2 ** 63):
            continue
        h, m, lo = x >> 80, (x >> 40) & (2 ** 40 - 1), x & (2 ** 40 - 1)
        assert lib.value(a, l1, l2, S) == lib.value(lo, m, h, S)
        ref = float(Fraction(x) / Fraction(2) ** S)
        assert abs(lib.value(a, l1, l2, S) - ref) <= 2 * np.spacing(abs(ref)) + 2.0 ** -S


def test_shift(lib):
    assert lib.shift(0) == 1000
    assert lib.shift(1023) == 80 - 1  # weights < 2
    assert lib.shift(1022) == 80      # weights < 1
    assert lib.shift(2046) == -1000 or lib.shift(2046) == 80 - 1024
    assert lib.expf_(1.0) == 1023 and lib.expf_(0.75) == 1022 and lib.expf_(0.0) == 0
