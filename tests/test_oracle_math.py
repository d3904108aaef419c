"""CPU: the fp32 transcendental recipes.

  * the product copy (paper_2605_10433_b200/csrc/qsg_math.cuh, compiled for
    the host with the same strict-IEEE flags) and the oracle's independent
    copy (oracle/qsg_oracle_math.h) agree bit-for-bit on ~1e6 arguments;
  * accuracy against libm in long double (via ctypes) on the decoder's
    argument ranges;
  * the exact identities the kernels rely on (exp_neg(-0) == 1,
    log1p_01(1) == float(ln 2), so logaddexp(x, x) == x + ln2f without a
    special case).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
FUNCS = {"exp_neg": 0, "log1p_01": 1, "log1p": 2, "expm1": 3, "logaddexp": 4, "vnF": 6}


@pytest.fixture(scope="module")
def host_math(tmp_path_factory):
    out = tmp_path_factory.mktemp("hm") / "libmath_host.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
                    "-mfma", "-o", str(out), os.path.join(HERE, "cpp", "math_host.cpp")], check=True)
    lib = C.CDLL(str(out))
    lib.qsg_math_host_batch.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
    lib.qsg_bp4_host.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]

    def run(name, x, y=None):
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.ascontiguousarray(y if y is not None else x, dtype=np.float32)
        o = np.empty_like(x)
        if name == "bp4":
            lib.qsg_bp4_host(x.ctypes.data, x.size, o.ctypes.data)
        else:
            lib.qsg_math_host_batch(FUNCS[name], x.ctypes.data, y.ctypes.data, o.ctypes.data, x.size)
        return o
    return run


def _args(name, rng, n=200_000):
    if name == "exp_neg":
        return np.concatenate([-rng.uniform(0, 87, n), -rng.uniform(0, 1e-3, n // 4), [0.0, -0.0, -87.0]]), None
    if name == "log1p_01":
        return np.concatenate([rng.uniform(0, 1, n), 10.0 ** rng.uniform(-30, 0, n // 2), [0.0, 1.0]]), None
    if name == "log1p":
        return np.concatenate([10.0 ** rng.uniform(-30, 13, n), [0.0, 1.0, 0.999999]]), None
    if name == "expm1":
        return np.concatenate([rng.uniform(1e-12, 64, n), 10.0 ** rng.uniform(-12, 0, n // 2)]), None
    if name == "vnF":  # (y, l0): message sums over the decoder's range, priors of p in [1e-4, 0.7]
        p = 10.0 ** rng.uniform(-4, np.log10(0.7), n)
        l0 = np.log(3.0 * (1.0 - p) / p)
        y = np.concatenate([rng.uniform(-700, 700, n // 2), rng.standard_normal(n - n // 2) * 10.0 ** rng.integers(-6, 2, n - n // 2)])
        y[:4] = [0.0, -0.0, 87.5, -87.5]
        return y, l0
    x = rng.uniform(-70, 70, n)
    y = x + rng.standard_normal(n) * 10.0 ** rng.integers(-8, 3, n)
    y[:1000] = x[:1000]  # exact ties exercise the x == y branch
    return x, y


@pytest.mark.parametrize("name", list(FUNCS))
def test_product_and_oracle_recipes_bit_identical(oracle, host_math, name):
    rng = np.random.default_rng(FUNCS[name])
    x, y = _args(name, rng)
    a = oracle.math32(name, x, y)
    b = host_math(name, x, y)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def _libm_long_double():
    lib = C.CDLL("libm.so.6")
    for fn in ("expl", "log1pl", "expm1l"):
        getattr(lib, fn).restype = C.c_longdouble
        getattr(lib, fn).argtypes = [C.c_longdouble]
    return lib


def _ulp_err(got, ref):
    ref32 = np.float32(ref)
    ulp = np.spacing(np.abs(ref32)).astype(np.float64)
    return np.abs(got.astype(np.float64) - ref) / np.maximum(ulp, np.float64(np.finfo(np.float32).tiny))


@pytest.mark.parametrize("name,max_ulp", [("exp_neg", 2.0), ("log1p_01", 2.0), ("log1p", 2.5),
                                          ("expm1", 3.0), ("logaddexp", 2.0)])
def test_recipe_accuracy(oracle, name, max_ulp):
    L = _libm_long_double()
    rng = np.random.default_rng(99)
    x, y = _args(name, rng, 20_000)
    x32 = x.astype(np.float32)
    y32 = None if y is None else y.astype(np.float32)
    got = oracle.math32(name, x32, y32)
    xs = x32.astype(np.float64)
    if name == "exp_neg":
        ref = np.array([float(L.expl(v)) for v in xs])
    elif name in ("log1p_01", "log1p"):
        ref = np.array([float(L.log1pl(v)) for v in xs])
    elif name == "expm1":
        ref = np.array([float(L.expm1l(v)) for v in xs])
    else:
        ys = y32.astype(np.float64)
        mx = np.maximum(xs, ys)
        tail = np.array([float(L.log1pl(L.expl(-abs(a - b)))) for a, b in zip(xs, ys)])
        ref = mx + tail
        # the final max + tail addition cancels when the result is near 0
        # (in the reference's float64 formula too): measure in ulps of the
        # larger addend
        scale = np.spacing(np.maximum(np.abs(mx), tail).astype(np.float32)).astype(np.float64)
        assert (np.abs(got.astype(np.float64) - ref) / scale).max() <= max_ulp
        return
    err = _ulp_err(got, ref)
    mask = np.abs(ref) > 1e-30
    assert err[mask].max() <= max_ulp, (name, err[mask].max())


def test_vn_factor_accuracy(oracle):
    """F(y) = log((1 + e^-l0 e^-y) / (1 + e^-y)), the qubit-update factor
    (V[X] = b_Z + F(S_Z)): error <= 2.5e-7 + 1 ulp(F) against the literal
    two-logaddexp form evaluated in long double, over |y| <= 700 and priors
    of p in [1e-4, 0.7] (|F| <= |l0| <= 10.3)."""
    L = _libm_long_double()
    rng = np.random.default_rng(7)
    y, l0 = _args("vnF", rng, 20_000)
    y32, l032 = y.astype(np.float32), l0.astype(np.float32)
    got = oracle.math32("vnF", y32, l032).astype(np.float64)

    def lae0(z):  # logaddexp(0, z)
        return max(z, 0.0) + float(L.log1pl(L.expl(-abs(z))))
    ref = np.array([lae0(-(float(a) + float(b))) - lae0(-float(b)) for a, b in zip(l032, y32)])
    err = np.abs(got - ref) / (2.5e-7 + np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64))
    assert err.max() <= 1.0, (err.max(), y32[err.argmax()], l032[err.argmax()])


def test_exact_identities(oracle, host_math):
    assert oracle.math32("exp_neg", [0.0])[0] == 1.0 and oracle.math32("exp_neg", [-0.0])[0] == 1.0
    ln2f = np.float32(np.log(2.0))
    assert oracle.math32("log1p_01", [1.0])[0] == ln2f
    x = np.float32([3.25, -7.5, 0.0, 64.0])
    assert np.array_equal(host_math("logaddexp", x, x), x + ln2f)
    assert np.array_equal(oracle.math32("logaddexp", x, x), x + ln2f)


def _bp4_checks(rng, count):
    """Random check inputs x_k = min(|v_k|, 64): degrees 1-32, a mix of
    small (near-zero, the phi-sum's cancelling regime), moderate and large
    magnitudes, exact zeros and the 64 clip."""
    out = []
    for _ in range(count):
        d = int(rng.choice([1, 2, 3, 4, 6, 8, 10, 12, 16, 24, 32]))
        kind = rng.random(d)
        x = np.where(kind < 0.25, rng.exponential(0.05, d),
                     np.where(kind < 0.5, rng.uniform(0.0, 3.0, d), rng.uniform(0.0, 64.0, d)))
        x[rng.random(d) < 0.03] = 0.0
        x[rng.random(d) < 0.03] = 64.0
        out.append(x.astype(np.float32))
    return out


def test_bp4_product_and_oracle_recipes_bit_identical(oracle, host_math):
    """The BP4 check recipe (qsg_math.cuh bp4_mags) and the oracle's copy
    (qo_bp4_mags) agree bit for bit."""
    for x in _bp4_checks(np.random.default_rng(5), 20_000):
        a, b = oracle.bp4_mags(x), host_math("bp4", x)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), x


def test_bp4_check_accuracy(oracle):
    """Product-form BP4 magnitudes against the exact value of the
    reference's formula phi(clip(sum_k phi(x_k) - phi(x_e), 1e-12, 50))
    (decoder.py:318-323, phi = log1p(2/expm1), inputs floored at 1e-12),
    evaluated in 40-digit arithmetic: |err| <= 5e-7 max(|ref|, 1) (measured
    2.3e-7; the float64 formula itself is off by 5.5e-6 here).  Against
    the same formula in float64 -- the reference's own arithmetic, whose
    sum - phi_e cancels when one small input dominates -- the agreement is
    the north_star message tolerance, 1e-5 with the unit floor."""
    import math
    import mpmath as mp
    mp.mp.dps = 40

    def phi_mp(v):
        return mp.log1p(2 / mp.expm1(mp.mpf(max(float(v), 1e-12))))

    def phi_64(v):
        return math.log1p(2.0 / math.expm1(max(float(v), 1e-12)))
    worst = worst64 = 0.0
    for x in _bp4_checks(np.random.default_rng(6), 1500):
        got = oracle.bp4_mags(x).astype(np.float64)
        ph = [phi_mp(v) for v in x]
        tot = mp.fsum(ph)
        p64 = [phi_64(v) for v in x]
        t64 = sum(p64)
        for e in range(len(x)):
            ref = float(phi_mp(min(max(tot - ph[e], mp.mpf(1e-12)), 50)))
            worst = max(worst, abs(got[e] - ref) / max(abs(ref), 1.0))
            r64 = phi_64(min(max(t64 - p64[e], 1e-12), 50.0))
            worst64 = max(worst64, abs(got[e] - r64) / max(abs(r64), 1.0))
    assert worst <= 5e-7, worst
    assert worst64 <= 1e-5, worst64
