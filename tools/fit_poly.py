"""Fit the fp32 polynomial coefficients used by the shared math recipes.

Run: python tools/fit_poly.py  (prints the coefficient tables quoted in
paper_2605_10433_b200/csrc/qsg_math.cuh and oracle/qsg_oracle_math.h).

Each fit is a weighted least-squares fit on Chebyshev nodes for *relative*
error (close to minimax), done in mpmath at 50 digits, then rounded to the
nearest float32.  The fp32 accuracy of the full recipes (range reduction +
Horner + scaling) is measured by tests/test_oracle_math.py against libm in
long double, not here.
"""
import mpmath as mp
import numpy as np

mp.mp.dps = 50


def fit(fn, lo, hi, deg, fixed=()):
    """Coefficients c[len(fixed)..deg] of sum c_k x^k ~ fn(x), relative error.

    ``fixed`` pins the leading low-order coefficients (c0, c1, ...).
    """
    nodes = 400
    xs = [mp.mpf(lo) + (mp.mpf(hi) - mp.mpf(lo)) * (1 - mp.cos(mp.pi * (i + 0.5) / nodes)) / 2
          for i in range(nodes)]
    nf = len(fixed)
    A = mp.matrix(nodes, deg + 1 - nf)
    b = mp.matrix(nodes, 1)
    for r, x in enumerate(xs):
        y = fn(x)
        w = 1 / abs(y) if y != 0 else mp.mpf(1)
        rhs = y - sum(fixed[k] * x ** k for k in range(nf))
        for c in range(nf, deg + 1):
            A[r, c - nf] = x ** c * w
        b[r] = rhs * w
    sol = mp.lu_solve(A.T * A, A.T * b)
    coeffs = list(fixed) + [sol[i] for i in range(deg + 1 - nf)]
    f32 = [float(np.float32(float(c))) for c in coeffs]
    # relative error of the (exact-arithmetic) fp32-rounded polynomial
    err = 0
    for x in xs:
        y = fn(x)
        p = sum(mp.mpf(f32[k]) * x ** k for k in range(deg + 1))
        if y != 0:
            err = max(err, abs((p - y) / y))
    return f32, float(err)


def show(name, f32, err):
    print(f"{name}: max rel err (exact arith) = {err:.3e}")
    for k, c in enumerate(f32):
        print(f"   c{k} = {np.float32(c)!r:>16}  ({np.float32(c).view(np.uint32):#010x})")


if __name__ == "__main__":
    h = float(mp.log(2) / 2) + 1e-6
    # exp(r) on [-h, h], c0 = c1 = 1
    show("exp", *fit(mp.exp, -h, h, 6, fixed=(1, 1)))
    # expm1(r) = r + r^2 Q(r): fit Q on [-h, h]
    q = lambda r: (mp.expm1(r) - r) / (r * r) if r != 0 else mp.mpf(1) / 2
    show("expm1 Q", *fit(q, -h, h, 5))
    # log1p(t) = t * P(t) on [0, 1], P(0) = 1
    p = lambda t: mp.log1p(t) / t if t != 0 else mp.mpf(1)
    for deg in (9, 10, 11):
        show(f"log1p P deg{deg}", *fit(p, 0, 1, deg, fixed=(1,)))


def fit_phi():
    """Division-free phi(x) = log1p(2/expm1(x)) pieces (BP4, qsg_math phi):
      x >= ln2:  t = e^-x, phi = 2 atanh(t) = 2t + 2t u S(u), u = t^2 in [0, 1/4]
      x <  ln2:  phi = ln2 - log(x) + v H(v),  v = x^2 in [0, ln2^2]
                 (v H(v) = log((x/2) coth(x/2)), an even analytic function)"""
    S = lambda u: (mp.atanh(mp.sqrt(u)) / mp.sqrt(u) - 1) / u if u != 0 else mp.mpf(1) / 3
    Hf = lambda v: mp.log((mp.sqrt(v) / 2) * mp.coth(mp.sqrt(v) / 2)) / v if v != 0 else mp.mpf(1) / 12
    for deg in (5, 6, 7):
        show(f"phi S deg{deg}", *fit(S, 0, 0.25, deg))
    for deg in (2, 3, 4):
        show(f"phi H deg{deg}", *fit(Hf, 0, float(mp.log(2) ** 2), deg))


if __name__ == "__main__" and "phi" in __import__("sys").argv:
    fit_phi()
