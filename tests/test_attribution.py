"""CPU: every frame whose outcome differs between the fp32 restatement (which
the GPU matches bit-for-bit, tests/test_gpu_parity.py) and float64 reference
arithmetic is attributed to an exact/near tie broken by fp32 rounding
(oracle/attribution.py), on the frozen reference batches and on a larger
[[254,28]] sample at the chaotic p = 0.08 point."""
from __future__ import annotations

import os
from types import SimpleNamespace as NS

import numpy as np
import pytest

from conftest import GB126, GB254, SMALL

GAIN = NS(alpha_min=0.30, alpha_max=0.50, eta_unsat=1.10)
VARIANTS = {"bp4": {}, "ms": {}, "sms": {"alpha": 0.75}, "sagms": {"gain": GAIN}}
CODES = {"small": SMALL, "gb126": GB126, "gb254": GB254}
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def cfg(variant, l_max, vn_mode="marginal"):
    kw = VARIANTS[variant]
    return NS(variant=variant, l_max=l_max, vn_mode=vn_mode, alpha=kw.get("alpha"), gain=kw.get("gain"))


def _diff_frames(oracle, g, syn, l0, c):
    r32 = oracle.decode(g, syn, l0, c, precision=32)
    r64 = oracle.decode(g, syn, l0, c, precision=64)
    return np.nonzero((r32.success != r64.success) | (r32.iterations != r64.iterations)
                      | (r32.e_hat != r64.e_hat).any(axis=1))[0]


@pytest.mark.parametrize("cname", list(CODES))
@pytest.mark.parametrize("vn_mode", ["marginal", "additive"])
@pytest.mark.parametrize("variant", list(VARIANTS))
def test_golden_batches_attributed(oracle, cname, vn_mode, variant):
    from oracle.attribution import attribute
    b = np.load(os.path.join(GOLD, "golden_batches.npz"))
    g = oracle.Graph(oracle.gb_graph(*CODES[cname]))
    syn = b[f"{cname}/syndromes"]
    eps, lmax = b[f"{cname}/meta"]
    c = cfg(variant, int(lmax), vn_mode)
    l0 = oracle.prior_llr(float(eps))
    for f in _diff_frames(oracle, g, syn, l0, c)[:12]:
        a = attribute(g, syn[f], l0, c, frame=int(f))
        assert a.attributed, a


def test_chaotic_point_sample_attributed(oracle):
    from oracle.attribution import attribute
    g = oracle.Graph(oracle.gb_graph(*GB254))
    e = oracle.sample_errors(254, 0.08, 0, 0, 1024)
    syn = oracle.syndromes_of(g, e)
    l0 = oracle.prior_llr(0.08)
    kinds = {}
    for variant in ("sagms", "sms", "bp4"):
        c = cfg(variant, 100)
        for f in _diff_frames(oracle, g, syn, l0, c)[:10]:
            a = attribute(g, syn[f], l0, c, frame=int(f))
            kinds[a.kind] = kinds.get(a.kind, 0) + 1
            assert a.attributed, a
