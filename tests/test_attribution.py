"""CPU: every frame whose outcome differs between the fp32 restatement (which
the GPU matches bit-for-bit, tests/test_gpu_parity.py) and float64 reference
arithmetic is attributed to an exact/near tie broken by fp32 rounding or to
gradual rounding growth (oracle/attribution.py):

  * ALL differing frames of the frozen reference batches (889 frames over
    3 codes x 4 decoders x 2 VN modes);
  * a frozen random sample of the outcome flips at the chaotic configs[1]
    point p = 0.08 (tests/golden/flips_p008.json, tools/attribution_sample.py):
    200 per SMS alpha and BP4, every SAGMS flip in 2^17 frames.  Each frame is
    re-derived as a flip here before it is attributed.
"""
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
    for f in _diff_frames(oracle, g, syn, l0, c):
        a = attribute(g, syn[f], l0, c, frame=int(f))
        assert a.attributed, a


FLIPS = os.path.join(GOLD, "flips_p008.json")


def _dec(name):
    alpha = float(name[3:]) if name.startswith("sms") else None
    variant = "sms" if name.startswith("sms") else name
    return NS(variant=variant, l_max=100, vn_mode="marginal", alpha=alpha, gain=GAIN if name == "sagms" else None)


@pytest.mark.parametrize("name", ["bp4", "sms0.5", "sms0.75", "sms1.0", "sagms"])
def test_chaotic_point_flip_sample_attributed(oracle, name):
    import json
    from oracle.attribution import attribute
    d = json.load(open(FLIPS))
    rec = d["decoders"][name]
    frames = rec["sample"]
    assert len(frames) == min(200, rec["flips"]) and rec["flips"] > 0
    g = oracle.Graph(oracle.gb_graph(*d["code"]))
    l0 = oracle.prior_llr(0.08)
    c = _dec(name)
    kinds = {}
    for f in frames:
        e = oracle.sample_errors(254, 0.08, 0, f, 1)
        syn = oracle.syndromes_of(g, e)
        r32 = oracle.decode(g, syn, l0, c, precision=32)
        r64 = oracle.decode(g, syn, l0, c, precision=64)
        assert r32.success[0] != r64.success[0] or r32.iterations[0] != r64.iterations[0], f
        a = attribute(g, syn[0], l0, c, frame=f)
        assert a.attributed, a
        kinds[a.kind] = kinds.get(a.kind, 0) + 1
    # no bucket is a catch-all: rounding-growth frames all passed the
    # gradual-amplification bound (attribute(max_growth=100))
    assert sum(kinds.values()) == len(frames)
