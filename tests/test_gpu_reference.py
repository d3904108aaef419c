"""GPU against the REFERENCE's own frozen outputs (tests/golden/, produced by
tests/golden/make_golden.py from /root/reference in the build container):

  * fp32 GPU messages within 1e-5 (relative, unit floor) of the reference's
    float64 snapshots on the first update(s);
  * GPU outcomes on the frozen batches equal the reference's except frames
    attributed to ties broken by fp32 rounding (checked on CPU by
    tests/test_attribution.py against the bit-identical fp32 restatement);
  * the FER protocol on the device (run_point / run_sweep) reproduces the
    reference's FerPoints and byte-identical results.json / fer.tsv.
"""
from __future__ import annotations

import json
import os
from dataclasses import asdict
from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import GB126, GB254, SMALL, TOY

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
CODES = {"small": SMALL, "gb126": GB126, "gb254": GB254}
VARIANTS = {"bp4": {}, "ms": {}, "sms": {"alpha": 0.75}, "sagms": {"gain": (0.30, 0.50, 1.10)}}


@pytest.fixture(scope="module")
def P():
    import paper_2605_10433_b200 as P
    assert torch.cuda.is_available()
    return P


def _cfg(P, variant, l_max, vn_mode="marginal"):
    kw = dict(VARIANTS[variant])
    if "gain" in kw:
        kw["gain"] = P.GainParams(*kw["gain"])
    return P.DecoderConfig(variant, l_max=l_max, vn_mode=vn_mode, **kw)


@pytest.mark.parametrize("cname", ["gb126", "gb254"])
@pytest.mark.parametrize("vn_mode", ["marginal", "additive"])
@pytest.mark.parametrize("variant", list(VARIANTS))
def test_gpu_messages_vs_reference_fp64(P, cname, vn_mode, variant):
    tr = np.load(GOLD / "golden_traces.npz")
    g = P.gb_graph(P.GbSpec(*CODES[cname]))
    syn = tr[f"{cname}/syndromes"]
    cfg = _cfg(P, variant, 3, vn_mode)
    nit = 2
    for f in range(3):
        r = P.decode(None, g, syn[f], P.prior_llr(0.06), cfg, capture_messages=True, early_stop=False)
        for k in range(nit):
            for side, got in (("vn", r.message_trace[k].vn_to_cn), ("cn", r.message_trace[k].cn_to_vn)):
                ref = tr[f"{cname}/{variant}/{vn_mode}/{side}"][f, k]
                err = np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)
                assert err.max() <= 1e-5, (f, k, side, float(err.max()))


@pytest.mark.parametrize("cname", list(CODES))
@pytest.mark.parametrize("vn_mode", ["marginal", "additive"])
@pytest.mark.parametrize("variant", list(VARIANTS))
def test_gpu_outcomes_vs_reference_batches(P, oracle, cname, vn_mode, variant):
    b = np.load(GOLD / "golden_batches.npz")
    g = P.gb_graph(P.GbSpec(*CODES[cname]))
    syn = b[f"{cname}/syndromes"]
    eps, lmax = b[f"{cname}/meta"]
    key = f"{cname}/{variant}/{vn_mode}"
    cfg = _cfg(P, variant, int(lmax), vn_mode)
    got = P.decode_batch(g, syn, P.prior_llr(float(eps)), cfg, collect_gamma=True)
    same = (got.success == b[key + "/success"]) & (got.iterations == b[key + "/iterations"]) \
        & (got.e_hat == b[key + "/e_hat"]).all(axis=1)
    # frames that differ from the float64 reference are exactly the frames
    # where the fp32 restatement differs from float64 arithmetic (each one
    # attributed on CPU); everywhere else the GPU reproduces the reference
    r32 = oracle.decode(g, syn, P.prior_llr(float(eps)).llr, cfg, precision=32, trace=True)
    assert np.array_equal(got.success, r32.success) and np.array_equal(got.iterations, r32.iterations)
    for a, c in zip(got.gamma_traces, r32.gamma_traces(g.m)):
        assert np.array_equal(a, c)
    r64 = oracle.decode(g, syn, P.prior_llr(float(eps)).llr, cfg, precision=64, trace=True)
    diff64 = (r32.success != r64.success) | (r32.iterations != r64.iterations) | (r32.e_hat != r64.e_hat).any(axis=1)
    if variant == "bp4":
        # numpy's BP4 uses SIMD expm1/log1p, so the fp64 restatement matches
        # the reference's outcomes on all but <= 2% of frames (iterations
        # only, tests/test_oracle_pins.py).  The frames where the GPU differs
        # from the reference are exactly the fp32-vs-fp64 frames (each one
        # attributed on CPU) except those where the fp64 restatement itself
        # differs from the reference's libm -- a complete partition:
        ref64 = (r64.success != b[key + "/success"]) | (r64.iterations != b[key + "/iterations"]) \
            | (r64.e_hat != b[key + "/e_hat"]).any(axis=1)
        assert not (~same & ~diff64).any()
        assert not (same & diff64 & ~ref64).any()
        assert ref64.mean() <= 0.02 and not (r64.success != b[key + "/success"]).any()
    else:
        assert np.array_equal(~same, diff64)
        # where fp32 and fp64 trajectories coincide, the GPU's gamma traces
        # are the reference's
        lens = b[key + "/gamma_len"]
        gam = np.split(b[key + "/gamma"], np.cumsum(lens)[:-1])
        for f, (t32, t64) in enumerate(zip(r32.gamma_traces(g.m), r64.gamma_traces(g.m))):
            if np.array_equal(t32, t64):
                assert np.array_equal(got.gamma_traces[f], gam[f])


def test_config1_on_gpu_matches_reference_golden(P):
    gold = json.loads((GOLD / "golden_config1.json").read_text())
    g = P.gb_graph(P.GbSpec(*GB254))
    cfg = _cfg(P, "sagms", 100)
    fails, iters = P.decode_frames(g, cfg, 0.05, 0.05, 0, 0, 10_000)
    assert np.nonzero(fails)[0].tolist() == gold["fail_frames"]
    assert int(iters.sum()) == gold["sum_iterations"]
    assert int((iters == 100).sum()) == gold["frames_at_lmax"]


def _sweep(P, code_id, variant, eps, seed, **kw):
    dkw = {"alpha": 0.5} if variant == "sms" else ({"gain": P.GainParams(0.3, 0.5, 1.1)} if variant == "sagms" else {})
    base = dict(code_id=code_id, decoder=P.DecoderConfig(variant, l_max=kw.pop("l_max", 4), **dkw),
                epsilon_list=tuple(eps), seed=seed, target_failures=50, max_frames=100_000)
    base.update(kw)
    return P.SweepConfig(**base)


def test_run_point_on_gpu_matches_reference(P):
    gold = json.loads((GOLD / "golden_harness.json").read_text())
    toy, small = P.gb_graph(P.GbSpec(*TOY)), P.gb_graph(P.GbSpec(*SMALL))
    cases = {
        "toy_ms_lmax1_eps05": (toy, _sweep(P, "toy", "ms", (0.5,), 2718, l_max=1), 0.5),
        "small_sagms_eps025": (small, _sweep(P, "gb-10-2", "sagms", (0.25,), 31, l_max=4, target_failures=40), 0.25),
        "small_ms_cap": (small, _sweep(P, "gb-10-2", "ms", (0.001,), 5, l_max=8, target_failures=500,
                                       max_frames=64), 0.001),
    }
    for name, (g, cfg, eps) in cases.items():
        assert asdict(P.run_point(g, cfg, eps)) == gold[name]["point"], name


def test_run_sweep_on_gpu_byte_identical(P, tmp_path):
    gold = json.loads((GOLD / "golden_harness.json").read_text())["sweep_sms"]
    small = P.gb_graph(P.GbSpec(*SMALL))
    cfg = _sweep(P, "gb-10-2", "sms", (0.3, 0.2, 0.25), 13, l_max=4, target_failures=20)
    P.run_sweep(small, cfg, out_dir=tmp_path)
    assert (tmp_path / "results.json").read_text() == gold["results_json"]
    assert (tmp_path / "fer.tsv").read_text() == gold["fer_tsv"]
    assert sorted(os.listdir(tmp_path / "points")) == gold["points"]


def test_decode_trace_sink_records(P):
    """Reference test_decoder.py:477-497 on the device trace mode."""
    g = P.gb_graph(P.GbSpec(*SMALL))
    e = np.zeros(g.n, np.uint8)
    e[1] = 1
    s = g.syndromes_of(e)[0]
    recs = []
    P.decode(None, g, s, P.prior_llr(0.1), _cfg(P, "sagms", 6), trace_sink=recs.append)
    assert recs
    for rec in recs:
        assert set(rec) == {"iteration", "gamma", "alpha_eff", "magnitude_hist"}
        assert 0.0 <= rec["gamma"] <= 1.0
        assert rec["alpha_eff"]["min"] <= rec["alpha_eff"]["max"] <= 1.0
        assert sum(rec["magnitude_hist"]["counts"]) == g.edge_count


def test_weight1_outcomes(P):
    """Reference test_decoder.py:230-260: the twinned [[6,2]] code fails all
    18 weight-1 syndromes (bp4, both VN modes); the twin-free [[10,2]] code
    decodes all of them for every variant."""
    toy, small = P.gb_graph(P.GbSpec(*TOY)), P.gb_graph(P.GbSpec(*SMALL))
    prior = P.prior_llr(0.05)

    def weight1(g):
        e = np.zeros((3 * g.n, g.n), np.uint8)
        for j in range(g.n):
            for p in (1, 2, 3):
                e[3 * j + p - 1, j] = p
        return g.syndromes_of(e)
    for vn in ("marginal", "additive"):
        r = P.decode_batch(toy, weight1(toy), prior, P.DecoderConfig("bp4", l_max=8, vn_mode=vn))
        assert not r.success.any()
    syn = weight1(small)
    for variant in VARIANTS:
        r = P.decode_batch(small, syn, prior, _cfg(P, variant, 8))
        assert r.success.all(), variant
        assert not (small.syndromes_of(r.e_hat) ^ syn).any()


def test_degenerate_equivalences_bit_identical(P):
    """Reference test_decoder.py:293-334 / acceptance criterion 4:
    sagms(.5,.5,1) == sms(.5) and sms(1) == ms, outcomes and messages."""
    g = P.gb_graph(P.GbSpec(*GB126))
    e = P.sample_errors(P.DepolarizingChannel(0.08, 314), g.n, 0, 1000)
    syn = g.syndromes_of(e)
    prior = P.prior_llr(0.08)
    pairs = [(P.DecoderConfig("sagms", l_max=8, gain=P.GainParams(0.5, 0.5, 1.0)), P.DecoderConfig("sms", l_max=8, alpha=0.5)),
             (P.DecoderConfig("sms", l_max=8, alpha=1.0), P.DecoderConfig("ms", l_max=8))]
    for a, b in pairs:
        ra, rb = P.decode_batch(g, syn, prior, a), P.decode_batch(g, syn, prior, b)
        assert np.array_equal(ra.success, rb.success) and np.array_equal(ra.e_hat, rb.e_hat)
        assert np.array_equal(ra.iterations, rb.iterations)
        ta = P.decode(None, g, syn[0], prior, a, capture_messages=True, early_stop=False)
        tb = P.decode(None, g, syn[0], prior, b, capture_messages=True, early_stop=False)
        for sa, sb in zip(ta.message_trace, tb.message_trace):
            assert np.array_equal(sa.vn_to_cn, sb.vn_to_cn) and np.array_equal(sa.cn_to_vn, sb.cn_to_vn)


def test_sharded_point_on_device_matches_reference(P):
    """dist.run_point_sharded with the device FER unit (world size 1 here;
    the multi-rank exchange is covered on CPU by tests/test_dist.py) and
    dist.fer_counters give the reference's FerPoint / counts."""
    from paper_2605_10433_b200 import dist as D
    gold = json.loads((GOLD / "golden_harness.json").read_text())
    small = P.gb_graph(P.GbSpec(*SMALL))
    g = P.GainParams(0.3, 0.5, 1.1)
    sweep = P.SweepConfig(code_id="gb-10-2", decoder=P.DecoderConfig("sagms", l_max=4, gain=g),
                          epsilon_list=(0.25,), seed=31, target_failures=40, max_frames=100_000)
    for chunk in (5, 1 << 20):
        pt = D.run_point_sharded(small, sweep, 0.25, chunk=chunk)
        assert asdict(pt) == gold["small_sagms_eps025"]["point"]
    cfg = P.DecoderConfig("sagms", l_max=8, gain=g)
    cnt = D.fer_counters(small, cfg, 0.2, 0.2, 7, 3, 1001)
    fails, iters = P.decode_frames(small, cfg, 0.2, 0.2, 7, 3, 1001)
    assert cnt.cpu().tolist() == [1001, int(fails.sum()), int(iters.sum()), small.edge_count * (int(iters.sum()) - 1001)]
