"""CPU: host-side logic that wraps the GPU path -- config validation
(decoder.py:62-112), the FER protocol (harness.py:102-356: Wilson interval,
canonical JSON, digest, ordered stop rule, persistence), code utilities.
The protocol tests swap the GPU FER unit for the CPU oracle (the checker)
so they run without a GPU; the -m gpu tests run the same protocol on the
device."""
from __future__ import annotations

import json
import math
import os
from pathlib import Path

import numpy as np
import pytest

import paper_2605_10433_b200 as P
from paper_2605_10433_b200 import harness as H
from conftest import GB126, GB254, SMALL, TOY

GOLD = Path(__file__).resolve().parent / "golden"


def test_gain_and_config_validation():
    P.GainParams(0.3, 0.5, 1.1)
    P.GainParams(0.5, 0.5, 1.0)
    for bad in [(0.6, 0.5, 1.1), (0.3, 0.5, 0.9), (0.3, 0.95, 1.10)]:
        with pytest.raises(ValueError):
            P.GainParams(*bad)
    for kw in [dict(variant="nms"), dict(variant="bp4", l_max=0), dict(variant="sms"),
               dict(variant="sms", alpha=1.5), dict(variant="sagms"), dict(variant="bp4", vn_mode="joint")]:
        with pytest.raises(ValueError):
            P.DecoderConfig(**kw)


def test_effective_gain_and_ratio():
    g = P.GainParams(0.30, 0.50, 1.10)
    assert P.effective_gain(0.0, 0, g) == pytest.approx(0.50)
    assert P.effective_gain(1.0, 0, g) == pytest.approx(0.30)
    assert P.effective_gain(0.5, 1, g) == pytest.approx(0.44)
    assert P.effective_gain(0.0, 1, g) == pytest.approx(0.55)
    with pytest.raises(ValueError):
        P.effective_gain(1.5, 0, g)
    r = np.zeros(126, np.uint8)
    r[:63] = 1
    assert P.syndrome_ratio(r) == 0.5


def test_wilson_interval():
    def textbook(f, n, z=1.959964):
        ph = f / n
        a, b, c = 1 + z * z / n, -(2 * ph + z * z / n), ph * ph
        lo, hi = sorted(np.roots([a, b, c]).real)
        return max(0.0, lo), min(1.0, hi)
    for f, n in [(500, 10**6), (1, 2), (0, 100), (100, 100), (7, 31)]:
        got, want = P.wilson_interval(f, n), textbook(f, n)
        assert got[0] == pytest.approx(want[0], abs=1e-9) and got[1] == pytest.approx(want[1], abs=1e-9)
    lo, hi = P.wilson_interval(500, 1_000_000)
    assert (hi - lo) / 2 / 5e-4 <= 0.09
    with pytest.raises(ValueError):
        P.wilson_interval(5, 4)


def _sweep(code_id="toy", variant="ms", eps=(0.5,), seed=99, **kw):
    dkw = {"alpha": 0.5} if variant == "sms" else ({"gain": P.GainParams(0.3, 0.5, 1.1)} if variant == "sagms" else {})
    base = dict(code_id=code_id, decoder=P.DecoderConfig(variant, l_max=kw.pop("l_max", 4), **dkw),
                epsilon_list=tuple(eps), seed=seed, target_failures=50, max_frames=100_000)
    base.update(kw)
    return P.SweepConfig(**base)


def test_canonical_json_and_digest():
    text = H.canonical_json({"b": 0.1, "a": [1, 2.5, None, True], "c": {"y": "s", "x": 2}})
    assert text == H.canonical_json(json.loads(text)) and "0.10000000000000001" in text
    assert P.config_digest(_sweep(workers=1)) == P.config_digest(_sweep(workers=8))
    assert P.config_digest(_sweep(seed=100)) != P.config_digest(_sweep())


def test_digest_equals_reference(reference):
    """Same SweepConfig -> same SHA-256 digest as the reference, so persisted
    point files are interchangeable (harness.py:156-158)."""
    from qsagms.decoder import DecoderConfig, GainParams
    from qsagms.harness import SweepConfig, config_digest
    ours = _sweep("gb-10-2", "sagms", (0.25, 0.2), 777, l_max=8, target_failures=120)
    ref = SweepConfig(code_id="gb-10-2", decoder=DecoderConfig("sagms", l_max=8, gain=GainParams(0.3, 0.5, 1.1)),
                      epsilon_list=(0.25, 0.2), seed=777, target_failures=120, max_frames=100_000)
    assert P.config_digest(ours) == config_digest(ref)


@pytest.fixture
def cpu_fer_unit(monkeypatch, oracle):
    """Run the FER protocol on the oracle (harness.FRAME_UNIT hook; protocol
    test on CPU)."""
    def unit(graph, cfg, eps, eps0, seed, start, count):
        f, it, _, _ = oracle.frames(oracle.Graph(graph), cfg, eps, eps0, seed, start, count, precision=64)
        return f, it
    monkeypatch.setattr(H, "FRAME_UNIT", unit)


@pytest.mark.parametrize("batch", [1 << 20, 7, 4096])
def test_run_point_matches_reference_golden(cpu_fer_unit, batch):
    gold = json.loads((GOLD / "golden_harness.json").read_text())
    toy, small = P.gb_graph(P.GbSpec(*TOY)), P.gb_graph(P.GbSpec(*SMALL))
    cases = {
        "toy_ms_lmax1_eps05": (toy, _sweep("toy", "ms", (0.5,), 2718, l_max=1), 0.5),
        "small_sagms_eps025": (small, _sweep("gb-10-2", "sagms", (0.25,), 31, l_max=4, target_failures=40), 0.25),
        "small_ms_cap": (small, _sweep("gb-10-2", "ms", (0.001,), 5, l_max=8, target_failures=500, max_frames=64), 0.001),
    }
    for name, (g, cfg, eps) in cases.items():
        p = H.run_point(g, cfg, eps, batch_frames=batch)
        want = gold[name]["point"]
        from dataclasses import asdict
        assert asdict(p) == want, name
    assert gold["toy_ms_lmax1_eps05"]["point"]["frames"] == 56  # reference test_harness.py:131-141


def test_run_sweep_byte_identical_to_reference(cpu_fer_unit, tmp_path):
    gold = json.loads((GOLD / "golden_harness.json").read_text())["sweep_sms"]
    small = P.gb_graph(P.GbSpec(*SMALL))
    cfg = _sweep("gb-10-2", "sms", (0.3, 0.2, 0.25), 13, l_max=4, target_failures=20)
    P.run_sweep(small, cfg, out_dir=tmp_path)
    assert (tmp_path / "results.json").read_text() == gold["results_json"]
    assert (tmp_path / "fer.tsv").read_text() == gold["fer_tsv"]
    assert sorted(os.listdir(tmp_path / "points")) == gold["points"]
    # resume: delete one point, rerun recomputes it identically
    pf = sorted((tmp_path / "points").glob("*.json"))
    keep = pf[1].read_bytes()
    pf[0].unlink()
    P.run_sweep(small, cfg, out_dir=tmp_path)
    assert pf[1].read_bytes() == keep and (tmp_path / "results.json").read_text() == gold["results_json"]


def test_code_dimensions():
    assert P.gb_dimension(P.GbSpec(*GB126)) == 28
    assert P.gb_dimension(P.GbSpec(*GB254)) == 28
    g = P.gb_graph(P.GbSpec(*GB126))
    assert P.code_dimension(g) == 28 and P.check_commute(g)
    assert P.code_dimension(P.gb_graph(P.GbSpec(*SMALL))) == 2


def test_random_gb_spec():
    for ell, w in [(63, 5), (127, 3), (127, 8), (255, 5)]:
        s = P.random_gb_spec(ell, w, seed=0)
        assert s == P.random_gb_spec(ell, w, seed=0)
        assert len(s.a_exponents) == w and s.a_exponents[0] == 0 and s.b_exponents[0] == 0
        assert P.gb_dimension(s) > 0
        assert P.gb_graph(s).kind in (0, w)


# random_gb_spec(ell, w, seed=0) for every BASELINE config-3/4/5 code: the
# generator is the builder's definition (the reference ships none), so its
# exact output is pinned here -- any change to the draw rule shows up.
PINNED_RANDOM_GB = {
    (63, 5): ((0, 17, 32, 39, 51), (0, 1, 11, 41, 50)),
    (127, 5): ((0, 10, 34, 56, 88), (0, 3, 90, 108, 117)),
    (255, 5): ((0, 20, 72, 105, 187), (0, 30, 34, 47, 234)),
    (511, 5): ((0, 5, 200, 397, 418), (0, 81, 284, 347, 418)),
    (127, 3): ((0, 9, 74), (0, 13, 80)),
    (127, 4): ((0, 65, 80, 106), (0, 3, 6, 10)),
    (127, 6): ((0, 34, 39, 64, 79, 104), (0, 63, 77, 80, 100, 114)),
    (127, 8): ((0, 6, 10, 34, 39, 63, 78, 103), (0, 68, 70, 73, 78, 89, 118, 126)),
}


def test_random_gb_spec_pinned_codes():
    for (ell, w), (a, b) in PINNED_RANDOM_GB.items():
        s = P.random_gb_spec(ell, w, seed=0)
        assert (s.ell, s.a_exponents, s.b_exponents) == (ell, a, b), (ell, w)
        k = P.gb_dimension(s)
        assert k > 0 and k == P.code_dimension(P.gb_graph(s))
        assert P.check_commute(P.gb_graph(s))


def test_load_qpc_validates_commutation(tmp_path):
    """load_code(validate=True) raises OrthogonalityError for rows that do
    not commute (code.py:375-377, :96-97); validate=False loads them."""
    (tmp_path / "anti.qpc").write_text("QPC 1\nn=2 m=2\n0: 0:X 1:X\n1: 0:Z\n")
    with pytest.raises(P.OrthogonalityError):
        P.load_qpc(tmp_path / "anti.qpc")
    g = P.load_qpc(tmp_path / "anti.qpc", validate=False)
    assert g.m == 2 and not P.check_commute(g)
    # X X / Z Z commute (two anticommuting positions)
    (tmp_path / "ok.qpc").write_text("QPC 1\nn=2 m=2\n0: 0:X 1:X\n1: 0:Z 1:Z\n")
    assert P.check_commute(P.load_qpc(tmp_path / "ok.qpc"))
    assert issubclass(P.OrthogonalityError, ValueError) and P.load_code is P.load_qpc


def test_load_qpc_validation_matches_reference(reference, tmp_path):
    from qsagms.code import OrthogonalityError, load_code
    rng = np.random.default_rng(11)
    seen = set()
    for t in range(40):
        n, m = 6, 4
        while True:  # every qubit covered (the layout compiler rejects isolated qubits)
            picks = [sorted(rng.choice(n, size=rng.integers(2, 5), replace=False).tolist()) for _ in range(m)]
            if len(set(sum(picks, []))) == n:
                break
        rows = [" ".join(f"{j}:{'XZY'[rng.integers(0, 3)]}" for j in cols) for cols in picks]
        text = "QPC 1\nn=6 m=4\n" + "".join(f"{i}: {r}\n" for i, r in enumerate(rows))
        (tmp_path / f"r{t}.qpc").write_text(text)
        try:
            load_code(tmp_path / f"r{t}.qpc")
            ref_ok = True
        except OrthogonalityError:
            ref_ok = False
        try:
            P.load_qpc(tmp_path / f"r{t}.qpc")
            ours = True
        except P.OrthogonalityError:
            ours = False
        assert ours == ref_ok, text
        seen.add(ours)
    assert seen == {True, False}


def test_qpc_roundtrip(tmp_path):
    g = P.gb_graph(P.GbSpec(*GB126))
    P.save_qpc(g, tmp_path / "c.qpc")
    h = P.load_qpc(tmp_path / "c.qpc")
    assert np.array_equal(h.edge_vn, g.edge_vn) and h.gb == P.GbSpec(*GB126)
    (tmp_path / "bad.qpc").write_text("QPC 1\nn=3 m=1\n0: 0:X 0:Z\n")
    with pytest.raises(P.CodeFormatError) as e:
        P.load_qpc(tmp_path / "bad.qpc")
    assert e.value.line == 3


def test_marginal_init_formula():
    from paper_2605_10433_b200.decoder import marginal_init
    l0 = P.prior_llr(0.1).llr
    assert marginal_init(l0) == pytest.approx(math.log((0.9 + 0.1 / 3) / (2 * 0.1 / 3)), abs=1e-12)


def test_install_routes_reference_harness(reference, monkeypatch, oracle):
    """install(qsagms.harness) swaps the reference's FER unit
    (harness.py:207-213 resolves _decode_frames by global name): the
    reference's own run_point then calls ours.  Here ours is backed by the
    CPU oracle (no GPU in this container); the result equals the
    reference's own run_point."""
    import qsagms.harness as RH
    from qsagms.code import GbSpec, build_gb, tanner_graph
    from qsagms.decoder import DecoderConfig

    Hm = build_gb(GbSpec(3, (0, 1), (0, 2)))
    g = tanner_graph(Hm)
    cfg = RH.SweepConfig(code_id="toy", decoder=DecoderConfig("ms", l_max=1), epsilon_list=(0.5,), seed=2718,
                         target_failures=50, max_frames=100_000)
    want = RH.run_point(Hm, g, cfg, 0.5)
    calls = []

    def unit(graph, dcfg, eps, eps0, seed, start, count):
        calls.append(count)
        f, it, _, _ = oracle.frames(oracle.Graph(graph), dcfg, eps, eps0, seed, start, count, precision=64)
        return f, it
    monkeypatch.setattr(H, "decode_frames", unit)
    monkeypatch.setattr(RH, "BATCH_FRAMES", RH.BATCH_FRAMES)  # restored after the test
    original = RH._decode_frames
    try:
        P.install(RH)
        assert RH._decode_frames is H.decode_frames is unit and RH.BATCH_FRAMES == 1 << 20
        got = RH.run_point(Hm, g, cfg, 0.5)
        P.install(RH, batch_frames=7)  # any batching gives the same point (harness.py:40)
        got7 = RH.run_point(Hm, g, cfg, 0.5)
    finally:
        RH._decode_frames = original
    assert calls and got == want == got7 and (got.frames, got.failures) == (56, 50)
