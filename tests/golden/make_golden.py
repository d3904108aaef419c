"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
(/root/reference/pkg/src/qsagms, imported in place) in this container.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are frozen here:
  golden_config1.json   BASELINE config 1 outcome summary
  golden_batches.npz    syndromes + reference outcomes (success, iterations,
                        e_hat, gamma) for several codes x variants x VN modes
  golden_traces.npz     reference float64 message snapshots (first 3
                        iterations) for the 1e-5 message check on the GPU
  golden_harness.json   run_point / run_sweep outputs (points, results.json
                        and fer.tsv bytes) for the protocol drop-in tests
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from qsagms.channel import DepolarizingChannel, prior_llr, sample_error  # noqa: E402
from qsagms.code import GbSpec, build_gb, tanner_graph  # noqa: E402
from qsagms.decoder import DecoderConfig, GainParams, _kernel_for, decode, decode_batch  # noqa: E402
from qsagms.harness import SweepConfig, run_point, run_sweep  # noqa: E402

HERE = Path(__file__).resolve().parent
GAIN = GainParams(0.30, 0.50, 1.10)
CODES = {
    "small": (5, (0, 1), (0, 2)),
    "gb126": (63, (0, 1, 14, 16, 22), (0, 3, 13, 20, 42)),
    "gb254": (127, (0, 15, 20, 28, 66), (0, 58, 59, 100, 121)),
}
VARIANTS = [("bp4", {}), ("ms", {}), ("sms", {"alpha": 0.75}), ("sagms", {"gain": GAIN})]


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def errors(H, eps, seed, start, count):
    ch = DepolarizingChannel(eps, seed)
    return np.stack([sample_error(ch, H.n, stream_id=f) for f in range(start, start + count)])


def config1():
    H = build_gb(GbSpec(*CODES["gb254"]))
    g = tanner_graph(H)
    e = errors(H, 0.05, 0, 0, 10_000)
    syn = _kernel_for(g).syndromes_of(e)
    cfg = DecoderConfig("sagms", l_max=100, gain=GAIN)
    r = decode_batch(g, syn, prior_llr(0.05), cfg)
    out = {
        "errors_sha16": digest(e), "syndromes_sha16": digest(syn), "ehat_sha16": digest(r.e_hat),
        "fail_frames": np.nonzero(~r.success)[0].tolist(), "sum_iterations": int(r.iterations.sum()),
        "iteration_hist_0_15": np.bincount(r.iterations, minlength=101)[:16].tolist(),
        "frames_at_lmax": int((r.iterations == 100).sum()),
    }
    (HERE / "golden_config1.json").write_text(json.dumps(out, indent=1) + "\n")


def batches():
    arrays = {}
    for cname, spec, eps, B, lmax in [("small", CODES["small"], 0.12, 200, 12),
                                      ("gb126", CODES["gb126"], 0.06, 200, 20),
                                      ("gb254", CODES["gb254"], 0.08, 120, 30)]:
        H = build_gb(GbSpec(*spec))
        g = tanner_graph(H)
        e = errors(H, eps, 21, 0, B)
        syn = _kernel_for(g).syndromes_of(e)
        arrays[f"{cname}/syndromes"] = syn
        arrays[f"{cname}/meta"] = np.array([eps, lmax])
        for vn in ("marginal", "additive"):
            for v, kw in VARIANTS:
                cfg = DecoderConfig(v, l_max=lmax, vn_mode=vn, **kw)
                r = decode_batch(g, syn, prior_llr(eps), cfg, collect_gamma=True)
                key = f"{cname}/{v}/{vn}"
                arrays[key + "/success"] = r.success
                arrays[key + "/iterations"] = r.iterations
                arrays[key + "/e_hat"] = r.e_hat
                arrays[key + "/gamma_len"] = np.array([len(t) for t in r.gamma_traces])
                arrays[key + "/gamma"] = np.concatenate(r.gamma_traces)
    np.savez_compressed(HERE / "golden_batches.npz", **arrays)


def traces():
    arrays = {}
    for cname in ("gb126", "gb254"):
        H = build_gb(GbSpec(*CODES[cname]))
        g = tanner_graph(H)
        e = errors(H, 0.06, 5, 0, 3)
        syn = _kernel_for(g).syndromes_of(e)
        arrays[f"{cname}/syndromes"] = syn
        for vn in ("marginal", "additive"):
            for v, kw in VARIANTS:
                cfg = DecoderConfig(v, l_max=3, vn_mode=vn, **kw)
                vs, cs = [], []
                for f in range(3):
                    r = decode(H, g, syn[f], prior_llr(0.06), cfg, capture_messages=True, early_stop=False)
                    vs.append(np.stack([s.vn_to_cn for s in r.message_trace]))
                    cs.append(np.stack([s.cn_to_vn for s in r.message_trace]))
                arrays[f"{cname}/{v}/{vn}/vn"] = np.stack(vs)
                arrays[f"{cname}/{v}/{vn}/cn"] = np.stack(cs)
    np.savez_compressed(HERE / "golden_traces.npz", **arrays)


def harness():
    out = {}
    toy = build_gb(GbSpec(3, (0, 1), (0, 2)))
    small = build_gb(GbSpec(*CODES["small"]))

    def sweep(code_id, variant, eps, seed, **kw):
        dkw = {"alpha": 0.5} if variant == "sms" else ({"gain": GainParams(0.3, 0.5, 1.1)} if variant == "sagms" else {})
        base = dict(code_id=code_id, decoder=DecoderConfig(variant, l_max=kw.pop("l_max", 4), **dkw),
                    epsilon_list=tuple(eps), seed=seed, target_failures=50, max_frames=100_000)
        base.update(kw)
        return SweepConfig(**base)

    cases = {
        # reference tests/test_harness.py:131-141 frozen outcome (56, 50)
        "toy_ms_lmax1_eps05": (toy, sweep("toy", "ms", (0.5,), 2718, l_max=1), 0.5),
        "small_sagms_eps025": (small, sweep("gb-10-2", "sagms", (0.25,), 31, l_max=4, target_failures=40), 0.25),
        "small_ms_cap": (small, sweep("gb-10-2", "ms", (0.001,), 5, l_max=8, target_failures=500, max_frames=64), 0.001),
        "small_ms_fixed_prior": (small, sweep("gb-10-2", "ms", (0.2,), 8, l_max=4, target_failures=30,
                                             epsilon0_mode="fixed", epsilon0=0.1), 0.2),
        # fixed prior where fp32 and fp64 decide every frame alike (the MS
        # case above is tie-dominated: DESIGN.md section 8, tests/test_gpu_dropin.py)
        "small_sagms_fixed_prior": (small, sweep("gb-10-2", "sagms", (0.2,), 8, l_max=4, target_failures=30,
                                                epsilon0_mode="fixed", epsilon0=0.1), 0.2),
    }
    for name, (H, cfg, eps) in cases.items():
        p = run_point(H, tanner_graph(H), cfg, eps)
        out[name] = {"point": p.__dict__ if hasattr(p, "__dict__") else None}
        from dataclasses import asdict
        out[name]["point"] = asdict(p)
    cfg = sweep("gb-10-2", "sms", (0.3, 0.2, 0.25), 13, l_max=4, target_failures=20)
    with tempfile.TemporaryDirectory() as td:
        run_sweep(small, tanner_graph(small), cfg, out_dir=td)
        out["sweep_sms"] = {
            "results_json": (Path(td) / "results.json").read_text(),
            "fer_tsv": (Path(td) / "fer.tsv").read_text(),
            "points": sorted(os.listdir(Path(td) / "points")),
        }
    (HERE / "golden_harness.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    config1()
    batches()
    traces()
    harness()
    print("golden fixtures written to", HERE)
