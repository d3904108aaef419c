"""Measure every BASELINE.json config on one B200 (device-timed, CUDA events).

    python tools/configs_bench.py [--out gpurun_out/configs.json] [--frames-scale 1.0]

Per (config, code, decoder, p) point: frames, failures, FER with 95% Wilson
interval, mean iterations, device ms (median of 3 timed launches), decoded
frames/s and CN-edge updates/s,
and the kernel kind used.  Config 1 is also checked against the reference's
golden outcome (tests/golden/golden_config1.json).  Random GB codes of
configs 3-4 come from paper_2605_10433_b200.random_gb_spec(ell, w, seed=0)
(the reference ships no generator).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_10433_b200 as P  # noqa: E402

GB254 = P.GbSpec(127, (0, 15, 20, 28, 66), (0, 58, 59, 100, 121))
G = P.GainParams(0.30, 0.50, 1.10)


def dec(name, l_max):
    if name == "bp4":
        return P.DecoderConfig("bp4", l_max=l_max)
    if name == "sagms":
        return P.DecoderConfig("sagms", l_max=l_max, gain=G)
    if name.startswith("sms"):
        return P.DecoderConfig("sms", l_max=l_max, alpha=float(name[3:]))
    return P.DecoderConfig("ms", l_max=l_max)


def point(graph, name, p, frames, l_max, seed=0):
    dg = P.device_graph(graph)
    cfg = dec(name, l_max)
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    P.decode_frames_device(dg, cfg, p, p, seed, 0, min(frames, 1 << 16), counters=cnt, want_frames=False)
    torch.cuda.synchronize()
    times = []
    for _ in range(3):  # median of 3 (short launches are sensitive to clock ramp)
        cnt.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        P.decode_frames_device(dg, cfg, p, p, seed, 0, frames, counters=cnt, want_frames=False)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    ms = sorted(times)[1]
    fr, fails, its, upd = (int(x) for x in cnt.cpu().tolist())
    lo, hi = P.wilson_interval(fails, fr)
    return {"decoder": name, "p": p, "frames": fr, "failures": fails, "fer": fails / fr,
            "wilson95": [lo, hi], "mean_iterations": its / fr, "device_ms": ms,
            "frames_per_s": fr / ms * 1e3, "cn_edge_updates_per_s": upd / ms * 1e3,
            "kernel_kind": dg.kind, "threads_per_frame": dg.threads}


def code_desc(spec, g):
    return {"ell": spec.ell, "a": list(spec.a_exponents), "b": list(spec.b_exponents), "n": g.n,
            "k": P.gb_dimension(spec), "E": g.edge_count}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.json"))
    ap.add_argument("--frames-scale", type=float, default=1.0)
    args = ap.parse_args()
    sc = lambda n: max(1024, int(n * args.frames_scale))  # noqa: E731
    out = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "configs": {}}
    g254 = P.gb_graph(GB254)

    # config 1 (+ golden)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden_config1.json")))
    fails, iters = P.decode_frames(g254, dec("sagms", 100), 0.05, 0.05, 0, 0, 10_000)
    c1 = point(g254, "sagms", 0.05, 10_000, 100)
    c1["golden_match"] = (fails.nonzero()[0].tolist() == gold["fail_frames"]
                          and int(iters.sum()) == gold["sum_iterations"])
    out["configs"]["1"] = {"code": code_desc(GB254, g254), "points": [c1]}

    # config 2
    pts = []
    for p in (0.02, 0.04, 0.06, 0.08, 0.10):
        for name in ("bp4", "sms0.5", "sms0.625", "sms0.75", "sms0.875", "sms1.0", "sagms"):
            pts.append(point(g254, name, p, sc(1 << 20), 100))
    out["configs"]["2"] = {"code": code_desc(GB254, g254), "points": pts}

    # config 3: random GB w=5, l in {63,127,255,511}, SAGMS and SMS(0.75), p=0.05, l_max 64
    c3 = []
    for ell in (63, 127, 255, 511):
        spec = P.random_gb_spec(ell, 5, seed=0)
        g = P.gb_graph(spec)
        c3.append({"code": code_desc(spec, g),
                   "points": [point(g, name, 0.05, sc(1 << 20), 64) for name in ("sagms", "sms0.75")]})
    out["configs"]["3"] = c3

    # config 4: random GB l=127, w in {3,4,5,6,8}, p=0.04, l_max 100
    c4 = []
    for w in (3, 4, 5, 6, 8):
        spec = P.random_gb_spec(127, w, seed=0)
        g = P.gb_graph(spec)
        c4.append({"code": code_desc(spec, g),
                   "points": [point(g, name, 0.04, sc(1 << 20), 100)
                              for name in ("sms0.5", "sms0.75", "sms1.0", "sagms", "bp4")]})
    out["configs"]["4"] = c4

    # config 5: [[254,28]] and a random w=5 l=511 code (the draw BASELINE.md
    # section 2.2 measured on CPU) at p=0.03 / 0.08, SAGMS, 2^22 frames (1 GPU here)
    spec511 = P.GbSpec(511, (0, 5, 200, 397, 418), (0, 81, 284, 347, 418))
    g511 = P.gb_graph(spec511)
    out["configs"]["5"] = [
        {"code": code_desc(GB254, g254), "points": [point(g254, "sagms", p, sc(1 << 22), 100) for p in (0.03, 0.08)]},
        {"code": code_desc(spec511, g511), "points": [point(g511, "sagms", p, sc(1 << 22), 100) for p in (0.03, 0.08)]},
    ]
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({"config1_golden_match": c1["golden_match"],
                      "config2_frames_per_s_total": sum(p["frames"] for p in pts) / sum(p["device_ms"] for p in pts) * 1e3}))


if __name__ == "__main__":
    main()
