"""FER match on shared frames: GPU outcomes vs the reference's float64
arithmetic (the fp64 oracle, bit-exact with the reference for the min-sum
family -- tests/test_oracle_pins.py).

    python tools/fer_match.py gpu  --frames 32768      # on the B200 box
    python tools/fer_match.py cpu  --frames 32768      # here: oracle fp64 + compare

For every BASELINE configs[1] point the GPU decodes frames [0, F) and the
per-frame fail flags are stored; the CPU side decodes the same frames with
the fp64 restatement and reports both FERs, their 95% Wilson intervals, the
paired flip counts, and whether each FER lies in the other's interval.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PS = (0.02, 0.04, 0.06, 0.08, 0.10)
NAMES = ("bp4", "sms0.5", "sms0.625", "sms0.75", "sms0.875", "sms1.0", "sagms")
CODE = (127, (0, 15, 20, 28, 66), (0, 58, 59, 100, 121))


def cfg_ns(name):
    from types import SimpleNamespace as NS
    gain = NS(alpha_min=0.30, alpha_max=0.50, eta_unsat=1.10) if name == "sagms" else None
    alpha = float(name[3:]) if name.startswith("sms") else None
    variant = "sms" if name.startswith("sms") else name
    return NS(variant=variant, l_max=100, vn_mode="marginal", alpha=alpha, gain=gain)


def gpu(frames, out, names=NAMES):
    import paper_2605_10433_b200 as P
    g = P.gb_graph(P.GbSpec(*CODE))
    res = {}
    for p in PS:
        for name in names:
            c = cfg_ns(name)
            dcfg = P.DecoderConfig(c.variant, l_max=100, alpha=c.alpha,
                                   gain=P.GainParams(0.30, 0.50, 1.10) if c.gain else None)
            f, it = P.decode_frames(g, dcfg, p, p, 0, 0, frames)
            res[f"{name}@{p}/fails"] = f
            res[f"{name}@{p}/iters"] = it.astype(np.uint8)  # <= l_max = 100
    np.savez_compressed(out, **res)


def cpu(frames, gpu_npz, out, nthreads=None, fp32=True, names=NAMES, ref_cache=None):
    """fp64 oracle on the same frames; rows are written after every point so
    a long run can be inspected (and is kept) while it progresses."""
    from oracle import oracle as O
    from paper_2605_10433_b200.harness import wilson_interval
    g = O.Graph(O.gb_graph(*CODE))
    d = np.load(gpu_npz)
    rows = []

    def dump(done):
        summary = {"points": len(rows), "complete": done,
                   "all_gpu_fer_in_ref_ci": all(r["gpu_fer_in_ref_ci"] for r in rows),
                   "total_flipped_frames": sum(r["frames_flipped"] for r in rows),
                   "total_frames": sum(r["frames"] for r in rows)}
        if fp32:
            summary["all_gpu_equal_fp32_oracle"] = all(r["gpu_equals_fp32_oracle"] for r in rows)
        with open(out, "w") as fh:
            json.dump({"summary": summary, "rows": rows}, fh, indent=1)
        return summary

    kw = {"nthreads": nthreads} if nthreads else {}
    for p in PS:
        for name in names:
            gf = d[f"{name}@{p}/fails"][:frames]
            git = d[f"{name}@{p}/iters"][:frames].astype(np.int64)
            key = f"{name}@{p}/{frames}"
            cache = dict(np.load(ref_cache)) if ref_cache and os.path.exists(ref_cache) else {}
            if key + "/fails" in cache:  # fp64 outcomes depend only on (decoder, p, frames)
                of, oit = cache[key + "/fails"].astype(bool), cache[key + "/iters"].astype(np.int64)
            else:
                of, oit, _, _ = O.frames(g, cfg_ns(name), p, p, 0, 0, frames, precision=64, **kw)
                if ref_cache:
                    cache[key + "/fails"], cache[key + "/iters"] = of.astype(np.uint8), oit.astype(np.uint8)
                    np.savez_compressed(ref_cache, **cache)
            n = len(gf)
            fg, fo = int(gf.sum()), int(of.sum())
            lg, hg = wilson_interval(fg, n)
            lo, ho = wilson_interval(fo, n)
            row = {"point": f"{name}@{p}", "frames": n, "gpu_failures": fg, "ref64_failures": fo,
                   "gpu_fer": fg / n, "ref64_fer": fo / n, "gpu_wilson95": [lg, hg],
                   "ref64_wilson95": [lo, ho], "gpu_fer_in_ref_ci": lo <= fg / n <= ho,
                   "frames_flipped": int((gf != of).sum()),
                   "gpu_only_failures": int((gf & ~of.astype(bool)).sum()),
                   "ref64_only_failures": int((~gf.astype(bool) & of.astype(bool)).sum()),
                   "frames_iterations_differ": int((git != oit).sum()),
                   "mean_iterations_gpu": float(git.mean()), "mean_iterations_ref64": float(oit.mean())}
            if fp32:
                o32, _, _, _ = O.frames(g, cfg_ns(name), p, p, 0, 0, frames, precision=32, **kw)
                row["gpu_equals_fp32_oracle"] = bool(np.array_equal(gf, o32))
            rows.append(row)
            dump(False)
            print(row["point"], fg, fo, row["gpu_fer_in_ref_ci"], flush=True)
    print(json.dumps(dump(True)))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=("gpu", "cpu"))
    ap.add_argument("--frames", type=int, default=32768)
    ap.add_argument("--gpu-npz", default=os.path.join(ROOT, "gpurun_out", "fer_gpu.npz"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "fer_match_r01.json"))
    ap.add_argument("--threads", type=int, default=None)
    ap.add_argument("--names", default=",".join(NAMES), help="comma-separated decoder subset")
    ap.add_argument("--ref-cache", default=None, help="npz cache of the fp64 outcomes (reused across GPU builds)")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32-oracle equality column")
    a = ap.parse_args()
    if a.mode == "gpu":
        gpu(a.frames, a.gpu_npz, names=a.names.split(","))
    else:
        cpu(a.frames, a.gpu_npz, a.out, nthreads=a.threads, fp32=not a.no_fp32, names=a.names.split(","),
            ref_cache=a.ref_cache)
