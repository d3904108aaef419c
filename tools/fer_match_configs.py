"""FER match for BASELINE configs 3-5: GPU outcomes vs the reference's
float64 arithmetic on shared frames (the fp64 oracle, bit-exact with the
reference for the min-sum family -- tests/test_oracle_pins.py).

    python tools/fer_match_configs.py gpu [--only c3,c4,c5]   # B200 box: fail bits + iterations
    python tools/fer_match_configs.py ref [--only ...]        # here: fp64 oracle, cached per point
    python tools/fer_match_configs.py compare --out profiles/fer_match_configs345_r02.json

Points (BASELINE.json configs[2..4], seed 0, matched eps0, marginal VN; `--only c2`
adds configs[1], the 35-point [[254,28]] sweep, at its own 2^20 frames per point):
  C3  random GB l in {63,127,255,511}, w=5; SAGMS(0.30,0.50,1.10), SMS 0.75; p=0.05; l_max 64
  C4  random GB l=127, w in {3,4,5,6,8}; SMS {0.5,0.75,1.0}, SAGMS, BP4; p=0.04; l_max 100
  C5  [[254,28]] and random GB l=511 w=5; SAGMS; p in {0.03,0.08}; l_max 100
Frames: 2^20 per C3/C4 point (the config's own count).  C5's workload is
2^22 frames; the GPU decodes all of them, the fp64 comparison covers the
first 2^20.

Per point the compare step reports both FERs with 95% Wilson intervals
(harness.py:102-125), whether the GPU FER lies inside the fp64 interval, the
paired flips (GPU-only / fp64-only failures) and their balance in sigma
((a - b) / sqrt(a + b), McNemar), and frames whose iteration count differs.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GB254 = (127, (0, 15, 20, 28, 66), (0, 58, 59, 100, 121))
CACHE = os.path.join(ROOT, "cache", "fer64")


def spec_of(code):
    """code = "gb254" or (ell, w) of random_gb_spec(ell, w, seed=0)."""
    if code == "gb254":
        return GB254
    from paper_2605_10433_b200.codes import random_gb_spec
    s = random_gb_spec(code[0], code[1], 0)
    return (s.ell, tuple(s.a_exponents), tuple(s.b_exponents))


def code_name(code):
    return "gb254" if code == "gb254" else f"l{code[0]}w{code[1]}"


def points(only=("c3", "c4", "c5")):
    """(config, code, decoder, p, l_max, gpu_frames, ref_frames)."""
    out = []
    if "c2" in only:  # BASELINE configs[1] at its own size; cheapest points first
        for p in (0.02, 0.04, 0.06, 0.08, 0.10):
            for name in ("sagms", "sms0.5", "sms0.625", "sms0.75", "sms0.875", "sms1.0", "bp4"):
                out.append(("c2", "gb254", name, p, 100, 1 << 20, 1 << 20))
    if "c3" in only:
        for ell in (63, 127, 255, 511):
            for name in ("sagms", "sms0.75"):
                out.append(("c3", (ell, 5), name, 0.05, 64, 1 << 20, 1 << 20))
    if "c4" in only:
        for w in (3, 4, 5, 6, 8):
            for name in ("sms0.5", "sms0.75", "sms1.0", "sagms", "bp4"):
                out.append(("c4", (127, w), name, 0.04, 100, 1 << 20, 1 << 20))
    if "c5" in only:
        for code in ("gb254", (511, 5)):
            for p in (0.03, 0.08):
                # the l = 511, p = 0.08 point first ran at 2^18 reference frames
                # (QSG_FER_C5_SHORT=1 reproduces that); now at the full 2^20
                short = os.environ.get("QSG_FER_C5_SHORT") and code != "gb254" and p == 0.08
                ref = 1 << 18 if short else 1 << 20
                out.append(("c5", code, "sagms", p, 100, 1 << 22, ref))
    return out


def key(pt):
    cfg, code, name, p, l_max, _, _ = pt
    return f"{cfg}_{code_name(code)}_{name}_p{p}_L{l_max}"


def cfg_ns(name, l_max):
    from types import SimpleNamespace as NS
    gain = NS(alpha_min=0.30, alpha_max=0.50, eta_unsat=1.10) if name == "sagms" else None
    alpha = float(name[3:]) if name.startswith("sms") else None
    variant = "sms" if name.startswith("sms") else name
    return NS(variant=variant, l_max=l_max, vn_mode="marginal", alpha=alpha, gain=gain)


def gpu(only, out_dir):
    import torch

    import paper_2605_10433_b200 as P
    os.makedirs(out_dir, exist_ok=True)
    for pt in points(only):
        cfg, code, name, p, l_max, nf, _ = pt
        ell, a, b = spec_of(code)
        g = P.gb_graph(P.GbSpec(ell, a, b))
        c = cfg_ns(name, l_max)
        dcfg = P.DecoderConfig(c.variant, l_max=l_max, alpha=c.alpha,
                               gain=P.GainParams(0.30, 0.50, 1.10) if c.gain else None)
        t = time.perf_counter()
        fails, iters, _ = P.decode_frames_device(g, dcfg, p, p, 0, 0, nf)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        f = fails.cpu().numpy().astype(bool)
        it = iters.cpu().numpy().astype(np.uint8)  # <= l_max <= 100
        np.savez_compressed(os.path.join(out_dir, key(pt) + ".npz"), fails=np.packbits(f), iters=it,
                            frames=np.int64(nf))
        print(key(pt), nf, int(f.sum()), f"{dt:.2f}s", flush=True)


def ref(only, threads, p_only=None, cache=None):
    from oracle import oracle as O
    cache = cache or CACHE
    os.makedirs(cache, exist_ok=True)
    for pt in points(only):
        cfg, code, name, p, l_max, _, nr = pt
        if p_only is not None and p != p_only:
            continue
        path = os.path.join(cache, key(pt) + f"_{nr}.npz")
        if os.path.exists(path):
            continue
        ell, a, b = spec_of(code)
        g = O.Graph(O.gb_graph(ell, a, b))
        t = time.perf_counter()
        fails, iters, _, cnt = O.frames(g, cfg_ns(name, l_max), p, p, 0, 0, nr, precision=64, nthreads=threads)
        dt = time.perf_counter() - t
        np.savez_compressed(path + ".tmp.npz", fails=np.packbits(fails), iters=iters.astype(np.uint8),
                            frames=np.int64(nr))
        os.replace(path + ".tmp.npz", path)
        print(key(pt), nr, int(fails.sum()), f"{dt:.1f}s", flush=True)


def compare_point(gf, git, of, oit):
    from paper_2605_10433_b200.harness import wilson_interval
    n = len(gf)
    fg, fo = int(gf.sum()), int(of.sum())
    lg, hg = wilson_interval(fg, n)
    lo, ho = wilson_interval(fo, n)
    a = int((gf & ~of).sum())
    b = int((~gf & of).sum())
    sigma = (a - b) / math.sqrt(a + b) if a + b else 0.0
    return {"frames": n, "gpu_failures": fg, "ref64_failures": fo, "gpu_fer": fg / n, "ref64_fer": fo / n,
            "gpu_wilson95": [lg, hg], "ref64_wilson95": [lo, ho], "gpu_fer_in_ref_ci": bool(lo <= fg / n <= ho),
            "gpu_only_failures": a, "ref64_only_failures": b, "flip_balance_sigma": round(sigma, 3),
            "frames_iterations_differ": int((git != oit).sum()),
            "mean_iterations_gpu": float(git.mean()), "mean_iterations_ref64": float(oit.mean())}


def compare(only, gpu_dir, out, update=False):
    """update: keep the rows already in ``out`` and replace only those whose
    GPU and fp64 outcome files are both present (the fp64 cache of a long
    study does not have to be complete to refresh a few points)."""
    rows = []
    old = {}
    if update and os.path.exists(out):
        with open(out) as fh:
            old = {r["point"]: r for r in json.load(fh)["rows"]}
    for pt in points(only):
        cfg, code, name, p, l_max, nf, nr = pt
        gpath = os.path.join(gpu_dir, key(pt) + ".npz")
        rpath = os.path.join(CACHE, key(pt) + f"_{nr}.npz")
        if not (os.path.exists(gpath) and os.path.exists(rpath)):
            if key(pt) in old:
                rows.append(old[key(pt)])
            else:
                print("missing", key(pt), os.path.exists(gpath), os.path.exists(rpath))
            continue
        gd, rd = np.load(gpath), np.load(rpath)
        gfa = np.unpackbits(gd["fails"])[:nf].astype(bool)
        gita = gd["iters"].astype(np.int64)
        of = np.unpackbits(rd["fails"])[:nr].astype(bool)
        oit = rd["iters"].astype(np.int64)
        row = {"point": key(pt), "config": cfg, "code": spec_of(code), "decoder": name, "p": p,
               "l_max": l_max}
        row.update(compare_point(gfa[:nr], gita[:nr], of, oit))
        if nf > nr:  # the GPU's full workload, for the record
            from paper_2605_10433_b200.harness import wilson_interval
            fg = int(gfa.sum())
            row["gpu_full"] = {"frames": nf, "failures": fg, "fer": fg / nf,
                               "wilson95": list(wilson_interval(fg, nf)), "mean_iterations": float(gita.mean())}
        rows.append(row)
    summary = {"points": len(rows), "frames_compared": sum(r["frames"] for r in rows),
               "all_gpu_fer_in_ref_ci": all(r["gpu_fer_in_ref_ci"] for r in rows),
               "max_abs_flip_balance_sigma": max((abs(r["flip_balance_sigma"]) for r in rows), default=0.0),
               "total_flipped_frames": sum(r["gpu_only_failures"] + r["ref64_only_failures"] for r in rows)}
    with open(out, "w") as fh:
        json.dump({"summary": summary, "rows": rows}, fh, indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=("gpu", "ref", "compare", "list"))
    ap.add_argument("--only", default="c3,c4,c5")
    ap.add_argument("--gpu-dir", default=os.path.join(ROOT, "gpurun_out", "fer_cfg"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "fer_match_configs345_r02.json"))
    ap.add_argument("--threads", type=int, default=None)
    ap.add_argument("--p-only", type=float, default=None, help="ref: only the points at this p")
    ap.add_argument("--cache-dir", default=None, help="ref: where the fp64 outcomes are cached")
    ap.add_argument("--update", action="store_true", help="compare: refresh only the rows whose files exist")
    a = ap.parse_args()
    only = tuple(a.only.split(","))
    if a.mode == "gpu":
        gpu(only, a.gpu_dir)
    elif a.mode == "ref":
        ref(only, a.threads, a.p_only, a.cache_dir)
    elif a.mode == "list":
        for pt in points(only):
            print(key(pt), pt[5], pt[6])
    else:
        compare(only, a.gpu_dir, a.out, a.update)
