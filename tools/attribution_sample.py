"""Draw the attribution sample of fp32-vs-fp64 outcome flips at the chaotic
configs[1] point p = 0.08 ([[254,28]], l_max 100, seed 0, matched eps0).

For each decoder the fp32 restatement (== the GPU bit for bit) and the fp64
restatement (== the reference's arithmetic) decode frames [0, N); frames
whose (fails, iterations) differ are the flips.  A seeded random sample of
up to 200 of them per decoder (all of them when fewer) is frozen in
tests/golden/flips_p008.json; tests/test_attribution.py re-derives each one
as a flip and attributes it (oracle/attribution.py).

    python tools/attribution_sample.py [--threads 8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from types import SimpleNamespace as NS

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GB254 = (127, (0, 15, 20, 28, 66), (0, 58, 59, 100, 121))
GAIN = NS(alpha_min=0.30, alpha_max=0.50, eta_unsat=1.10)
# decoder -> frames searched (SAGMS flips are rare: ~15 per 2^18 frames)
SEARCH = {"bp4": 1 << 14, "sms0.5": 1 << 14, "sms0.75": 1 << 14, "sms1.0": 1 << 14, "sagms": 1 << 17}


def cfg_ns(name):
    alpha = float(name[3:]) if name.startswith("sms") else None
    variant = "sms" if name.startswith("sms") else name
    return NS(variant=variant, l_max=100, vn_mode="marginal", alpha=alpha, gain=GAIN if name == "sagms" else None)


def main():
    from oracle import oracle as O
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=None)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "flips_p008.json"))
    a = ap.parse_args()
    g = O.Graph(O.gb_graph(*GB254))
    rng = np.random.default_rng(8)
    out = {"code": GB254, "p": 0.08, "l_max": 100, "seed": 0, "decoders": {}}
    for name, n in SEARCH.items():
        c = cfg_ns(name)
        f32, i32, _, _ = O.frames(g, c, 0.08, 0.08, 0, 0, n, precision=32, nthreads=a.threads)
        f64, i64, _, _ = O.frames(g, c, 0.08, 0.08, 0, 0, n, precision=64, nthreads=a.threads)
        flips = np.nonzero((f32 != f64) | (i32 != i64))[0]
        pick = flips if len(flips) <= 200 else np.sort(rng.choice(flips, size=200, replace=False))
        out["decoders"][name] = {"searched": n, "flips": int(len(flips)),
                                 "outcome_flips": int((f32 != f64).sum()),
                                 "sample": [int(x) for x in pick]}
        print(name, n, len(flips), int((f32 != f64).sum()), flush=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=0)


if __name__ == "__main__":
    main()
