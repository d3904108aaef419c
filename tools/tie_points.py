"""Tie-dominated points (dev tool, CPU): fp32 restatement (== the GPU) vs
float64 restatement (== the reference's arithmetic) on the reference's
[[10,2]] harness test code, where symmetric cycles make whole classes of
frames decide on exact ties.  For every decoder and
prior, failures in fp32 and fp64 on the same frames, and the attribution
kinds of the first 40 differing frames.

    python tools/tie_points.py [--frames 20000] [--out profiles/tie_points_r02.json]
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import sys
from types import SimpleNamespace as NS

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SMALL = (5, (0, 1), (0, 2))
GAIN = NS(alpha_min=0.3, alpha_max=0.5, eta_unsat=1.1)
DECODERS = {"ms": NS(variant="ms", l_max=4, vn_mode="marginal", alpha=None, gain=None),
            "sms0.75": NS(variant="sms", l_max=4, vn_mode="marginal", alpha=0.75, gain=None),
            "sms1.0": NS(variant="sms", l_max=4, vn_mode="marginal", alpha=1.0, gain=None),
            "sagms": NS(variant="sagms", l_max=4, vn_mode="marginal", alpha=None, gain=GAIN)}


def main():
    from oracle import oracle as O
    from oracle.attribution import attribute
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=20000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "tie_points_r02.json"))
    a = ap.parse_args()
    g = O.Graph(O.gb_graph(*SMALL))
    eps, seed, n = 0.2, 8, a.frames
    e = O.sample_errors(g.n, eps, seed, 0, n)
    syn = O.syndromes_of(g, e)
    rows = []
    for name, cfg in DECODERS.items():
        for eps0 in (0.1, 0.2, 0.3):
            f32 = O.frames(g, cfg, eps, eps0, seed, 0, n, precision=32)[0]
            f64 = O.frames(g, cfg, eps, eps0, seed, 0, n, precision=64)[0]
            diff = np.nonzero(f32 != f64)[0]
            kinds = collections.Counter(
                attribute(g, syn[f], O.prior_llr(eps0), cfg, frame=int(f)).kind for f in diff[:40])
            rows.append({"decoder": name, "epsilon": eps, "epsilon0": eps0, "frames": n,
                         "fp32_failures": int(f32.sum()), "fp64_failures": int(f64.sum()),
                         "frames_differing": int(len(diff)), "attribution_first_40": dict(kinds)})
            print(rows[-1], flush=True)
    with open(a.out, "w") as fh:
        json.dump({"code": SMALL, "seed": seed, "note": "[[10,2]] GB code of the reference's harness "
                   "tests; fp32 == GPU bit for bit, fp64 == the reference's arithmetic", "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
