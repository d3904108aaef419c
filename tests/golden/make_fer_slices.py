"""fp64 outcome slices for the FER-criterion GPU test (tests/test_gpu_fer.py).

For every BASELINE config-3/4/5 point of tools/fer_match_configs.py, the
first 2^15 frames (seed 0, frames 0..32767 -- the same frames the GPU
decodes first) are decoded by the oracle's float64 restatement, which is
bit-exact with the reference's own arithmetic for the min-sum family
(tests/test_oracle_pins.py) and pinned to the reference's BP4 outcomes.
Stored: packed failure bits and iteration counts per point.

    python tests/golden/make_fer_slices.py [--threads N]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

SLICE = 1 << 15
OUT = os.path.join(HERE, "fer_slices_c345.npz")


def main():
    import fer_match_configs as F
    from oracle import oracle as O
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=None)
    a = ap.parse_args()
    arrays = {}
    for pt in F.points():
        cfg, code, name, p, l_max, _, _ = pt
        ell, aa, bb = F.spec_of(code)
        g = O.Graph(O.gb_graph(ell, aa, bb))
        t = time.perf_counter()
        fails, iters, _, _ = O.frames(g, F.cfg_ns(name, l_max), p, p, 0, 0, SLICE, precision=64,
                                      nthreads=a.threads)
        k = F.key(pt)
        arrays[k + "/fails"] = np.packbits(fails)
        arrays[k + "/iters"] = iters.astype(np.uint8)
        print(k, int(fails.sum()), f"{time.perf_counter() - t:.1f}s", flush=True)
    np.savez_compressed(OUT, **arrays)


if __name__ == "__main__":
    main()
