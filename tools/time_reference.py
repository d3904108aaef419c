"""Time the REFERENCE itself (numpy, /root/reference/pkg/src/qsagms) on the
BASELINE configs[1] points, single core, in the build container (the
reference cannot travel to the GPU box; bench.py's reference arm times the
C port of it there).

    OMP_NUM_THREADS=1 python tools/time_reference.py [--frames 256]

For every (decoder, p) point: reference _decode_frames on frames [0, F)
(Philox sampling + syndromes + decode_batch, the reference FER unit).
Writes profiles/reference_numpy_r01.json.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=256)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "reference_numpy_r01.json"))
    a = ap.parse_args()
    from qsagms.code import GbSpec, build_gb, tanner_graph
    from qsagms.decoder import DecoderConfig, GainParams
    from qsagms.harness import _decode_frames
    H = build_gb(GbSpec(127, (0, 15, 20, 28, 66), (0, 58, 59, 100, 121)))
    g = tanner_graph(H)
    decs = [("bp4", DecoderConfig("bp4", l_max=100))]
    decs += [(f"sms{al}", DecoderConfig("sms", l_max=100, alpha=al)) for al in (0.5, 0.625, 0.75, 0.875, 1.0)]
    decs.append(("sagms", DecoderConfig("sagms", l_max=100, gain=GainParams(0.30, 0.50, 1.10))))
    rows, tot_frames, tot_time, tot_upd = [], 0, 0.0, 0
    for p in (0.02, 0.04, 0.06, 0.08, 0.10):
        for name, cfg in decs:
            t0 = time.perf_counter()
            fails, iters = _decode_frames(g, cfg, p, p, 0, 0, a.frames)
            dt = time.perf_counter() - t0
            upd = g.edge_count * int((iters - 1).sum())
            rows.append({"point": f"{name}@{p}", "frames": a.frames, "seconds": dt,
                         "frames_per_s": a.frames / dt, "cn_edge_updates_per_s": upd / dt,
                         "failures": int(fails.sum()), "mean_iterations": float(iters.mean())})
            tot_frames += a.frames
            tot_time += dt
            tot_upd += upd
            print(rows[-1], flush=True)
    out = {"what": "reference qsagms._decode_frames (numpy float64), 1 core, build container CPU",
           "cpu": platform.processor() or platform.machine(), "omp_threads": os.environ.get("OMP_NUM_THREADS"),
           "frames_per_point": a.frames, "total_frames": tot_frames, "total_seconds": tot_time,
           "frames_per_s": tot_frames / tot_time, "cn_edge_updates_per_s": tot_upd / tot_time, "rows": rows}
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: out[k] for k in ("frames_per_s", "cn_edge_updates_per_s", "total_seconds")}))


if __name__ == "__main__":
    main()
