"""Off-bench throughput probes (dev tool): run_point (pipelined 2^20-frame
batches, ordered stop rule) and the reference harness's 4096-frame calls."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_10433_b200 as P  # noqa: E402
from paper_2605_10433_b200 import harness as H  # noqa: E402

g = P.gb_graph(P.GbSpec(127, (0, 15, 20, 28, 66), (0, 58, 59, 100, 121)))
cfg = P.DecoderConfig("sagms", l_max=100, gain=P.GainParams(0.30, 0.50, 1.10))
for p in (0.02, 0.05):
    sc = P.SweepConfig("gb-254-28", cfg, (p,), 0, target_failures=10**9, max_frames=1 << 24)
    P.run_point(g, sc, p)
    torch.cuda.synchronize()
    t = time.perf_counter()
    pt = P.run_point(g, sc, p)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    # the same frames as device-only launches
    t = time.perf_counter()
    for s in range(0, 1 << 24, 1 << 20):
        H.decode_frames_device(g, cfg, p, p, 0, s, 1 << 20)
    torch.cuda.synchronize()
    dd = time.perf_counter() - t
    # batch iteration alone (no stop-rule bookkeeping)
    t = time.perf_counter()
    for fails, iters in H.frame_batches(g, cfg, p, p, 0, 1 << 24, 1 << 20):
        pass
    db = time.perf_counter() - t
    print(f"p={p}: run_point {pt.frames / dt:.3g} frames/s; frame_batches {(1 << 24) / db:.3g}; "
          f"device-only launches {(1 << 24) / dd:.3g}")
for _ in range(3):
    P.decode_frames(g, cfg, 0.05, 0.05, 0, 0, 4096)
t = time.perf_counter()
for i in range(200):
    P.decode_frames(g, cfg, 0.05, 0.05, 0, i * 4096, 4096)
dt = (time.perf_counter() - t) / 200
print(f"decode_frames 4096 p=0.05: {dt * 1e3:.3f} ms per call, {4096 / dt:.3g} frames/s")
