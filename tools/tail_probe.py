"""Per-launch fixed cost of the persistent decode kernel (dev tool): time
decode_frames_device for growing frame counts from frame 0 and fit
T(N) = c N + D.  python tools/tail_probe.py CODE VARIANT P [log2 counts]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10433_b200 as P  # noqa: E402

codes = {"254": (127, (0, 15, 20, 28, 66), (0, 58, 59, 100, 121)),
         "1022": (511, (0, 5, 200, 397, 418), (0, 81, 284, 347, 418))}
G = P.GainParams(0.3, 0.5, 1.1)
cfgs = {"sagms": P.DecoderConfig("sagms", l_max=100, gain=G), "bp4": P.DecoderConfig("bp4", l_max=100),
        "sms": P.DecoderConfig("sms", l_max=100, alpha=0.75)}
code, var, p = sys.argv[1], sys.argv[2], float(sys.argv[3])
logs = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [16, 17, 18, 19, 20, 21, 22]
g = P.device_graph(P.gb_graph(P.GbSpec(*codes[code])))
cfg = cfgs[var]
P.decode_frames_device(g, cfg, p, p, 0, 0, 1 << 16, want_frames=False)
rows = []
for lg in logs:
    n = 1 << lg
    ts = []
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        P.decode_frames_device(g, cfg, p, p, 0, 0, n, want_frames=False)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    rows.append((n, min(ts)))
    print(f"code={code} {var} p={p} frames=2^{lg} ms={min(ts):.3f} ns/frame={min(ts) * 1e6 / n:.2f}", flush=True)
N = np.array([r[0] for r in rows], float)
T = np.array([r[1] for r in rows], float)
c, d = np.polyfit(N, T, 1)
print(f"fit: {c * 1e6:.3f} ns/frame + {d:.3f} ms per launch", flush=True)
