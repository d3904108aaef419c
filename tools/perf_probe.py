"""Quick device-timed throughput probe of qsg_decode_frames (dev tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_10433_b200 as P

codes = {"254": (127, (0, 15, 20, 28, 66), (0, 58, 59, 100, 121)),
         "1022": (511, (0, 5, 200, 397, 418), (0, 81, 284, 347, 418))}
G = P.GainParams(0.3, 0.5, 1.1)
cfgs = {"sagms": P.DecoderConfig("sagms", l_max=100, gain=G), "sms": P.DecoderConfig("sms", l_max=100, alpha=0.75),
        "bp4": P.DecoderConfig("bp4", l_max=100), "sms": P.DecoderConfig("sms", l_max=100, alpha=0.75), "sagms_add": P.DecoderConfig("sagms", l_max=100, gain=G, vn_mode="additive")}
frames = int(os.environ.get("FRAMES", 1 << 20))
for code in sys.argv[1].split(","):
    # "254", "1022", or "rgb<ell>w<w>" for random_gb_spec(ell, w, seed=0)
    if code.startswith("rgb"):
        ell, w = code[3:].split("w")
        g = P.gb_graph(P.random_gb_spec(int(ell), int(w), seed=0))
    else:
        g = P.gb_graph(P.GbSpec(*codes[code]))
    dg = P.device_graph(g)
    for name in sys.argv[2].split(","):
        for p in [float(x) for x in sys.argv[3].split(",")]:
            cfg = cfgs[name]
            cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
            P.decode_frames_device(g, cfg, p, p, 0, 0, min(frames, 65536), counters=cnt, want_frames=False)
            torch.cuda.synchronize()
            cnt.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            P.decode_frames_device(g, cfg, p, p, 0, 0, frames, counters=cnt, want_frames=False)
            e.record(); torch.cuda.synchronize()
            ms = s.elapsed_time(e)
            c = cnt.cpu().tolist()
            print(f"code={code} {name} p={p} frames={c[0]} fails={c[1]} mean_it={c[2]/c[0]:.3f} "
                  f"ms={ms:.2f} frames/s={c[0]/ms*1e3:.4g} cn_upd/s={c[3]/ms*1e3:.4g} kind={dg.kind} T={dg.threads}", flush=True)
