import sys, os, torch
sys.path.insert(0, "/root/repo")
import paper_2605_10433_b200 as P
spec = P.random_gb_spec(127, 5, seed=0)
g = P.gb_graph(spec); dg = P.device_graph(g)
G = P.GainParams(0.3, 0.5, 1.1)
cfgs = {"sagms": P.DecoderConfig("sagms", l_max=64, gain=G), "sms0.75": P.DecoderConfig("sms", l_max=64, alpha=0.75)}
for frames in (1 << 20, 1 << 22):
    for rep in range(3):
        for name, cfg in cfgs.items():
            cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); s.record()
            P.decode_frames_device(dg, cfg, 0.05, 0.05, 0, 0, frames, counters=cnt, want_frames=False)
            e.record(); torch.cuda.synchronize()
            ms = s.elapsed_time(e); c = cnt.cpu().tolist()
            print(frames, rep, name, f"ms={ms:.1f} it={c[2]/c[0]:.2f} upd/s={c[3]/ms*1e3:.3g} f/s={c[0]/ms*1e3:.3g}", flush=True)
