"""Randomised GPU-vs-oracle stress (dev tool, needs a GPU): random GB codes
(l, w) across every kernel shape, random decoders / p / l_max / seeds;
outcomes, iterations and e_hat must match the fp32 oracle bit for bit."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_10433_b200 as P  # noqa: E402
from oracle import oracle  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
cases = int(sys.argv[2]) if len(sys.argv) > 2 else 40
bad = 0
for i in range(cases):
    ell = int(rng.choice([33, 47, 63, 64, 96, 127, 128, 129, 150, 191, 200, 255, 256, 257, 300, 511, 512]))
    w = int(rng.choice([2, 3, 4, 5, 6, 8]))
    if w >= ell // 2:
        continue
    if rng.random() < 0.35:
        # generic kernels: |a| != |b| GB rows, or rows with random Pauli symbols (Y-type edges)
        wb = int(rng.integers(2, 9))
        a = tuple(sorted(rng.choice(ell, size=w, replace=False).tolist()))
        b = tuple(sorted(rng.choice(ell, size=wb, replace=False).tolist()))
        if rng.random() < 0.5 or w == wb:
            n = 2 * ell
            rows = []
            for i in range(int(rng.integers(ell // 2, 2 * ell))):
                cols = sorted(rng.choice(n, size=int(rng.integers(2, 17)), replace=False).tolist())
                rows.append([(c, int(rng.integers(1, 4))) for c in cols])
            used = {c for r in rows for c, _ in r}
            if len(used) < n:  # every qubit needs an edge
                rows.append([(c, 2) for c in sorted(set(range(n)) - used)][:32])
                used = {c for r in rows for c, _ in r}
                if len(used) < n:
                    continue
            g = P.csr_graph(n, rows)
        else:
            g = P.gb_graph(P.GbSpec(ell, a, b))
    else:
        try:
            spec = P.random_gb_spec(ell, w, seed=int(rng.integers(1 << 30)))
        except Exception as exc:  # no k > 0 code found quickly
            print("skip", ell, w, exc)
            continue
        g = P.gb_graph(spec)
    variant = str(rng.choice(["bp4", "ms", "sms", "sagms"]))
    kw = {"alpha": float(rng.choice([0.5, 0.75, 1.0]))} if variant == "sms" else {}
    if variant == "sagms":
        kw["gain"] = P.GainParams(0.3, 0.5, 1.1)
    cfg = P.DecoderConfig(variant, l_max=int(rng.integers(1, 60)),
                          vn_mode=str(rng.choice(["marginal", "additive"])), **kw)
    p = float(rng.uniform(0.01, 0.14))
    seed, start, count = int(rng.integers(1 << 40)), int(rng.integers(1 << 20)), int(rng.integers(1, 400))
    f, it, eh = P.decode_frames_device(g, cfg, p, p, seed, start, count, want_ehat=True)
    of, oi, oe, _ = oracle.frames(g, cfg, p, p, seed, start, count, want_ehat=True)
    ok = (np.array_equal(f.cpu().numpy().astype(bool), of) and np.array_equal(it.cpu().numpy(), oi)
          and np.array_equal(eh.cpu().numpy(), oe))
    # the same frames without e_hat: the lean kernel instance where one exists
    f2, it2, _ = P.decode_frames_device(g, cfg, p, p, seed, start, count)
    ok = ok and np.array_equal(f2.cpu().numpy().astype(bool), of) and np.array_equal(it2.cpu().numpy(), oi)
    bad += not ok
    print(f"{'ok ' if ok else 'BAD'} l={ell} w={w} kind={g.kind} T={g.threads} {variant} {cfg.vn_mode} l_max={cfg.l_max} "
          f"p={p:.3f} frames={count}", flush=True)
print("STRESS_FAILURES", bad)
sys.exit(1 if bad else 0)
