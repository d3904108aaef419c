"""Build tests/golden/fer64_config2.json: per BASELINE configs[1] point, the
failure count of the reference's float64 arithmetic on frames [0, F) (seed 0,
matched eps0) -- what bench.py's `fer_check` compares the GPU's failure
counts with (dev tool; rerun after tools/fer_match_configs.py ref --only c2).

Source, per point, the largest available of:
  cache/fer64/c2_gb254_<decoder>_p<p>_L100_<F>.npz   (fer_match_configs.py ref)
  profiles/fer_match_256k_r01.json                   (2^18 frames, same oracle)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
PS = (0.02, 0.04, 0.06, 0.08, 0.10)
NAMES = ("bp4", "sms0.5", "sms0.625", "sms0.75", "sms0.875", "sms1.0", "sagms")


def main():
    old = {r["point"]: r for r in json.load(open(os.path.join(ROOT, "profiles", "fer_match_256k_r01.json")))["rows"]}
    out = {}
    for p in PS:
        for name in NAMES:
            path = os.path.join(ROOT, "cache", "fer64", f"c2_gb254_{name}_p{p}_L100_{1 << 20}.npz")
            if os.path.exists(path):
                d = np.load(path)
                fails = np.unpackbits(d["fails"])[: 1 << 20]
                out[f"{name}@{p}"] = {"frames": 1 << 20, "ref64_failures": int(fails.sum()),
                                      "ref64_sum_iterations": int(d["iters"].astype(np.int64).sum())}
            else:
                r = old[f"{name}@{p}"]
                out[f"{name}@{p}"] = {"frames": r["frames"], "ref64_failures": r["ref64_failures"]}
    doc = {"note": "float64 restatement of the reference (oracle precision=64; bit-exact with the reference for the "
                   "min-sum family, tests/test_oracle_pins.py) on frames [0, frames) of each BASELINE configs[1] "
                   "point: [[254,28]], seed 0, matched eps0, l_max 100, marginal VN.  tools/make_fer64_fixture.py",
           "points": out}
    with open(os.path.join(ROOT, "tests", "golden", "fer64_config2.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    n20 = sum(1 for v in out.values() if v["frames"] == 1 << 20)
    print(f"{len(out)} points, {n20} at 2^20 frames")


if __name__ == "__main__":
    main()
