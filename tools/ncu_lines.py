"""Per-source-line profile of one kernel from an ncu report (dev tool).

ncu's CLI exports per-SASS-instruction metrics (source page, sass view) but
not the CUDA-line view; this joins them with the line table nvdisasm -g
prints for the same function in the build's object file.

    python tools/ncu_lines.py REPORT.ncu-rep build/csrc/qsg_inst_w5.o MANGLED_NAME [--top 40]

Prints, per source line (innermost location, inlined bodies included), warp
instructions executed and stall samples, sorted by samples, plus per-region
totals for the line ranges given with --region name:lo-hi.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import os
import re
import subprocess
import tempfile


def sass_lines(obj, fn):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True, check=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
    lines = txt.splitlines()
    start = lines.index(f"{fn}:")
    amap, cur = {}, None
    for ln in lines[start + 1:]:
        if re.match(r"^\S+:$", ln) and not ln.startswith(".text." + fn) and not ln.startswith(".L"):
            break
        m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if m:
            amap[int(m.group(1), 16)] = (cur, m.group(2).strip())
    return amap


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("obj")
    ap.add_argument("fn")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--region", action="append", default=[])
    a = ap.parse_args()
    amap = sass_lines(a.obj, a.fn)
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ia, ie, isamp = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    per = collections.defaultdict(lambda: [0, 0])
    tot_i = tot_s = 0
    base = None
    for r in rows[2:]:
        try:
            addr = int(r[ia], 16)
            n, s = int(r[ie] or 0), int(r[isamp] or 0)
        except (ValueError, IndexError):
            continue
        if base is None:
            base = addr
        loc = amap.get(addr - base, (("?", 0), ""))[0]
        per[loc][0] += n
        per[loc][1] += s
        tot_i += n
        tot_s += s
    srcs = {}
    for (f, _), _v in per.items():
        p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2605_10433_b200", "csrc", f)
        if f not in srcs and os.path.exists(p):
            srcs[f] = open(p).read().splitlines()
    print(f"total warp instructions {tot_i}, stall samples {tot_s}")
    for loc, (n, s) in sorted(per.items(), key=lambda kv: -kv[1][1])[:a.top]:
        f, line = loc
        text = srcs.get(f, [""] * (line + 1))[line - 1].strip() if f in srcs and line else ""
        print(f"{100 * s / max(tot_s, 1):5.1f}% samp {100 * n / max(tot_i, 1):5.1f}% inst  {f}:{line:<5d} {text[:90]}")
    for reg in a.region:
        name, rng = reg.split(":")
        f, lohi = rng.rsplit("@", 1) if "@" in rng else ("qsg_kernel.cuh", rng)
        lo, hi = (int(x) for x in lohi.split("-"))
        n = sum(v[0] for (ff, ln), v in per.items() if ff == f and lo <= ln <= hi)
        s = sum(v[1] for (ff, ln), v in per.items() if ff == f and lo <= ln <= hi)
        print(f"region {name:20s} {100 * s / max(tot_s, 1):5.1f}% samples {100 * n / max(tot_i, 1):5.1f}% instructions")


if __name__ == "__main__":
    main()
