"""Tabulate tools/ab3.sh output: min ms per (point, library) (dev tool)."""
import collections
import re
import sys

d = collections.defaultdict(lambda: collections.defaultdict(list))
libs = []
lib = None
for ln in open(sys.argv[1]):
    m = re.match(r"== (\S+) \(rep", ln)
    if m:
        lib = m.group(1).split("/")[-1]
        if lib not in libs:
            libs.append(lib)
        continue
    m = re.search(r"code=(\S+) (\S+) p=(\S+) .* ms=(\S+) frames/s", ln)
    if m:
        d[(m.group(1), m.group(2), m.group(3))][lib].append(float(m.group(4)))
print("point".ljust(26), " ".join(x[:10].rjust(10) for x in libs))
for k, v in d.items():
    b = min(v[libs[0]])
    print(str(k).ljust(26), " ".join(f"{min(v[x]):6.2f}{b / min(v[x]):5.3f}"[:10].rjust(10) if v[x] else " " * 10 for x in libs))
