"""List local-memory (spill) instructions of one kernel with their source
lines (dev tool).  python tools/spills.py build/csrc/qsg_inst_w5.o MANGLED_NAME"""
import os
import re
import subprocess
import sys
import tempfile

obj, fn = sys.argv[1], sys.argv[2]
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True, check=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
lines = txt.splitlines()
i = lines.index(fn + ":")
cur = None
for ln in lines[i + 1:]:
    if re.match(r"^_Z\S+:$", ln):
        break
    m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if re.search(r"\b(STL|LDL)\b", ln):
        print(cur, ln.strip()[:90])
