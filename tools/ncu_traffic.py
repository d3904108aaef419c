"""Write profiles/ncu_traffic.json from one `ncu --set full` capture of the
dominant min-sum kernel and one of the BP4 kernel (dev tool).  bench.py
reports the hardware counters it holds only when its build_id equals the
running library's qsg_build_id() (tools/gpu_session.sh records the id of
the build each capture ran on).

    python tools/ncu_traffic.py MINSUM.ncu-rep BP4.ncu-rep BUILD_ID_FILE [--launch "..."]
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    vals = {}
    for h, u, v in zip(r[0], r[1], r[2]):
        try:
            vals[h] = float(v.replace(",", "")) * scale.get(u, 1.0)
        except ValueError:
            vals[h] = v
    return r[2][r[0].index("Kernel Name")], vals


def f(d, k):
    return float(d[k])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("minsum")
    ap.add_argument("bp4")
    ap.add_argument("build_id_file")
    ap.add_argument("--launch", default="tools/perf_probe.py 254 <variant> <p>, 131072 frames")
    a = ap.parse_args()
    bid = open(a.build_id_file).read().strip()
    name, m = raw(a.minsum)
    bname, b = raw(a.bp4)
    rd, wr = f(m, "dram__bytes_read.sum"), f(m, "dram__bytes_write.sum")
    out = {
        "build_id": bid,
        "kernel": name,
        "launch": a.launch,
        "report": os.path.basename(a.minsum),
        "dram_bytes_read": rd, "dram_bytes_write": wr, "bytes_per_launch": rd + wr,
        "issue_slots_busy": round(f(m, "sm__inst_issued.avg.pct_of_peak_sustained_active") / 100, 4),
        "alu_pipe": round(f(m, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active") / 100, 4),
        "lsu_pipe": round(f(m, "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active") / 100, 4),
        "fma_pipe_cycles_active": round(f(m, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active") / 100, 4),
        "bp4": {
            "kernel": bname, "report": os.path.basename(a.bp4),
            "issue_slots_busy": round(f(b, "sm__inst_issued.avg.pct_of_peak_sustained_active") / 100, 4),
            "fma_pipe_cycles_active": round(f(b, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active") / 100, 4),
            "alu_pipe": round(f(b, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active") / 100, 4),
            "dram_bytes": f(b, "dram__bytes_read.sum") + f(b, "dram__bytes_write.sum"),
        },
        "source": "ncu --set full --clock-control none --import-source on (tools/gpu_session.sh STEPS=ncu)",
        "note": "issue_slots_busy = sm__inst_issued share of SMSP issue slots; *_pipe = "
                "sm__inst_executed_pipe_* share; fma_pipe_cycles_active = sm__pipe_fma_cycles_active share",
    }
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as fh:
        json.dump(out, fh, indent=1)
        fh.write("\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
