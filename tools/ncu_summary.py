"""Summarise an ncu report: SOL, issue, pipes, occupancy, smem conflicts,
and the SASS opcode mix / hottest regions (dev tool; output goes to
profiles/)."""
import collections
import csv
import io
import subprocess
import sys


def run(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    out = []
    det = list(csv.reader(io.StringIO(run(rep, "--page", "details", "--csv"))))
    hdr = det[0]
    keep = ("Duration", "SM Frequency", "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active",
            "Achieved Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Block Size",
            "Grid Size", "Theoretical Occupancy", "Eligible Warps Per Scheduler", "No Eligible",
            "DRAM Throughput", "L1/TEX Cache Throughput", "Warp Cycles Per Issued Instruction")
    for row in det[1:]:
        d = dict(zip(hdr, row))
        if d.get("Metric Name") in keep:
            out.append(f"{d['Metric Name']:40s} {d['Metric Value']:>16s} {d['Metric Unit']}")
    raw = list(csv.reader(io.StringIO(run(rep, "--page", "raw", "--csv"))))
    rh, ru, rv = raw[0], raw[1], raw[2]
    for h, u, v in zip(rh, ru, rv):
        if h in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                 "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                 "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                 "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "gpu__time_duration.sum"):
            out.append(f"{h:60s} {v:>16s} {u}")
    sass = list(csv.reader(io.StringIO(run(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    sh = sass[1]
    ia, isrc = sh.index("Instructions Executed"), sh.index("Source")
    tot, byop = 0, collections.Counter()
    for r in sass[2:]:
        try:
            n = int(r[ia] or 0)
        except ValueError:
            continue
        toks = r[isrc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        byop[op.split(".")[0]] += n
        tot += n
    out.append(f"warp-level instructions executed: {tot}")
    for op, n in byop.most_common(24):
        out.append(f"  {op:10s} {n:14d} {100 * n / tot:5.1f}%")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
