"""Benchmark of the GB-QLDPC decode hot path (BASELINE.json configs[1]).

One step = one full pass of BASELINE configs[1] on every GPU: the [[254,28]]
GB code, p in {0.02, 0.04, 0.06, 0.08, 0.10} x {BP4, SMS alpha in {0.5,
0.625, 0.75, 0.875, 1.0}, SAGMS (0.30, 0.50, 1.10)}, 2^20 frames per point
per GPU, l_max 100, fp32 messages, marginal qubit update, seed 0.  Frames are
sampled on device (Philox keyed by (seed, frame), bit-identical to the
reference's sample_error), decoded by the persistent sm_100a kernel, and the
per-point counters {frames, failures, sum iterations, CN-edge updates} are
summed over ranks with one NCCL all-reduce per point.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the CPU oracle port (oracle/, the reference's
algorithm restated in C, all host threads) on a bounded sample of the same
workload (the first frames of every point).

Every run also measures the north-star scaling workload, BASELINE configs[4]
(`strong_config5` in the JSON line): [[254,28]] and the random l=511 w=5 GB
code, SAGMS, p in {0.03, 0.08}, l_max 100, a FIXED 2^22 frames per point
sharded contiguously over the N ranks (strong scaling), the four points
launched back to back with ONE all-reduce of the counter block at the end
and no host synchronisation in between.

With --gpus N > 1 and no torchrun environment (WORLD_SIZE unset) the script
re-executes itself under torch.distributed.run with N local ranks
(rendezvous on 127.0.0.1).  NCCL's init log (NCCL_DEBUG=INFO,
NCCL_DEBUG_SUBSYS=INIT unless set) records the communicator's rank count.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CODE = (127, (0, 15, 20, 28, 66), (0, 58, 59, 100, 121))
PS = (0.02, 0.04, 0.06, 0.08, 0.10)
SMS_ALPHAS = (0.5, 0.625, 0.75, 0.875, 1.0)
FRAMES_PER_POINT = int(os.environ.get("QSG_BENCH_FRAMES", 1 << 20))  # override: tests only
L_MAX = 100
SEED = 0
CPU_SAMPLE_FRAMES = int(os.environ.get("QSG_BENCH_CPU_SAMPLE", 1024))  # per point, for the CPU legs
METRIC = "decoded frames/s and CN-edge updates/s per GPU & 8×B200 (% roofline), FER match"
# Algorithmic ops per CN-edge update: ALU + MUFU-class
# ops of the reference algorithm, the numerator of roofline.achieved.
OPS_PER_EDGE = {"sagms": 30.3 + 4, "sms": 30.0 + 4, "ms": 29.0 + 4, "bp4": 34.1 + 10}
# FP32-pipe lane operations per BP4 CN-edge update of the fp32 recipe
# (check side 36.6: exponential 11, prefix/suffix 3.6, merge 4, reciprocal 3
# (its MUFU seed runs on the XU pipe), ratio 1, logarithm 14; qubit side 10.0
# per edge: 14 sum / belief adds, 2 x 37 for the factor pair, 2 + 10 output
# adds per 10 edges); DESIGN.md section 5
BP4_FP32_OPS = 46.6


# BASELINE configs[4] (strong scaling): GbSpec args, p values, total frames per point
C5_CODES = (("[[254,28]]", CODE), ("l511w5", (511, (0, 5, 200, 397, 418), (0, 81, 284, 347, 418))))
C5_PS = (0.03, 0.08)
C5_FRAMES = int(os.environ.get("QSG_BENCH_C5_FRAMES", 1 << 22))  # override: tests only


def decoders(P):
    out = [("bp4", P.DecoderConfig("bp4", l_max=L_MAX))]
    out += [(f"sms{a}", P.DecoderConfig("sms", l_max=L_MAX, alpha=a)) for a in SMS_ALPHAS]
    out.append(("sagms", P.DecoderConfig("sagms", l_max=L_MAX, gain=P.GainParams(0.30, 0.50, 1.10))))
    return out


def workload_desc():
    return ("configs[1]: [[254,28]] GB (l=127) sweep p in {0.02,0.04,0.06,0.08,0.10} x "
            "{BP4, SMS a in {0.5,0.625,0.75,0.875,1.0}, SAGMS(0.30,0.50,1.10)}, "
            + ("2^20" if FRAMES_PER_POINT == 1 << 20 else str(FRAMES_PER_POINT))
            + " frames/point/GPU, l_max=100, fp32, marginal VN, seed 0")


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_leg(P_or_none, steps, warmup, nthreads):
    """The oracle port on a bounded sample: first CPU_SAMPLE_FRAMES frames of
    every point.  Returns (frames/s, cn_updates/s, per-point outcomes, wall)."""
    from oracle import oracle as O
    g = O.gb_graph(*CODE)
    cfgs = _plain_decoders()
    outcomes = {}
    frames = upd = 0
    t0 = time.perf_counter()
    for p in PS:
        for name, cfg in cfgs:
            f, it, _, cnt = O.frames(g, cfg, p, p, SEED, 0, CPU_SAMPLE_FRAMES, nthreads=nthreads)
            outcomes[(name, p)] = (f, it)
            frames += int(cnt[0])
            upd += int(cnt[3])
    wall = time.perf_counter() - t0
    return frames / wall, upd / wall, outcomes, wall, frames


def _plain_decoders():
    """Decoder configs without importing the GPU package (reference arm)."""
    from types import SimpleNamespace as NS
    gain = NS(alpha_min=0.30, alpha_max=0.50, eta_unsat=1.10)
    out = [("bp4", NS(variant="bp4", l_max=L_MAX, alpha=None, gain=None, vn_mode="marginal"))]
    out += [(f"sms{a}", NS(variant="sms", l_max=L_MAX, alpha=a, gain=None, vn_mode="marginal"))
            for a in SMS_ALPHAS]
    out.append(("sagms", NS(variant="sagms", l_max=L_MAX, alpha=None, gain=gain, vn_mode="marginal")))
    return out


def run_reference(args, rank):
    if rank != 0:
        return
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    nthreads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_leg(None, 1, 0, nthreads)
    vals, upds, walls, frames = [], [], [], 0
    for _ in range(args.steps):
        v, u, _, wall, fr = cpu_leg(None, 1, 0, nthreads)
        vals.append(v); upds.append(u); walls.append(wall); frames = fr
    value = sum(frames for _ in vals) / sum(walls)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(walls) / len(walls), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (Philox frames, seed 0)",
        "config": {"workload": workload_desc(), "sample": f"first {CPU_SAMPLE_FRAMES} frames of each "
                   "of the 35 points per step", "frames_per_step": frames},
        "cn_edge_updates_per_s": sum(u * w for u, w in zip(upds, walls)) / sum(walls),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": nthreads, "kind": "port",
                         "sample": f"{frames} frames/step: first {CPU_SAMPLE_FRAMES} frames of each of "
                                   "the 35 (decoder, p) points; oracle/qsg_oracle.c fp32, pthreads"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def flush_l2(buf):
    buf.fill_(1)


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_10433_b200 as P

    dev_index = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    g = P.gb_graph(P.GbSpec(*CODE))
    dg = P.device_graph(g, dev)
    decs = decoders(P)
    points = [(name, cfg, p) for p in PS for name, cfg in decs]
    base = rank * FRAMES_PER_POINT
    counters = torch.zeros((len(points), 4), dtype=torch.int64, device=dev)
    l2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step(record=None):
        counters.zero_()
        for k, (name, cfg, p) in enumerate(points):
            if record is not None:
                record[k][0].record()
            P.decode_frames_device(dg, cfg, p, p, SEED, base, FRAMES_PER_POINT, counters=counters[k],
                                   want_frames=False)
            if record is not None:
                record[k][1].record()
        if world > 1:
            dist.all_reduce(counters)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, launch_ms = [], [[0.0, 0.0] for _ in points]
    sampler = ClockSampler(dev_index)
    with sampler:
        for _ in range(args.steps):
            flush_l2(l2)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in points]
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            step(ev)
            s1.record()
            torch.cuda.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            for k in range(len(points)):
                launch_ms[k][0] += ev[k][0].elapsed_time(ev[k][1])
        # a timed region shorter than nvidia-smi's start-up plus one sampling
        # period (reduced test workloads) would leave no clock sample: keep
        # the same load running, untimed, until the first sample arrives
        # (single rank only: step() holds a collective when world > 1)
        t_wait = time.perf_counter()
        while world == 1 and not sampler.lines and sampler.proc and time.perf_counter() - t_wait < 5.0:
            step()
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    cnt = counters.cpu().numpy()  # last step, already summed over ranks
    frames_step = int(cnt[:, 0].sum())
    upd_step = int(cnt[:, 3].sum())
    value = frames_step * args.steps / (total_ms / 1e3)
    clocks = sampler.summary()

    # ---- e2e through the public API with host inputs, every rank ----
    # Inputs: the step's syndromes (uint8, one byte per check -- the
    # reference decode_batch format), generated once outside the timed region
    # and held in pinned host memory; every timed step copies them H2D,
    # decodes (decode_batch_device), and reads success + iterations back.
    from paper_2605_10433_b200 import _native

    def host_syndromes(p):
        e = P.sample_errors_device(g.n, p, SEED, base, FRAMES_PER_POINT, device=dev)
        syn = torch.empty((FRAMES_PER_POINT, g.m), dtype=torch.uint8, device=dev)
        _native.check(_native.lib().qsg_syndromes_of(dg.handle, e.data_ptr(), FRAMES_PER_POINT, syn.data_ptr(),
                                                     torch.cuda.current_stream(dev).cuda_stream))
        del e
        # bit-pack (setup only): distinct bits, so an int32 sum is an OR
        nwd = (g.m + 31) // 32
        shifts = torch.arange(32, dtype=torch.int32, device=dev)
        words = torch.empty((FRAMES_PER_POINT, nwd), dtype=torch.int32, device=dev)
        for c0 in range(0, FRAMES_PER_POINT, 1 << 17):
            pad = torch.zeros((min(1 << 17, FRAMES_PER_POINT - c0), nwd * 32), dtype=torch.int32, device=dev)
            pad[:, :g.m] = syn[c0:c0 + pad.shape[0]]
            words[c0:c0 + pad.shape[0]] = (pad.view(pad.shape[0], nwd, 32) << shifts).sum(-1, dtype=torch.int32)
        h_syn = torch.empty(syn.shape, dtype=torch.uint8, pin_memory=True)
        h_words = torch.empty(words.shape, dtype=torch.int32, pin_memory=True)
        h_syn.copy_(syn)
        h_words.copy_(words)
        return h_syn, h_words

    hosts = {p: host_syndromes(p) for p in PS}
    h_out = torch.empty((len(points), 9 * FRAMES_PER_POINT), dtype=torch.uint8, pin_memory=True)

    h_outs = [(h_out[k, 8 * FRAMES_PER_POINT:], h_out[k, : 8 * FRAMES_PER_POINT].view(torch.int64))
              for k in range(len(points))]

    def e2e_run(packed):
        # decode_host_batches: H2D of point k+1 overlaps the decode of point k
        # (side stream, double buffer); results land in pinned host memory
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        batches = [P.HostBatch(hosts[p][1] if packed else hosts[p][0], P.prior_llr(p).llr, cfg, packed=packed)
                   for name, cfg, p in points]
        P.decode_host_batches(dg, batches, device=dev, outputs=h_outs)
        ms = (time.perf_counter() - t0) * 1e3
        h2d = sum(b.syndromes.numel() * b.syndromes.element_size() for b in batches)
        d2h = 9 * FRAMES_PER_POINT * len(points)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, h2d, d2h

    # the _decode_frames drop-in (inputs are (seed, start, count) only; one
    # untimed pass, then the median of up to 3)
    def frames_run():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for name, cfg, p in points:
            P.decode_frames(dg, cfg, p, p, SEED, base, FRAMES_PER_POINT)
        return (time.perf_counter() - t0) * 1e3

    frames_run()
    frames_ms = statistics.median(frames_run() for _ in range(max(1, min(args.steps, 3))))
    e2e_run(False)  # untimed: first-touch of the pinned outputs and device buffers
    e2e_runs = [e2e_run(False) for _ in range(max(1, args.steps))]
    e2e_ms = statistics.median(r[0] for r in e2e_runs)
    e2e_value = frames_step / (e2e_ms / 1e3)
    e2e_h2d, e2e_d2h = e2e_runs[0][1] * world, e2e_runs[0][2] * world
    packed_runs = [e2e_run(True) for _ in range(max(1, min(args.steps, 3)))]
    packed_ms = statistics.median(r[0] for r in packed_runs)
    # the e2e decodes must agree with the device-timed step (same frames)
    if world == 1:
        assert int(h_out[:, 8 * FRAMES_PER_POINT:].sum()) == int(cnt[:, 0].sum() - cnt[:, 1].sum())

    c5 = strong_config5(args, rank, world, dev, l2)
    if rank != 0:
        return
    fer_check = fer_criterion(P, dg, points, dev)
    # ---- roofline of the dominant kernel (min-sum marginal, bicycle W=5) ----
    mins = [k for k, (name, _, _) in enumerate(points) if name != "bp4"]
    ms_mins = sum(launch_ms[k][0] for k in mins) / args.steps
    ops = sum(cnt[k, 3] / world * OPS_PER_EDGE["sagms" if points[k][0] == "sagms" else "sms"]
              for k in mins)
    f_sm = (clocks["sm_mhz"] or 1965.0) * 1e6
    peak = dg_sms() * 128 * f_sm
    achieved = ops / (ms_mins / 1e3)
    # hardware counters of the committed ncu capture, used only when it was
    # taken on THIS build (qsg_build_id(): hash of the kernel sources and flags)
    traffic = issue_busy = None
    bp4_hw = {}
    tj = {}
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tj = json.load(fh)
    build_id = P._native.lib().qsg_build_id().decode()
    ncu_match = tj.get("build_id") == build_id
    if ncu_match:
        traffic = tj.get("bytes_per_launch")
        issue_busy = tj.get("issue_slots_busy")
        bp4_hw = tj.get("bp4", {})
    share = ms_mins / (sum(l[0] for l in launch_ms) / args.steps)
    # the BP4 launches (the rest of the step): against the same issue roof
    # (SURVEY 8(d)'s 44.1 ops per edge) and against the pipe that binds them,
    # the FP32 pipe (ncu: math-pipe throttle is their top stall): the fp32
    # recipe performs BP4_FP32_OPS FP32-pipe lane operations per CN-edge
    # update, peak 128 per SM per clock
    bp4s = [k for k, (name, _, _) in enumerate(points) if name == "bp4"]
    ms_bp4 = sum(launch_ms[k][0] for k in bp4s) / args.steps
    upd_bp4 = sum(cnt[k, 3] / world for k in bp4s)
    bp4_rate = upd_bp4 / (ms_bp4 / 1e3)
    bp4_line = {"achieved": bp4_rate * OPS_PER_EDGE["bp4"] / 1e9, "peak": peak / 1e9,
                "unit": "Gop/s", "frac": bp4_rate * OPS_PER_EDGE["bp4"] / peak,
                "cn_edge_updates_per_s": bp4_rate,
                "fp32_pipe": {"bound": "fp32 pipe", "ops_per_cn_edge_update": BP4_FP32_OPS,
                              "achieved": bp4_rate * BP4_FP32_OPS / 1e9, "peak": peak / 1e9, "unit": "Gop/s",
                              "frac": bp4_rate * BP4_FP32_OPS / peak,
                              "ncu_fma_pipe_cycles_active": bp4_hw.get("fma_pipe_cycles_active"),
                              "ncu_issue_slots_busy": bp4_hw.get("issue_slots_busy")},
                "kernel": "qsg::decode_kernel<5,32,true,false,256,lean> (BP4, marginal VN)",
                "share_of_step": ms_bp4 / (sum(l[0] for l in launch_ms) / args.steps)}

    # ---- CPU baseline on a bounded sample + per-frame parity on that sample ----
    cpu = {}
    parity = None
    if world == 1 and not args.no_cpu:
        nthreads = os.cpu_count() or 1
        v, u, outcomes, wall, fr = cpu_leg(None, 1, 0, nthreads)
        cpu = {"value": v, "unit": "frames/s", "cores": nthreads, "kind": "port",
               "sample": f"{fr} frames: first {CPU_SAMPLE_FRAMES} frames of each of the 35 "
                         "(decoder, p) points; oracle/qsg_oracle.c fp32, pthreads",
               "cn_edge_updates_per_s": u, "wall_s": wall}
        same = 0
        for name, cfg, p in points:
            f, it = P.decode_frames(dg, cfg, p, p, SEED, 0, CPU_SAMPLE_FRAMES)
            of, oit = outcomes[(name, p)]
            same += int(np.array_equal(f, of) and np.array_equal(it, oit))
        parity = f"{same}/{len(points)} points bit-exact vs oracle on the CPU sample"

    fer = {f"{name}@{p}": round(float(cnt[k, 1] / cnt[k, 0]), 6) for k, (name, _, p) in enumerate(points)
           if name in ("sagms", "bp4", "sms0.75")}
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (on-device Philox frames keyed (seed 0, frame), reference sampler)",
        "config": {"workload": workload_desc(), "points": len(points),
                   "frames_per_point_per_gpu": FRAMES_PER_POINT, "frames_per_step": frames_step,
                   "l2": "flushed (256 MiB device write) before every timed step",
                   "parallelism": f"dp{world} (contiguous frame shards, NCCL all-reduce of counters per point)"},
        "cn_edge_updates_per_s": upd_step * args.steps / (total_ms / 1e3),
        "mean_iterations": float(cnt[:, 2].sum() / cnt[:, 0].sum()),
        "gpu_launches": len(points) * args.steps,
        "roofline": {"bound": "issue", "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "Gop/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "qsg::decode_kernel<5,32,false,false,256,lean> (min-sum family, marginal VN, n_pad 256)",
                     "ops_per_cn_edge_update": "SURVEY.md 8(d): SAGMS 34.3, SMS 34.0",
                     "peak_basis": "148 SMs x 128 lane-instr/clk x measured median SM clock",
                     "share_of_step": share,
                     "ncu_issue_slots_busy": issue_busy,
                     "ncu_build_id": tj.get("build_id"), "build_id": build_id, "ncu_build_match": ncu_match},
        "roofline_bp4": bp4_line,
        "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": int(e2e_h2d),
                "d2h_bytes_per_step": int(e2e_d2h),
                "api": "decode_host_batches: uint8 syndromes (reference decode_batch format) in pinned host "
                       "memory -> device (H2D of point k+1 overlapping the decode of point k) -> success + "
                       "iterations back to pinned host, every point of the step"},
        "e2e_packed": {"value": frames_step / (packed_ms / 1e3), "unit": "frames/s",
                       "h2d_bytes_per_step": int(packed_runs[0][1] * world),
                       "d2h_bytes_per_step": int(packed_runs[0][2] * world),
                       "api": "decode_host_batches(packed): bit-packed syndromes (32 B/frame)"},
        "e2e_frames": {"value": frames_step / world / (frames_ms / 1e3) * world, "unit": "frames/s",
                       "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 9 * FRAMES_PER_POINT * len(points) * world,
                       "api": "decode_frames, the qsagms.harness._decode_frames drop-in (inputs are seed/start/count; "
                              "sampling is part of the path)"},
        "clocks": clocks,
        "fer": fer,
    }
    line["strong_config5"] = c5
    if fer_check:
        line["fer_check"] = fer_check
    if cpu:
        line["cpu_baseline"] = cpu
    if parity:
        line["parity"] = parity
    print(json.dumps(line), flush=True)


def fer_criterion(P, dg, points, dev):
    """north_star's FER criterion inside the bench run (untimed): every
    configs[1] point decoded on the frames [0, F) of the committed float64
    reference counts (tests/golden/fer64_config2.json: the reference's fp64
    arithmetic on the same Philox frames, F = 2^20 where available); the GPU
    FER must lie inside the reference's 95% Wilson interval
    (harness.py:102-125)."""
    import torch
    path = os.path.join(ROOT, "tests", "golden", "fer64_config2.json")
    if not os.path.exists(path) or FRAMES_PER_POINT != 1 << 20:
        return None
    with open(path) as fh:
        ref = json.load(fh)["points"]
    cnt = torch.zeros((len(points), 4), dtype=torch.int64, device=dev)
    for k, (name, cfg, p) in enumerate(points):
        P.decode_frames_device(dg, cfg, p, p, SEED, 0, ref[f"{name}@{p}"]["frames"], counters=cnt[k],
                               want_frames=False)
    c = cnt.cpu().numpy()
    inside, rows, worst = 0, 0, None
    for k, (name, cfg, p) in enumerate(points):
        r = ref[f"{name}@{p}"]
        n, fg, fo = int(c[k, 0]), int(c[k, 1]), r["ref64_failures"]
        assert n == r["frames"]
        lo, hi = P.wilson_interval(fo, n)
        ok = lo <= fg / n <= hi
        inside += int(ok)
        rows += 1
        # distance from the reference FER in units of the interval's half-width
        d = abs(fg - fo) / max(1e-300, n * (hi - lo) / 2)
        if worst is None or d > worst["half_widths"]:
            worst = {"point": f"{name}@{p}", "frames": n, "gpu_failures": fg, "ref64_failures": fo,
                     "ref64_wilson95": [lo, hi], "half_widths": round(d, 3)}
    return {"points": rows, "inside_ref64_wilson95": inside, "all_inside": inside == rows,
            "frames_per_point": sorted({v["frames"] for v in ref.values()}), "worst": worst,
            "reference": "tests/golden/fer64_config2.json: the reference's float64 arithmetic on the same frames"}


def strong_config5(args, rank, world, dev, l2):
    """BASELINE configs[4]: a fixed 2^22 frames per point, sharded over the
    ranks; all four points back to back, one all-reduce, max over ranks.
    On one GPU also a proxy of the 8-GPU step: each of the 8 shards of every
    point timed alone (CUDA events), the step of the slowest shard summed over
    the points -> t(2^22) / (8 x max-shard time)."""
    import torch
    import torch.distributed as dist

    import paper_2605_10433_b200 as P
    from paper_2605_10433_b200.dist import shard_range
    cfg = P.DecoderConfig("sagms", l_max=L_MAX, gain=P.GainParams(0.30, 0.50, 1.10))
    pts = []
    for cname, spec in C5_CODES:
        dg = P.device_graph(P.gb_graph(P.GbSpec(*spec)), dev)
        for p in C5_PS:
            pts.append((cname, dg, p))
    lo, n = shard_range(rank, world, 0, C5_FRAMES)
    cnt = torch.zeros((len(pts), 4), dtype=torch.int64, device=dev)

    def step():
        cnt.zero_()
        for k, (_, dg, p) in enumerate(pts):
            P.decode_frames_device(dg, cfg, p, p, SEED, lo, n, counters=cnt[k], want_frames=False)
        if world > 1:
            dist.all_reduce(cnt)

    for _ in range(max(1, args.warmup)):
        step()
    times = []
    for _ in range(args.steps):
        flush_l2(l2)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    t = torch.tensor(times, dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.mean())
    c = cnt.cpu().numpy()
    frames = int(c[:, 0].sum())
    out = {"value": frames / (ms / 1e3), "unit": "frames/s", "scaling": "strong", "n_gpus": world,
           "ms_per_step": ms, "frames_per_step": frames,
           "cn_edge_updates_per_s": float(c[:, 3].sum()) / (ms / 1e3),
           "workload": "configs[4]: [[254,28]] + random GB l=511 w=5 (seed 0), SAGMS(0.30,0.50,1.10), "
                       "p in {0.03,0.08}, l_max 100, 2^22 frames/point in total sharded over the ranks, "
                       "4 points back to back + one NCCL all-reduce per step, max over ranks",
           "points": [{"code": cname, "p": p, "frames": int(c[k, 0]), "failures": int(c[k, 1]),
                       "fer": float(c[k, 1] / max(1, c[k, 0])), "mean_iterations": float(c[k, 2] / max(1, c[k, 0]))}
                      for k, (cname, _, p) in enumerate(pts)]}
    if world == 1:
        # one-GPU proxy of the 8-way split: shard r of 8 of every point alone
        shard_ms = [[0.0] * len(pts) for _ in range(8)]
        for rep in range(2):  # first pass warms each shard's launch
            for r in range(8):
                slo, sn = shard_range(r, 8, 0, C5_FRAMES)
                for k, (_, dg, p) in enumerate(pts):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    P.decode_frames_device(dg, cfg, p, p, SEED, slo, sn, counters=None, want_frames=False)
                    e1.record()
                    torch.cuda.synchronize()
                    if rep:
                        shard_ms[r][k] = e0.elapsed_time(e1)
        per_rank = [sum(x) for x in shard_ms]
        # and per point: t(2^22 frames) / (8 x slowest 2^19-frame shard)
        full_ms = []
        for k, (_, dg, p) in enumerate(pts):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            P.decode_frames_device(dg, cfg, p, p, SEED, 0, C5_FRAMES, counters=None, want_frames=False)
            e1.record()
            torch.cuda.synchronize()
            full_ms.append(e0.elapsed_time(e1))
        out["proxy_8way"] = {
            "shard_ms_max_over_8": max(per_rank), "shard_ms_min_over_8": min(per_rank),
            "efficiency": ms / (8 * max(per_rank)),
            "per_point": [{"code": cname, "p": p, "full_ms": full_ms[k],
                           "shard_ms_max": max(shard_ms[r][k] for r in range(8)),
                           "efficiency": full_ms[k] / (8 * max(shard_ms[r][k] for r in range(8)))}
                          for k, (cname, _, p) in enumerate(pts)],
            "note": "t(2^22 frames on 1 GPU) / (8 x slowest 1/8 shard timed alone): the strong-scaling "
                    "efficiency an 8-GPU run would reach with zero collective cost"}
    return out


def dg_sms():
    import torch
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def spawn(n):
    """Re-execute this script under torch.distributed.run with n local ranks
    (one process per GPU), rendezvous on 127.0.0.1 at a free port."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execve(sys.executable, cmd, env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn(args.gpus)  # does not return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        dev_index = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(dev_index)
        # QSG_BENCH_BACKEND=gloo exercises the multi-rank logic on one GPU
        backend = os.environ.get("QSG_BENCH_BACKEND", "nccl")
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init log: nranks visible
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
