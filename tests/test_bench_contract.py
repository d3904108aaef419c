"""The bench.py output contract (one JSON line with the driver's keys).
The reference arm (CPU oracle port) runs here; the GPU arm in -m gpu."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, env=env, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "3"], {"QSG_BENCH_CPU_SAMPLE": "16"})
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "frames/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = _run(["--steps", "1", "--warmup", "3"], {"QSG_BENCH_FRAMES": "16384", "QSG_BENCH_CPU_SAMPLE": "32"})
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["gpu_launches"] == 35 and d["value"] > 0 and d["n_gpus"] == 1
    r = d["roofline"]
    # frac is achieved / peak of the same line; peak = 148 SMs x 128 x the
    # sampled SM clock; a 16k-frame point still keeps the SMs busy enough
    # for a third of the full-size figure
    assert r["bound"] == "issue" and r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-12)
    assert r["peak"] == pytest.approx(148 * 128 * d["clocks"]["sm_mhz"] * 1e6 / 1e9, rel=1e-9)
    assert 0.3 < r["frac"] < 1.3 and 0.5 < r["share_of_step"] < 1.0
    # hardware counters only from a capture of this very build
    assert r["ncu_build_match"] == (r["ncu_build_id"] == r["build_id"])
    if not r["ncu_build_match"]:
        assert r["ncu_issue_slots_busy"] is None and r["traffic"] is None
    b = d["roofline_bp4"]["fp32_pipe"]
    assert b["frac"] == pytest.approx(b["achieved"] / b["peak"], rel=1e-12) and 0.2 < b["frac"] < 1.0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["value"] > 0 and d["parity"].startswith("35/35")
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


@pytest.mark.gpu
def test_gpu_arm_two_ranks_on_one_gpu():
    """The N > 1 code path of bench.py (sharded frames, counter all-reduce,
    max-over-ranks timing, e2e on every rank) under torchrun with 2 ranks.
    The pool has one GPU per box, so both ranks share it and talk over gloo
    (QSG_BENCH_BACKEND); the N-GPU driver run uses NCCL."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, QSG_BENCH_FRAMES="16384", QSG_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--steps", "1", "--warmup", "3", "--no-cpu"],
                         capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["frames_per_step"] == 2 * 35 * 16384
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and "cpu_baseline" not in d


@pytest.mark.gpu
def test_gpu_arm_self_spawns_ranks():
    """`python bench.py --gpus 2` without a torchrun environment re-executes
    itself under torch.distributed.run with 2 local ranks (the driver may
    launch either way).  On this one-GPU pool both ranks share cuda:0 and
    use gloo; the line reports both ranks and the strong-scaling config-5
    leg sharded over them."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                              "MASTER_PORT")}
    env.update(QSG_BENCH_FRAMES="16384", QSG_BENCH_C5_FRAMES="65536", QSG_BENCH_BACKEND="gloo")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                          "--warmup", "3", "--no-cpu"], capture_output=True, text=True, env=env, timeout=900,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["frames_per_step"] == 2 * 35 * 16384
    c5 = d["strong_config5"]
    assert c5["n_gpus"] == 2 and c5["scaling"] == "strong" and c5["frames_per_step"] == 4 * 65536
    assert all(pt["frames"] == 65536 for pt in c5["points"])
