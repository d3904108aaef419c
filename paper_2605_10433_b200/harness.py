"""Monte-Carlo FER loop on the GPU (mirrors pkg/src/qsagms/harness.py).

``decode_frames`` is the drop-in replacement of the reference's FER-loop
unit ``_decode_frames`` (harness.py:172-182): the reference resolves that
function by module-global name at call time (harness.py:207-213), so
``install(qsagms.harness)`` makes the reference's own ``run_point`` /
``run_sweep`` / CLI decode on the GPU.  ``run_point`` / ``run_sweep`` here
reproduce the reference protocol (ordered stop rule, Wilson interval,
digest, resumable JSON/TSV artifacts) with large device batches; batching
never changes results because frame f is keyed by (seed, f).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import logging
import math
from dataclasses import asdict, dataclass
from pathlib import Path
from statistics import NormalDist

import numpy as np
import torch

from . import __version__, _native
from .device import decoder_cfg_struct, device_graph, ptr, stream_ptr

log = logging.getLogger("paper_2605_10433_b200.harness")

#: Frames per device launch in run_point (results do not depend on it).
GPU_BATCH_FRAMES = 1 << 20


def decode_frames_device(graph, decoder_cfg, epsilon, epsilon0, seed, start, count, *,
                         counters: torch.Tensor | None = None, want_frames: bool = True,
                         want_ehat: bool = False, device=None):
    """Sample, decode and summarise frames [start, start+count) on the GPU.

    Returns device tensors (fails uint8, iterations int64, e_hat uint8 or
    None).  ``counters`` (int64[4] on the device) accumulates {frames,
    failures, sum iterations, sum CN-edge updates} without a host sync.
    """
    dg = device_graph(graph, device)
    dev = dg.device
    fails = torch.empty(count, dtype=torch.uint8, device=dev) if want_frames else None
    iters = torch.empty(count, dtype=torch.int64, device=dev) if want_frames else None
    ehat = torch.empty((count, dg.n), dtype=torch.uint8, device=dev) if want_ehat else None
    c = decoder_cfg_struct(decoder_cfg, True)
    _native.check(_native.lib().qsg_decode_frames(
        dg.handle, C.byref(c), float(epsilon), float(epsilon0), int(seed) & (2**64 - 1),
        int(start), int(count), ptr(fails), ptr(iters), ptr(ehat), ptr(counters), stream_ptr(dev)))
    return fails, iters, ehat


_PINNED: dict = {}


def _pinned(nbytes: int) -> torch.Tensor:
    """Grow-only pinned host staging buffer (one per thread and device)."""
    import threading
    key = (threading.get_ident(), torch.cuda.current_device())
    buf = _PINNED.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        _PINNED[key] = buf
    return buf


def decode_frames(graph, decoder_cfg, epsilon, epsilon0, seed, start, count):
    """Drop-in for ``qsagms.harness._decode_frames``: returns numpy
    (fails bool[count], iterations int64[count]).  Results come back through
    a pinned staging buffer with one stream synchronisation."""
    fails, iters, _ = decode_frames_device(graph, decoder_cfg, epsilon, epsilon0, seed, start, count)
    stage = _pinned(9 * count)
    it_h = stage[: 8 * count].view(torch.int64)
    f_h = stage[8 * count: 9 * count]
    it_h.copy_(iters, non_blocking=True)
    f_h.copy_(fails, non_blocking=True)
    torch.cuda.current_stream(iters.device).synchronize()
    return f_h.numpy().astype(bool), it_h.numpy().copy()


def install(harness_module, batch_frames: int | None = 1 << 20) -> None:
    """Route a reference harness module's FER loop through the GPU, e.g.
    ``install(qsagms.harness)``; run it with workers=1 (the GPU is the
    parallelism).

    ``batch_frames`` also sets the harness's ``BATCH_FRAMES`` (4096 by
    default, harness.py:40-41: "has no effect on results, only on
    scheduling"): a 4096-frame call is latency-bound on the GPU by its
    slowest (l_max-iteration) frame, 2^20 frames fill all 148 SMs.  None
    leaves it unchanged."""
    harness_module._decode_frames = globals()["decode_frames"]
    if batch_frames is not None and hasattr(harness_module, "BATCH_FRAMES"):
        harness_module.BATCH_FRAMES = int(batch_frames)


# -- protocol (harness.py:44-158, 248-356) ----------------------------------------

@dataclass(frozen=True)
class SweepConfig:
    code_id: str
    decoder: object
    epsilon_list: tuple[float, ...]
    seed: int
    epsilon0_mode: str = "matched"
    epsilon0: float | None = None
    target_failures: int = 500
    max_frames: int = 20_000_000
    workers: int = 1

    def __post_init__(self):
        if self.epsilon0_mode not in ("matched", "fixed"):
            raise ValueError("epsilon0_mode must be 'matched' or 'fixed'")
        if self.epsilon0_mode == "fixed" and self.epsilon0 is None:
            raise ValueError("fixed mode needs epsilon0")
        if not self.epsilon_list:
            raise ValueError("epsilon_list is empty")
        if any(not 0.0 < e < 1.0 for e in self.epsilon_list):
            raise ValueError("epsilon values must lie in (0, 1)")
        if self.target_failures < 1:
            raise ValueError("target_failures must be at least 1")
        if self.max_frames < 1:
            raise ValueError("max_frames must be at least 1")
        if self.workers < 1:
            raise ValueError("workers must be at least 1")


@dataclass(frozen=True)
class FerPoint:
    epsilon: float
    epsilon0: float
    frames: int
    failures: int
    fer: float
    wilson_low: float
    wilson_high: float
    mean_iterations: float
    cap_hit: bool
    config_digest: str
    seed: int


WILSON_Z_95 = 1.959964


def wilson_interval(failures: int, frames: int, confidence: float = 0.95) -> tuple[float, float]:
    """Wilson score interval clamped to [0, 1] and containing the estimate
    (harness.py:102-125)."""
    if frames < 1:
        raise ValueError("frames must be at least 1")
    if not 0 <= failures <= frames:
        raise ValueError("failures must lie in [0, frames]")
    z = WILSON_Z_95 if confidence == 0.95 else NormalDist().inv_cdf(0.5 + confidence / 2.0)
    n = float(frames)
    p = failures / n
    denom = 1.0 + z * z / n
    center = (p + z * z / (2.0 * n)) / denom
    half = z * math.sqrt(p * (1.0 - p) / n + z * z / (4.0 * n * n)) / denom
    return max(0.0, min(float(center - half), p)), min(1.0, max(float(center + half), p))


def canonical_json(obj) -> str:
    """Sorted keys, floats at 17 significant digits (harness.py:128-147)."""
    if isinstance(obj, dict):
        return "{" + ", ".join(f"{json.dumps(k)}: {canonical_json(v)}" for k, v in sorted(obj.items())) + "}"
    if isinstance(obj, (list, tuple)):
        return "[" + ", ".join(canonical_json(v) for v in obj) + "]"
    if isinstance(obj, bool) or obj is None:
        return json.dumps(obj)
    if isinstance(obj, float):
        return format(obj, ".17g")
    if isinstance(obj, (int, str)):
        return json.dumps(obj)
    raise TypeError(f"cannot serialize {type(obj)!r}")


def _config_dict(cfg: SweepConfig) -> dict:
    d = asdict(cfg)
    d.pop("workers")
    return d


def config_digest(cfg: SweepConfig) -> str:
    return hashlib.sha256(canonical_json(_config_dict(cfg)).encode()).hexdigest()


#: Optional FER unit with the ``_decode_frames`` signature used by
#: run_point / run_sweep instead of the device pipeline (e.g. the CPU oracle
#: in the protocol tests).  None: the GPU.
FRAME_UNIT = None


def frame_batches(graph, decoder_cfg, epsilon, epsilon0, seed, stop, batch_frames):
    """Yield (fails, iterations) numpy arrays for frames [0, stop) in order,
    batch by batch, keeping the next batch's launch queued on the device
    while the current one is handed back (speculative, like the reference's
    worker pool: a consumer that stops early discards it, harness.py:200-246).
    Two persistent pinned staging buffers; one event per batch."""
    if FRAME_UNIT is not None:
        for start in range(0, stop, batch_frames):
            yield FRAME_UNIT(graph, decoder_cfg, epsilon, epsilon0, seed, start, min(batch_frames, stop - start))
        return
    dg = device_graph(graph)
    n = min(batch_frames, stop)
    stages = [torch.empty(9 * n, dtype=torch.uint8, pin_memory=True) for _ in range(2)] if n else []
    inflight = []

    def launch(start, k):
        count = min(batch_frames, stop - start)
        fails, iters, _ = decode_frames_device(dg, decoder_cfg, epsilon, epsilon0, seed, start, count)
        st = stages[k % 2]
        st[: 8 * count].view(torch.int64).copy_(iters, non_blocking=True)
        st[8 * count: 9 * count].copy_(fails, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(dg.device))
        inflight.append((ev, st, count))

    starts = list(range(0, stop, batch_frames))
    try:
        for k, start in enumerate(starts[:2]):
            launch(start, k)
        for k in range(len(starts)):
            ev, st, count = inflight.pop(0)
            ev.synchronize()
            fails = st[8 * count: 9 * count].numpy().astype(bool)
            iters = st[: 8 * count].view(torch.int64).numpy().copy()
            if k + 2 < len(starts):
                launch(starts[k + 2], k + 2)  # reuses this batch's staging buffer (already copied out)
            yield fails, iters
    finally:  # a consumer that stopped early: let the speculative copies land before the buffers go
        for ev, _, _ in inflight:
            ev.synchronize()


def run_point(graph, cfg: SweepConfig, epsilon: float, batch_frames: int = GPU_BATCH_FRAMES) -> FerPoint:
    """FER at one noise level under the ordered stop rule (harness.py:248-293):
    stop at the smallest frame index where cumulative failures reach the
    target, else at max_frames."""
    eps0 = epsilon if cfg.epsilon0_mode == "matched" else float(cfg.epsilon0)
    digest = config_digest(cfg)
    frames = failures = iter_sum = 0
    start = 0
    batches = frame_batches(graph, cfg.decoder, epsilon, eps0, cfg.seed, cfg.max_frames, batch_frames)
    for fails, iters in batches:
        count = len(fails)
        nfail = int(np.count_nonzero(fails))
        if failures + nfail >= cfg.target_failures:  # the stop frame is in this batch
            cum = np.cumsum(fails)
            stop = int(np.nonzero(failures + cum >= cfg.target_failures)[0][0]) + 1
            frames = start + stop
            failures += int(cum[stop - 1])
            iter_sum += int(iters[:stop].sum())
            break
        frames = start + count
        failures += nfail
        iter_sum += int(iters.sum())
        start += count
    batches.close()
    low, high = wilson_interval(failures, frames)
    point = FerPoint(epsilon=epsilon, epsilon0=eps0, frames=frames, failures=failures,
                     fer=failures / frames, wilson_low=low, wilson_high=high,
                     mean_iterations=iter_sum / frames, cap_hit=failures < cfg.target_failures,
                     config_digest=digest, seed=cfg.seed)
    log.info("point eps=%g fer=%g (%d/%d frames) CI=[%g, %g]%s", epsilon, point.fer, failures,
             frames, low, high, " cap-hit" if point.cap_hit else "")
    return point


def _payload(point: FerPoint, cfg: SweepConfig) -> dict:
    return {"point": asdict(point), "config": _config_dict(cfg), "version": __version__}


def _point_path(out_dir: Path, digest: str, k: int) -> Path:
    return out_dir / "points" / f"point_{digest[:12]}_{k:03d}.json"


def run_sweep(graph, cfg: SweepConfig, out_dir=None) -> list[FerPoint]:
    """Every noise point of cfg with per-point JSON reuse and aggregate
    results.json / fer.tsv (harness.py:308-356)."""
    digest = config_digest(cfg)
    out = Path(out_dir) if out_dir is not None else None
    points = []
    for k, eps in enumerate(cfg.epsilon_list):
        if out is not None:
            pf = _point_path(out, digest, k)
            if pf.exists():
                try:
                    payload = json.loads(pf.read_text(encoding="utf-8"))
                    if payload["point"]["config_digest"] == digest:
                        points.append(FerPoint(**payload["point"]))
                        continue
                except (KeyError, TypeError, ValueError) as exc:
                    raise OSError(f"unreadable point file {pf}: {exc}") from exc
        point = run_point(graph, cfg, eps)
        points.append(point)
        if out is not None:
            pf = _point_path(out, digest, k)
            pf.parent.mkdir(parents=True, exist_ok=True)
            pf.write_text(canonical_json(_payload(point, cfg)) + "\n", encoding="utf-8", newline="\n")
    if out is not None:
        out.mkdir(parents=True, exist_ok=True)
        (out / "results.json").write_text(canonical_json([_payload(p, cfg) for p in points]) + "\n",
                                          encoding="utf-8", newline="\n")
        (out / "fer.tsv").write_text("".join(f"{p.epsilon:.17g}\t{p.fer:.17g}\n"
                                             for p in sorted(points, key=lambda p: p.epsilon)),
                                     encoding="utf-8", newline="\n")
    return points
