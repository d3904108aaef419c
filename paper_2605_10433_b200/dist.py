"""Multi-GPU FER points: one process per GPU, frames sharded contiguously.

Frame f is keyed by (seed, f), so any partition of the frame range gives
bit-identical per-frame results (reference harness.py:1-11).  Two modes:

  * ``fer_counters``: fixed frame budget (BASELINE configs 2-5).  Each rank
    decodes its shard with device-side counters and ONE all-reduce(sum) of
    int64[4] {frames, failures, sum iterations, CN-edge updates} per point
    (NCCL over NVLink; latency-bound, ~32 bytes).
  * ``run_point_sharded``: the reference's ordered stop rule
    (harness.py:262-270) across ranks.  Frames are processed in rounds of
    world x chunk; each rank decodes its contiguous sub-range, the ranks
    all-gather their (failures, sum iterations) scalars, and only the rank
    whose prefix crosses the target searches its own fail flags (on its
    device) for the stop frame and broadcasts it; frames past the stop index
    are discarded as the reference does for speculative batches.

The per-rank FER unit is pluggable (``unit``) so the host logic is testable
with the gloo backend on CPU; the product path uses ``decode_frames_device``
on the rank's GPU with NCCL.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .harness import FerPoint, SweepConfig, config_digest, decode_frames_device, wilson_interval


def shard_range(rank: int, world: int, start: int, count: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of frames [start, start+count) for ``rank``."""
    lo = start + count * rank // world
    hi = start + count * (rank + 1) // world
    return lo, hi - lo


def _world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def gpu_unit(graph, cfg, eps, eps0, seed, start, count, device=None):
    """Default FER unit: (fails uint8, iterations int64) device tensors."""
    fails, iters, _ = decode_frames_device(graph, cfg, eps, eps0, seed, start, count, device=device)
    return fails, iters


def fer_counters(graph, cfg, eps, eps0, seed, start, count, *, unit=None, device=None) -> torch.Tensor:
    """Global {frames, failures, sum iterations, CN-edge updates} over all
    ranks for frames [start, start+count) (one all-reduce)."""
    rank, world = _world()
    lo, n = shard_range(rank, world, start, count)
    if unit is None:
        cnt = torch.zeros(4, dtype=torch.int64, device=device or torch.device("cuda", torch.cuda.current_device()))
        decode_frames_device(graph, cfg, eps, eps0, seed, lo, n, counters=cnt, want_frames=False, device=device)
    else:
        fails, iters = unit(graph, cfg, eps, eps0, seed, lo, n)
        E = int(graph.edge_count if hasattr(graph, "edge_count") else graph.E)
        cnt = torch.tensor([n, int(fails.sum()), int(iters.sum()), E * (int(iters.sum()) - n)],
                           dtype=torch.int64)
    if world > 1:
        dist.all_reduce(cnt)
    return cnt


@dataclass
class ShardedStats:
    frames: int
    failures: int
    iter_sum: int


def run_point_sharded(graph, cfg: SweepConfig, epsilon: float, *, chunk: int = 1 << 20, unit=None,
                      device=None) -> FerPoint:
    """run_point (harness.py:248-293) with frames sharded over all ranks and
    the exact ordered stop rule; every rank returns the same FerPoint.

    Per round of world x chunk frames only scalars cross ranks: ONE
    all-gather of each rank's (failures, sum iterations).  If the global
    cumulative count reaches the target inside the round, the first rank
    whose prefix crosses it finds its local stop frame and iteration prefix
    on its own device and broadcasts those two numbers -- frames past the
    stop are discarded, as the reference does for speculative batches."""
    rank, world = _world()
    unit = unit or (lambda *a: gpu_unit(*a, device=device))
    eps0 = epsilon if cfg.epsilon0_mode == "matched" else float(cfg.epsilon0)

    def launch(start):
        """Decode this rank's shard of the round at ``start`` and queue the
        scalar all-gather (both stream-ordered, no host sync)."""
        count = min(chunk * world, cfg.max_frames - start)
        lo, n = shard_range(rank, world, start, count)
        fails, iters = unit(graph, cfg.decoder, epsilon, eps0, cfg.seed, lo, n)
        fails = fails.to(torch.int64)
        iters = iters.to(torch.int64)
        mine = torch.stack([fails.sum(), iters.sum()]) if n else torch.zeros(2, dtype=torch.int64,
                                                                             device=fails.device)
        allv = [mine]
        if world > 1:
            allv = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(allv, mine)
        return start, count, fails, iters, mine, allv

    frames = failures = iter_sum = 0
    nxt = launch(0) if cfg.max_frames > 0 else None
    while nxt is not None:
        start, count, fails, iters, mine, allv = nxt
        # speculative: the next round is queued before this one is inspected
        nxt = launch(start + count) if start + count < cfg.max_frames else None
        per = torch.stack(allv).cpu().tolist()
        before = failures
        crossing = None
        for r, (nf, _) in enumerate(per):
            if before + nf >= cfg.target_failures:
                crossing = r
                break
            before += nf
        if crossing is None:
            frames = start + count
            failures = before
            iter_sum += sum(ni for _, ni in per)
            continue
        # the crossing rank locates the stop frame inside its shard
        if rank == crossing:
            cum = torch.cumsum(fails, 0)
            k = int(torch.nonzero(before + cum >= cfg.target_failures)[0, 0])
            info = torch.tensor([k, int(iters[: k + 1].sum())], dtype=torch.int64, device=mine.device)
        else:
            info = torch.zeros(2, dtype=torch.int64, device=mine.device)
        if world > 1:
            dist.broadcast(info, src=crossing)
        k, it_prefix = (int(x) for x in info.cpu().tolist())
        lo_c, _ = shard_range(crossing, world, start, count)
        frames = lo_c + k + 1
        # failures grow by at most one per frame, so the first crossing frame
        # brings the cumulative count to exactly the target
        failures = cfg.target_failures
        iter_sum += sum(ni for _, ni in per[:crossing]) + it_prefix
        break
    low, high = wilson_interval(failures, frames)
    return FerPoint(epsilon=epsilon, epsilon0=eps0, frames=frames, failures=failures,
                    fer=failures / frames, wilson_low=low, wilson_high=high,
                    mean_iterations=iter_sum / frames, cap_hit=failures < cfg.target_failures,
                    config_digest=config_digest(cfg), seed=cfg.seed)
