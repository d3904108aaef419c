"""CPU, world_size 2 (gloo): the multi-rank host logic of the N>1 path --
contiguous frame shards, the counter all-reduce and the exact distributed
stop rule -- with the CPU oracle as each rank's FER unit (the -m gpu runs and
bench.py use the device unit and NCCL)."""
from __future__ import annotations

import json
import os
import socket
from dataclasses import asdict
from pathlib import Path

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, SMALL, TOY

GOLD = Path(__file__).resolve().parent / "golden"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_unit(graph, cfg, eps, eps0, seed, start, count):
    from oracle import oracle as O
    f, it, _, _ = O.frames(O.Graph(graph), cfg, eps, eps0, seed, start, count, precision=64, nthreads=2)
    return torch.from_numpy(f.astype("uint8")), torch.from_numpy(it)


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2605_10433_b200 as P
    from paper_2605_10433_b200 import dist as D
    small = P.gb_graph(P.GbSpec(*SMALL))
    toy = P.gb_graph(P.GbSpec(*TOY))
    cfg = P.DecoderConfig("sagms", l_max=8, gain=P.GainParams(0.3, 0.5, 1.1))
    cnt = D.fer_counters(small, cfg, 0.2, 0.2, 7, 3, 1001, unit=_oracle_unit)
    g = P.GainParams(0.3, 0.5, 1.1)
    sweep = P.SweepConfig(code_id="gb-10-2", decoder=P.DecoderConfig("sagms", l_max=4, gain=g),
                          epsilon_list=(0.25,), seed=31, target_failures=40, max_frames=100_000)
    p1 = D.run_point_sharded(small, sweep, 0.25, chunk=5, unit=_oracle_unit)
    sweep2 = P.SweepConfig(code_id="toy", decoder=P.DecoderConfig("ms", l_max=1), epsilon_list=(0.5,),
                           seed=2718, target_failures=50, max_frames=100_000)
    p2 = D.run_point_sharded(toy, sweep2, 0.5, chunk=3, unit=_oracle_unit)
    # the stop frame (index 55) in rank 1's shard: last element (chunk 4) and
    # first element (chunk 1); and a cap-hit point (target never reached)
    p3 = D.run_point_sharded(toy, sweep2, 0.5, chunk=4, unit=_oracle_unit)
    p4 = D.run_point_sharded(toy, sweep2, 0.5, chunk=1, unit=_oracle_unit)
    sweep3 = P.SweepConfig(code_id="toy", decoder=P.DecoderConfig("ms", l_max=1), epsilon_list=(0.5,),
                           seed=2718, target_failures=50, max_frames=41)
    p5 = D.run_point_sharded(toy, sweep3, 0.5, chunk=7, unit=_oracle_unit)
    out[rank] = {"cnt": cnt.tolist(), "p1": asdict(p1), "p2": asdict(p2), "p3": asdict(p3), "p4": asdict(p4),
                 "p5": asdict(p5)}
    dist.destroy_process_group()


def test_two_rank_gloo(oracle):
    world = 2
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    import paper_2605_10433_b200 as P
    from types import SimpleNamespace as NS
    # single-process oracle over the whole range
    g = oracle.gb_graph(*SMALL)
    cfg = NS(variant="sagms", l_max=8, vn_mode="marginal", alpha=None,
             gain=NS(alpha_min=0.3, alpha_max=0.5, eta_unsat=1.1))
    f, it, _, c = oracle.frames(g, cfg, 0.2, 0.2, 7, 3, 1001, precision=64)
    for r in range(world):
        assert out[r]["cnt"] == c.tolist()
    gold = json.loads((GOLD / "golden_harness.json").read_text())
    from paper_2605_10433_b200 import harness as H
    H.FRAME_UNIT = lambda *a: tuple(x.numpy() for x in _oracle_unit(*a))
    try:
        toy = P.gb_graph(P.GbSpec(*TOY))
        capped = H.run_point(toy, P.SweepConfig(code_id="toy", decoder=P.DecoderConfig("ms", l_max=1),
                                                epsilon_list=(0.5,), seed=2718, target_failures=50,
                                                max_frames=41), 0.5)
    finally:
        H.FRAME_UNIT = None
    for r in range(world):
        assert out[r]["p1"] == gold["small_sagms_eps025"]["point"]
        assert out[r]["p2"] == gold["toy_ms_lmax1_eps05"]["point"]
        assert out[r]["p3"] == out[r]["p4"] == gold["toy_ms_lmax1_eps05"]["point"]
        assert out[r]["p5"] == asdict(capped) and capped.cap_hit and capped.frames == 41
    assert P.dist.shard_range(0, 3, 10, 8) == (10, 2) and P.dist.shard_range(2, 3, 10, 8) == (15, 3)
