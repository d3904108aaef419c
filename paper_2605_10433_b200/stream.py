"""Pipelined decoding of host-resident syndrome batches.

A sweep decodes many independent batches (one per (decoder, p) point, or
successive chunks of one point).  ``decode_host_batches`` overlaps the
host-to-device copy of batch i+1 (a side stream, double-buffered) with the
decode of batch i (the caller's current stream) and returns each batch's
success flags and iteration counts in pinned host memory -- the
``decode_batch`` contract (decoder.py:374-485) applied to a stream of
batches, with the PCIe transfer hidden behind the kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .decoder import decode_batch_device, decode_batch_packed_device
from .device import device_graph, require_cuda


@dataclass
class HostBatch:
    """One batch: syndromes in host memory (pinned for a true async copy),
    uint8 (B, m) or, with ``packed``, int32/uint32 words (B, ceil(m/32));
    the prior LLR l0 and the decoder configuration."""

    syndromes: torch.Tensor
    l0: float
    cfg: object
    packed: bool = False


_COPY_STREAMS: dict = {}


def _copy_stream(dev: torch.device) -> torch.cuda.Stream:
    """One side stream per device for the host-to-device copies."""
    s = _COPY_STREAMS.get(dev.index)
    if s is None:
        s = _COPY_STREAMS[dev.index] = torch.cuda.Stream(dev)
    return s


def decode_host_batches(graph, batches, *, device=None, early_stop: bool = True, outputs=None):
    """Decode ``batches`` (an iterable of HostBatch) with copy/compute overlap.

    Returns a list of (success uint8 (B,), iterations int64 (B,)) pinned host
    tensors, valid after this call returns (it synchronises once at the end).
    ``outputs`` may supply those tensors (one pair per batch) to avoid
    allocating pinned memory per call.
    """
    dev = require_cuda(device)
    dg = device_graph(graph, dev)
    comp = torch.cuda.current_stream(dev)
    copy = _copy_stream(dev)
    copy.wait_stream(comp)  # buffers from earlier work on the caller's stream
    bufs: dict = {}
    ready = [torch.cuda.Event(), torch.cuda.Event()]
    free = [None, None]
    results = []
    for i, b in enumerate(batches):
        slot = i & 1
        src = b.syndromes
        key = (slot, b.packed, tuple(src.shape), src.dtype)
        buf = bufs.get(key)
        if buf is None:
            buf = bufs[key] = torch.empty(src.shape, dtype=src.dtype, device=dev)
        with torch.cuda.stream(copy):
            if free[slot] is not None:
                copy.wait_event(free[slot])
            buf.copy_(src, non_blocking=True)
            ready[slot].record(copy)
        comp.wait_event(ready[slot])
        if b.packed:
            out = decode_batch_packed_device(dg, buf, b.l0, b.cfg)
        else:
            out = decode_batch_device(dg, buf, b.l0, b.cfg, early_stop=early_stop, e_hat=False)
        ev = torch.cuda.Event()
        ev.record(comp)
        free[slot] = ev
        n = src.shape[0]
        if outputs is not None:
            succ, iters = outputs[i]
        else:
            succ = torch.empty(n, dtype=torch.uint8, pin_memory=True)
            iters = torch.empty(n, dtype=torch.int64, pin_memory=True)
        succ.copy_(out["success"], non_blocking=True)
        iters.copy_(out["iterations"], non_blocking=True)
        results.append((succ, iters))
    comp.synchronize()
    return results
