"""Decoder API mirroring the reference's ``qsagms.decoder``.

``decode_batch`` and ``decode`` keep the reference signatures, dtypes and
error behaviour (pkg/src/qsagms/decoder.py:374-559) but every decode runs in
the sm_100a kernels of ``libqsg.so`` (fp32 messages; see DESIGN.md for the
numerics contract).  Config objects may be this module's or the reference's.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .channel import ChannelPrior
from .device import decoder_cfg_struct, device_graph, ptr, stream_ptr

VARIANTS = ("bp4", "ms", "sms", "sagms")
VN_MODES = ("marginal", "additive")
LLR_CLIP = 64.0


@dataclass(frozen=True)
class GainParams:
    """SAGMS ramp (alpha_min, alpha_max) and unsatisfied-check boost
    (decoder.py:62-88), with the stability constraint alpha_max*eta <= 1."""

    alpha_min: float
    alpha_max: float
    eta_unsat: float

    def __post_init__(self):
        if not 0.0 < self.alpha_min <= self.alpha_max <= 1.0:
            raise ValueError("need 0 < alpha_min <= alpha_max <= 1, got "
                             f"({self.alpha_min}, {self.alpha_max})")
        if self.eta_unsat < 1.0:
            raise ValueError(f"eta_unsat must be >= 1, got {self.eta_unsat}")
        if self.alpha_max * self.eta_unsat > 1.0:
            raise ValueError("stability constraint alpha_max*eta_unsat <= 1 violated: "
                             f"{self.alpha_max}*{self.eta_unsat} = "
                             f"{self.alpha_max * self.eta_unsat}")


@dataclass(frozen=True)
class DecoderConfig:
    """Variant, iteration budget and qubit-update mode (decoder.py:91-112)."""

    variant: str
    l_max: int = 8
    alpha: float | None = None
    gain: GainParams | None = None
    vn_mode: str = "marginal"

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"variant must be one of {VARIANTS}, got {self.variant!r}")
        if self.vn_mode not in VN_MODES:
            raise ValueError(f"vn_mode must be one of {VN_MODES}, got {self.vn_mode!r}")
        if self.l_max < 1:
            raise ValueError("l_max must be at least 1")
        if self.variant == "sms" and (self.alpha is None or not 0.0 < self.alpha <= 1.0):
            raise ValueError(f"sms requires alpha in (0, 1], got {self.alpha}")
        if self.variant == "sagms" and self.gain is None:
            raise ValueError("sagms requires GainParams")


@dataclass
class EdgeMessageState:
    """Per-edge message snapshot in canonical edge order."""

    vn_to_cn: np.ndarray
    cn_to_vn: np.ndarray
    iteration: int


@dataclass
class DecodeResult:
    success: bool
    e_hat: np.ndarray
    iterations_used: int
    gamma_trace: np.ndarray
    message_trace: list[EdgeMessageState] | None = None


@dataclass
class BatchDecodeResult:
    success: np.ndarray
    e_hat: np.ndarray
    iterations: np.ndarray
    gamma_traces: list[np.ndarray] | None = None
    message_trace: list[EdgeMessageState] | None = None


def syndrome_ratio(residual) -> float:
    """Fraction of unsatisfied checks (decoder.py:157-162)."""
    residual = np.asarray(residual)
    if residual.size < 1:
        raise ValueError("residual syndrome must have at least one bit")
    return float(np.count_nonzero(residual)) / residual.size


def effective_gain(gamma: float, s_tilde_bit: int, p: GainParams) -> float:
    """Per-check SAGMS gain (decoder.py:165-170)."""
    if not 0.0 <= gamma <= 1.0:
        raise ValueError(f"gamma must lie in [0, 1], got {gamma}")
    base = p.alpha_max - (p.alpha_max - p.alpha_min) * gamma
    return base * p.eta_unsat if s_tilde_bit else base


def decode_batch_device(graph, syndromes: torch.Tensor, l0: float, cfg, *, early_stop=True,
                        e_hat=True, collect_gamma=False, capture_messages=False):
    """Device-tensor form of decode_batch: syndromes uint8 (B, m) on the GPU.

    Returns a dict of device tensors: success (uint8 B), iterations (int64 B),
    e_hat (uint8 B x n, optional) and, when requested, unsat (int32 B x l_max),
    counts (int32 B x 2), vn_msgs / cn_msgs (float32 B x l_max x E).
    """
    dg = device_graph(graph, syndromes.device if syndromes.is_cuda else None)
    dev = dg.device
    if syndromes.dim() != 2 or syndromes.shape[1] != dg.m:
        raise ValueError(f"syndromes must have shape (B, {dg.m})")
    syn = syndromes.to(device=dev, dtype=torch.uint8).contiguous()
    B = syn.shape[0]
    L = int(cfg.l_max)
    out = {
        "success": torch.empty(B, dtype=torch.uint8, device=dev),
        "iterations": torch.empty(B, dtype=torch.int64, device=dev),
        "e_hat": torch.empty((B, dg.n), dtype=torch.uint8, device=dev) if e_hat else None,
    }
    trace = None
    if collect_gamma or capture_messages:
        out["unsat"] = torch.zeros((B, L), dtype=torch.int32, device=dev)
        out["counts"] = torch.zeros((B, 2), dtype=torch.int32, device=dev)
        if capture_messages:
            out["vn_msgs"] = torch.zeros((B, L, dg.E), dtype=torch.float32, device=dev)
            out["cn_msgs"] = torch.zeros((B, L, dg.E), dtype=torch.float32, device=dev)
        trace = _native.Trace(ptr(out["unsat"]), ptr(out.get("vn_msgs")), ptr(out.get("cn_msgs")),
                              ptr(out["counts"]))
    c = decoder_cfg_struct(cfg, early_stop)
    import ctypes as C
    _native.check(_native.lib().qsg_decode_syndromes(
        dg.handle, C.byref(c), float(l0), ptr(syn), B, ptr(out["success"]), ptr(out["e_hat"]),
        ptr(out["iterations"]), C.byref(trace) if trace is not None else None, stream_ptr(dev)))
    return out


_STAGE: dict = {}


def _stage(key, nbytes: int) -> torch.Tensor:
    """Grow-only pinned host staging buffer per (thread, device, role)."""
    import threading
    k = (threading.get_ident(), torch.cuda.current_device(), key)
    buf = _STAGE.get(k)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        _STAGE[k] = buf
    return buf


def _pinned_from(a: np.ndarray) -> torch.Tensor:
    """A numpy array staged in pinned memory (for an asynchronous H2D copy);
    valid until the next call on this thread."""
    a = np.ascontiguousarray(a)
    buf = _stage("in", a.nbytes)[: a.nbytes]
    np.copyto(buf.numpy().view(a.dtype).reshape(a.shape), a)
    return buf.view(torch.from_numpy(a[:0].reshape(-1)).dtype).view(a.shape)


def _to_host(tensors: dict) -> dict:
    """Device tensors -> fresh numpy arrays through one pinned staging
    buffer and one stream sync."""
    total = sum((t.numel() * t.element_size() + 15) // 16 * 16 for t in tensors.values())
    buf = _stage("out", total)
    views, off = {}, 0
    for k, t in tensors.items():
        nb = t.numel() * t.element_size()
        v = buf[off: off + nb].view(t.dtype).view(t.shape)
        v.copy_(t, non_blocking=True)
        views[k] = v
        off += (nb + 15) // 16 * 16
    if tensors:
        torch.cuda.current_stream(next(iter(tensors.values())).device).synchronize()
    return {k: v.numpy().copy() for k, v in views.items()}


def decode_batch(graph, syndromes, prior: ChannelPrior, cfg, *, early_stop: bool = True,
                 collect_gamma: bool = False, capture_messages: bool = False) -> BatchDecodeResult:
    """Decode a batch of syndromes (decoder.py:374-485) on the GPU.

    Frames are independent: results are bit-identical for any batching.
    ``capture_messages`` is limited to single-frame batches, as in the
    reference.
    """
    syn = np.asarray(syndromes, dtype=np.uint8)
    if syn.ndim != 2 or syn.shape[1] != int(graph.m):
        raise ValueError(f"syndromes must have shape (B, {int(graph.m)})")
    if capture_messages and syn.shape[0] != 1:
        raise ValueError("capture_messages requires a single-frame batch")
    dg = device_graph(graph)
    # pinned staging both ways (torch caches pinned blocks) and one sync:
    # pageable copies of B x m and B x n bytes cost ~4x more than the decode
    d_syn = _pinned_from(syn).to(dg.device, non_blocking=True)
    out = decode_batch_device(dg, d_syn, prior.llr, cfg,
                              early_stop=early_stop, collect_gamma=collect_gamma,
                              capture_messages=capture_messages)
    host = _to_host({k: out[k] for k in ("success", "e_hat", "iterations")})
    res = BatchDecodeResult(
        success=host["success"].astype(bool),
        e_hat=host["e_hat"],
        iterations=host["iterations"],
    )
    if collect_gamma or capture_messages:
        unsat = out["unsat"].cpu().numpy()
        counts = out["counts"].cpu().numpy()
        m = dg.m
        if collect_gamma:
            res.gamma_traces = [unsat[b, : counts[b, 0]] / m for b in range(len(counts))]
        if capture_messages:
            vn = out["vn_msgs"].cpu().numpy().astype(np.float64)
            cn = out["cn_msgs"].cpu().numpy().astype(np.float64)
            res.message_trace = [EdgeMessageState(vn_to_cn=vn[0, k], cn_to_vn=cn[0, k], iteration=k + 1)
                                 for k in range(counts[0, 1])]
    return res


def pack_syndromes(syndromes) -> np.ndarray:
    """(B, m) syndrome bits -> (B, ceil(m/32)) uint32, bit i of row b at
    word i // 32, bit i % 32 (the qsg_decode_syndromes_packed wire format)."""
    syn = np.asarray(syndromes, dtype=np.uint8) != 0
    B, m = syn.shape
    pad = np.zeros((B, (m + 31) // 32 * 32), dtype=bool)
    pad[:, :m] = syn
    return np.packbits(pad, axis=1, bitorder="little").view("<u4").reshape(B, -1).astype(np.uint32)


def decode_batch_packed_device(graph, syn_words: torch.Tensor, l0: float, cfg, *, e_hat=False):
    """decode_batch from bit-packed device syndromes (uint32/int32 (B, ceil(m/32)))."""
    import ctypes as C
    dg = device_graph(graph, syn_words.device if syn_words.is_cuda else None)
    dev = dg.device
    if syn_words.dim() != 2 or syn_words.shape[1] != (dg.m + 31) // 32:
        raise ValueError(f"packed syndromes must have shape (B, {(dg.m + 31) // 32})")
    words = syn_words.to(device=dev).contiguous()
    B = words.shape[0]
    out = {"success": torch.empty(B, dtype=torch.uint8, device=dev),
           "iterations": torch.empty(B, dtype=torch.int64, device=dev),
           "e_hat": torch.empty((B, dg.n), dtype=torch.uint8, device=dev) if e_hat else None}
    c = decoder_cfg_struct(cfg, True)
    _native.check(_native.lib().qsg_decode_syndromes_packed(
        dg.handle, C.byref(c), float(l0), ptr(words), B, ptr(out["success"]), ptr(out["e_hat"]),
        ptr(out["iterations"]), stream_ptr(dev)))
    return out


def decode_batch_packed(graph, syn_words, prior: ChannelPrior, cfg) -> BatchDecodeResult:
    """decode_batch for bit-packed syndromes (see pack_syndromes)."""
    dg = device_graph(graph)
    w = np.ascontiguousarray(syn_words, dtype=np.uint32).view(np.int32)
    out = decode_batch_packed_device(dg, _pinned_from(w).to(dg.device, non_blocking=True), prior.llr, cfg,
                                     e_hat=True)
    host = _to_host({k: out[k] for k in ("success", "e_hat", "iterations")})
    return BatchDecodeResult(success=host["success"].astype(bool), e_hat=host["e_hat"],
                             iterations=host["iterations"])


def decode(H, graph, s, prior: ChannelPrior, cfg, *, early_stop: bool = True,
           capture_messages: bool = False, trace_sink=None) -> DecodeResult:
    """Single-syndrome decode with gamma trace and optional per-iteration
    records (decoder.py:488-559).  ``H`` may be None (the graph is used to
    re-verify a reported success)."""
    s = np.asarray(s, dtype=np.uint8)
    m = int(graph.m)
    if s.shape != (m,):
        raise ValueError(f"syndrome must have length m={m}")
    want = capture_messages or trace_sink is not None
    batch = decode_batch(graph, s[None, :], prior, cfg, early_stop=early_stop, collect_gamma=True,
                         capture_messages=want)
    gamma_trace = batch.gamma_traces[0]
    res = DecodeResult(success=bool(batch.success[0]), e_hat=batch.e_hat[0],
                       iterations_used=int(batch.iterations[0]), gamma_trace=gamma_trace,
                       message_trace=batch.message_trace if capture_messages else None)
    if res.success:
        dg = device_graph(graph)
        if (dg.graph.syndromes_of(res.e_hat[None, :])[0] ^ s).any():
            raise RuntimeError("internal inconsistency: reported success with nonzero residual")
    if trace_sink is not None and batch.message_trace:
        for st in batch.message_trace:
            ell = st.iteration
            gamma = float(gamma_trace[ell - 1]) if ell - 1 < len(gamma_trace) else 0.0
            if cfg.variant == "sagms":
                gs = {"min": effective_gain(gamma, 0, cfg.gain), "max": effective_gain(gamma, 1, cfg.gain)}
            elif cfg.variant == "sms":
                gs = {"min": cfg.alpha, "max": cfg.alpha}
            else:
                gs = {"min": 1.0, "max": 1.0}
            counts, edges = np.histogram(np.abs(st.vn_to_cn), bins=16, range=(0.0, LLR_CLIP))
            trace_sink({"iteration": ell, "gamma": gamma, "alpha_eff": gs,
                        "magnitude_hist": {"bin_edges": edges.tolist(), "counts": counts.tolist()}})
    return res


def marginal_init(l0: float) -> float:
    """Initial marginal-mode message (decoder.py:255-261)."""
    return math.log1p(math.exp(-l0)) + l0 - math.log(2.0)
