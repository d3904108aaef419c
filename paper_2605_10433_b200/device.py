"""Device-resident graph handles and buffer plumbing.

PyTorch is used only for device memory and streams; every computation is a
``libqsg.so`` kernel launched through the C ABI (include/qsg.h).
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _native
from .codes import CodeGraph, as_code_graph

VARIANT_CODES = {"bp4": 0, "ms": 1, "sms": 2, "sagms": 3}
VN_MODE_CODES = {"marginal": 0, "additive": 1}


def require_cuda(device=None) -> torch.device:
    """The decode path has no CPU fallback: fail loudly without a GPU."""
    if not torch.cuda.is_available():
        raise _native.NativeError("qsg decode requires a CUDA device (no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       torch.device(device).index or 0)
    return dev


class DeviceGraph:
    """A ``qsg_graph*`` uploaded to one device (immutable, shareable)."""

    def __init__(self, graph, device=None):
        self.graph: CodeGraph = as_code_graph(graph)
        self.device = require_cuda(device)
        g = self.graph
        L = _native.lib()
        self._cn_ptr = np.ascontiguousarray(g.cn_ptr, dtype=np.int64)
        self._ev = np.ascontiguousarray(g.edge_vn, dtype=np.int64)
        self._es = np.ascontiguousarray(g.edge_sym, dtype=np.uint8)
        h = C.c_void_p()
        _native.check(L.qsg_graph_create_csr(g.n, g.m, self._cn_ptr.ctypes.data, self._ev.ctypes.data,
                                             self._es.ctypes.data, self.device.index, C.byref(h)))
        self.handle = h
        n, m, dcm, dvm, kind, thr = (C.c_int32() for _ in range(6))
        E = C.c_int64()
        _native.check(L.qsg_graph_info(h, C.byref(n), C.byref(m), C.byref(E), C.byref(dcm),
                                       C.byref(dvm), C.byref(kind), C.byref(thr)))
        self.n, self.m, self.E = n.value, m.value, E.value
        self.kind, self.threads = kind.value, thr.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _native._lib is not None:
            _native._lib.qsg_graph_destroy(h)
            self.handle = None


_CACHE: dict = {}
_CACHE_LOCK = threading.Lock()


def device_graph(graph, device=None) -> DeviceGraph:
    """Per-(graph object, device) cache, like the reference's _kernel_for
    (decoder.py:362-371) but keyed by identity and bounded."""
    if isinstance(graph, DeviceGraph):
        return graph
    dev = require_cuda(device)
    key = (id(graph), dev.index)
    with _CACHE_LOCK:
        hit = _CACHE.get(key)
        if hit is not None and hit[0] is graph:
            return hit[1]
        dg = DeviceGraph(graph, dev)
        if len(_CACHE) >= 16:
            _CACHE.pop(next(iter(_CACHE)))
        _CACHE[key] = (graph, dg)
        return dg


def decoder_cfg_struct(cfg, early_stop: bool = True) -> _native.DecoderCfg:
    """Flatten a DecoderConfig (this package's or the reference's)."""
    gain = getattr(cfg, "gain", None)
    alpha = getattr(cfg, "alpha", None)
    try:
        variant = VARIANT_CODES[cfg.variant]
        vn_mode = VN_MODE_CODES[cfg.vn_mode]
    except KeyError as exc:
        raise ValueError(f"unknown decoder option {exc}") from None
    return _native.DecoderCfg(
        variant, vn_mode, int(cfg.l_max), 1 if early_stop else 0,
        float(alpha) if alpha is not None else 0.0,
        float(gain.alpha_min) if gain is not None else 0.0,
        float(gain.alpha_max) if gain is not None else 0.0,
        float(gain.eta_unsat) if gain is not None else 0.0,
    )


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()
