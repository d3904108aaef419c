"""ctypes binding of the C ABI in ``include/qsg.h`` (``libqsg.so``).

The library is built in-tree (``paper_2605_10433_b200/csrc/Makefile``, see
``__graft_entry__.build``).  There is no CPU fallback: if the shared library
is missing or a CUDA device is unavailable, every decode entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
# QSG_LIB overrides the library path (A/B timing of two builds in one process
# tree; tools/ only).
LIB_PATH = os.environ.get("QSG_LIB") or os.path.join(HERE, "libqsg.so")
CSRC = os.path.join(HERE, "csrc")

QSG_OK = 0
QSG_EINVAL = -1
QSG_ECUDA = -2
QSG_ENOMEM = -3
QSG_EUNSUPPORTED = -4

#: Every symbol include/qsg.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "qsg_graph_create_gb", "qsg_graph_create_csr", "qsg_graph_destroy", "qsg_graph_info",
    "qsg_graph_export", "qsg_decode_syndromes", "qsg_decode_syndromes_packed", "qsg_decode_frames",
    "qsg_sample_errors",
    "qsg_syndromes_of", "qsg_graph_check_commute", "qsg_last_error", "qsg_abi_version",
    "qsg_build_id",
)


class DecoderCfg(C.Structure):
    """``qsg_decoder_cfg``."""

    _fields_ = [
        ("variant", C.c_int32), ("vn_mode", C.c_int32), ("l_max", C.c_int32),
        ("early_stop", C.c_int32), ("alpha", C.c_double), ("alpha_min", C.c_double),
        ("alpha_max", C.c_double), ("eta_unsat", C.c_double),
    ]


class Trace(C.Structure):
    """``qsg_trace`` (device pointers)."""

    _fields_ = [("unsat", C.c_void_p), ("vn_msgs", C.c_void_p),
                ("cn_msgs", C.c_void_p), ("counts", C.c_void_p)]


class NativeError(RuntimeError):
    pass


_lib = None


def build(verbose: bool = False) -> str:
    """Compile libqsg.so for sm_100a (nvcc cross-compiles without a GPU)."""
    out = subprocess.run(["make", "-C", CSRC, f"-j{os.cpu_count() or 4}"],
                         capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise NativeError(f"libqsg build failed:\n{out.stdout}\n{out.stderr}")
    return LIB_PATH


def lib():
    """Load libqsg.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, dbl, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_uint64
        L.qsg_graph_create_gb.argtypes = [i32, vp, i32, vp, i32, i32, C.POINTER(vp)]
        L.qsg_graph_create_csr.argtypes = [i32, i32, vp, vp, vp, i32, C.POINTER(vp)]
        L.qsg_graph_destroy.argtypes = [vp]
        L.qsg_graph_info.argtypes = [vp] + [vp] * 7
        L.qsg_graph_export.argtypes = [vp] * 7
        L.qsg_decode_syndromes.argtypes = [vp, vp, dbl, vp, i64, vp, vp, vp, vp, vp]
        L.qsg_decode_syndromes_packed.argtypes = [vp, vp, dbl, vp, i64, vp, vp, vp, vp]
        L.qsg_decode_frames.argtypes = [vp, vp, dbl, dbl, u64, i64, i64, vp, vp, vp, vp, vp]
        L.qsg_sample_errors.argtypes = [i32, dbl, u64, i64, i64, vp, i32, vp]
        L.qsg_syndromes_of.argtypes = [vp, vp, i64, vp, vp]
        L.qsg_graph_check_commute.argtypes = [vp, vp, vp]
        L.qsg_last_error.restype = C.c_char_p
        L.qsg_last_error.argtypes = []
        L.qsg_abi_version.argtypes = []
        L.qsg_build_id.restype = C.c_char_p
        L.qsg_build_id.argtypes = []
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a qsg status to the reference's exception types."""
    if rc == QSG_OK:
        return
    msg = lib().qsg_last_error().decode()
    if rc == QSG_EINVAL:
        raise ValueError(msg)
    raise NativeError(f"qsg error {rc}: {msg}")
