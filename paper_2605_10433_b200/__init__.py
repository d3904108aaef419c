"""B200-native batched Monte-Carlo decoder for generalized-bicycle QLDPC codes.

Drop-in for the hot path of the reference package ``qsagms`` (arXiv
2605.10433): depolarizing sampling -> syndrome -> flooding BP4 / MS / SMS /
SAGMS decode with early termination, run by hand-written sm_100a kernels in
``libqsg.so`` behind the C ABI of ``include/qsg.h``.  The Python names below
mirror the reference's public API (pkg/src/qsagms/__init__.py:63-114) for the
decode path.
"""

#: Version of the qsagms API (and persisted artifact format) mirrored here.
__version__ = "0.1.0"

from .channel import (  # noqa: E402
    ChannelPrior,
    DepolarizingChannel,
    prior_llr,
    sample_error,
    sample_errors,
    sample_errors_device,
)
from .codes import (  # noqa: E402
    CodeFormatError,
    CodeGraph,
    GbSpec,
    as_code_graph,
    OrthogonalityError,
    check_commute,
    check_commute_device,
    code_dimension,
    csr_graph,
    gb_dimension,
    gb_graph,
    load_qpc,
    random_gb_spec,
    save_qpc,
)
from .decoder import (  # noqa: E402
    BatchDecodeResult,
    DecodeResult,
    DecoderConfig,
    EdgeMessageState,
    GainParams,
    decode,
    decode_batch,
    decode_batch_device,
    decode_batch_packed,
    decode_batch_packed_device,
    effective_gain,
    pack_syndromes,
    syndrome_ratio,
)
from . import dist  # noqa: E402,F401
from .stream import HostBatch, decode_host_batches  # noqa: E402
from .device import DeviceGraph, device_graph  # noqa: E402
from .harness import (  # noqa: E402
    FerPoint,
    SweepConfig,
    config_digest,
    decode_frames,
    decode_frames_device,
    install,
    run_point,
    run_sweep,
    wilson_interval,
)

# reference spelling of the graph builders and code I/O
build_gb_graph = gb_graph
tanner_graph = as_code_graph
load_code = load_qpc

__all__ = [
    "__version__", "ChannelPrior", "DepolarizingChannel", "prior_llr", "sample_error",
    "sample_errors", "sample_errors_device", "CodeFormatError", "CodeGraph", "GbSpec",
    "as_code_graph", "check_commute", "check_commute_device", "OrthogonalityError", "code_dimension", "csr_graph", "gb_dimension", "gb_graph",
    "load_qpc", "random_gb_spec", "save_qpc", "BatchDecodeResult", "DecodeResult",
    "DecoderConfig", "EdgeMessageState", "GainParams", "decode", "decode_batch",
    "decode_batch_device", "decode_batch_packed", "decode_batch_packed_device", "pack_syndromes",
    "effective_gain", "syndrome_ratio", "DeviceGraph", "device_graph",
    "FerPoint", "SweepConfig", "config_digest", "decode_frames", "decode_frames_device",
    "install", "run_point", "run_sweep", "wilson_interval", "build_gb_graph", "tanner_graph",
    "HostBatch", "decode_host_batches", "load_code",
]
