"""CPU: the C-ABI library builds for sm_100a, loads without a GPU, exports
every symbol include/qsg.h declares, and its host-only layout compiler
(device -1) reproduces the reference's TannerGraph arrays.  No decode is
launched here (no GPU); the decode entry points are exercised by the -m gpu
tests."""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import GB126, GB254, GB1022, ROOT, SMALL, TOY, make_tree_rows


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "qsg.h")).read()
    return sorted(set(re.findall(r"\b(qsg_[a-z0-9_]+)\s*\(", text)))


def test_header_and_exports(tmp_path):
    from paper_2605_10433_b200 import _native
    L = _native.lib()
    syms = declared_symbols()
    assert set(syms) == set(_native.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (qsg_[a-z0-9_]+)", out))
    assert set(syms) <= exported
    for s in syms:
        assert hasattr(L, s)
    assert L.qsg_abi_version() == 1
    # the header compiles as C (plain pointers and sizes, no torch types)
    src = tmp_path / "h.c"
    src.write_text('#include "qsg.h"\nint main(void){return QSG_OK;}\n')
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-c",
                    str(src), "-o", str(tmp_path / "h.o")], check=True)


def test_kernels_are_sm100a():
    """The fatbin holds sm_100a SASS for the decode kernels."""
    from paper_2605_10433_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH], capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    for ln in sass.splitlines():
        if "Function : " in ln:
            cur = ln.split("Function : ")[1].strip()
            funcs[cur] = []
        elif cur:
            funcs[cur].append(ln)
    # the BASELINE configs[1] kernels (W = 5, one warp per frame, n_pad 256)
    # (lean instances, the ones the bench launches: template flag LEAN = true)
    ms = "\n".join(funcs["_ZN3qsg13decode_kernelILi5ELi32ELb0ELb0ELi256ELb1EEEvNS_7KParamsE"])
    bp4 = "\n".join(funcs["_ZN3qsg13decode_kernelILi5ELi32ELb1ELb0ELi256ELb1EEEvNS_7KParamsE"])
    full = [funcs["_ZN3qsg13decode_kernelILi5ELi32ELb0ELb0ELi256ELb0EEEvNS_7KParamsE"],
            funcs["_ZN3qsg13decode_kernelILi5ELi32ELb1ELb0ELi256ELb0EEEvNS_7KParamsE"]]
    # the lean instances fold the run-time options: markedly less code
    assert len(ms.splitlines()) < 0.8 * len(full[0]) and len(bp4.splitlines()) < 0.8 * len(full[1])
    # min-sum: min1/min2 with the sign product riding on min (FMNMX), paired
    # qubit factors (FFMA2), frame queue (ATOMG), ballot-packed bitmaps (VOTE)
    for op in ("FMNMX", "FFMA2", "ATOMG", "VOTE", "LDS.U16", "SHFL"):
        assert op in ms, op
    # BP4: product-form recipe on FFMA2 / FMUL2.  Neither kernel uses the
    # hardware approximations MUFU.EX2 / LG2 (the fp32 recipes must be
    # reproducible by the CPU oracle; the only MUFU is the RCP seed of integer /
    # double divisions outside the recipes), and neither spills
    for op in ("FFMA2", "FMUL2"):
        assert op in bp4, op
    for k in (ms, bp4, "\n".join(full[0]), "\n".join(full[1])):
        assert "MUFU.EX2" not in k and "MUFU.LG2" not in k
        assert "STL" not in k and "LDL" not in k


@pytest.mark.parametrize("spec,kind", [(TOY, 0), (SMALL, 0), (GB126, 5), (GB254, 5), (GB1022, 5),
                                       ((127, (0, 15, 20), (0, 58, 59, 100)), 0)])
def test_layout_compiler_host_only(oracle, spec, kind):
    import paper_2605_10433_b200 as P
    g = P.gb_graph(P.GbSpec(*spec))
    o = oracle.gb_graph(*spec)
    for k in ("edge_cn", "edge_vn", "edge_sym", "cn_ptr", "vn_order", "vn_ptr", "vn_inverse"):
        assert np.array_equal(getattr(g, k), getattr(o, k)), k
    assert g.kind == kind


@pytest.mark.parametrize("ell,threads", [(63, 32), (127, 32), (128, 32), (129, 64), (255, 64), (256, 64),
                                         (257, 128), (511, 128)])
def test_threads_per_frame_rule(ell, threads):
    """Bicycle kernels use about four circulant indices per thread: 32
    threads for l <= 128, 64 for l <= 256, else 128."""
    import paper_2605_10433_b200 as P
    g = P.gb_graph(P.GbSpec(ell, (0, 1, 3, 7, 12), (0, 2, 5, 9, 14)))
    assert g.kind == 5 and g.threads == threads


def test_layout_compiler_vs_reference(reference):
    import paper_2605_10433_b200 as P
    from qsagms.code import GbSpec, build_gb, load_code, tanner_graph
    for spec in (TOY, SMALL, GB126, GB254, GB1022):
        r = tanner_graph(build_gb(GbSpec(*spec)))
        g = P.gb_graph(P.GbSpec(*spec))
        for k in ("edge_cn", "edge_vn", "edge_sym", "cn_ptr", "vn_order", "vn_ptr", "vn_inverse"):
            assert np.array_equal(getattr(g, k), getattr(r, k)), (spec, k)
    qpc = "/root/reference/pkg/codes/gb-126-28.qpc"
    r = tanner_graph(load_code(qpc))
    g = P.load_qpc(qpc)
    assert np.array_equal(g.edge_vn, r.edge_vn) and np.array_equal(g.cn_ptr, r.cn_ptr)
    assert g.gb == P.GbSpec(*GB126)


def test_generic_csr_graph(oracle):
    import paper_2605_10433_b200 as P
    rng = np.random.default_rng(3)
    n, rows = make_tree_rows(rng, 11)
    g = P.csr_graph(n, rows)
    o = oracle.tanner_arrays(n, rows)
    for k in ("edge_cn", "edge_vn", "edge_sym", "cn_ptr", "vn_order", "vn_ptr"):
        assert np.array_equal(getattr(g, k), getattr(o, k))
    assert g.kind == 0


def test_invalid_arguments_map_to_value_error():
    import paper_2605_10433_b200 as P
    with pytest.raises(ValueError):
        P.csr_graph(3, [[(0, 1), (0, 2)]])        # columns not strictly increasing
    with pytest.raises(ValueError):
        P.csr_graph(3, [[(0, 1), (5, 2)]])        # column out of range
    with pytest.raises(ValueError):
        P.csr_graph(3, [[(0, 1), (1, 4)]])        # not a Pauli
    with pytest.raises(ValueError):
        P.csr_graph(3, [[(0, 1), (1, 2)]])        # qubit 2 isolated
    with pytest.raises(ValueError):
        P.GbSpec(5, (0, 0), (1,))
    from paper_2605_10433_b200 import _native
    L = _native.lib()
    h = C.c_void_p()
    a = np.array([0, 7], dtype=np.int32)
    assert L.qsg_graph_create_gb(5, a.ctypes.data, 2, a.ctypes.data, 1, -1, C.byref(h)) == _native.QSG_EINVAL
    assert b"exponents" in L.qsg_last_error()


def test_decode_without_gpu_fails_loudly():
    """No CPU fallback: the decode entry points refuse to run without CUDA."""
    import torch

    import paper_2605_10433_b200 as P
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = P.gb_graph(P.GbSpec(*SMALL))
    cfg = P.DecoderConfig("ms", l_max=4)
    with pytest.raises(RuntimeError):
        P.decode_frames(g, cfg, 0.1, 0.1, 0, 0, 4)
    with pytest.raises(RuntimeError):
        P.decode_batch(g, np.zeros((2, g.m), np.uint8), P.prior_llr(0.1), cfg)
    with pytest.raises(RuntimeError):
        P.decode_host_batches(g, [P.HostBatch(torch.zeros((2, g.m), dtype=torch.uint8), 1.0, cfg)])
