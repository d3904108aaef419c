// Internal declarations shared by the C-ABI translation unit and the kernel
// instantiation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "qsg_kernel.cuh"

namespace qsg {

// Kernel envelope compiled into the library.
constexpr int kBicycleWs[] = {2, 3, 4, 5, 6, 8};
constexpr int kThreadCounts[] = {32, 128};

// Returns the __global__ function for (W, T, bp4, additive) or nullptr.
void *kernel_ptr(int W, int T, bool bp4, bool additive, int np, bool lean);
void *kernel_ptr_w0(int T, bool bp4, bool additive, int np, bool lean);
void *kernel_ptr_w2(int T, bool bp4, bool additive, int np, bool lean);
void *kernel_ptr_w3(int T, bool bp4, bool additive, int np, bool lean);
void *kernel_ptr_w4(int T, bool bp4, bool additive, int np, bool lean);
void *kernel_ptr_w5(int T, bool bp4, bool additive, int np, bool lean);
void *kernel_ptr_w6(int T, bool bp4, bool additive, int np, bool lean);
void *kernel_ptr_w8(int T, bool bp4, bool additive, int np, bool lean);

struct LaunchCfg {
    int groups = 0;        // groups (frames in flight) per CTA
    int ctas_per_sm = 0;
    size_t smem = 0;
    bool ok = false;
    // the same number of frames per SM in the fewest, largest CTAs (used when
    // the batch fills every SM: one table copy per SM, warps spread evenly
    // over the four schedulers); 0 when it is the configuration above
    int big_groups = 0, big_ctas_per_sm = 0;
    size_t big_smem = 0;
};

}  // namespace qsg

// The opaque handle of include/qsg.h.
struct qsg_graph {
    int device = 0;
    int32_t n = 0, m = 0;
    int64_t E = 0;
    int32_t dc_max = 0, dv_max = 0, kind = 0, threads = 32;
    int32_t n_pad = 0, log2_npad = 0, m_pad = 0, row_words = 0;
    int32_t ell = 0, nw = 0, lpw = 0, gb_a[8] = {0}, gb_b[8] = {0};  // bicycle kernels
    uint32_t off_ehat = 0, off_bits = 0, off_synw = 0, off_resw = 0, off_scratch = 0;
    int32_t num_sms = 0;
    // canonical TannerGraph arrays (host)
    std::vector<int64_t> edge_cn, edge_vn, cn_ptr, vn_order, vn_ptr;
    std::vector<uint8_t> edge_sym;
    // device tables
    uint32_t *d_cn_tab = nullptr;
    uint32_t *d_cn_tab_x = nullptr;  // bicycle: rows in exponent order (min-sum kernels)
    uint8_t *d_vn_sym = nullptr, *d_vn_deg = nullptr;
    int32_t *d_slot_edge = nullptr;
    int32_t *d_cn_ptr = nullptr, *d_edge_vn = nullptr;
    uint8_t *d_edge_sym = nullptr;
    uint32_t tab_bytes = 0, group_bytes = 0;
    // launch configurations cached per kernel instance
    std::mutex mu;
    qsg::LaunchCfg cfg_cache[2][2][2];  // [bp4][additive][lean]
    // frame-queue counter per stream: launches on one stream are ordered, so
    // one 8-byte counter (re-zeroed before each launch) serves them all; no
    // per-launch allocation (the stream-ordered pool returns freed memory at
    // every synchronisation, making a per-launch cudaMallocAsync cost
    // ~200 us after each sync)
    std::unordered_map<cudaStream_t, unsigned long long *> queues;
};
