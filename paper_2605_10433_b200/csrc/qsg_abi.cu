// C ABI (include/qsg.h): Tanner-graph layout compiler, launch configuration
// and the entry points that replace the reference's FER-loop unit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/qsg.h"
#include "qsg_internal.h"

namespace {

thread_local std::string g_last_error = "ok";

int fail(int code, const std::string &msg)
{
    g_last_error = msg;
    return code;
}

#define QSG_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t err_ = (call);                                                      \
        if (err_ != cudaSuccess)                                                        \
            return fail(QSG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(err_)); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        if (dev < 0) return;  // host-only graph: no CUDA calls at all
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

int next_pow2(int x)
{
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

template <typename T>
int upload(T **dst, const std::vector<T> &src)
{
    QSG_CUDA(cudaMalloc((void **)dst, std::max<size_t>(src.size(), 1) * sizeof(T)));
    if (!src.empty()) QSG_CUDA(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
    return QSG_OK;
}

void free_device(qsg_graph *g)
{
    cudaFree(g->d_cn_tab); cudaFree(g->d_cn_tab_x);
    for (auto &q : g->queues) cudaFree(q.second);
    g->queues.clear();
    cudaFree(g->d_vn_sym); cudaFree(g->d_vn_deg); cudaFree(g->d_slot_edge);
    cudaFree(g->d_cn_ptr); cudaFree(g->d_edge_vn); cudaFree(g->d_edge_sym);
}

bool bicycle_w_supported(int w)
{
    for (int x : qsg::kBicycleWs)
        if (x == w) return true;
    return false;
}

// Rows of build_gb (code.py:201-231) as canonical CSR: rows 0..ell-1 are X
// on [A|B] (columns (i + a_k), ell + (i + b_k)), rows ell..2ell-1 are Z on
// [B^T|A^T] (columns (i - b_k), ell + (i - a_k)), each row sorted.
void gb_rows(int32_t ell, const int32_t *a, int32_t wa, const int32_t *b, int32_t wb,
             std::vector<int64_t> &cn_ptr, std::vector<int64_t> &edge_vn, std::vector<uint8_t> &edge_sym)
{
    auto circ = [&](const int32_t *x, int w, int row, int sign) {
        std::vector<int64_t> cols(w);
        for (int k = 0; k < w; ++k) cols[k] = (((int64_t)row + sign * (int64_t)x[k]) % ell + ell) % ell;
        std::sort(cols.begin(), cols.end());
        return cols;
    };
    cn_ptr.assign(1, 0);
    edge_vn.clear();
    edge_sym.clear();
    for (int i = 0; i < ell; ++i) {
        for (int64_t c : circ(a, wa, i, 1)) { edge_vn.push_back(c); edge_sym.push_back(1); }
        for (int64_t c : circ(b, wb, i, 1)) { edge_vn.push_back(ell + c); edge_sym.push_back(1); }
        cn_ptr.push_back((int64_t)edge_vn.size());
    }
    for (int i = 0; i < ell; ++i) {
        for (int64_t c : circ(b, wb, i, -1)) { edge_vn.push_back(c); edge_sym.push_back(2); }
        for (int64_t c : circ(a, wa, i, -1)) { edge_vn.push_back(ell + c); edge_sym.push_back(2); }
        cn_ptr.push_back((int64_t)edge_vn.size());
    }
}

// ---- layout compiler ---------------------------------------------------------
// Input: canonical CSR (TannerGraph order, code.py:150-191).  Output: the
// TannerGraph arrays (kept for export), the qubit-major slot layout
// (slot = s * n_pad + j for the s-th edge of qubit j), the k-major check
// slot table, and the kernel kind (generic or bicycle W).
int compile_layout(qsg_graph *g, int32_t n, int32_t m, const int64_t *cn_ptr, const int64_t *edge_vn,
                   const uint8_t *edge_sym)
{
    if (n < 1 || m < 1) return fail(QSG_EINVAL, "n and m must be positive");
    if (!cn_ptr || !edge_vn || !edge_sym) return fail(QSG_EINVAL, "null CSR array");
    if (cn_ptr[0] != 0) return fail(QSG_EINVAL, "cn_ptr[0] must be 0");
    const int64_t E = cn_ptr[m];
    if (E < 1) return fail(QSG_EINVAL, "graph has no edges");
    g->n = n; g->m = m; g->E = E;
    g->cn_ptr.assign(cn_ptr, cn_ptr + m + 1);
    g->edge_vn.assign(edge_vn, edge_vn + E);
    g->edge_sym.assign(edge_sym, edge_sym + E);
    g->edge_cn.resize(E);
    std::vector<int64_t> vdeg(n, 0);
    int32_t dc_max = 0;
    for (int i = 0; i < m; ++i) {
        if (cn_ptr[i + 1] <= cn_ptr[i]) return fail(QSG_EINVAL, "graph has isolated checks");
        dc_max = std::max<int32_t>(dc_max, (int32_t)(cn_ptr[i + 1] - cn_ptr[i]));
        int64_t prev = -1;
        for (int64_t e = cn_ptr[i]; e < cn_ptr[i + 1]; ++e) {
            const int64_t j = edge_vn[e];
            if (j < 0 || j >= n) return fail(QSG_EINVAL, "row " + std::to_string(i) + ": column out of range");
            if (j <= prev) return fail(QSG_EINVAL, "row " + std::to_string(i) + ": columns not strictly increasing");
            if (edge_sym[e] < 1 || edge_sym[e] > 3) return fail(QSG_EINVAL, "symbol is not a nonzero Pauli");
            prev = j;
            g->edge_cn[e] = i;
            vdeg[j]++;
        }
    }
    int32_t dv_max = 0;
    g->vn_ptr.assign(n + 1, 0);
    for (int j = 0; j < n; ++j) {
        if (vdeg[j] == 0) return fail(QSG_EINVAL, "graph has isolated qubits");
        dv_max = std::max<int32_t>(dv_max, (int32_t)vdeg[j]);
        g->vn_ptr[j + 1] = g->vn_ptr[j] + vdeg[j];
    }
    // vn_order: edges of each qubit in ascending check (= canonical) order
    g->vn_order.assign(E, 0);
    std::vector<int64_t> fill(g->vn_ptr.begin(), g->vn_ptr.end() - 1);
    std::vector<int32_t> pos_in_vn(E);
    for (int64_t e = 0; e < E; ++e) {
        const int64_t j = edge_vn[e];
        pos_in_vn[e] = (int32_t)(fill[j] - g->vn_ptr[j]);
        g->vn_order[fill[j]++] = e;
    }
    g->dc_max = dc_max;
    g->dv_max = dv_max;
    g->n_pad = next_pow2(std::max(n, 32));
    g->log2_npad = 0;
    while ((1 << g->log2_npad) < g->n_pad) ++g->log2_npad;
    g->m_pad = (m + 31) / 32 * 32;

    // kernel kind: generalized-bicycle circulant codes (code.py:201-231) with
    // |a| = |b| = W get the specialised kernels; everything else the generic
    // table-driven ones.
    int kind = 0;
    if (n % 2 == 0 && m == n && n / 2 >= 32 && dv_max % 2 == 0 && bicycle_w_supported(dv_max / 2) &&
        (int64_t)dv_max * g->n_pad <= 65536) {
        const int32_t ell = n / 2, W = dv_max / 2;
        std::vector<int32_t> a, b;
        for (int64_t e = cn_ptr[0]; e < cn_ptr[1]; ++e)
            (edge_vn[e] < ell ? a : b).push_back((int32_t)(edge_vn[e] < ell ? edge_vn[e] : edge_vn[e] - ell));
        if ((int)a.size() == W && (int)b.size() == W) {
            std::vector<int64_t> cp, ev;
            std::vector<uint8_t> es;
            gb_rows(ell, a.data(), W, b.data(), W, cp, ev, es);
            bool same = (int64_t)ev.size() == E;
            for (int i = 0; same && i <= m; ++i) same = cp[i] == cn_ptr[i];
            for (int64_t e = 0; same && e < E; ++e) same = ev[e] == edge_vn[e] && es[e] == edge_sym[e];
            if (same) {
                kind = W;
                g->ell = ell;
                for (int k = 0; k < W; ++k) { g->gb_a[k] = a[k]; g->gb_b[k] = b[k]; }
            }
        }
    }
    // threads per frame: every thread of a generic kernel owns <= 32 checks
    // (register bit masks)
    const int nodes = std::max(n, m);
    if (nodes <= 32 * 12) g->threads = 32;
    else if (m <= 128 * 32) g->threads = 128;
    else return fail(QSG_EUNSUPPORTED, "more than 4096 checks");
    // bicycle kernels: about four circulant indices per thread (measured:
    // l = 127 fastest on 32 threads, l = 160-255 on 64, l = 320-511 on 128)
    if (kind > 0) g->threads = g->ell <= 128 ? 32 : (g->ell <= 256 ? 64 : 128);
    if (const char *env = std::getenv("QSG_THREADS")) {  // diagnostics: force 32 / 64 / 128 (bicycle)
        const int t = std::atoi(env);
        if (kind > 0 && (t == 32 || t == 64 || t == 128)) g->threads = t;
    }
    if (kind > 0) {
        g->nw = (g->ell + 31) / 32;
        const int lpw = g->threads / (2 * g->nw);  // lanes per syndrome word
        if (lpw < 1) {
            // too few threads for one lane per syndrome word (only reachable
            // through QSG_THREADS): the generic kernels, with their own
            // thread rule and no circulant description
            kind = 0;
            g->ell = g->nw = g->lpw = 0;
            for (int k = 0; k < 8; ++k) g->gb_a[k] = g->gb_b[k] = 0;
            if (nodes <= 32 * 12) g->threads = 32;
            else if (m <= 128 * 32) g->threads = 128;
            else return fail(QSG_EUNSUPPORTED, "more than 4096 checks");
        } else {
            int p2 = 1;
            while (p2 * 2 <= lpw && p2 * 2 <= 32) p2 *= 2;
            g->lpw = p2;
        }
    }
    g->kind = kind;
    if (kind == 0) {
        if (dc_max > qsg::kGenericMaxDeg || dv_max > qsg::kGenericMaxDeg)
            return fail(QSG_EUNSUPPORTED, "node degree exceeds the generic kernel limit (32)");
        if ((int64_t)dv_max * g->n_pad * 4 >= (1 << 24))
            return fail(QSG_EUNSUPPORTED, "graph too large for 24-bit slot offsets");
    }

    // check table: one row of row_words (odd) u32 per check: byte offsets of
    // the check's edges in canonical order (generic rows also carry the edge
    // symbol in bits 30-31) and an info word at index dc_max (bicycle: 1 for
    // X checks, 0 for Z checks; generic: the degree).
    const int mp = g->m_pad, np_ = g->n_pad;
    // bicycle rows: 2W u16 slot indices (W words, made odd); generic rows:
    // dc_max u32 entries + info word (made odd)
    int rw = kind > 0 ? kind : dc_max + 1;
    if (rw % 2 == 0) ++rw;
    g->row_words = rw;
    std::vector<uint32_t> cn_tab((size_t)mp * rw, 0);
    std::vector<uint8_t> vn_sym((size_t)dv_max * np_, 0), vn_deg(np_, 0);
    std::vector<int32_t> slot_edge((size_t)dv_max * np_, -1);
    for (int i = 0; i < m; ++i) {
        uint32_t *row = &cn_tab[(size_t)i * rw];
        uint16_t *row16 = reinterpret_cast<uint16_t *>(row);
        if (kind == 0) row[dc_max] = (uint32_t)(cn_ptr[i + 1] - cn_ptr[i]);
        for (int64_t e = cn_ptr[i]; e < cn_ptr[i + 1]; ++e) {
            const int k = (int)(e - cn_ptr[i]);
            const uint32_t slot = (uint32_t)pos_in_vn[e] * np_ + (uint32_t)edge_vn[e];
            if (kind > 0) row16[k] = (uint16_t)slot;
            else row[k] = slot * 4u | (uint32_t)edge_sym[e] << 30;
            slot_edge[slot] = (int32_t)e;
        }
    }
    for (int j = 0; j < n; ++j) {
        vn_deg[j] = (uint8_t)vdeg[j];
        for (int64_t q = g->vn_ptr[j]; q < g->vn_ptr[j + 1]; ++q)
            vn_sym[(size_t)(q - g->vn_ptr[j]) * np_ + j] = edge_sym[g->vn_order[q]];
    }
    if (g->device < 0) {
        g->tab_bytes = g->group_bytes = 0;
        return QSG_OK;
    }
    int rc;
    if ((rc = upload(&g->d_cn_tab, cn_tab)) || (rc = upload(&g->d_slot_edge, slot_edge))) return rc;
    if (kind > 0) {
        // Min-sum checks are order-free (min1/min2 with multiplicity, sign
        // XOR), so their rows can list edges in exponent order: X check c
        // at columns c + a_k, l + c + b_k; Z check c at c - b_k, l + c - a_k
        // (mod l).  Lanes (consecutive c) then touch consecutive qubits:
        // ~1.1 shared-memory wavefronts per access instead of ~1.75 with the
        // row-sorted canonical order, whose position k jumps between
        // exponents across the wrap.  BP4 keeps the canonical order (its
        // prefix / suffix products round order-dependently, and the oracle
        // multiplies in canonical order).
        const int l = g->ell, W = kind;
        std::vector<uint32_t> tab_x((size_t)mp * rw, 0);
        for (int i = 0; i < m; ++i) {
            const bool zc = i >= l;
            const int c = zc ? i - l : i;
            uint16_t *row16 = reinterpret_cast<uint16_t *>(&tab_x[(size_t)i * rw]);
            for (int k = 0; k < 2 * W; ++k) {
                const bool left = k < W;
                const int e = left ? (zc ? g->gb_b[k] : g->gb_a[k]) : (zc ? g->gb_a[k - W] : g->gb_b[k - W]);
                const int col = (left ? 0 : l) + (zc ? ((c - e) % l + l) % l : (c + e) % l);
                int64_t hit = -1;
                for (int64_t q = cn_ptr[i]; q < cn_ptr[i + 1]; ++q)
                    if (edge_vn[q] == col) hit = q;
                if (hit < 0) return fail(QSG_EINVAL, "internal: bicycle row does not match its exponents");
                row16[k] = (uint16_t)((uint32_t)pos_in_vn[hit] * np_ + (uint32_t)col);
            }
        }
        if ((rc = upload(&g->d_cn_tab_x, tab_x))) return rc;
    }
    if (kind == 0) {
        if ((rc = upload(&g->d_vn_sym, vn_sym)) || (rc = upload(&g->d_vn_deg, vn_deg))) return rc;
    }
    std::vector<int32_t> cp32(g->cn_ptr.begin(), g->cn_ptr.end()), ev32(g->edge_vn.begin(), g->edge_vn.end());
    if ((rc = upload(&g->d_cn_ptr, cp32)) || (rc = upload(&g->d_edge_vn, ev32)) ||
        (rc = upload(&g->d_edge_sym, g->edge_sym)))
        return rc;

    // shared-memory footprint
    size_t tab = (size_t)mp * rw * 4;
    if (kind == 0) tab += (size_t)dv_max * np_ + np_;
    if (kind > 0) tab += 16 * 4;  // circulant exponents
    g->tab_bytes = (uint32_t)((tab + 15) / 16 * 16);
    const int T = g->threads;
    size_t off = (size_t)dv_max * np_ * 4;             // messages
    g->off_ehat = (uint32_t)off;
    if (kind == 0) off += (size_t)np_ * 4;             // bicycle: aliases the messages
    g->off_bits = (uint32_t)off; off += (size_t)16 * (g->nw + 1);
    g->off_synw = (uint32_t)off; off += (size_t)8 * g->nw;
    g->off_resw = (uint32_t)off; off += (size_t)8 * g->nw;
    off = (off + 7) / 8 * 8;
    // scratch: group_sum slots, the frame index (8 B), the per-group tallies (24 B)
    g->off_scratch = (uint32_t)off; off += 2 * (T / 32) * 4 + 8 + 24;
    g->group_bytes = (uint32_t)((off + 15) / 16 * 16);
    return QSG_OK;
}

int validate_cfg(const qsg_decoder_cfg *c)
{
    if (!c) return fail(QSG_EINVAL, "null decoder config");
    if (c->variant < QSG_BP4 || c->variant > QSG_SAGMS) return fail(QSG_EINVAL, "unknown variant");
    if (c->vn_mode != QSG_VN_MARGINAL && c->vn_mode != QSG_VN_ADDITIVE) return fail(QSG_EINVAL, "unknown vn_mode");
    if (c->l_max < 1) return fail(QSG_EINVAL, "l_max must be at least 1");
    if (c->variant == QSG_SMS && !(c->alpha > 0.0 && c->alpha <= 1.0))
        return fail(QSG_EINVAL, "sms requires alpha in (0, 1]");
    if (c->variant == QSG_SAGMS) {  // GainParams.__post_init__, decoder.py:75-88
        if (!(0.0 < c->alpha_min && c->alpha_min <= c->alpha_max && c->alpha_max <= 1.0))
            return fail(QSG_EINVAL, "need 0 < alpha_min <= alpha_max <= 1");
        if (!(c->eta_unsat >= 1.0)) return fail(QSG_EINVAL, "eta_unsat must be >= 1");
        if (c->alpha_max * c->eta_unsat > 1.0) return fail(QSG_EINVAL, "stability constraint alpha_max*eta_unsat <= 1 violated");
    }
    return QSG_OK;
}

// u >= t  <=>  (w >> 11) >= ceil(t * 2^53)  (channel.py:70-75, exact).
void thresholds(double eps, uint64_t K[3])
{
    const double t_x = 1.0 - eps, t_y = 1.0 - eps + eps / 3.0, t_z = 1.0 - eps / 3.0;
    K[0] = (uint64_t)std::ceil(t_x * 9007199254740992.0);
    K[1] = (uint64_t)std::ceil(t_y * 9007199254740992.0);
    K[2] = (uint64_t)std::ceil(t_z * 9007199254740992.0);
}

// The dynamic shared-memory limit is an attribute of the kernel FUNCTION
// (per device), and many graphs share one function; it is raised once to the
// device's opt-in maximum and never lowered, so no graph's launch can find it
// set below its own footprint by another graph (or another thread).  The
// launch's own smem argument still decides occupancy.
std::mutex g_attr_mu;
std::vector<std::pair<void *, int>> g_attr_done;

int raise_smem_limit(void *fn, int device, int max_smem)
{
    std::lock_guard<std::mutex> lock(g_attr_mu);
    for (const auto &d : g_attr_done)
        if (d.first == fn && d.second == device) return QSG_OK;
    QSG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
    g_attr_done.emplace_back(fn, device);
    return QSG_OK;
}

// Pick groups-per-CTA maximising resident frames per SM for one kernel.
int launch_cfg(qsg_graph *g, bool bp4, bool add, bool lean, void *fn, qsg::LaunchCfg *out)
{
    int max_smem = 0;
    QSG_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device));
    int rc = raise_smem_limit(fn, g->device, max_smem);
    if (rc) return rc;
    std::lock_guard<std::mutex> lock(g->mu);
    qsg::LaunchCfg &c = g->cfg_cache[bp4][add][lean];
    if (c.ok) { *out = c; return QSG_OK; }
    const int T = g->threads;
    cudaFuncAttributes fa;
    QSG_CUDA(cudaFuncGetAttributes(&fa, fn));
    // at most 640 threads per CTA, and no more than the register budget
    // (__maxnreg__, reg_budget in qsg_kernel.cuh) lets one CTA hold
    int gmax = std::min(640, fa.maxThreadsPerBlock) / T;
    int cap_sm = 1 << 30;         // QSG_MAX_FRAMES_PER_SM: tuning/diagnostics only
    if (const char *env = std::getenv("QSG_MAX_FRAMES_PER_SM")) cap_sm = std::max(1, std::atoi(env));
    int force_g = 0;              // QSG_GROUPS: tuning/diagnostics only
    if (const char *env = std::getenv("QSG_GROUPS")) force_g = std::atoi(env);
    qsg::LaunchCfg best;
    for (int G = 1; G <= gmax; ++G) {
        if (force_g > 0 && G != std::min(force_g, gmax)) continue;
        const size_t smem = g->tab_bytes + (size_t)G * g->group_bytes;
        if (smem > (size_t)max_smem) break;
        int nb = 0;
        QSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, G * T, smem));
        nb = std::min(nb, cap_sm / G);
        if (nb * G > best.ctas_per_sm * best.groups) {
            best.groups = G; best.ctas_per_sm = nb; best.smem = smem; best.ok = nb > 0;
            best.big_groups = 0;
        } else if (nb > 0 && nb * G == best.ctas_per_sm * best.groups) {
            best.big_groups = G; best.big_ctas_per_sm = nb; best.big_smem = smem;  // same frames, larger CTAs
        }
    }
    if (!best.ok) return fail(QSG_EUNSUPPORTED, "graph does not fit in shared memory");
    if (std::getenv("QSG_VERBOSE"))  // diagnostics
        std::fprintf(stderr, "qsg launch_cfg: kind %d T %d bp4 %d regs %d groups %d ctas/SM %d smem %zu (group %u, tab %u); "
                     "full batches: groups %d ctas/SM %d\n",
                     g->kind, T, (int)bp4, fa.numRegs, best.groups, best.ctas_per_sm, best.smem, g->group_bytes,
                     g->tab_bytes, best.big_groups ? best.big_groups : best.groups,
                     best.big_groups ? best.big_ctas_per_sm : best.ctas_per_sm);
    c = best;
    *out = best;
    return QSG_OK;
}

// (threads, n_pad) pairs with a compile-time qubit stride: the shapes that
// have a lean instance (qsg_inst.cuh)
bool lean_kernel_exists(const qsg_graph *g)
{
    if (g->kind <= 0) return false;
    const int T = g->threads, np = g->n_pad;
    return (T == 32 && (np == 256 || np == 128)) || (T == 64 && np == 512) || (T == 128 && (np == 512 || np == 1024));
}

int launch_decode(qsg_graph *g, const qsg_decoder_cfg *cfg, qsg::KParams &p, cudaStream_t st)
{
    const bool bp4 = cfg->variant == QSG_BP4, add = cfg->vn_mode == QSG_VN_ADDITIVE;
    if (!bp4 && g->d_cn_tab_x) p.cn_tab = g->d_cn_tab_x;
    // the lean instance (qsg_kernel.cuh) serves the production shape: no
    // traces, no e_hat, early stop, closed-form first iteration, 4 lanes per
    // syndrome word, gains from the table; QSG_NO_LEAN=1 disables it (tests)
    static const bool no_lean = std::getenv("QSG_NO_LEAN") != nullptr;
    const bool lean = !no_lean && lean_kernel_exists(g) && !add && p.first_fast && p.early_stop && !p.out_ehat &&
                      !p.tr_unsat && !p.tr_vn && !p.tr_cn && !p.tr_counts && g->lpw == 4 && p.m < qsg::kGainTab;
    void *fn = qsg::kernel_ptr(g->kind, g->threads, bp4, add,
                               g->kind > 0 ? g->n_pad : std::max(g->dc_max, g->dv_max), lean);
    if (!fn) return fail(QSG_EUNSUPPORTED, "no kernel for this graph kind");
    qsg::LaunchCfg lc;
    int rc = launch_cfg(g, bp4, add, lean, fn, &lc);
    if (rc) return rc;
    if (p.count == 0) return QSG_OK;
    // a batch that fills every SM runs in the largest CTAs holding the same
    // number of frames per SM (+1-1.5% measured: one table copy per SM, an
    // even spread of the warps over the schedulers); smaller batches keep
    // the small CTAs, which reach more SMs
    if (lc.big_groups > 0 && p.count >= (int64_t)lc.big_groups * lc.big_ctas_per_sm * g->num_sms) {
        lc.groups = lc.big_groups; lc.ctas_per_sm = lc.big_ctas_per_sm; lc.smem = lc.big_smem;
    }
    const int64_t want = (p.count + lc.groups - 1) / lc.groups;
    const int grid = (int)std::min<int64_t>(want, (int64_t)lc.ctas_per_sm * g->num_sms);
    unsigned long long *queue = nullptr;
    // the zeroing of the stream's frame-queue counter and the launch that
    // consumes it are enqueued under the graph lock, so two host threads
    // sharing (graph, stream) cannot interleave memset, memset, kernel, kernel
    std::lock_guard<std::mutex> lock(g->mu);
    auto it = g->queues.find(st);
    if (it == g->queues.end()) {
        QSG_CUDA(cudaMalloc((void **)&queue, sizeof(unsigned long long)));
        g->queues.emplace(st, queue);
    } else {
        queue = it->second;
    }
    QSG_CUDA(cudaMemsetAsync(queue, 0, sizeof(unsigned long long), st));
    p.queue = queue;
    p.zero = 0;  // queue_fetch: opaque zero offset (keeps the frame-queue atomic un-aggregated)
    p.groups = lc.groups;
    void *args[] = {&p};
    cudaError_t err = cudaLaunchKernel(fn, dim3(grid), dim3(lc.groups * g->threads), args, lc.smem, st);
    if (err != cudaSuccess) return fail(QSG_ECUDA, std::string("decode launch: ") + cudaGetErrorString(err));
    return QSG_OK;
}

void fill_graph_params(const qsg_graph *g, qsg::KParams &p)
{
    p.cn_tab = g->d_cn_tab;
    p.vn_sym = g->d_vn_sym; p.vn_deg = g->d_vn_deg; p.slot_edge = g->d_slot_edge;
    p.n = g->n; p.m = g->m; p.n_pad = g->n_pad; p.log2_npad = g->log2_npad; p.m_pad = g->m_pad;
    p.dc_max = g->dc_max; p.dv_max = g->dv_max; p.row_words = g->row_words; p.E = g->E;
    p.ell = g->ell; p.nw = g->nw; p.lpw = g->lpw;
    for (int k = 0; k < 8; ++k) { p.gb_a[k] = g->gb_a[k]; p.gb_b[k] = g->gb_b[k]; }
    p.off_ehat = g->off_ehat; p.off_bits = g->off_bits; p.off_synw = g->off_synw;
    p.off_resw = g->off_resw; p.off_scratch = g->off_scratch;
    p.tab_bytes = g->tab_bytes; p.group_bytes = g->group_bytes;
}

void fill_cfg_params(const qsg_decoder_cfg *c, double l0, qsg::KParams &p)
{
    p.gain_mode = c->variant == QSG_SMS ? 1 : (c->variant == QSG_SAGMS ? 2 : 0);
    p.l_max = c->l_max;
    p.early_stop = c->early_stop ? 1 : 0;
    p.l0 = (float)l0;
    // vn_F constant from the fp32 prior, in double (the oracle's qo_vn_kapc)
    p.kapc = (float)std::exp(-(double)p.l0);
    // decoder.py:405-406 (marginal init :255-261), double then one rounding
    double v0 = c->vn_mode == QSG_VN_MARGINAL ? std::log1p(std::exp(-l0)) + l0 - 0.6931471805599453 : l0;
    v0 = std::min(64.0, std::max(-64.0, v0));
    p.v0 = (float)v0;
    p.alpha = (float)c->alpha;
    p.amin = c->alpha_min; p.amax = c->alpha_max; p.eta = c->eta_unsat;
    // first check update in closed form (decode_kernel, cn_phase_first):
    // bicycle kernels with v0 > 0; BP4 magnitudes by the shared recipe
    p.first_fast = (p.ell > 0 && p.v0 > 0.0f && p.dv_max <= 16) ? 1 : 0;  // bicycle: D = 2W <= 16
    if (p.first_fast && c->variant == QSG_BP4) {
        const int D = p.dv_max;  // bicycle: every check and qubit has degree 2W
        float x[16], mag[16];
        for (int k = 0; k < D; ++k) x[k] = std::min(p.v0, 64.0f);
        qsg::bp4_mags(x, D, mag);
        for (int k = 0; k < D; ++k) p.first_bp4[k] = qsg::f2u(mag[k]);
    }
    // SAGMS gains per unsat count (decoder.py:464-465), the kernel's double
    // recipe evaluated here once instead of a double division per iteration
    // and frame; volatile keeps each product rounded (no contraction)
    p.use_gtab = (p.gain_mode == 2 && p.m < qsg::kGainTab) ? 1 : 0;
    if (p.gain_mode != 2 && p.m < qsg::kGainTab) {
        // lean kernels read the gains of every variant from the table
        const float gc = p.gain_mode == 1 ? p.alpha : 1.0f;
        for (int u = 0; u <= p.m; ++u) p.gtab[2 * u] = p.gtab[2 * u + 1] = gc;
    }
    if (p.use_gtab) {
        for (int u = 0; u <= p.m; ++u) {
            const double gamma = (double)u / (double)p.m;
            volatile double prod = (p.amax - p.amin) * gamma;
            const double base = p.amax - prod;
            volatile double b1 = base * 1.0, be = base * p.eta;
            p.gtab[2 * u] = (float)b1;
            p.gtab[2 * u + 1] = (float)be;
        }
    }
}

// ---- standalone sampling / syndrome kernels ----------------------------------
__global__ void sample_kernel(int32_t n, uint64_t seed, int64_t start, int64_t count, uint64_t kx,
                              uint64_t ky, uint64_t kz, uint8_t *out)
{
    const int nblk = (n + 3) >> 2;
    const int64_t total = count * nblk;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = t / nblk;
        const int b = (int)(t - f * nblk);
        const qsg::U64x4 w = qsg::philox4x64_10((uint64_t)b + 1, seed, (uint64_t)(start + f));
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (4 * b + q < n) out[f * n + 4 * b + q] = qsg::pauli_from_word(w.v[q], kx, ky, kz);
    }
}

__global__ void syndrome_kernel(int32_t n, int32_t m, const int32_t *cn_ptr, const int32_t *edge_vn,
                                const uint8_t *edge_sym, const uint8_t *e, int64_t B, uint8_t *syn)
{
    const int64_t total = B * m;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / m;
        const int i = (int)(t - b * m);
        uint32_t x = 0;
        for (int k = cn_ptr[i]; k < cn_ptr[i + 1]; ++k) {
            const uint32_t c = e[b * n + edge_vn[k]], s = edge_sym[k];
            x ^= ((c & 1u) & (s >> 1)) ^ ((c >> 1) & (s & 1u));
        }
        syn[t] = (uint8_t)x;
    }
}

// Row commutation (pauli.py:120-144 check_orthogonality, decoder-independent
// code validation): one thread per check i visits every check k > i sharing
// a column with it through the qubit lists, and evaluates the pair ONCE --
// at their first shared column -- by merging the two sorted rows and XORing
// trace_inner over the shared columns (pauli.py symplectic form: X=1, Z=2,
// Y=3; two Paulis anticommute iff x1 z2 ^ z1 x2).  O(m d_c d_v (2 d_c))
// instead of the reference's O(m^2) pair scan.  The lowest anticommuting pair
// (i * m + k) is kept with atomicMin, so the report is deterministic.
__global__ void commute_kernel(int32_t m, const int32_t *cn_ptr, const int32_t *edge_vn, const uint8_t *edge_sym,
                               const int32_t *vn_ptr, const int32_t *vn_order, const int32_t *edge_cn,
                               unsigned long long *first_bad)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const int b0 = cn_ptr[i], b1 = cn_ptr[i + 1];
        for (int e = b0; e < b1; ++e) {
            const int j = edge_vn[e];
            for (int q = vn_ptr[j]; q < vn_ptr[j + 1]; ++q) {
                const int e2 = vn_order[q];
                const int k = edge_cn[e2];
                if (k <= i) continue;
                // merge rows i and k: parity over shared columns, first shared column
                int a = b0, b = cn_ptr[k];
                const int a1 = b1, bend = cn_ptr[k + 1];
                int first = -1;
                uint32_t par = 0;
                while (a < a1 && b < bend) {
                    const int ca = edge_vn[a], cb = edge_vn[b];
                    if (ca < cb) { ++a; continue; }
                    if (cb < ca) { ++b; continue; }
                    if (first < 0) first = ca;
                    const uint32_t s = edge_sym[a], t = edge_sym[b];
                    par ^= ((s & 1u) & (t >> 1)) ^ ((s >> 1) & (t & 1u));
                    ++a; ++b;
                }
                if (first == j && par)
                    atomicMin(first_bad, (unsigned long long)i * (unsigned long long)m + (unsigned long long)k);
            }
        }
    }
}

int create_common(int32_t device, qsg_graph **out, qsg_graph **g)
{
    if (!out) return fail(QSG_EINVAL, "null output handle");
    *out = nullptr;
    if (device >= 0) {  // device -1: host-only layout (export/inspection, no decode)
        int ndev = 0;
        QSG_CUDA(cudaGetDeviceCount(&ndev));
        if (device >= ndev) return fail(QSG_EINVAL, "invalid device ordinal");
    } else if (device != -1) {
        return fail(QSG_EINVAL, "invalid device ordinal");
    }
    *g = new (std::nothrow) qsg_graph();
    if (!*g) return fail(QSG_ENOMEM, "host allocation failed");
    (*g)->device = device;
    if (device >= 0) {
        cudaError_t err = cudaDeviceGetAttribute(&(*g)->num_sms, cudaDevAttrMultiProcessorCount, device);
        if (err != cudaSuccess) {
            delete *g;
            return fail(QSG_ECUDA, std::string("cudaDeviceGetAttribute: ") + cudaGetErrorString(err));
        }
    }
    return QSG_OK;
}

}  // namespace

namespace qsg {
void *kernel_ptr(int W, int T, bool bp4, bool additive, int np, bool lean)
{
    switch (W) {
    case 0: return kernel_ptr_w0(T, bp4, additive, np, lean);
    case 2: return kernel_ptr_w2(T, bp4, additive, np, lean);
    case 3: return kernel_ptr_w3(T, bp4, additive, np, lean);
    case 4: return kernel_ptr_w4(T, bp4, additive, np, lean);
    case 5: return kernel_ptr_w5(T, bp4, additive, np, lean);
    case 6: return kernel_ptr_w6(T, bp4, additive, np, lean);
    case 8: return kernel_ptr_w8(T, bp4, additive, np, lean);
    default: return nullptr;
    }
}
}  // namespace qsg

extern "C" {

int qsg_abi_version(void) { return QSG_ABI_VERSION; }

#ifndef QSG_BUILD_ID
#define QSG_BUILD_ID "unknown"
#endif
const char *qsg_build_id(void) { return QSG_BUILD_ID; }

const char *qsg_last_error(void) { return g_last_error.c_str(); }

int qsg_graph_create_csr(int32_t n, int32_t m, const int64_t *cn_ptr, const int64_t *edge_vn,
                         const uint8_t *edge_sym, int32_t device, qsg_graph **out)
{
    qsg_graph *g = nullptr;
    int rc = create_common(device, out, &g);
    if (rc) return rc;
    DeviceGuard dg(device);
    rc = compile_layout(g, n, m, cn_ptr, edge_vn, edge_sym);
    if (rc) {
        if (device >= 0) free_device(g);
        delete g;
        return rc;
    }
    *out = g;
    return QSG_OK;
}

int qsg_graph_create_gb(int32_t ell, const int32_t *a, int32_t wa, const int32_t *b, int32_t wb,
                        int32_t device, qsg_graph **out)
{
    if (ell < 1) return fail(QSG_EINVAL, "ell must be positive");
    if (!a || !b || wa < 1 || wb < 1) return fail(QSG_EINVAL, "exponent set is empty");
    for (int pass = 0; pass < 2; ++pass) {  // GbSpec.__post_init__, code.py:56-65
        const int32_t *x = pass ? b : a;
        const int32_t w = pass ? wb : wa;
        for (int i = 0; i < w; ++i) {
            if (x[i] < 0 || x[i] >= ell) return fail(QSG_EINVAL, "exponents must lie in [0, ell)");
            for (int k = 0; k < i; ++k)
                if (x[k] == x[i]) return fail(QSG_EINVAL, "duplicate exponent");
        }
    }
    const int32_t m = 2 * ell, n = 2 * ell;
    std::vector<int64_t> cn_ptr, edge_vn;
    std::vector<uint8_t> edge_sym;
    gb_rows(ell, a, wa, b, wb, cn_ptr, edge_vn, edge_sym);
    return qsg_graph_create_csr(n, m, cn_ptr.data(), edge_vn.data(), edge_sym.data(), device, out);
}

int qsg_graph_destroy(qsg_graph *g)
{
    if (!g) return QSG_OK;
    if (g->device >= 0) {
        DeviceGuard dg(g->device);
        free_device(g);
    }
    delete g;
    return QSG_OK;
}

int qsg_graph_info(const qsg_graph *g, int32_t *n, int32_t *m, int64_t *E, int32_t *dc_max,
                   int32_t *dv_max, int32_t *kind, int32_t *threads)
{
    if (!g) return fail(QSG_EINVAL, "null graph");
    if (n) *n = g->n;
    if (m) *m = g->m;
    if (E) *E = g->E;
    if (dc_max) *dc_max = g->dc_max;
    if (dv_max) *dv_max = g->dv_max;
    if (kind) *kind = g->kind;
    if (threads) *threads = g->threads;
    return QSG_OK;
}

int qsg_graph_export(const qsg_graph *g, int64_t *edge_cn, int64_t *edge_vn, uint8_t *edge_sym,
                     int64_t *cn_ptr, int64_t *vn_order, int64_t *vn_ptr)
{
    if (!g) return fail(QSG_EINVAL, "null graph");
    auto cp = [](auto *dst, const auto &v) {
        if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(edge_cn, g->edge_cn); cp(edge_vn, g->edge_vn); cp(edge_sym, g->edge_sym);
    cp(cn_ptr, g->cn_ptr); cp(vn_order, g->vn_order); cp(vn_ptr, g->vn_ptr);
    return QSG_OK;
}

int qsg_graph_check_commute(const qsg_graph *g, int32_t *commutes, int64_t *bad_pair)
{
    if (!g) return fail(QSG_EINVAL, "null graph");
    if (g->device < 0) return fail(QSG_EINVAL, "graph was created host-only (device -1)");
    if (!commutes) return fail(QSG_EINVAL, "null output");
    DeviceGuard dg(g->device);
    std::vector<int32_t> vp(g->vn_ptr.begin(), g->vn_ptr.end()), vo(g->vn_order.begin(), g->vn_order.end()),
        ec(g->edge_cn.begin(), g->edge_cn.end());
    int32_t *d_vp = nullptr, *d_vo = nullptr, *d_ec = nullptr;
    unsigned long long *d_bad = nullptr;
    const unsigned long long none = ~0ull;
    unsigned long long bad = none;
    int rc = QSG_OK;
    cudaError_t err = cudaSuccess;
    if ((rc = upload(&d_vp, vp)) || (rc = upload(&d_vo, vo)) || (rc = upload(&d_ec, ec))) goto done;
    if ((err = cudaMalloc((void **)&d_bad, sizeof(bad))) != cudaSuccess ||
        (err = cudaMemcpy(d_bad, &none, sizeof(none), cudaMemcpyHostToDevice)) != cudaSuccess)
        goto done;
    commute_kernel<<<(g->m + 127) / 128, 128>>>(g->m, g->d_cn_ptr, g->d_edge_vn, g->d_edge_sym, d_vp, d_vo, d_ec,
                                                  d_bad);
    if ((err = cudaGetLastError()) != cudaSuccess ||
        (err = cudaMemcpy(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost)) != cudaSuccess)
        goto done;
    *commutes = bad == none ? 1 : 0;
    if (bad_pair) {
        bad_pair[0] = bad == none ? -1 : (int64_t)(bad / (unsigned long long)g->m);
        bad_pair[1] = bad == none ? -1 : (int64_t)(bad % (unsigned long long)g->m);
    }
done:
    cudaFree(d_vp); cudaFree(d_vo); cudaFree(d_ec); cudaFree(d_bad);
    if (rc) return rc;
    if (err != cudaSuccess) return fail(QSG_ECUDA, std::string("check_commute: ") + cudaGetErrorString(err));
    return QSG_OK;
}

int qsg_decode_syndromes(const qsg_graph *gc, const qsg_decoder_cfg *cfg, double l0,
                         const uint8_t *syndromes_dev, int64_t B, uint8_t *success_dev,
                         uint8_t *e_hat_dev, int64_t *iterations_dev, const qsg_trace *trace,
                         void *stream)
{
    qsg_graph *g = const_cast<qsg_graph *>(gc);
    if (!g) return fail(QSG_EINVAL, "null graph");
    if (g->device < 0) return fail(QSG_EINVAL, "graph was created host-only (device -1)");
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (B < 0) return fail(QSG_EINVAL, "negative batch size");
    if (B > 0 && (!syndromes_dev || !success_dev || !iterations_dev)) return fail(QSG_EINVAL, "null buffer");
    if (!std::isfinite(l0)) return fail(QSG_EINVAL, "prior llr must be finite");
    DeviceGuard dg(g->device);
    qsg::KParams p{};
    fill_graph_params(g, p);
    fill_cfg_params(cfg, l0, p);
    p.sample = 0;
    p.syn_in = syndromes_dev;
    p.count = B;
    p.out_flag = success_dev;
    p.out_iters = iterations_dev;
    p.out_ehat = e_hat_dev;
    if (trace) {
        p.tr_unsat = trace->unsat; p.tr_vn = trace->vn_msgs; p.tr_cn = trace->cn_msgs;
        p.tr_counts = trace->counts;
    }
    return launch_decode(g, cfg, p, (cudaStream_t)stream);
}

int qsg_decode_syndromes_packed(const qsg_graph *gc, const qsg_decoder_cfg *cfg, double l0,
                                const uint32_t *syn_words_dev, int64_t B, uint8_t *success_dev,
                                uint8_t *e_hat_dev, int64_t *iterations_dev, void *stream)
{
    qsg_graph *g = const_cast<qsg_graph *>(gc);
    if (!g) return fail(QSG_EINVAL, "null graph");
    if (g->device < 0) return fail(QSG_EINVAL, "graph was created host-only (device -1)");
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (B < 0) return fail(QSG_EINVAL, "negative batch size");
    if (B > 0 && (!syn_words_dev || !success_dev || !iterations_dev)) return fail(QSG_EINVAL, "null buffer");
    if (!std::isfinite(l0)) return fail(QSG_EINVAL, "prior llr must be finite");
    DeviceGuard dg(g->device);
    qsg::KParams p{};
    fill_graph_params(g, p);
    fill_cfg_params(cfg, l0, p);
    p.sample = 0;
    p.syn_words = syn_words_dev;
    p.syn_wpf = (g->m + 31) / 32;
    p.count = B;
    p.out_flag = success_dev;
    p.out_iters = iterations_dev;
    p.out_ehat = e_hat_dev;
    return launch_decode(g, cfg, p, (cudaStream_t)stream);
}

int qsg_decode_frames(const qsg_graph *gc, const qsg_decoder_cfg *cfg, double epsilon, double epsilon0,
                      uint64_t seed, int64_t start, int64_t count, uint8_t *fails_dev,
                      int64_t *iterations_dev, uint8_t *e_hat_dev, int64_t *counters_dev, void *stream)
{
    qsg_graph *g = const_cast<qsg_graph *>(gc);
    if (!g) return fail(QSG_EINVAL, "null graph");
    if (g->device < 0) return fail(QSG_EINVAL, "graph was created host-only (device -1)");
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (!(epsilon >= 0.0 && epsilon < 1.0)) return fail(QSG_EINVAL, "epsilon must lie in [0, 1)");
    if (!(epsilon0 > 0.0 && epsilon0 < 1.0)) return fail(QSG_EINVAL, "epsilon0 must lie in (0, 1)");
    if (count < 0 || start < 0) return fail(QSG_EINVAL, "negative frame range");
    DeviceGuard dg(g->device);
    qsg::KParams p{};
    fill_graph_params(g, p);
    // prior_llr, channel.py:48-52
    fill_cfg_params(cfg, std::log(3.0 * (1.0 - epsilon0) / epsilon0), p);
    p.sample = 1;
    p.seed = seed;
    p.start = start;
    uint64_t K[3];
    thresholds(epsilon, K);
    p.kx = K[0]; p.ky = K[1]; p.kz = K[2];
    p.count = count;
    p.out_flag = fails_dev;
    p.out_iters = iterations_dev;
    p.out_ehat = e_hat_dev;
    p.counters = counters_dev;
    return launch_decode(g, cfg, p, (cudaStream_t)stream);
}

int qsg_sample_errors(int32_t n, double epsilon, uint64_t seed, int64_t start, int64_t count,
                      uint8_t *errors_dev, int32_t device, void *stream)
{
    if (n < 1) return fail(QSG_EINVAL, "n must be at least 1");
    if (!(epsilon >= 0.0 && epsilon < 1.0)) return fail(QSG_EINVAL, "epsilon must lie in [0, 1)");
    if (count < 0 || start < 0) return fail(QSG_EINVAL, "negative frame range");
    if (count == 0) return QSG_OK;
    if (!errors_dev) return fail(QSG_EINVAL, "null buffer");
    DeviceGuard dg(device);
    uint64_t K[3];
    thresholds(epsilon, K);
    const int64_t total = count * ((n + 3) / 4);
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
    sample_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(n, seed, start, count, K[0], K[1], K[2], errors_dev);
    QSG_CUDA(cudaGetLastError());
    return QSG_OK;
}

int qsg_syndromes_of(const qsg_graph *g, const uint8_t *e_dev, int64_t B, uint8_t *syn_dev, void *stream)
{
    if (!g) return fail(QSG_EINVAL, "null graph");
    if (g->device < 0) return fail(QSG_EINVAL, "graph was created host-only (device -1)");
    if (B < 0) return fail(QSG_EINVAL, "negative batch size");
    if (B == 0) return QSG_OK;
    if (!e_dev || !syn_dev) return fail(QSG_EINVAL, "null buffer");
    DeviceGuard dg(g->device);
    const int64_t total = B * g->m;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
    syndrome_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(g->n, g->m, g->d_cn_ptr, g->d_edge_vn,
                                                            g->d_edge_sym, e_dev, B, syn_dev);
    QSG_CUDA(cudaGetLastError());
    return QSG_OK;
}

}  // extern "C"
