// Persistent fused decode kernel for sm_100a.
//
// One "group" of T threads owns one frame at a time; a CTA holds G groups and
// every group pulls frame indices from a global atomic queue until the batch
// is exhausted (load balance across frames that stop after 2 or after 100
// iterations).  Per frame the group runs, entirely in shared memory:
//
//   sample (Philox, channel.py:55-76) -> syndrome (decoder.py:303-309) ->
//   for ell = 1..l_max (decoder.py:422-469):
//     R: residual = syndrome ^ synd(e_hat), unsat via popc + group reduce
//     exit on success / l_max; SAGMS gains from gamma (decoder.py:462-467)
//     C: check-node update (min1/min2/sign, or BP4 in the product domain),
//        decoder.py:311-338
//     V: qubit-node update (marginal or additive), decoder.py:340-359, which
//        also produces the next iteration's hard decision (the reduceat sums
//        of hard_decisions, decoder.py:292-301, are the same sums).
//
// Message storage: ONE fp32 word per edge, updated in place (each edge is
// owned by exactly one check and one qubit, and the C and V phases are
// separated by group barriers).  Slot of the s-th edge of qubit j (qubit
// order = ascending check index, code.py:171) is s * n_pad + j, so qubit
// reads/writes are unit-stride across the group (conflict-free).  Checks
// reach their edges through a per-graph table, one row of `row_words` (odd,
// so rows start in distinct banks) u32 words per check: generic rows hold
// byte offsets (+ the edge symbol) in canonical order and an info word at
// index dc_max; bicycle rows hold u16 slot indices, in canonical order for
// BP4 (the order of its prefix / suffix products) and in exponent order for
// the order-free min-sum update (consecutive checks -> consecutive qubits,
// few bank conflicts).  Generic kernels keep hard decisions as one u32 per qubit.
//
// The fp32 recipes (qsg_math.cuh) run scalar or, where two independent
// evaluations exist, paired on FFMA2 / FADD2 / FMUL2 (qsg_math2.cuh) with
// bit-identical results.
//
// W > 0 selects the generalized-bicycle specialisation (circulant A, B with
// |a| = |b| = W, code.py:201-231): degrees, masks and numpy's pairwise
// summation tree are compile-time constants, thread t owns circulant index c
// (check c, check l+c, qubit c, qubit l+c), and the residual syndrome is
// computed bit-sliced -- hard decisions are ballot-packed into four l-bit
// circulant bitmaps (x/z bits of each block) and every 32-check syndrome
// word is the XOR of 2W rotated 32-bit windows of them.  W == 0 is the
// generic table-driven path (any graph).
#pragma once

#include <stdint.h>

#include "qsg_math.cuh"
#include "qsg_math2.cuh"
#include "qsg_philox.cuh"

namespace qsg {

constexpr int kGenericMaxDeg = 32;
// SAGMS gain table: (g0, g1) per unsat count 0..m, for m < kGainTab
constexpr int kGainTab = 1025;

struct KParams {
    // graph tables (global; copied to shared memory per CTA)
    const uint32_t *cn_tab;    // [m_pad][row_words] byte offsets (+ sym << 30 generic) + info
    const uint8_t *vn_sym;     // [dv_max][n_pad] generic only
    const uint8_t *vn_deg;     // [n_pad]         generic only
    const int32_t *slot_edge;  // [dv_max*n_pad]  canonical edge per slot (traces)
    int32_t n, m, n_pad, log2_npad, m_pad, dc_max, dv_max, row_words;
    int64_t E;
    // generalized-bicycle circulant description (W > 0 kernels)
    int32_t ell, nw, lpw;       // circulant size, 32-bit words per block, lanes per word
    int32_t gb_a[8], gb_b[8];   // exponents of a(x), b(x)
    // decoder
    int32_t gain_mode;  // 0: none (bp4/ms), 1: constant alpha (sms), 2: sagms
    int32_t l_max, early_stop;
    float l0, v0, alpha;
    float kapc;  // e^-l0 (vn_F)
    double amin, amax, eta;
    int32_t first_fast;         // bicycle kernels, v0 > 0: first check update from the values below
    uint32_t first_bp4[16];     // BP4: the first update's output bits at row position k (v0 inputs, sign +)
    int32_t use_gtab;           // SAGMS: gains from gtab (host double, decoder.py:464-465) when m < kGainTab
    float gtab[2 * kGainTab];   // gtab[2u] = (float)base(u), gtab[2u+1] = (float)(base(u) * eta), u = unsat
    // input
    int32_t sample;  // 1: sample frames on device; 0: read syndromes
    uint64_t seed;
    int64_t start;
    uint64_t kx, ky, kz;
    const uint8_t *syn_in;      // syndromes, one byte per check (decode_batch)
    const uint32_t *syn_words;  // or bit-packed, syn_wpf words per frame
    int32_t syn_wpf;
    int64_t count;
    // outputs
    uint8_t *out_flag;  // fails (sample) or success (syndromes)
    int64_t *out_iters;
    uint8_t *out_ehat;
    int64_t *counters;
    unsigned long long *queue;
    int32_t zero;  // always 0 (queue_fetch)
    // traces (syndrome mode)
    int32_t *tr_unsat;
    float *tr_vn, *tr_cn;
    int32_t *tr_counts;
    // layout (byte offsets inside one group's shared-memory area)
    int32_t groups;  // groups per CTA
    uint32_t tab_bytes, group_bytes;
    uint32_t off_ehat, off_bits, off_synw, off_resw, off_scratch;
};

// Frame-queue fetch by one thread.  On a warp-uniform address ptxas turns
// any atomic add into a warp-aggregated one (leader vote, popc, and a
// shuffle of the result right after the atomic), which stalls the warp for
// the atomic's round trip at every frame start.  The address is therefore
// offset by threadIdx.x * KParams::zero (0 at run time, opaque to the
// compiler): a plain ATOMG whose result register is first read at the NEXT
// frame start, so the round trip overlaps the current frame.
__device__ __forceinline__ unsigned long long queue_fetch(unsigned long long *q, int32_t zero)
{
    return atomicAdd(q + threadIdx.x * (uint32_t)zero, 1ull);
}

// ---- optional-value arithmetic for compile-time masked reductions ---------
// np.add.reduceat over cv * anti_mask keeps the masked (+-0) entries in
// their tree positions; x + (+-0) == x, so dropping them from the tree is
// value-identical.  With compile-time presence flags the dead adds vanish.
struct OptF {
    float v;
    bool p;
};
__device__ __forceinline__ OptF oadd(OptF a, OptF b)
{
    if (!a.p) return b;
    if (!b.p) return a;
    return OptF{a.v + b.v, true};
}

// numpy pairwise_sum over a[0..N-1] (loops_utils.h.src), N <= 128.
template <int N>
__device__ __forceinline__ OptF pairwise_c(const OptF *a)
{
    if constexpr (N < 8) {
        OptF r{0.0f, false};
#pragma unroll
        for (int i = 0; i < N; ++i) r = oadd(r, a[i]);
        return r;
    } else {
        static_assert(N <= 128, "degree too large");
        OptF r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = a[k];
        constexpr int lim = N - (N % 8);
#pragma unroll
        for (int i = 8; i < lim; i += 8)
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = oadd(r[k], a[i + k]);
        OptF res = oadd(oadd(oadd(r[0], r[1]), oadd(r[2], r[3])),
                        oadd(oadd(r[4], r[5]), oadd(r[6], r[7])));
#pragma unroll
        for (int i = lim; i < N; ++i) res = oadd(res, a[i]);
        return res;
    }
}

// One reduceat segment: x0 + pairwise(x1..x_{N-1}).  Absent total -> 0.
template <int N>
__device__ __forceinline__ float segsum_c(const OptF *a)
{
    const OptF r = oadd(a[0], pairwise_c<N - 1>(a + 1));
    return r.p ? r.v : 0.0f;
}

// Runtime-length version for the generic path (masked entries are zeros).
__device__ __forceinline__ float pairwise_rt(const float *a, int n)
{
    if (n < 8) {
        float res = -0.0f;
        for (int i = 0; i < n; ++i) res += a[i];
        return res;
    }
    float r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = a[k];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] += a[i + k];
    float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
}
__device__ __forceinline__ float segsum_rt(const float *a, int n) { return a[0] + pairwise_rt(a + 1, n - 1); }

// segsum_rt for a run-time length d <= DM with every index compile-time (the
// generic kernels keep their per-node arrays in registers): the same numpy
// tree -- x0 + pairwise(x1..x_{d-1}), sequential below 8 elements, else 8
// strided accumulators, their tree and a sequential tail -- with the unused
// steps predicated off (adding -0.0 is an exact no-op).
template <int DM>
__device__ __forceinline__ float segsum_pred(const float (&x)[DM], int d)
{
    const int n = d - 1;  // length of the pairwise part x[1..d-1]
    float res = -0.0f;
    if (DM <= 8 || n < 8) {
#pragma unroll
        for (int k = 1; k < (DM < 8 ? DM : 8); ++k) res = res + (k <= n ? x[k] : -0.0f);
    } else {
        if constexpr (DM > 8) {
            float r[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = x[1 + k];
            const int lim = n - (n % 8);
#pragma unroll
            for (int i = 8; i + 8 <= DM - 1; i += 8)
#pragma unroll
                for (int k = 0; k < 8; ++k) r[k] = r[k] + (i < lim ? x[1 + i + k] : -0.0f);
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
#pragma unroll
            for (int i = 8; i < DM - 1; ++i) res = res + ((i >= lim && i < n) ? x[1 + i] : -0.0f);
        }
    }
    return x[0] + res;
}

// argmin over (0, mX, mZ, mY) with ties to the lowest code (np.argmin,
// decoder.py:301).
__device__ __forceinline__ uint32_t hard_decision(float mX, float mZ, float mY)
{
    float best = 0.0f;
    uint32_t e = 0;
    if (mX < best) { best = mX; e = 1; }
    if (mZ < best) { best = mZ; e = 2; }
    if (mY < best) { e = 3; }
    return e;
}

// The same argmin as the two bits the bicycle kernels ballot (x = code & 1,
// z = code >> 1), straight from the compares: Z beats {I, X} iff
// mZ < min(0, mX), Y beats all iff mY < min(0, mX, mZ), X needs mX < 0 and
// no Z win -- two FMNMX and four FSETP whose predicates feed VOTE directly
// (the code form costs three FSETP, two FSEL, three SEL and the bit tests).
struct HardXZ {
    bool x, z;
};
__device__ __forceinline__ HardXZ hard_xz(float mX, float mZ, float mY)
{
    const float t1 = fminf(0.0f, mX);
    const bool wz = mZ < t1;
    const bool wx = (mX < 0.0f) && !wz;
    const bool wy = mY < fminf(t1, mZ);
    return HardXZ{wy || wx, wy || wz};
}

// ---- group synchronisation ---------------------------------------------
template <int T>
__device__ __forceinline__ void group_sync(int g)
{
    if constexpr (T == 32) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(T) : "memory");
    }
}

template <int T>
__device__ __forceinline__ int group_sum(int v, int *scratch, int parity, int tid, int g)
{
    v = __reduce_add_sync(0xffffffffu, v);
    if constexpr (T == 32) {
        return v;
    } else {
        int *slot = scratch + parity * (T / 32);
        if ((tid & 31) == 0) slot[tid >> 5] = v;
        group_sync<T>(g);
        int s = 0;
#pragma unroll
        for (int w = 0; w < T / 32; ++w) s += slot[w];
        return s;
    }
}

// Shared-memory view of one group (frame) plus the per-CTA tables.
struct GroupMem {
    const uint32_t *tab;     // check rows (byte offsets into msg)
    const uint8_t *vn_sym;   // generic only
    const uint8_t *vn_deg;   // generic only
    const int32_t *gbexp;    // bicycle: a exponents [0, 8), b exponents [8, 16)
    unsigned char *msg;      // fp32 messages, slot-major
    uint32_t *ehat;          // generic only: one Pauli code per qubit
    uint32_t *bits;          // bicycle: XL, ZL, XR, ZR circulant bitmaps, nw+1 words each, word-interleaved (bidx)
    uint32_t *synw;          // bicycle: observed syndrome words (X checks, then Z checks)
    uint32_t *resw;          // bicycle: residual syndrome words
};

enum { kXL = 0, kZL = 1, kXR = 2, kZR = 3 };
// Bitmap word wd of block blk lives at gm.bits[4 * wd + blk]: the four words
// a warp ballots per 32-qubit step are one 16-byte store (the area is
// 16-byte aligned), and a bitmap is read with a stride of four words.
__device__ __forceinline__ int bidx(int blk, int wd) { return 4 * wd + blk; }
__device__ __forceinline__ void store_bits4(uint32_t *bits, int wd, uint32_t xl, uint32_t zl, uint32_t xr,
                                            uint32_t zr)
{
    *reinterpret_cast<uint4 *>(bits + 4 * wd) = make_uint4(xl, zl, xr, zr);
}

// ---- check-phase helpers ---------------------------------------------------
// The check phase is bound by the half-rate ALU pipe (FMNMX / FSETP / SEL /
// LOP3) and by issue; these helpers pin the cheapest forms: a plain 16-bit
// shared load (no PRMT unpacking of paired entries) and a single
// three-input LUT for the sign merge (the compiler otherwise splits it in
// two).  Moving the sign merge to the FMA pipe (IMAD.HI + IMAD) measured 5%
// slower: the extra issue slot costs more than the ALU relief.
__device__ __forceinline__ uint32_t lds_u16(const uint16_t *p)
{
    uint32_t v;
    asm("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}
__device__ __forceinline__ uint32_t sign_merge(uint32_t v, uint32_t mag)  // (v & 0x80000000) ^ mag
{
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x6a;" : "=r"(d) : "r"(v), "r"(0x80000000u), "r"(mag));
    return d;
}

// 32-bit shared-window addressing for the check phase: one LEA per edge
// (slot * 4 + frame base) instead of an offset add plus a window add.
// Volatile + clobber keep them ordered against the group barriers.
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float lds_a(uint32_t a)
{
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_a(uint32_t a, uint32_t v)
{
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// min(|a|, |b|) carrying sign(a) ^ sign(b): the check's sign product rides
// along the min1 reduction for free (FMNMX.XORSIGN).
__device__ __forceinline__ float min_xs(float a, float b)
{
    float d;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
// a ^ b kept opaque so the compiler cannot sink it below a select (which
// would turn 2 XORs per check into one per edge).
__device__ __forceinline__ uint32_t xor_pin(uint32_t a, uint32_t b)
{
    uint32_t d;
    asm("xor.b32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

__device__ __forceinline__ float lds_f(const unsigned char *base, uint32_t off)
{
    return *reinterpret_cast<const float *>(base + off);
}
__device__ __forceinline__ void sts_u(unsigned char *base, uint32_t off, uint32_t v)
{
    *reinterpret_cast<uint32_t *>(base + off) = v;
}

// ---- generic residual (table-driven, decoder.py:303-309) -------------------
// Bits of this thread's checks; bit t <-> check tid + t*T.
template <int T, int DM>
__device__ __forceinline__ uint32_t syndrome_bits_generic(const KParams &p, const GroupMem &gm, int tid)
{
    uint32_t bits = 0;
    const uint32_t jmask = (uint32_t)(p.n_pad - 1) << 2;
    const unsigned char *eb = reinterpret_cast<const unsigned char *>(gm.ehat);
    int t = 0;
#pragma unroll 1
    for (int i = tid; i < p.m; i += T, ++t) {
        const uint32_t *row = gm.tab + i * p.row_words;
        uint32_t x = 0;
        const int d = (int)row[p.dc_max];
#pragma unroll
        for (int k = 0; k < DM; ++k) {
            if (k < d) {
                const uint32_t ent = row[k];
                const uint32_t c = *reinterpret_cast<const uint32_t *>(eb + (ent & jmask));
                const uint32_t sym = ent >> 30;
                x ^= ((c & 1u) & (sym >> 1)) ^ ((c >> 1) & (sym & 1u));
            }
        }
        bits |= (x & 1u) << t;
    }
    return bits;
}

// ---- bit-sliced circulant syndrome (bicycle kernels) -----------------------
// Bits start..start+31 (indices mod l) of an l-bit circular bitmap B whose
// bits >= l are zero and which has one zero padding word (l >= 32).
__device__ __forceinline__ uint32_t circ_window(const uint32_t *B, int l, int start)
{
    const int q = start >> 5;
    uint32_t w = __funnelshift_r(B[4 * q], B[4 * (q + 1)], start & 31);  // words of one bitmap: stride 4
    const int n1 = l - start;
    if (n1 < 32) w |= B[0] << n1;
    return w;
}

// Syndrome words of the error held in the bitmaps (decoder.py:303-309 for
// the GB rows of code.py:216-223): X check c has parity
//   XOR_k z_L[c + a_k] ^ XOR_k z_R[c + b_k]          (indices mod l)
// and Z check l+c
//   XOR_k x_L[c - b_k] ^ XOR_k x_R[c - a_k].
// Word w < nw holds X checks 32w..32w+31, word nw + w the Z checks; T/(2 nw)
// lanes cooperate on a word and XOR-reduce with shuffles.  Writes
// out[w] = base[w] ^ parity (base may be null) and returns this thread's
// share of popc(out) (for the unsat count).
template <int W, int T>
__device__ __forceinline__ int circ_syndrome(const KParams &p, const GroupMem &gm, const uint32_t *base,
                                             uint32_t *out, int tid)
{
    const int nw = p.nw, l = p.ell;
    const int lpw = p.lpw;  // lanes per syndrome word (power of two <= 32, host-computed)
    const int w = tid / lpw, sub = tid - w * lpw;
    uint32_t acc = 0;
    bool zc = false;
    int ww = 0;
    if (w < 2 * nw) {
        zc = w >= nw;
        ww = zc ? w - nw : w;
        const uint32_t *BL = gm.bits + (zc ? kXL : kZL);
        const uint32_t *BR = gm.bits + (zc ? kXR : kZR);
        for (int k = sub; k < 2 * W; k += lpw) {
            const bool left = k < W;
            // X: left a_k, right b_k; Z: left -b_k, right -a_k
            const int e = gm.gbexp[(left != zc) ? k % W : 8 + k % W];
            int start = 32 * ww + (zc ? l - e : e);
            start = start >= l ? start - l : start;
            start = start >= l ? start - l : start;
            acc ^= circ_window(left ? BL : BR, l, start);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        if (o < lpw) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
    int cnt = 0;
    if (w < 2 * nw && sub == 0) {
        const int valid = l - 32 * ww;
        const uint32_t mask = valid >= 32 ? 0xffffffffu : ((1u << valid) - 1u);
        const uint32_t v = ((base ? base[w] : 0u) ^ acc) & mask;
        out[w] = v;
        cnt = __popc(v);
    }
    return cnt;
}

// The same syndrome with every loop-invariant part hoisted: a thread's word
// w, its 32-bit windows and the word's valid mask depend only on its lane
// and the code, so they are computed once per kernel, as shared-window byte
// addresses: lo[j] = address of B[q] | shift << 24, hi[j] = address of B[0]
// of that bitmap | wrap << 24, wrap = l - start when the window wraps, else
// 32 (PTX shl by >= 32 gives 0).  Unused windows point at a bitmap's zero
// padding word with shift 0 and wrap 32, so every window is evaluated
// without a branch.  Needs lpw >= 4 (at most ceil(2W / 4) windows per lane;
// the host guarantees it for every bicycle shape it builds, else
// circ_syndrome is used).
template <int W>
struct SynPlan {
    static constexpr int K = (2 * W + 3) / 4;
    uint32_t lo[K], hi[K];
    uint32_t mask;  // valid bits of word w (0 for idle lanes)
    int w;          // syndrome word (X words then Z words), -1 idle
    bool writer;    // first lane of its word
};

__device__ __forceinline__ uint32_t lds_u32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t n)  // x << n, 0 for n >= 32
{
    uint32_t d;
    asm("shl.b32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(n));
    return d;
}

template <int W, int T>
__device__ __forceinline__ SynPlan<W> syn_plan(const KParams &p, const GroupMem &gm, int tid)
{
    SynPlan<W> P;
    const int nw = p.nw, l = p.ell, lpw = p.lpw;
    const int w = tid / lpw, sub = tid - w * lpw;
    const uint32_t bits_s = smem_addr(gm.bits);
    const uint32_t zero = bits_s + 16u * (uint32_t)nw;  // XL padding word (always 0)
    P.w = -1; P.mask = 0u; P.writer = false;
#pragma unroll
    for (int j = 0; j < SynPlan<W>::K; ++j) {
        P.lo[j] = zero;
        P.hi[j] = zero | (32u << 24);
    }
    if (w < 2 * nw) {
        const bool zc = w >= nw;
        const int ww = zc ? w - nw : w;
        P.w = w;
        P.writer = sub == 0;
        const int valid = l - 32 * ww;
        P.mask = valid >= 32 ? 0xffffffffu : ((1u << valid) - 1u);
#pragma unroll
        for (int j = 0; j < SynPlan<W>::K; ++j) {
            const int k = sub + j * lpw;
            if (k < 2 * W) {
                const bool left = k < W;
                const int e = gm.gbexp[(left != zc) ? k % W : 8 + k % W];
                int start = 32 * ww + (zc ? l - e : e);
                start = start >= l ? start - l : start;
                start = start >= l ? start - l : start;
                const int blk = left ? (zc ? kXL : kZL) : (zc ? kXR : kZR);
                const uint32_t b0 = bits_s + 4u * (uint32_t)blk;
                const uint32_t n1 = (uint32_t)(l - start);
                P.lo[j] = (b0 + 16u * (uint32_t)(start >> 5)) | ((uint32_t)(start & 31) << 24);
                P.hi[j] = b0 | ((n1 < 32u ? n1 : 32u) << 24);
            }
        }
    }
    return P;
}

// BASE: out[w] = base[w] ^ parity (the residual against the observed
// syndrome); else out[w] = parity (a compile-time flag: a run-time null test
// of a shared-memory pointer costs eight instructions of generic-address
// arithmetic per iteration).
template <int W, int T, bool BASE>
__device__ __forceinline__ int circ_syndrome_plan(const SynPlan<W> &P, const GroupMem &gm, const uint32_t *base,
                                                  uint32_t *out, int lpw)
{
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < SynPlan<W>::K; ++j) {
        const uint32_t a = P.lo[j] & 0x00ffffffu, b = P.hi[j] & 0x00ffffffu;
        uint32_t x = __funnelshift_r(lds_u32(a), lds_u32(a + 16u), P.lo[j] >> 24);
        x |= shl_clamp(lds_u32(b), P.hi[j] >> 24);
        acc ^= x;
    }
    acc ^= __shfl_xor_sync(0xffffffffu, acc, 1);
    acc ^= __shfl_xor_sync(0xffffffffu, acc, 2);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1)
        if (o < lpw) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
    int cnt = 0;
    if (P.writer) {
        uint32_t v = acc;
        if constexpr (BASE) v ^= base[P.w];
        v &= P.mask;
        out[P.w] = v;
        cnt = __popc(v);
    }
    return cnt;
}

// Pack per-qubit Pauli codes (bytes in gm.ehat scratch) into the bitmaps.
template <int T>
__device__ __forceinline__ void bitmaps_from_bytes(const KParams &p, const GroupMem &gm, const uint8_t *e, int tid)
{
    const int l = p.ell;
    for (int c0 = tid & ~31; c0 < 32 * p.nw; c0 += T) {
        const int c = c0 + (tid & 31);
        const uint32_t eL = c < l ? e[c] : 0u, eR = c < l ? e[l + c] : 0u;
        const uint32_t xl = __ballot_sync(0xffffffffu, eL & 1u), zl = __ballot_sync(0xffffffffu, eL >> 1);
        const uint32_t xr = __ballot_sync(0xffffffffu, eR & 1u), zr = __ballot_sync(0xffffffffu, eR >> 1);
        if ((tid & 31) == 0) {
            const int wd = c0 >> 5;
            store_bits4(gm.bits, wd, xl, zl, xr, zr);
        }
    }
}

// ---- check-node phase (decoder.py:311-338) ---------------------------------
// Min-sum: the argmin edge gets min2 and all others min1, with ties at min1
// giving min2 == min1; so mag_e = (|v_e| == min1 ? min2 : min1) reproduces
// the first-argmin rule (:325-333) without tracking the index.  Signs: the
// extrinsic sign is (-1)^s_i * prod(sgn) * sgn_e (:314-316); messages are
// never -0.0, so sgn_e is the IEEE sign bit and the product is an XOR.
// Qubit->check messages are stored UNCLIPPED; the +-64 saturation of the
// qubit update (decoder.py:358) is applied here where they are consumed:
// every use is sign(v) or |clip(v)| = min(|v|, 64), and min1/min2 of the
// clipped magnitudes are min(min1, 64), min(min2, 64) (clip is monotone),
// with the |v_e| == min1 test unchanged whenever min1 < 64 and irrelevant
// (min2 == min1 == 64) otherwise.
// Split into the loads and the update so that callers can issue the loads
// of a second check before the first one's stores (the shared accesses are
// volatile asm, kept in program order).
template <int D>
__device__ __forceinline__ void cn_load(const uint16_t *row, uint32_t msg_s, uint32_t (&ad)[D], float (&v)[D])
{
#pragma unroll
    for (int k = 0; k < D; ++k) {
        ad[k] = msg_s + 4u * lds_u16(row + k);  // bicycle rows hold u16 slot indices
        v[k] = lds_a(ad[k]);
    }
}

template <int D, bool BP4>
__device__ __forceinline__ void cn_finish(const uint32_t (&ad)[D], const float (&v)[D], uint32_t sneg, float gain)
{
    if constexpr (BP4) {
        // product-form magnitudes (qsg_math.cuh bp4_mags, paired:
        // bp4_mags_fixed); the sign as in the min-sum branch
        uint32_t sx = sneg;
#pragma unroll
        for (int k = 0; k < D; ++k) sx ^= f2u(v[k]);
        const uint32_t sgn = sx & 0x80000000u;  // (-1)^s_i * prod sgn, as a sign bit
        float x[D], mag[D];
#pragma unroll
        for (int k = 0; k < D; ++k) x[k] = fminf(fabsf(v[k]), kClip);
        bp4_mags_fixed<D>(x, mag);
#pragma unroll
        for (int k = 0; k < D; ++k) sts_a(ad[k], (f2u(v[k]) & 0x80000000u) ^ f2u(mag[k]) ^ sgn);
    } else {
        // smallest and second smallest of |v| (with multiplicity), two at a
        // time: second' = min(second, max(min1, lo), hi).  min1 carries the
        // XOR of all message signs in its sign bit.
        float mn1, mn2;
        mn1 = min_xs(v[0], v[1]);
        mn2 = fmaxf(fabsf(v[0]), fabsf(v[1]));
#pragma unroll
        for (int k = 2; k + 1 < D; k += 2) {
            const float lo = min_xs(v[k], v[k + 1]), hi = fmaxf(fabsf(v[k]), fabsf(v[k + 1]));
            mn2 = fminf(fminf(mn2, fmaxf(fabsf(mn1), fabsf(lo))), hi);
            mn1 = min_xs(mn1, lo);
        }
        if constexpr (D % 2) {
            mn2 = fminf(mn2, fmaxf(fabsf(mn1), fabsf(v[D - 1])));
            mn1 = min_xs(mn1, v[D - 1]);
        }
        const uint32_t sgn = (f2u(mn1) ^ sneg) & 0x80000000u;  // (-1)^s_i * prod sgn
        const float a1 = fminf(fabsf(mn1), kClip), a2 = fminf(mn2, kClip);
        const uint32_t m1 = xor_pin(f2u(fminf(gain * a1, kClip)), sgn);
        const uint32_t m2 = xor_pin(f2u(fminf(gain * a2, kClip)), sgn);
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const uint32_t mag = fabsf(v[k]) == a1 ? m2 : m1;
            sts_a(ad[k], sign_merge(f2u(v[k]), mag));
        }
    }
}

// Both circulant halves (check c and l + c, qubit c and l + c) are inlined:
// more independent work per lane (+4-5% on the 128-thread min-sum kernels;
// +3.5% on BP4 at p >= 0.06 once its check update took the product form --
// the phi-sum form overflowed the instruction cache unrolled, -25%).

// First iteration (decoder.py:405-410): every qubit->check message is v0,
// so every check sees D equal inputs and its update is known in closed form:
// min-sum sends sign(s_i) gain_i min(v0, 64) on every edge (min1 = min2 =
// v0, sign product +), BP4 sends the product-form magnitude of D copies of
// min(v0, 64) at row position k (host-computed with the same recipe,
// KParams::first_bp4) with sign(s_i).  These are the words the general
// update stores (the -m gpu parity suite checks every frame bit for bit);
// the check phase of iteration 1 then costs a table load and a store per
// edge.  Needs v0 > 0 (then the hard decision of iteration 1 is I and the
// residual equals the syndrome).
template <int W, int T, bool BP4>
__device__ __forceinline__ void cn_phase_first(const KParams &p, const GroupMem &gm, float g0, float g1, int tid)
{
    constexpr int D = 2 * W;
    const int l = p.ell, nw = p.nw;
    const uint32_t msg_s = smem_addr(gm.msg);
    const float a = fminf(p.v0, kClip);
    const uint32_t m0 = f2u(fminf(g0 * a, kClip)), m1 = f2u(fminf(g1 * a, kClip));
#pragma unroll 1
    for (int c = tid; c < l; c += T) {
        const int bit = c & 31;
        // both checks' slot indices first: the stores are volatile (ordered
        // against the barriers), so a load issued after a store would wait
        // for it -- one table-load latency per edge otherwise
        uint32_t ad[2][D];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint16_t *row = reinterpret_cast<const uint16_t *>(gm.tab + (h * l + c) * p.row_words);
#pragma unroll
            for (int q = 0; q < D; ++q) ad[h][q] = msg_s + 4u * lds_u16(row + q);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int wd = h * nw + (c >> 5);
            const uint32_t s = (gm.synw[wd] >> bit) & 1u, r = (gm.resw[wd] >> bit) & 1u;
            const uint32_t sg = s << 31;
            const uint32_t ms = (r ? m1 : m0) ^ sg;
#pragma unroll
            for (int q = 0; q < D; ++q) sts_a(ad[h][q], BP4 ? (p.first_bp4[q] ^ sg) : ms);
        }
    }
}

template <int W, int T, bool BP4, int NP>
__device__ __forceinline__ void cn_phase(const KParams &p, const GroupMem &gm, uint32_t syn_bits,
                                         uint32_t res_bits, float g0, float g1, int tid)
{
    unsigned char *msg = gm.msg;
    if constexpr (W > 0) {
        const int l = p.ell, nw = p.nw;
        const uint32_t msg_s = smem_addr(msg);
#pragma unroll 1
        for (int c = tid; c < l; c += T) {
            // X check c and Z check l + c: both checks' loads first, then
            // the two updates
            constexpr int D = 2 * W;
            const int bit = c & 31;
            const int wd0 = c >> 5, wd1 = nw + (c >> 5);
            const uint32_t s0 = gm.synw[wd0] >> bit, r0 = gm.resw[wd0] >> bit;
            const uint32_t s1 = gm.synw[wd1] >> bit, r1 = gm.resw[wd1] >> bit;
            uint32_t ad0[D], ad1[D];
            float v0[D], v1[D];
#ifdef QSG_BP4_PAIR
            if constexpr (false) {
#else
            if constexpr (BP4) {
#endif
                // one check at a time: the product-form update is long enough
                // to hide its loads, and the second check's 2D live values
                // would push the kernel past its register budget
                cn_load<D>(reinterpret_cast<const uint16_t *>(gm.tab + c * p.row_words), msg_s, ad0, v0);
                cn_finish<D, BP4>(ad0, v0, s0 << 31, (r0 & 1u) ? g1 : g0);
                cn_load<D>(reinterpret_cast<const uint16_t *>(gm.tab + (l + c) * p.row_words), msg_s, ad1, v1);
                cn_finish<D, BP4>(ad1, v1, s1 << 31, (r1 & 1u) ? g1 : g0);
            } else {
                cn_load<D>(reinterpret_cast<const uint16_t *>(gm.tab + c * p.row_words), msg_s, ad0, v0);
                cn_load<D>(reinterpret_cast<const uint16_t *>(gm.tab + (l + c) * p.row_words), msg_s, ad1, v1);
                cn_finish<D, BP4>(ad0, v0, s0 << 31, (r0 & 1u) ? g1 : g0);
                cn_finish<D, BP4>(ad1, v1, s1 << 31, (r1 & 1u) ? g1 : g0);
            }
        }
    } else {
        constexpr uint32_t kAddr = 0x00ffffffu;  // generic entries carry sym << 30
        constexpr int DM = NP > 0 ? NP : kGenericMaxDeg;  // degree bound of this instantiation
        const uint32_t msg_s = smem_addr(msg);
        int t = 0;
#pragma unroll 1
        for (int i = tid; i < p.m; i += T, ++t) {
            const uint32_t *row = gm.tab + i * p.row_words;
            const uint32_t sneg = ((syn_bits >> t) & 1u) << 31;
            const float gain = ((res_bits >> t) & 1u) ? g1 : g0;
            const int d = (int)row[p.dc_max];
            uint32_t ad[DM];
            float v[DM];
            uint32_t sx = sneg;
#pragma unroll
            for (int k = 0; k < DM; ++k) {
                ad[k] = msg_s + (k < d ? (row[k] & kAddr) : 0u);
                v[k] = k < d ? lds_a(ad[k]) : __int_as_float(0x7f800000);  // +inf: neutral for min
                sx ^= k < d ? f2u(v[k]) : 0u;
            }
            const uint32_t sgn = sx & 0x80000000u;
            if constexpr (BP4) {
                // product-form magnitudes (qsg_math.cuh bp4_mags) for the
                // run-time degree d <= DM: the prefix (A, B) is kept per
                // edge, the suffix runs backwards alongside the merge (the
                // scalar recipe's operations; unused steps predicated off)
                uint32_t vs = 0;  // message sign bits
                float s[DM], A[DM], B[DM];
#pragma unroll
                for (int k = 0; k < DM; k += 2) {
                    vs |= (f2u(v[k]) >> 31) << k | (f2u(v[k + 1]) >> 31) << (k + 1);
                    const F2 e = exp_neg2(pk(-fminf(fabsf(v[k]), kClip), -fminf(fabsf(v[k + 1]), kClip)));
                    s[k] = lo(e); s[k + 1] = hi(e);
                }
                A[0] = 1.0f; B[0] = 0.0f;
#pragma unroll
                for (int j = 0; j + 1 < DM; ++j) {
                    const bool on = j + 1 < d;
                    A[j + 1] = on ? fmaf(s[j], B[j], A[j]) : A[j];
                    B[j + 1] = on ? fmaf(s[j], A[j], B[j]) : B[j];
                }
                float C = 1.0f, Dd = 0.0f;  // suffix of edge e (edges e+1 .. d-1)
#pragma unroll
                for (int e = DM - 1; e >= 1; e -= 2) {
                    // edges e and e - 1: ratios, then one paired logarithm
                    F2 eo[2] = {bc(1.0f), bc(1.0f)};
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int q = e - h;
                        if (q < d) {
                            const F2 t = mul2(bc(B[q]), pk(Dd, C));
                            eo[h] = fma2(bc(A[q]), pk(C, Dd), t);
                            const float Cn = fmaf(s[q], Dd, C), Dn = fmaf(s[q], C, Dd);
                            C = Cn; Dd = Dn;
                        }
                    }
                    const F2 m = bp4_out2(eo[0], eo[1]);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int q = e - h;
                        if (q < d) sts_a(ad[q], ((vs >> q) << 31) ^ f2u(h ? hi(m) : lo(m)) ^ sgn);
                    }
                }
            } else {
                float mn1 = __int_as_float(0x7f800000), mn2 = mn1;
#pragma unroll
                for (int k = 0; k < DM; ++k) {
                    const float a = fabsf(v[k]);
                    mn2 = fminf(mn2, fmaxf(mn1, a));
                    mn1 = fminf(mn1, a);
                }
                mn1 = fminf(mn1, kClip);
                mn2 = fminf(mn2, kClip);
                const uint32_t m1 = xor_pin(f2u(fminf(gain * mn1, kClip)), sgn);
                const uint32_t m2 = xor_pin(f2u(fminf(gain * mn2, kClip)), sgn);
#pragma unroll
                for (int k = 0; k < DM; ++k)
                    if (k < d) sts_a(ad[k], sign_merge(f2u(v[k]), fabsf(v[k]) == mn1 ? m2 : m1));
            }
        }
    }
}

// ---- qubit-node phase (decoder.py:340-359) + next hard decision ------------
// Marginal mode: both anticommuting beliefs of an edge contain that edge's
// own message c (b_a = l0 + tot_a - c), and logaddexp(u - c, v - c) =
// logaddexp(u, v) - c, so out = V[sym] - c with
//   V[S] = LAE(0, -(l0 + tot_S)) - LAE(-(l0 + tot_a1), -(l0 + tot_a2))
// computed once per qubit and symbol (the fp32 restatement's recipe; the
// oracle's fp32 path uses the same factorisation, its fp64 path the
// reference's literal per-edge form).  Returns the hard decision.
// NP > 0: the qubit stride n_pad is a compile-time constant, so the D column
// loads / stores use immediate offsets from one base (no address IMADs).
template <int W, int NP>
__device__ __forceinline__ void vn_load(uint32_t cs, uint32_t rowb, float (&c)[2 * W])
{
    if constexpr (NP > 0) rowb = 4u * NP;
#pragma unroll
    for (int s = 0; s < 2 * W; ++s) c[s] = lds_a(cs + s * rowb);
}

template <int W, bool ADD, int NP>
__device__ __forceinline__ HardXZ vn_finish(uint32_t cs, uint32_t rowb, const float (&c)[2 * W], float l0,
                                            float kapc)
{
    if constexpr (NP > 0) rowb = 4u * NP;
    constexpr int D = 2 * W;
    if constexpr (W <= 5 && !ADD) {
        // numpy's trees with the masks written out (segsum_c<D>): for d = 10
        //   S_X = x0 + P, S_Z = Q + z4, tot_Y = x0 + ((P + Q) + z4),
        //   P = (x1 + x2) + (x3 + x4), Q = (z0 + z1) + (z2 + z3);
        // for d <= 8 the sums run left to right,
        //   S_X = x0 + P, S_Z = Q + z_{W-1}, tot_Y = x0 + (((P + z0) + z1) ...),
        //   P = (x1 + x2) + ..., Q = (z0 + z1) + ... (W - 1 terms each).
        // P and Q, the two sums and the two beliefs therefore run as pairs
        // (x_{s+1}, z_s), (x0, z_{W-1}) on FADD2 -- the same additions in
        // half the issue slots -- and each pair is also the operand of its
        // two outgoing messages.
        F2 pr[W > 1 ? W - 1 : 1];
#pragma unroll
        for (int s = 0; s + 1 < W; ++s) pr[s] = pk(c[s + 1], c[W + s]);
        const F2 pe = pk(c[0], c[D - 1]);
        F2 PQ;
        float tY;
        if constexpr (W == 5) {
            PQ = add2(add2(pr[0], pr[1]), add2(pr[2], pr[3]));
            tY = c[0] + ((lo(PQ) + hi(PQ)) + c[D - 1]);
        } else {
            static_assert(W >= 2, "bicycle weight");
            PQ = pr[0];
#pragma unroll
            for (int s = 1; s + 1 < W; ++s) PQ = add2(PQ, pr[s]);
            float t = lo(PQ);
#pragma unroll
            for (int s = 0; s < W; ++s) t = t + c[W + s];
            tY = c[0] + t;
        }
        const F2 S = add2(pe, PQ);      // (S_X, S_Z)
        const F2 b2 = add2(bc(l0), S);  // (b_Z, b_X)
        const float bY = l0 + tY;
        const F2 v2 = add2(b2, vn_F2(hi(S), lo(S), bc(kapc)));  // (V[X], V[Z])
        const F2 oe = sub2(v2, pe);
        sts_a(cs, f2u(lo(oe)));  // clipped by the consumer
        sts_a(cs + (D - 1) * rowb, f2u(hi(oe)));
#pragma unroll
        for (int s = 0; s + 1 < W; ++s) {
            const F2 o = sub2(v2, pr[s]);
            sts_a(cs + (s + 1) * rowb, f2u(lo(o)));
            sts_a(cs + (W + s) * rowb, f2u(hi(o)));
        }
        return hard_xz(hi(b2), lo(b2), bY);
    }
    OptF ox[D], oz[D], oa[D];
#pragma unroll
    for (int s = 0; s < D; ++s) {
        // anti_X keeps Z-edges (z-bit), anti_Z keeps X-edges (x-bit)
        ox[s] = OptF{c[s], s >= W};
        oz[s] = OptF{c[s], s < W};
        oa[s] = OptF{c[s], true};
    }
    const float sZ = segsum_c<D>(ox), sX = segsum_c<D>(oz);  // tot_X, tot_Z
    const float bX = l0 + sZ;
    const float bZ = l0 + sX;
    const float tY = segsum_c<D>(oa);
    const float bY = l0 + tY;
    if constexpr (ADD) {
#pragma unroll
        for (int s = 0; s < D; ++s) sts_a(cs + s * rowb, f2u(l0 + (tY - c[s])));  // clipped by the consumer
    } else {
        // X-edge: self X, anti {Z, Y}; Z-edge: self Z, anti {X, Y}; no Y
        // edges, so V[X] = b_Z + F(S_Z), V[Z] = b_X + F(S_X) (vn_F)
        // both factors at once (FFMA2 / FADD2 / FMUL2, qsg_math2.cuh)
        const F2 v2 = add2(pk(bZ, bX), vn_F2(sZ, sX, bc(kapc)));
#pragma unroll
        for (int s = 0; s < W; ++s) {  // X-edge s and Z-edge W + s together
            const F2 o2 = sub2(v2, pk(c[s], c[W + s]));
            sts_a(cs + s * rowb, f2u(lo(o2)));  // clipped by the consumer
            sts_a(cs + (W + s) * rowb, f2u(hi(o2)));
        }
    }
    return hard_xz(bX, bZ, bY);
}

template <int W, bool ADD, int NP>
__device__ __forceinline__ HardXZ vn_update_fixed(unsigned char *col, uint32_t rowb, float l0, float kapc)
{
    const uint32_t cs = smem_addr(col);
    float c[2 * W];
    vn_load<W, NP>(cs, rowb, c);
    return vn_finish<W, ADD, NP>(cs, rowb, c, l0, kapc);
}

// First qubit update of the min-sum family (marginal VN, bicycle kernels
// with the closed-form first check update, W <= 5).  After iteration 1's
// check update every message is +A (satisfied check: g0 min(v0, 64)) or -B
// (unsatisfied: g1 min(v0, 64)), so a qubit's X-edge sum S_X (numpy tree
// x0 + ((x1 + x2) + (x3 + x4)) over its W X-edges) and F(S_X) depend only on
// the W-bit pattern of which of its X checks are unsatisfied -- likewise S_Z
// and F(S_Z) on the Z-edge pattern.  Lane p of every warp tabulates both for
// pattern p (2^W <= 32 patterns; the same fp32 recipes, so the table entries
// are bit-identical to the general update's values), and each qubit fetches
// its four values with shuffles instead of evaluating the exponential and
// two logarithms of vn_F2.  The Y-belief sum over all 2W edges, the hard
// decision and the outgoing messages V - c are computed as in vn_finish.
// Pattern bit (W - 1 - s) <-> edge s (the funnel-shift packing below).
template <int W>
struct FirstTab {
    float sx, fx, sz, fz;  // this lane's pattern: S_X, F(S_X), S_Z, F(S_Z)
};

template <int W>
__device__ __forceinline__ FirstTab<W> first_tab(float A, float nB, float kapc, uint32_t lane)
{
    constexpr int D = 2 * W;
    const uint32_t pat = lane & ((1u << W) - 1u);
    OptF ox[D], oz[D];
#pragma unroll
    for (int s = 0; s < W; ++s) {
        const float v = (pat >> (W - 1 - s)) & 1u ? nB : A;
        oz[s] = OptF{v, true};       // X-edge s (anti_Z keeps X-edges)
        oz[W + s] = OptF{0.0f, false};
        ox[s] = OptF{0.0f, false};
        ox[W + s] = OptF{v, true};   // Z-edge s
    }
    FirstTab<W> t;
    t.sz = segsum_c<D>(ox);
    t.sx = segsum_c<D>(oz);
    const F2 f = vn_F2(t.sz, t.sx, bc(kapc));
    t.fz = lo(f);
    t.fx = hi(f);
    return t;
}

// All 32 lanes must call this (shuffles); lanes without a qubit pass
// store = false (their loads read inside the group's area and are ignored).
template <int W, int NP>
__device__ __forceinline__ HardXZ vn_first_fixed(uint32_t cs, uint32_t rowb, float l0, const FirstTab<W> &t,
                                                   bool store)
{
    if constexpr (NP > 0) rowb = 4u * NP;
    constexpr int D = 2 * W;
    float c[D];
    vn_load<W, NP>(cs, rowb, c);
    uint32_t px = 0, pz = 0;
#pragma unroll
    for (int s = 0; s < W; ++s) {
        px = __funnelshift_l(f2u(c[s]), px, 1);      // (px << 1) | sign(c[s])
        pz = __funnelshift_l(f2u(c[W + s]), pz, 1);
    }
    const float sX = __shfl_sync(0xffffffffu, t.sx, (int)px), fX = __shfl_sync(0xffffffffu, t.fx, (int)px);
    const float sZ = __shfl_sync(0xffffffffu, t.sz, (int)pz), fZ = __shfl_sync(0xffffffffu, t.fz, (int)pz);
    OptF oa[D];
#pragma unroll
    for (int s = 0; s < D; ++s) oa[s] = OptF{c[s], true};
    const float bX = l0 + sZ, bZ = l0 + sX;
    const float bY = l0 + segsum_c<D>(oa);
    const F2 v2 = add2(pk(bZ, bX), pk(fZ, fX));
    if (store) {
#pragma unroll
        for (int s = 0; s < W; ++s) {
            const F2 o2 = sub2(v2, pk(c[s], c[W + s]));
            sts_a(cs + s * rowb, f2u(lo(o2)));
            sts_a(cs + (W + s) * rowb, f2u(hi(o2)));
        }
    }
    return hard_xz(bX, bZ, bY);
}

template <int W, int T, int NP>
__device__ __forceinline__ void vn_phase_first(const KParams &p, const GroupMem &gm, float g0, float g1, int tid)
{
    const uint32_t rowb = (uint32_t)p.n_pad * 4;
    const float a = fminf(p.v0, kClip);
    // the words cn_phase_first stored: +m0 (satisfied), -m1 (unsatisfied)
    const float A = fminf(g0 * a, kClip), nB = -fminf(g1 * a, kClip);
    const FirstTab<W> t = first_tab<W>(A, nB, p.kapc, (uint32_t)tid & 31u);
    const int l = p.ell;
    const float l0 = p.l0;
#pragma unroll 1
    for (int c0 = tid & ~31; c0 < l; c0 += T) {
        const int c = c0 + (tid & 31);
        const bool ok = c < l;
        const int cc = ok ? c : c0;  // idle lanes re-read a valid column, store nothing
        const HardXZ eL = vn_first_fixed<W, NP>(smem_addr(gm.msg + 4 * cc), rowb, l0, t, ok);
        const HardXZ eR = vn_first_fixed<W, NP>(smem_addr(gm.msg + 4 * (l + cc)), rowb, l0, t, ok);
        const uint32_t xl = __ballot_sync(0xffffffffu, ok && eL.x), zl = __ballot_sync(0xffffffffu, ok && eL.z);
        const uint32_t xr = __ballot_sync(0xffffffffu, ok && eR.x), zr = __ballot_sync(0xffffffffu, ok && eR.z);
        if ((tid & 31) == 0) {
            const int wd = c0 >> 5;
            store_bits4(gm.bits, wd, xl, zl, xr, zr);
        }
    }
}

template <int W, int T, bool BP4, bool ADD, int NP>
__device__ __forceinline__ void vn_phase(const KParams &p, const GroupMem &gm, int tid)
{
    const uint32_t rowb = (uint32_t)p.n_pad * 4;
    const float l0 = p.l0, kapc = p.kapc;
    unsigned char *msg = gm.msg;
    if constexpr (W > 0) {
        // thread owns qubits c and l + c; the warp ballots their hard
        // decisions into word c >> 5 of the circulant bitmaps
        const int l = p.ell;
        int c0 = tid & ~31;
        if constexpr (!BP4 && T > 32) {
            // two circulant indices (four qubits) per step while both are full
            // (min-sum, 64 / 128 threads: +1.5-2% at l = 255 / 511; one warp
            // at l = 127 measured -6% at low p)
#pragma unroll 1
            for (; c0 + T + 31 < l; c0 += 2 * T) {
                const int c = c0 + (tid & 31);
                const HardXZ a0 = vn_update_fixed<W, ADD, NP>(msg + 4 * c, rowb, l0, kapc);
                const HardXZ a1 = vn_update_fixed<W, ADD, NP>(msg + 4 * (l + c), rowb, l0, kapc);
                const HardXZ b0 = vn_update_fixed<W, ADD, NP>(msg + 4 * (c + T), rowb, l0, kapc);
                const HardXZ b1 = vn_update_fixed<W, ADD, NP>(msg + 4 * (l + c + T), rowb, l0, kapc);
                const uint32_t xl = __ballot_sync(0xffffffffu, a0.x), zl = __ballot_sync(0xffffffffu, a0.z);
                const uint32_t xr = __ballot_sync(0xffffffffu, a1.x), zr = __ballot_sync(0xffffffffu, a1.z);
                const uint32_t xl2 = __ballot_sync(0xffffffffu, b0.x), zl2 = __ballot_sync(0xffffffffu, b0.z);
                const uint32_t xr2 = __ballot_sync(0xffffffffu, b1.x), zr2 = __ballot_sync(0xffffffffu, b1.z);
                if ((tid & 31) == 0) {
                    const int wd = c0 >> 5, wd2 = (c0 + T) >> 5;
                    store_bits4(gm.bits, wd, xl, zl, xr, zr);
                    store_bits4(gm.bits, wd2, xl2, zl2, xr2, zr2);
                }
            }
        }
        if constexpr (T == 32 && !BP4) {
            // full 32-qubit steps without the c < l guard (its predicate
            // bookkeeping and reconvergence points): +0.5-0.9% on the
            // one-warp min-sum kernels; the BP4 kernels, whose code is larger,
            // lose 5% at p = 0.02 to the extra 3.7 KB (instruction cache)
#pragma unroll 1
            for (; c0 + 32 <= l; c0 += T) {
                const int c = c0 + (tid & 31);
                const HardXZ eL = vn_update_fixed<W, ADD, NP>(msg + 4 * c, rowb, l0, kapc);
                const HardXZ eR = vn_update_fixed<W, ADD, NP>(msg + 4 * (l + c), rowb, l0, kapc);
                const uint32_t xl = __ballot_sync(0xffffffffu, eL.x), zl = __ballot_sync(0xffffffffu, eL.z);
                const uint32_t xr = __ballot_sync(0xffffffffu, eR.x), zr = __ballot_sync(0xffffffffu, eR.z);
                if ((tid & 31) == 0) {
                    const int wd = c0 >> 5;
                    store_bits4(gm.bits, wd, xl, zl, xr, zr);
                }
            }
        }
#pragma unroll 1
        for (; c0 < l; c0 += T) {
            const int c = c0 + (tid & 31);
            HardXZ eL{false, false}, eR{false, false};
            if (c < l) {
                eL = vn_update_fixed<W, ADD, NP>(msg + 4 * c, rowb, l0, kapc);
                eR = vn_update_fixed<W, ADD, NP>(msg + 4 * (l + c), rowb, l0, kapc);
            }
            const uint32_t xl = __ballot_sync(0xffffffffu, eL.x), zl = __ballot_sync(0xffffffffu, eL.z);
            const uint32_t xr = __ballot_sync(0xffffffffu, eR.x), zr = __ballot_sync(0xffffffffu, eR.z);
            if ((tid & 31) == 0) {
                const int wd = c0 >> 5;
                store_bits4(gm.bits, wd, xl, zl, xr, zr);
            }
        }
    } else {
        constexpr int DM = NP > 0 ? NP : kGenericMaxDeg;  // degree bound of this instantiation
        const F2 kapc2 = bc(kapc);
#pragma unroll 1
        for (int j = tid; j < p.n; j += T) {
            const uint32_t cs = smem_addr(msg + 4 * j);
            const int d = gm.vn_deg[j];
            float c[DM], tmp[DM];
            uint32_t sym[DM];
            uint32_t any_y = 0;
#pragma unroll
            for (int s = 0; s < DM; ++s) {
                c[s] = s < d ? lds_a(cs + s * rowb) : 0.0f;
                sym[s] = s < d ? gm.vn_sym[s * p.n_pad + j] : 0u;
                any_y |= sym[s] == 3;
            }
            float b[4], tot[4];
#pragma unroll
            for (int e = 1; e <= 3; ++e) {
#pragma unroll
                for (int s = 0; s < DM; ++s) {
                    const uint32_t sx = sym[s] & 1u, sz = sym[s] >> 1;
                    const uint32_t a = e == 1 ? sz : (e == 2 ? sx : (sx ^ sz));
                    tmp[s] = a ? c[s] : 0.0f;
                }
                tot[e] = segsum_pred<DM>(tmp, d);
                b[e] = l0 + tot[e];
            }
            gm.ehat[j] = hard_decision(b[1], b[2], b[3]);
            if constexpr (ADD) {
                const float all = segsum_pred<DM>(c, d);
#pragma unroll
                for (int s = 0; s < DM; ++s)
                    if (s < d) sts_a(cs + s * rowb, f2u(l0 + (all - c[s])));  // clipped by the consumer
            } else {
                float V[4];
                if (!any_y) {  // b[1] - l0 = S_Z, b[2] - l0 = S_X exactly as summed
                    const F2 v2 = add2(pk(b[2], b[1]), vn_F2(tot[1], tot[2], kapc2));
                    V[1] = lo(v2);
                    V[2] = hi(v2);
                    V[3] = 0.0f;
                } else {
#pragma unroll
                    for (int S = 1; S <= 3; ++S) {
                        const int a1 = S == 1 ? 2 : 1, a2 = S == 3 ? 2 : 3;
                        V[S] = logaddexp(0.0f, -b[S]) - logaddexp(-b[a1], -b[a2]);
                    }
                }
#pragma unroll
                for (int s = 0; s < DM; ++s) {
                    const float vs = sym[s] == 1 ? V[1] : (sym[s] == 2 ? V[2] : V[3]);
                    if (s < d) sts_a(cs + s * rowb, f2u(vs - c[s]));  // clipped by the consumer
                }
            }
        }
    }
}

template <int T>
__device__ __forceinline__ void snapshot(const KParams &p, const unsigned char *msg, float *dst, int tid,
                                         bool clip)
{
    const int total = p.dv_max * p.n_pad;
    for (int s = tid; s < total; s += T) {
        const int e = p.slot_edge[s];
        if (e >= 0) {
            const float v = lds_f(msg, 4u * s);
            dst[e] = clip ? clip64(v) : v;
        }
    }
}

// current hard decision of qubit j
template <int W>
__device__ __forceinline__ uint8_t ehat_of(const KParams &p, const GroupMem &gm, int j)
{
    if constexpr (W > 0) {
        const bool right = j >= p.ell;
        const int c = right ? j - p.ell : j;
        const uint32_t x = gm.bits[bidx(right ? kXR : kXL, c >> 5)] >> (c & 31);
        const uint32_t z = gm.bits[bidx(right ? kZR : kZL, c >> 5)] >> (c & 31);
        return (uint8_t)((x & 1u) | ((z & 1u) << 1));
    } else {
        return (uint8_t)gm.ehat[j];
    }
}

// Threads-per-CTA bound per kernel, which sets its register budget (the
// register file is 16K 32-bit registers per SM sub-partition, so a bound of
// 5 warps per sub-partition gives 96 registers, 4 warps 128, 3 warps 168):
//  * bicycle W <= 5 min-sum: 640 (96 registers, 20 one-warp frames per SM,
//    which is also the shared-memory limit at l = 127);
//  * bicycle BP4 (W <= 5): 512 (128; its product-form check update needs a
//    few more than 96 -- spill-free, and +1-2% at p >= 0.06 despite 16
//    frames per SM instead of 20);
//  * W = 6 / 8: 512 / 384, whose 12 / 16 fp32 messages per qubit slot limit
//    the frames per SM by shared memory anyway (<= 18 / 13);
//  * generic kernels with degree bound >= 12: 256, their register arrays
//    (messages, addresses and, for BP4, prefix products per edge) need up to
//    the 255-register maximum; <= 8: 640.
#ifndef QSG_BP4_THREADS
#define QSG_BP4_THREADS 512
#endif
constexpr int max_threads(int W, bool BP4, int NP)
{
    if (W == 0) return NP >= 12 ? 256 : 640;
    return W == 8 ? 384 : (W == 6 ? 512 : (BP4 ? QSG_BP4_THREADS : 640));
}

// LEAN: the production shape of a bicycle launch, compiled without the
// run-time options the iteration loop otherwise tests every iteration --
// no traces / snapshots, no e_hat output, early stop on, the windowed
// syndrome plan with 4 lanes per word (every bicycle shape the host builds
// with about four circulant indices per thread), the closed-form first
// iteration (v0 > 0) and gains for every variant from KParams::gtab (the
// host fills it with 1 / alpha / the SAGMS recipe).  The host selects it
// when all of that holds (launch_decode); the serial
// syndrome -> reduce -> exit-test -> gains section between the qubit and
// check phases is ~40% shorter.  Results are identical by construction:
// the same phases run, only the option tests are folded.
template <int W, int T, bool BP4, bool ADD, int NP, bool LEAN = false>
__global__ void __launch_bounds__(max_threads(W, BP4, NP), W == 0 ? 1 : 0) decode_kernel(const KParams p)
{
    static_assert(!LEAN || (W > 0 && !ADD), "lean kernels: bicycle, marginal");
    extern __shared__ __align__(16) unsigned char smem[];
    // ---- per-CTA copy of the graph tables ----
    const uint32_t tabw = (uint32_t)p.m_pad * p.row_words;
    {
        uint32_t *dst = reinterpret_cast<uint32_t *>(smem);
        for (uint32_t w = threadIdx.x; w < tabw; w += blockDim.x) dst[w] = p.cn_tab[w];
        if constexpr (W == 0) {
            const uint32_t *vs = reinterpret_cast<const uint32_t *>(p.vn_sym);
            const uint32_t *vd = reinterpret_cast<const uint32_t *>(p.vn_deg);
            const uint32_t nsw = (uint32_t)p.dv_max * p.n_pad / 4, ndw = (uint32_t)p.n_pad / 4;
            for (uint32_t w = threadIdx.x; w < nsw; w += blockDim.x) dst[tabw + w] = vs[w];
            for (uint32_t w = threadIdx.x; w < ndw; w += blockDim.x) dst[tabw + nsw + w] = vd[w];
        } else {
            if (threadIdx.x < 16)
                dst[tabw + threadIdx.x] = (uint32_t)(threadIdx.x < 8 ? p.gb_a[threadIdx.x] : p.gb_b[threadIdx.x - 8]);
        }
    }
    __syncthreads();

    const int g = threadIdx.x / T, tid = threadIdx.x % T;
    unsigned char *gbase = smem + p.tab_bytes + (size_t)g * p.group_bytes;
    GroupMem gm;
    gm.tab = reinterpret_cast<const uint32_t *>(smem);
    gm.vn_sym = smem + (size_t)tabw * 4;
    gm.vn_deg = gm.vn_sym + (size_t)p.dv_max * p.n_pad;
    gm.gbexp = reinterpret_cast<const int32_t *>(smem + (size_t)tabw * 4);
    gm.msg = gbase;
    gm.ehat = reinterpret_cast<uint32_t *>(gbase + p.off_ehat);
    gm.bits = reinterpret_cast<uint32_t *>(gbase + p.off_bits);
    gm.synw = reinterpret_cast<uint32_t *>(gbase + p.off_synw);
    gm.resw = reinterpret_cast<uint32_t *>(gbase + p.off_resw);
    int *scratch = reinterpret_cast<int *>(gbase + p.off_scratch);  // 2*(T/32) ints
    long long *fslot = reinterpret_cast<long long *>(scratch + 2 * (T / 32));
    // per-group tallies {frames, failures, sum iterations}, kept by thread 0
    // in shared memory (three 64-bit registers live across the whole frame
    // loop cost the BP4 kernels their last spills)
    unsigned long long *tally = reinterpret_cast<unsigned long long *>(fslot + 1);

    const int n = p.n, m = p.m, np_ = p.n_pad;
    const int msg_words = p.dv_max * np_;
    if (tid == 0) tally[0] = tally[1] = tally[2] = 0ull;

    // hard decision with all-zero check messages: argmin(0, L0, L0, L0)
    const uint32_t hd0 = hard_decision(p.l0, p.l0, p.l0);
    // bicycle residual plan (loop-invariant syndrome windows), lpw >= 4
    const bool use_plan = LEAN || (W > 0 && p.lpw >= 4);
    const int lpw = LEAN ? 4 : p.lpw;
    SynPlan<(W > 0 ? W : 1)> plan;
    if constexpr (W > 0) {
        if (use_plan) plan = syn_plan<W, T>(p, gm, tid);
    }
    const bool capture = !LEAN && (p.tr_vn != nullptr || p.tr_cn != nullptr);

    // frame queue: the index of the NEXT frame is fetched as soon as the
    // current one is known, so the global atomic's round trip overlaps the
    // current frame's decode instead of stalling the group between frames
    long long f_next = 0;
    if (tid == 0) f_next = (long long)queue_fetch(p.queue, p.zero);
    while (true) {
        long long f;
        if constexpr (T == 32) {
            f = __shfl_sync(0xffffffffu, f_next, 0);
        } else {
            if (tid == 0) *fslot = f_next;
            group_sync<T>(g);
            f = *fslot;
            group_sync<T>(g);
        }
        if (f >= p.count) break;
        if (tid == 0) f_next = (long long)queue_fetch(p.queue, p.zero);

        // ---- frame input: observed syndrome ----
        uint32_t syn_bits = 0;
        if constexpr (W > 0) {
            // sampling scratch aliases the message area (initialised below,
            // after the bitmaps are built)
            uint8_t *eb = reinterpret_cast<uint8_t *>(gm.msg);
            if (p.sample) {
                const uint64_t key1 = (uint64_t)(p.start + f);
                const int nblk = (n + 3) >> 2;
                for (int b = tid; b < nblk; b += T) {
                    const U64x4 w = philox4x64_10((uint64_t)b + 1, p.seed, key1);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (4 * b + q < n) eb[4 * b + q] = pauli_from_word(w.v[q], p.kx, p.ky, p.kz);
                }
                if (tid < 4) gm.bits[bidx(tid, p.nw)] = 0u;  // padding words (the rest is written below)
                group_sync<T>(g);
                bitmaps_from_bytes<T>(p, gm, eb, tid);
                group_sync<T>(g);
                if (use_plan) circ_syndrome_plan<W, T, false>(plan, gm, nullptr, gm.synw, lpw);
                else circ_syndrome<W, T>(p, gm, nullptr, gm.synw, tid);
                group_sync<T>(g);  // every warp done reading the bitmaps before they are reset below
            } else if (p.syn_words) {
                // bit-packed rows: X checks are bits [0, l), Z checks [l, 2l)
                const uint32_t *row = p.syn_words + f * (long long)p.syn_wpf;
                const int l = p.ell;
                for (int w = tid; w < 2 * p.nw; w += T) {
                    const bool zc = w >= p.nw;
                    const int ww = zc ? w - p.nw : w;
                    const int start = (zc ? l : 0) + 32 * ww;
                    const int q = start >> 5;
                    const uint32_t hi = q + 1 < p.syn_wpf ? row[q + 1] : 0u;
                    const uint32_t v = __funnelshift_r(row[q], hi, start & 31);
                    const int valid = l - 32 * ww;
                    gm.synw[w] = valid >= 32 ? v : v & ((1u << valid) - 1u);
                }
            } else {
                // observed syndrome rows: X checks c < l, Z checks l + c
                const uint8_t *s_in = p.syn_in + f * (long long)m;
                const int l = p.ell;
                for (int c0 = tid & ~31; c0 < 32 * p.nw; c0 += T) {
                    const int c = c0 + (tid & 31);
                    const uint32_t bx = __ballot_sync(0xffffffffu, c < l && s_in[c] != 0);
                    const uint32_t bz = __ballot_sync(0xffffffffu, c < l && s_in[l + c] != 0);
                    if ((tid & 31) == 0) { gm.synw[c0 >> 5] = bx; gm.synw[p.nw + (c0 >> 5)] = bz; }
                }
            }
            // e_hat of iteration 1: hd0 on every qubit
            const int nw1 = p.nw + 1;
            for (int wd = tid; wd < nw1; wd += T) {
                const int valid = p.ell - 32 * wd;
                const uint32_t full = valid >= 32 ? 0xffffffffu : (valid > 0 ? (1u << valid) - 1u : 0u);
                const uint32_t x = (hd0 & 1u) ? full : 0u, z = (hd0 >> 1) ? full : 0u;
                store_bits4(gm.bits, wd, x, z, x, z);
            }
        } else {
            if (p.sample) {
                const uint64_t key1 = (uint64_t)(p.start + f);
                const int nblk = (n + 3) >> 2;
                for (int b = tid; b < nblk; b += T) {
                    const U64x4 w = philox4x64_10((uint64_t)b + 1, p.seed, key1);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (4 * b + q < n) gm.ehat[4 * b + q] = pauli_from_word(w.v[q], p.kx, p.ky, p.kz);
                }
                group_sync<T>(g);
                syn_bits = syndrome_bits_generic<T, (NP > 0 ? NP : kGenericMaxDeg)>(p, gm, tid);
                group_sync<T>(g);
            } else if (p.syn_words) {
                int t = 0;
                const uint32_t *row = p.syn_words + f * (long long)p.syn_wpf;
                for (int i = tid; i < m; i += T, ++t) syn_bits |= ((row[i >> 5] >> (i & 31)) & 1u) << t;
            } else {
                int t = 0;
                const uint8_t *s_in = p.syn_in + f * (long long)m;
                for (int i = tid; i < m; i += T, ++t) syn_bits |= (s_in[i] != 0 ? 1u : 0u) << t;
            }
            for (int j = tid; j < np_; j += T) gm.ehat[j] = hd0;
        }
        // the initial qubit->check messages (v0); not needed when the first
        // check update is the closed form, which writes every edge slot
        if (!LEAN && !(W > 0 && p.first_fast)) {
            const uint32_t v0b = f2u(p.v0);
            for (int s = tid; s < msg_words; s += T) sts_u(gm.msg, 4u * s, v0b);
        }
        group_sync<T>(g);

        int recorded = 0, success = 0, iters = p.l_max, n_gamma = 0, n_snap = 0;
        for (int ell = 1; ell <= p.l_max; ++ell) {
            uint32_t res = 0;
            int part;
            if constexpr (W > 0) {
                part = use_plan ? circ_syndrome_plan<W, T, true>(plan, gm, gm.synw, gm.resw, lpw)
                                : circ_syndrome<W, T>(p, gm, gm.synw, gm.resw, tid);
            } else {
                res = syn_bits ^ syndrome_bits_generic<T, (NP > 0 ? NP : kGenericMaxDeg)>(p, gm, tid);
                part = __popc(res);
            }
            const int unsat = group_sum<T>(part, scratch, ell & 1, tid, g);
            if constexpr (W > 0 && T == 32) __syncwarp();  // resw visible to the check phase
            float g0 = 1.0f, g1 = 1.0f;
            if constexpr (LEAN) {
                if (unsat == 0) { success = 1; iters = ell; break; }
                if (ell == p.l_max) break;
                g0 = p.gtab[2 * unsat];
                g1 = p.gtab[2 * unsat + 1];
            } else {
                if (p.tr_unsat && tid == 0) p.tr_unsat[f * p.l_max + n_gamma] = unsat;
                ++n_gamma;
                if (unsat == 0 && !recorded) {
                    success = 1;
                    iters = ell;
                    recorded = 1;
                    if (p.out_ehat)
                        for (int j = tid; j < n; j += T) p.out_ehat[f * n + j] = ehat_of<W>(p, gm, j);
                }
                if (p.early_stop && unsat == 0) break;
                if (ell == p.l_max) {
                    if (!recorded && p.out_ehat)
                        for (int j = tid; j < n; j += T) p.out_ehat[f * n + j] = ehat_of<W>(p, gm, j);
                    if (!capture) break;
                }
                if (p.gain_mode == 1) {
                    g0 = g1 = p.alpha;
                } else if (p.gain_mode == 2) {
                    if (p.use_gtab) {  // the same double recipe, tabulated per unsat count by the host
                        g0 = p.gtab[2 * unsat];
                        g1 = p.gtab[2 * unsat + 1];
                    } else {
                        const double gamma = (double)unsat / (double)m;
                        const double base = p.amax - (p.amax - p.amin) * gamma;
                        g0 = (float)(base * 1.0);
                        g1 = (float)(base * p.eta);
                    }
                }
            }
            if (W > 0 && ell == 1 && (LEAN || p.first_fast))
                cn_phase_first<(W > 0 ? W : 1), T, BP4>(p, gm, g0, g1, tid);
            else
                cn_phase<W, T, BP4, NP>(p, gm, syn_bits, res, g0, g1, tid);
            group_sync<T>(g);
            if (capture && p.tr_cn) snapshot<T>(p, gm.msg, p.tr_cn + (f * p.l_max + n_snap) * p.E, tid, false);
            if constexpr (W > 0 && W <= 5 && !BP4 && !ADD) {
                if (ell == 1 && (LEAN || p.first_fast))
                    vn_phase_first<(W > 0 ? W : 1), T, NP>(p, gm, g0, g1, tid);
                else
                    vn_phase<W, T, BP4, ADD, NP>(p, gm, tid);
            } else {
                vn_phase<W, T, BP4, ADD, NP>(p, gm, tid);
            }
            group_sync<T>(g);
            if (capture) {
                if (p.tr_vn) snapshot<T>(p, gm.msg, p.tr_vn + (f * p.l_max + n_snap) * p.E, tid, true);
                ++n_snap;
            }
        }
        if (tid == 0) {
            if (p.out_flag) p.out_flag[f] = (uint8_t)(p.sample ? !success : success);
            if (p.out_iters) p.out_iters[f] = iters;
            if (!LEAN && p.tr_counts) { p.tr_counts[2 * f] = n_gamma; p.tr_counts[2 * f + 1] = n_snap; }
            tally[0] += 1ull;
            tally[1] += (unsigned long long)!success;
            tally[2] += (unsigned long long)iters;
        }
        group_sync<T>(g);  // group memory reuse by the next frame
    }
    if (p.counters && tid == 0 && tally[0]) {
        const unsigned long long c_frames = tally[0], c_iters = tally[2];
        atomicAdd((unsigned long long *)&p.counters[0], c_frames);
        atomicAdd((unsigned long long *)&p.counters[1], tally[1]);
        atomicAdd((unsigned long long *)&p.counters[2], c_iters);
        atomicAdd((unsigned long long *)&p.counters[3], (unsigned long long)p.E * (c_iters - c_frames));
    }
}

}  // namespace qsg
