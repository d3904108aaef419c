/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle (checker) for the GB-QLDPC decode
 * hot path; see qsg_oracle.h for the function map to the reference.
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -mfma, no fast-math).
 */
#include "qsg_oracle.h"
#include "qsg_oracle_math.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- Philox4x64-10 exactly as numpy.random.Philox (channel.py:63-65) ----
 * counter (c, 0, 0, 0) with c starting at 1 (numpy increments before each
 * block), key (seed, stream_id); block b yields words 4b..4b+3. */
#define PH_M0 0xD2E7470EE14C6C93ULL
#define PH_M1 0xCA5A826395121157ULL
#define PH_W0 0x9E3779B97F4A7C15ULL
#define PH_W1 0xBB67AE8584CAA73BULL

static inline uint64_t mulhilo(uint64_t a, uint64_t b, uint64_t *hi)
{
    unsigned __int128 p = (unsigned __int128)a * b;
    *hi = (uint64_t)(p >> 64);
    return (uint64_t)p;
}

void qsgo_philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4])
{
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += PH_W0; k1 += PH_W1; }
        uint64_t hi0, hi1;
        uint64_t lo0 = mulhilo(PH_M0, c0, &hi0);
        uint64_t lo1 = mulhilo(PH_M1, c2, &hi1);
        uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* u = (word >> 11) * 2^-53 >= t  <=>  (word >> 11) >= ceil(t * 2^53);
 * t * 2^53 is exact in double, so the integer thresholds are exact. */
static void thresholds(double eps, uint64_t K[3])
{
    double t_x = 1.0 - eps, t_y = 1.0 - eps + eps / 3.0, t_z = 1.0 - eps / 3.0;
    K[0] = (uint64_t)ceil(t_x * 9007199254740992.0);
    K[1] = (uint64_t)ceil(t_y * 9007199254740992.0);
    K[2] = (uint64_t)ceil(t_z * 9007199254740992.0);
}

/* sample_error for frames start..start+count-1 (channel.py:55-76).  The
 * assignment order I, X(1), Y(3), Z(2) with later masks overriding earlier
 * ones follows :73-75. */
int qsgo_sample_errors(int32_t n, double eps, uint64_t seed, int64_t start, int64_t count,
                       uint8_t *out)
{
    if (n < 1 || count < 0 || !(eps >= 0.0 && eps < 1.0)) return -1;
    uint64_t K[3];
    thresholds(eps, K);
    for (int64_t f = 0; f < count; ++f) {
        uint64_t key[2] = {seed, (uint64_t)(start + f)};
        uint8_t *e = out + f * n;
        for (int32_t b = 0; 4 * b < n; ++b) {
            uint64_t ctr[4] = {(uint64_t)b + 1, 0, 0, 0}, w[4];
            qsgo_philox4x64_10(ctr, key, w);
            for (int q = 0; q < 4 && 4 * b + q < n; ++q) {
                uint64_t k = w[q] >> 11;
                uint8_t c = 0;
                if (eps != 0.0) {
                    if (k >= K[0] && k < K[1]) c = 1;
                    if (k >= K[1] && k < K[2]) c = 3;
                    if (k >= K[2]) c = 2;
                }
                e[4 * b + q] = c;
            }
        }
    }
    return 0;
}

/* _Kernel.syndromes_of (decoder.py:303-309). */
void qsgo_syndromes_of(const qsgo_graph *g, const uint8_t *e, int64_t B, uint8_t *syn)
{
    for (int64_t b = 0; b < B; ++b) {
        const uint8_t *eb = e + b * g->n;
        for (int i = 0; i < g->m; ++i) {
            int x = 0;
            for (int64_t k = g->cn_ptr[i]; k < g->cn_ptr[i + 1]; ++k) {
                int c = eb[g->edge_vn[k]], s = g->edge_sym[k];
                x ^= ((c & 1) & (s >> 1)) ^ ((c >> 1) & (s & 1));
            }
            syn[b * g->m + i] = (uint8_t)x;
        }
    }
}

/* ---- fp32 restatement ---- */
#define REAL float
#define SFX 32
#define TRACE_T qsgo_trace32
#define LAE(x, y) qo_logaddexp((x), (y))
#define MAXR(a, b) fmaxf((a), (b))
#define ABSR(x) fabsf(x)
#define VN_FACTORED 1
#define BP4_PRODUCT 1
#include "qsg_oracle_body.h"
#undef REAL
#undef SFX
#undef TRACE_T
#undef LAE
#undef PHI
#undef MAXR
#undef ABSR
#undef VN_FACTORED
#undef BP4_PRODUCT

/* ---- fp64 with glibc: the reference's own arithmetic ---- */
static inline double lae64(double x, double y) /* npy_logaddexp */
{
    if (x == y) return x + 0.6931471805599453;
    double d = x - y;
    if (d > 0) return x + log1p(exp(-d));
    return y + log1p(exp(d));
}
#define REAL double
#define SFX 64
#define TRACE_T qsgo_trace64
#define LAE(x, y) lae64((x), (y))
#define PHI(x) log1p(2.0 / expm1(x))
#define MAXR(a, b) fmax((a), (b))
#define ABSR(x) fabs(x)
#define VN_FACTORED 0
#define BP4_PRODUCT 0
#include "qsg_oracle_body.h"

/* One BP4 check: output magnitudes for input magnitudes x[0..d) (fp32 recipe). */
void qsgo_bp4_mags(const float *x, int32_t d, float *out)
{
    if (d >= 1 && d <= QO_BP4_MAXD) qo_bp4_mags(x, (int)d, out);
}

void qsgo_math32_batch(int32_t which, const float *x, const float *y, float *out, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) {
        switch (which) {
        case 0: out[i] = qo_exp_neg(x[i]); break;
        case 1: out[i] = qo_log1p_01(x[i]); break;
        case 2: out[i] = qo_log1p(x[i]); break;
        case 3: out[i] = qo_expm1(x[i]); break;
        case 4: out[i] = qo_logaddexp(x[i], y[i]); break;
        case 6: out[i] = qo_vnF(x[i], qo_vn_kapc(y[i])); break;
        default: out[i] = NAN;
        }
    }
}
