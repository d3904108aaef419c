/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the batched GB-QLDPC decode
 * path.  Used by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
 * leg as the checker; never linked into the product.
 *
 * A plain-C restatement of the reference's hot path
 * (/root/reference/pkg/src/qsagms):
 *   qsgo_sample_errors   channel.py:55-76   (Philox4x64-10, inverse CDF)
 *   qsgo_syndromes_of    decoder.py:303-309
 *   qsgo{32,64}_decode   decoder.py:374-485 with _Kernel :264-359
 *   qsgo{32,64}_frames   harness.py:172-182 (_decode_frames)
 * The 64 suffix is float64 with glibc transcendentals (the reference's own
 * arithmetic; bit-exact with numpy for ms/sms/sagms, within ulps for bp4
 * whose numpy expm1/log1p are SIMD kernels).  The 32 suffix is the fp32
 * restatement the GPU is required to match bit-for-bit.
 */
#ifndef QSG_ORACLE_H
#define QSG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* TannerGraph arrays (code.py:118-191), canonical row-major edge order. */
typedef struct qsgo_graph {
    int32_t n, m;
    int64_t E;
    const int64_t *edge_cn, *edge_vn;
    const uint8_t *edge_sym;
    const int64_t *cn_ptr;   /* m+1 */
    const int64_t *vn_order; /* E   */
    const int64_t *vn_ptr;   /* n+1 */
} qsgo_graph;

/* variant: 0 bp4, 1 ms, 2 sms, 3 sagms (decoder.py:49 order);
 * vn_mode: 0 marginal, 1 additive (decoder.py:50). */
typedef struct qsgo_cfg {
    int32_t variant, vn_mode, l_max, early_stop;
    double alpha, alpha_min, alpha_max, eta_unsat;
} qsgo_cfg;

/* Optional per-frame traces.  unsat: B x l_max ints (gamma = unsat/m);
 * vn_msgs / cn_msgs: B x l_max x E snapshots after each executed update
 * (capture_messages semantics, decoder.py:454-475); counts: B x 2
 * (#gamma entries, #snapshots).  Any pointer may be NULL. */
typedef struct qsgo_trace32 {
    int32_t *unsat; float *vn_msgs; float *cn_msgs; int32_t *counts;
} qsgo_trace32;
typedef struct qsgo_trace64 {
    int32_t *unsat; double *vn_msgs; double *cn_msgs; int32_t *counts;
} qsgo_trace64;

int qsgo_sample_errors(int32_t n, double epsilon, uint64_t seed, int64_t start,
                       int64_t count, uint8_t *out);
void qsgo_philox4x64_10(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]);
void qsgo_syndromes_of(const qsgo_graph *g, const uint8_t *e, int64_t B, uint8_t *syn);

int qsgo32_decode(const qsgo_graph *g, const qsgo_cfg *cfg, double l0,
                  const uint8_t *syn, int64_t B, uint8_t *success, uint8_t *e_hat,
                  int64_t *iterations, const qsgo_trace32 *trace, int32_t nthreads);
int qsgo64_decode(const qsgo_graph *g, const qsgo_cfg *cfg, double l0,
                  const uint8_t *syn, int64_t B, uint8_t *success, uint8_t *e_hat,
                  int64_t *iterations, const qsgo_trace64 *trace, int32_t nthreads);

/* _decode_frames: sample frames [start, start+count) with (seed, frame),
 * syndrome, decode with prior llr(epsilon0).  fails/iterations/e_hat may be
 * NULL; counters (may be NULL) accumulate {frames, failures, sum iterations,
 * sum E*(iterations-1)}. */
int qsgo32_frames(const qsgo_graph *g, const qsgo_cfg *cfg, double epsilon,
                  double epsilon0, uint64_t seed, int64_t start, int64_t count,
                  uint8_t *fails, int64_t *iterations, uint8_t *e_hat,
                  int64_t *counters, int32_t nthreads);
int qsgo64_frames(const qsgo_graph *g, const qsgo_cfg *cfg, double epsilon,
                  double epsilon0, uint64_t seed, int64_t start, int64_t count,
                  uint8_t *fails, int64_t *iterations, uint8_t *e_hat,
                  int64_t *counters, int32_t nthreads);

/* fp32 recipe entry points, exposed so tests can measure their accuracy and
 * compare them with the CUDA copy. */
void qsgo_math32_batch(int32_t which, const float *x, const float *y, float *out, int64_t n);
void qsgo_bp4_mags(const float *x, int32_t d, float *out);

#ifdef __cplusplus
}
#endif
#endif
