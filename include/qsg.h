/*
 * qsg -- C ABI of the B200 (sm_100a) batched GB-QLDPC Monte-Carlo decoder.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/qsagms).  The reference has no plugin registry;
 * its operator surface is two Python functions, and each entry point below
 * replaces one of them (or a piece they call):
 *
 *   qsg_decode_frames    <- harness._decode_frames      harness.py:172-182
 *                           (sample_error channel.py:55-76 x count,
 *                            _Kernel.syndromes_of decoder.py:303-309,
 *                            decode_batch decoder.py:374-485)
 *   qsg_decode_syndromes <- decoder.decode_batch        decoder.py:374-485
 *   qsg_decode_syndromes_packed  same, bit-packed syndrome wire format
 *                           (+ collect_gamma / capture_messages traces used
 *                            by decoder.decode          decoder.py:488-559)
 *   qsg_sample_errors    <- channel.sample_error        channel.py:55-76
 *   qsg_syndromes_of     <- _Kernel.syndromes_of        decoder.py:303-309
 *   qsg_graph_create_*   <- code.build_gb + code.tanner_graph
 *                                                       code.py:150-231
 *   qsg_graph_export     <- TannerGraph flat arrays     code.py:118-147
 *
 * Conventions: plain pointers and sizes only.  Buffers named *_dev are device
 * pointers (any allocator; e.g. torch tensors used as buffers) on the graph's
 * device; `stream` is a cudaStream_t (NULL = legacy default stream) and all
 * device work is enqueued on it (no host synchronisation unless stated).
 * Pauli codes follow pauli.py:28-31 (I=0, X=1, Z=2, Y=3).  Every function
 * returns QSG_OK or a negative status; qsg_last_error() gives a thread-local
 * message.  The Python layer maps QSG_EINVAL to ValueError (the reference's
 * config / shape errors, decoder.py:76-112, :396-402) and the others to
 * RuntimeError.  Graph handles are immutable after creation and may be shared
 * by concurrent calls on different streams.
 */
#ifndef QSG_H
#define QSG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSG_ABI_VERSION 1

#define QSG_OK 0
#define QSG_EINVAL (-1)       /* invalid argument / config (ValueError)      */
#define QSG_ECUDA (-2)        /* CUDA runtime failure (RuntimeError)          */
#define QSG_ENOMEM (-3)       /* host or device allocation failure            */
#define QSG_EUNSUPPORTED (-4) /* graph outside the compiled kernel envelope   */

/* decoder.py:49 VARIANTS order and :50 VN_MODES order. */
enum { QSG_BP4 = 0, QSG_MS = 1, QSG_SMS = 2, QSG_SAGMS = 3 };
enum { QSG_VN_MARGINAL = 0, QSG_VN_ADDITIVE = 1 };

/* DecoderConfig + GainParams (decoder.py:62-112) flattened.  Validated with
 * the reference's rules; alpha is used by sms, alpha_min/alpha_max/eta_unsat
 * by sagms.  early_stop mirrors decode_batch(early_stop=...). */
typedef struct qsg_decoder_cfg {
    int32_t variant;
    int32_t vn_mode;
    int32_t l_max;
    int32_t early_stop;
    double alpha;
    double alpha_min;
    double alpha_max;
    double eta_unsat;
} qsg_decoder_cfg;

typedef struct qsg_graph qsg_graph;

/* Generalized-bicycle code from circulant exponents (code.py:201-231):
 * rows 0..ell-1 are X on [A|B], rows ell..2ell-1 are Z on [B^T|A^T].
 * Exponents must be distinct and in [0, ell).  Commutation holds by
 * construction (circulants commute). */
int qsg_graph_create_gb(int32_t ell, const int32_t *a, int32_t wa, const int32_t *b,
                        int32_t wb, int32_t device, qsg_graph **out);

/* Arbitrary check matrix as canonical CSR (TannerGraph order: row-major,
 * strictly increasing columns per row; edge_sym in {1,2,3}).  cn_ptr has
 * m+1 entries.  Every check and qubit needs degree >= 1 (decoder.py:274-277). */
int qsg_graph_create_csr(int32_t n, int32_t m, const int64_t *cn_ptr, const int64_t *edge_vn,
                         const uint8_t *edge_sym, int32_t device, qsg_graph **out);

int qsg_graph_destroy(qsg_graph *g);

/* kind: 0 = generic table-driven kernels, W > 0 = "bicycle" kernels
 * (every node of degree 2W, each qubit's edges X-then-Z, W each, every check
 * single-symbol).  threads: threads cooperating on one frame. */
int qsg_graph_info(const qsg_graph *g, int32_t *n, int32_t *m, int64_t *E, int32_t *dc_max,
                   int32_t *dv_max, int32_t *kind, int32_t *threads);

/* TannerGraph flat arrays (code.py:150-191) into host buffers sized E
 * (edge_cn, edge_vn, edge_sym, vn_order), m+1 (cn_ptr), n+1 (vn_ptr).
 * Any pointer may be NULL. */
int qsg_graph_export(const qsg_graph *g, int64_t *edge_cn, int64_t *edge_vn, uint8_t *edge_sym,
                     int64_t *cn_ptr, int64_t *vn_order, int64_t *vn_ptr);

/* Row commutation of the check matrix on the graph's device (the
 * stabilizer validation of SparseCheckMatrix.validate, code.py:80-97, via
 * pauli.check_orthogonality, pauli.py:120-144), in O(m d_c d_v d_c) rather
 * than the reference's O(m^2) pair scan.  Synchronous (setup-time call).
 * *commutes = 1 iff every pair of rows commutes; bad_pair (int64[2], may be
 * NULL) receives the lowest anticommuting pair (i, k), i < k, or (-1, -1). */
int qsg_graph_check_commute(const qsg_graph *g, int32_t *commutes, int64_t *bad_pair);

/* Optional per-frame traces of qsg_decode_syndromes (device buffers, any may
 * be NULL):
 *   unsat[B * l_max]         residual weight per executed iteration
 *                            (gamma = unsat / m, decoder.py:425-431)
 *   vn_msgs, cn_msgs[B * l_max * E]  message snapshots in canonical edge
 *                            order after each executed update (capture_messages,
 *                            decoder.py:470-475; includes the final update at
 *                            l_max as the reference does)
 *   counts[B * 2]            (#unsat entries, #snapshots) per frame */
typedef struct qsg_trace {
    int32_t *unsat;
    float *vn_msgs;
    float *cn_msgs;
    int32_t *counts;
} qsg_trace;

/* decode_batch: syndromes_dev uint8[B*m] (nonzero = 1) decoded with prior
 * LLR l0 (= ln(3(1-e0)/e0), channel.py:48-52).  Outputs uint8 success[B],
 * uint8 e_hat[B*n] (failures carry the last iteration's estimate), int64
 * iterations[B] (l_max on failure).  e_hat_dev and trace may be NULL. */
int qsg_decode_syndromes(const qsg_graph *g, const qsg_decoder_cfg *cfg, double l0,
                         const uint8_t *syndromes_dev, int64_t B, uint8_t *success_dev,
                         uint8_t *e_hat_dev, int64_t *iterations_dev, const qsg_trace *trace,
                         void *stream);

/* decode_batch with bit-packed syndromes (32x less input traffic than one
 * byte per check): syn_words_dev uint32[B * ceil(m/32)], bit i of frame b is
 * (syn_words[b * ceil(m/32) + i/32] >> (i % 32)) & 1.  Outputs as in
 * qsg_decode_syndromes (no traces). */
int qsg_decode_syndromes_packed(const qsg_graph *g, const qsg_decoder_cfg *cfg, double l0,
                                const uint32_t *syn_words_dev, int64_t B, uint8_t *success_dev,
                                uint8_t *e_hat_dev, int64_t *iterations_dev, void *stream);

/* _decode_frames: frames [start, start+count) sampled on device with
 * Philox4x64-10 keyed (seed, frame) exactly like sample_error, syndromes,
 * decoded with prior llr(epsilon0).  Per-frame outputs (each may be NULL):
 * uint8 fails[count], int64 iterations[count], uint8 e_hat[count*n].
 * counters_dev (may be NULL) is int64[4] and is ACCUMULATED (not zeroed):
 * {frames, failures, sum iterations, sum E*(iterations-1) CN-edge updates}. */
int qsg_decode_frames(const qsg_graph *g, const qsg_decoder_cfg *cfg, double epsilon,
                      double epsilon0, uint64_t seed, int64_t start, int64_t count,
                      uint8_t *fails_dev, int64_t *iterations_dev, uint8_t *e_hat_dev,
                      int64_t *counters_dev, void *stream);

/* sample_error for frames [start, start+count): uint8 errors[count*n]. */
int qsg_sample_errors(int32_t n, double epsilon, uint64_t seed, int64_t start, int64_t count,
                      uint8_t *errors_dev, int32_t device, void *stream);

/* syndromes_of: uint8 e[B*n] -> uint8 syn[B*m]. */
int qsg_syndromes_of(const qsg_graph *g, const uint8_t *e_dev, int64_t B, uint8_t *syn_dev,
                     void *stream);

/* Thread-local description of the last failure (never NULL). */
const char *qsg_last_error(void);
int qsg_abi_version(void);
/* Hash of the kernel sources and build flags the library was compiled from
 * (16 hex digits).  Not a reference interface: profiles/ncu_traffic.json
 * records the id its ncu capture was taken on, and bench.py refuses
 * hardware counters from a different build. */
const char *qsg_build_id(void);

#ifdef __cplusplus
}
#endif
#endif
