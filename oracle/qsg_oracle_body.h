/*
 * TEST INFRASTRUCTURE ONLY -- oracle decode body, included twice by
 * qsg_oracle.c (REAL = float with the fp32 recipes, REAL = double with
 * glibc).  Follows /root/reference/pkg/src/qsagms/decoder.py operation by
 * operation on canonical (row-major) edge arrays, including the masked
 * reductions (cv * anti mask, then numpy's pairwise reduceat tree).
 *
 * Required macros: REAL, SFX (32 or 64), TRACE_T, LAE(x, y), PHI(x),
 *                  MAXR(a, b), ABSR(x), VN_FACTORED (0 = literal decoder.py:348-357)
 */

#define QO_CAT2(a, b) a##b
#define QO_CAT(a, b) QO_CAT2(a, b)
#define QF(name) QO_CAT(QO_CAT(qsgo, SFX), name)

/* numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src): n < 8
 * sequential from -0.0; n <= 128 eight strided accumulators combined as
 * ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then a sequential tail; larger n
 * split at a multiple of 8 near n/2.  Verified against np.add.reduceat in
 * tests/test_oracle_pins.py. */
static REAL QF(_pairwise)(const REAL *a, int64_t n)
{
    if (n < 8) {
        REAL res = (REAL)-0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    }
    if (n <= 128) {
        REAL r[8];
        for (int k = 0; k < 8; ++k) r[k] = a[k];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; ++k) r[k] += a[i + k];
        REAL res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return QF(_pairwise)(a, n2) + QF(_pairwise)(a + n2, n - n2);
}

/* One np.add.reduceat segment: out = x0; out += pairwise(x1..). */
static REAL QF(_segsum)(const REAL *x, int64_t d)
{
    return x[0] + QF(_pairwise)(x + 1, d - 1);
}

static REAL QF(_clip)(REAL x, REAL lo, REAL hi)
{
    return x < lo ? lo : (x > hi ? hi : x);
}

/* anticommutation mask of candidate error e in {1 X, 2 Z, 3 Y} against an
 * edge symbol (decoder.py:279-283): X vs z-bit, Z vs x-bit, Y vs x^z. */
static inline REAL QF(_anti)(int e, uint8_t sym)
{
    int sx = sym & 1, sz = sym >> 1;
    int a = e == 1 ? sz : (e == 2 ? sx : (sx ^ sz));
    return (REAL)a;
}

typedef struct {
    REAL *vmsg, *cmsg, *cv, *tmp, *ph, *gains;
    uint8_t *ehat, *resid;
} QF(_scratch);

/* decode one frame: decode_batch (decoder.py:374-485) for B = 1 with the
 * early_stop / capture semantics of the batched driver. */
static void QF(_decode_one)(const qsgo_graph *g, const qsgo_cfg *cfg, REAL l0, REAL v0,
                            const uint8_t *syn, uint8_t *succ_out, uint8_t *ehat_out,
                            int64_t *iters_out, int32_t *tr_unsat, REAL *tr_vn,
                            REAL *tr_cn, int32_t *tr_counts, QF(_scratch) *s)
{
    const int64_t E = g->E;
    const int n = g->n, m = g->m;
    const REAL CLIP = (REAL)64.0;
    const int capture = (tr_vn != NULL || tr_cn != NULL);
#if VN_FACTORED
    const float kapc = qo_vn_kapc((float)l0);
#endif
    for (int64_t e = 0; e < E; ++e) { s->vmsg[e] = v0; s->cmsg[e] = (REAL)0.0; }
    int recorded = 0, success = 0, n_gamma = 0, n_snap = 0;
    int64_t iters = cfg->l_max;

    for (int ell = 1; ell <= cfg->l_max; ++ell) {
        /* _Kernel.hard_decisions, decoder.py:292-301 */
        for (int j = 0; j < n; ++j) {
            int64_t p0 = g->vn_ptr[j], d = g->vn_ptr[j + 1] - p0;
            for (int64_t q = 0; q < d; ++q) s->cv[q] = s->cmsg[g->vn_order[p0 + q]];
            REAL best = (REAL)0.0;
            int arg = 0;
            for (int e = 1; e <= 3; ++e) {
                for (int64_t q = 0; q < d; ++q)
                    s->tmp[q] = s->cv[q] * QF(_anti)(e, g->edge_sym[g->vn_order[p0 + q]]);
                REAL metric = l0 + QF(_segsum)(s->tmp, d);
                if (metric < best) { best = metric; arg = e; }
            }
            s->ehat[j] = (uint8_t)arg;
        }
        /* residual = syn ^ syndromes_of(e_hat), decoder.py:424, :303-309 */
        int64_t unsat = 0;
        for (int i = 0; i < m; ++i) {
            int x = 0;
            for (int64_t e = g->cn_ptr[i]; e < g->cn_ptr[i + 1]; ++e) {
                int c = s->ehat[g->edge_vn[e]], sym = g->edge_sym[e];
                x ^= ((c & 1) & (sym >> 1)) ^ ((c >> 1) & (sym & 1));
            }
            s->resid[i] = (uint8_t)((syn[i] != 0) ^ x);
            unsat += s->resid[i];
        }
        if (tr_unsat) tr_unsat[n_gamma] = (int32_t)unsat;
        n_gamma++;
        if (unsat == 0 && !recorded) { /* decoder.py:432-439 */
            success = 1;
            iters = ell;
            recorded = 1;
            if (ehat_out) memcpy(ehat_out, s->ehat, (size_t)n);
        }
        if (cfg->early_stop && unsat == 0) break; /* :441-445 (B = 1) */
        if (ell == cfg->l_max) {                  /* :454-460 */
            if (!recorded && ehat_out) memcpy(ehat_out, s->ehat, (size_t)n);
            if (!capture) break;
        }
        /* gains, decoder.py:462-467 */
        if (cfg->variant == 3) {
            double gamma = (double)unsat / (double)m;
            double base = cfg->alpha_max - (cfg->alpha_max - cfg->alpha_min) * gamma;
            for (int i = 0; i < m; ++i)
                s->gains[i] = (REAL)(s->resid[i] == 1 ? base * cfg->eta_unsat : base * 1.0);
        }
        /* _Kernel.cn_step, decoder.py:311-338 */
        for (int i = 0; i < m; ++i) {
            int64_t p0 = g->cn_ptr[i], d = g->cn_ptr[i + 1] - p0;
            REAL syn_sign = (REAL)1.0 - (REAL)2.0 * (REAL)(syn[i] != 0);
            REAL prod = (REAL)1.0;
            for (int64_t q = 0; q < d; ++q) prod *= (s->vmsg[p0 + q] < (REAL)0.0) ? (REAL)-1.0 : (REAL)1.0;
            if (cfg->variant == 0) { /* bp4 :318-323 */
#if BP4_PRODUCT
                /* fp32 restatement: the same magnitudes in the product
                 * domain (qo_bp4_mags); vmsg is clipped to +-64 already */
                for (int64_t q = 0; q < d; ++q) s->ph[q] = ABSR(s->vmsg[p0 + q]);
                qo_bp4_mags(s->ph, (int)d, s->tmp);
                for (int64_t q = 0; q < d; ++q) {
                    REAL v = s->vmsg[p0 + q];
                    REAL sg = (v < (REAL)0.0) ? (REAL)-1.0 : (REAL)1.0;
                    s->cmsg[p0 + q] = QF(_clip)((syn_sign * prod) * sg * s->tmp[q], -CLIP, CLIP);
                }
#else
                for (int64_t q = 0; q < d; ++q)
                    s->ph[q] = PHI(MAXR(ABSR(s->vmsg[p0 + q]), (REAL)1e-12));
                REAL total = QF(_segsum)(s->ph, d);
                for (int64_t q = 0; q < d; ++q) {
                    REAL v = s->vmsg[p0 + q];
                    REAL sg = (v < (REAL)0.0) ? (REAL)-1.0 : (REAL)1.0;
                    REAL ext = QF(_clip)(total - s->ph[q], (REAL)1e-12, (REAL)50.0);
                    REAL mag = PHI(ext);
                    s->cmsg[p0 + q] = QF(_clip)((syn_sign * prod) * sg * mag, -CLIP, CLIP);
                }
#endif
            } else { /* min-sum family :324-337 */
                REAL min1 = (REAL)INFINITY;
                for (int64_t q = 0; q < d; ++q) {
                    REAL a = ABSR(s->vmsg[p0 + q]);
                    if (a < min1) min1 = a;
                }
                int64_t first = -1;
                for (int64_t q = 0; q < d; ++q)
                    if (ABSR(s->vmsg[p0 + q]) == min1) { first = q; break; }
                REAL min2 = (REAL)INFINITY;
                for (int64_t q = 0; q < d; ++q) {
                    REAL a = q == first ? (REAL)INFINITY : ABSR(s->vmsg[p0 + q]);
                    if (a < min2) min2 = a;
                }
                for (int64_t q = 0; q < d; ++q) {
                    REAL v = s->vmsg[p0 + q];
                    REAL sg = (v < (REAL)0.0) ? (REAL)-1.0 : (REAL)1.0;
                    REAL mag = q == first ? min2 : min1;
                    if (cfg->variant == 2) mag = (REAL)cfg->alpha * mag;
                    else if (cfg->variant == 3) mag = s->gains[i] * mag;
                    s->cmsg[p0 + q] = QF(_clip)((syn_sign * prod) * sg * mag, -CLIP, CLIP);
                }
            }
        }
        /* _Kernel.vn_step, decoder.py:340-359 */
        for (int j = 0; j < n; ++j) {
            int64_t p0 = g->vn_ptr[j], d = g->vn_ptr[j + 1] - p0;
            for (int64_t q = 0; q < d; ++q) s->cv[q] = s->cmsg[g->vn_order[p0 + q]];
            if (cfg->vn_mode == 1) { /* additive :344-346 */
                REAL tot = QF(_segsum)(s->cv, d);
                for (int64_t q = 0; q < d; ++q)
                    s->vmsg[g->vn_order[p0 + q]] = QF(_clip)(l0 + (tot - s->cv[q]), -CLIP, CLIP);
            } else { /* marginal :348-357 */
                REAL tot[4];
                for (int e = 1; e <= 3; ++e) {
                    for (int64_t q = 0; q < d; ++q)
                        s->tmp[q] = s->cv[q] * QF(_anti)(e, g->edge_sym[g->vn_order[p0 + q]]);
                    tot[e] = QF(_segsum)(s->tmp, d);
                }
#if VN_FACTORED
                /* fp32 restatement: both anticommuting beliefs of an edge
                 * contain its own message c, and logaddexp(u - c, v - c) =
                 * logaddexp(u, v) - c, so out = V[sym] - c with V[S] =
                 * LAE(0, -(l0 + tot_S)) - LAE(-(l0 + tot_a1), -(l0 + tot_a2))
                 * once per qubit and symbol (a1/a2 as selected at :355-356). */
                REAL V[4];
                int has_y = 0;
                for (int64_t q = 0; q < d; ++q) has_y |= g->edge_sym[g->vn_order[p0 + q]] == 3;
                if (!has_y) {
                    /* no Y-type edge: tot[1] = S_Z, tot[2] = S_X and
                     * V[X] = (l0 + S_X) + F(S_Z), V[Z] = (l0 + S_Z) + F(S_X)
                     * (qo_vnF, the kernels' vn_F) */
                    V[1] = (l0 + tot[2]) + qo_vnF(tot[1], kapc);
                    V[2] = (l0 + tot[1]) + qo_vnF(tot[2], kapc);
                    V[3] = (REAL)0.0;
                } else {
                    for (int S = 1; S <= 3; ++S) {
                        int a1 = S == 1 ? 2 : 1, a2 = S == 3 ? 2 : 3;
                        V[S] = LAE((REAL)0.0, -(l0 + tot[S])) - LAE(-(l0 + tot[a1]), -(l0 + tot[a2]));
                    }
                }
                for (int64_t q = 0; q < d; ++q) {
                    uint8_t sym = g->edge_sym[g->vn_order[p0 + q]];
                    s->vmsg[g->vn_order[p0 + q]] = QF(_clip)(V[sym] - s->cv[q], -CLIP, CLIP);
                }
#else
                for (int64_t q = 0; q < d; ++q) {
                    uint8_t sym = g->edge_sym[g->vn_order[p0 + q]];
                    REAL c = s->cv[q], b[4];
                    for (int e = 1; e <= 3; ++e) b[e] = l0 + (tot[e] - QF(_anti)(e, sym) * c);
                    REAL b_self = sym == 1 ? b[1] : (sym == 3 ? b[3] : b[2]);
                    REAL b_a1 = sym == 1 ? b[2] : b[1];
                    REAL b_a2 = sym == 3 ? b[2] : b[3];
                    REAL out = LAE((REAL)0.0, -b_self) - LAE(-b_a1, -b_a2);
                    s->vmsg[g->vn_order[p0 + q]] = QF(_clip)(out, -CLIP, CLIP);
                }
#endif
            }
        }
        if (capture) {
            if (tr_vn) memcpy(tr_vn + (int64_t)n_snap * E, s->vmsg, sizeof(REAL) * (size_t)E);
            if (tr_cn) memcpy(tr_cn + (int64_t)n_snap * E, s->cmsg, sizeof(REAL) * (size_t)E);
            n_snap++;
        }
    }
    if (succ_out) *succ_out = (uint8_t)success;
    if (iters_out) *iters_out = iters;
    if (tr_counts) { tr_counts[0] = n_gamma; tr_counts[1] = n_snap; }
}

static int QF(_scratch_alloc)(const qsgo_graph *g, QF(_scratch) *s)
{
    int64_t dmax = 1;
    for (int i = 0; i < g->m; ++i) {
        int64_t d = g->cn_ptr[i + 1] - g->cn_ptr[i];
        if (d > dmax) dmax = d;
    }
    for (int j = 0; j < g->n; ++j) {
        int64_t d = g->vn_ptr[j + 1] - g->vn_ptr[j];
        if (d > dmax) dmax = d;
    }
    s->vmsg = (REAL *)malloc(sizeof(REAL) * (size_t)(g->E + 1));
    s->cmsg = (REAL *)malloc(sizeof(REAL) * (size_t)(g->E + 1));
    s->cv = (REAL *)malloc(sizeof(REAL) * (size_t)dmax);
    s->tmp = (REAL *)malloc(sizeof(REAL) * (size_t)dmax);
    s->ph = (REAL *)malloc(sizeof(REAL) * (size_t)dmax);
    s->gains = (REAL *)malloc(sizeof(REAL) * (size_t)(g->m + 1));
    s->ehat = (uint8_t *)malloc((size_t)g->n + 1);
    s->resid = (uint8_t *)malloc((size_t)g->m + 1);
    return s->vmsg && s->cmsg && s->cv && s->tmp && s->ph && s->gains && s->ehat && s->resid;
}

static void QF(_scratch_free)(QF(_scratch) *s)
{
    free(s->vmsg); free(s->cmsg); free(s->cv); free(s->tmp);
    free(s->ph); free(s->gains); free(s->ehat); free(s->resid);
}

/* initial message, decoder.py:405-406 with _marginal_init :255-261 (in
 * double, as the reference, then rounded once to REAL). */
static REAL QF(_v0)(const qsgo_cfg *cfg, double l0)
{
    double v0 = cfg->vn_mode == 0 ? log1p(exp(-l0)) + l0 - 0.6931471805599453 : l0;
    v0 = v0 < -64.0 ? -64.0 : (v0 > 64.0 ? 64.0 : v0);
    return (REAL)v0;
}

typedef struct {
    const qsgo_graph *g; const qsgo_cfg *cfg; double l0;
    const uint8_t *syn; int64_t lo, hi;
    uint8_t *success; uint8_t *e_hat; int64_t *iterations; const TRACE_T *trace;
    int ok;
} QF(_job);

static void *QF(_worker)(void *arg)
{
    QF(_job) *jb = (QF(_job) *)arg;
    const qsgo_graph *g = jb->g;
    QF(_scratch) s;
    jb->ok = QF(_scratch_alloc)(g, &s);
    if (!jb->ok) { QF(_scratch_free)(&s); return NULL; }
    REAL l0 = (REAL)jb->l0, v0 = QF(_v0)(jb->cfg, jb->l0);
    const int L = jb->cfg->l_max;
    for (int64_t b = jb->lo; b < jb->hi; ++b) {
        const TRACE_T *t = jb->trace;
        QF(_decode_one)(g, jb->cfg, l0, v0, jb->syn + b * g->m,
                        jb->success ? jb->success + b : NULL,
                        jb->e_hat ? jb->e_hat + b * g->n : NULL,
                        jb->iterations ? jb->iterations + b : NULL,
                        t && t->unsat ? t->unsat + b * L : NULL,
                        t && t->vn_msgs ? t->vn_msgs + b * L * g->E : NULL,
                        t && t->cn_msgs ? t->cn_msgs + b * L * g->E : NULL,
                        t && t->counts ? t->counts + 2 * b : NULL, &s);
    }
    QF(_scratch_free)(&s);
    return NULL;
}

int QF(_decode)(const qsgo_graph *g, const qsgo_cfg *cfg, double l0, const uint8_t *syn,
                int64_t B, uint8_t *success, uint8_t *e_hat, int64_t *iterations,
                const TRACE_T *trace, int32_t nthreads)
{
    if (!g || !cfg || B < 0 || (B > 0 && !syn) || cfg->l_max < 1) return -1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > B) nthreads = (int32_t)(B > 0 ? B : 1);
    QF(_job) jobs[256];
    pthread_t th[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (QF(_job)){g, cfg, l0, syn, B * t / nthreads, B * (t + 1) / nthreads,
                             success, e_hat, iterations, trace, 0};
    }
    if (nthreads == 1) {
        QF(_worker)(&jobs[0]);
        return jobs[0].ok ? 0 : -3;
    }
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, QF(_worker), &jobs[t]);
    int ok = 1;
    for (int t = 0; t < nthreads; ++t) { pthread_join(th[t], NULL); ok &= jobs[t].ok; }
    return ok ? 0 : -3;
}

/* harness._decode_frames, harness.py:172-182 (with device-style counters). */
int QF(_frames)(const qsgo_graph *g, const qsgo_cfg *cfg, double epsilon, double epsilon0,
                uint64_t seed, int64_t start, int64_t count, uint8_t *fails,
                int64_t *iterations, uint8_t *e_hat, int64_t *counters, int32_t nthreads)
{
    if (!g || count < 0 || !(epsilon0 > 0.0 && epsilon0 < 1.0)) return -1;
    uint8_t *err = (uint8_t *)malloc((size_t)(count * g->n + 1));
    uint8_t *syn = (uint8_t *)malloc((size_t)(count * g->m + 1));
    uint8_t *succ = (uint8_t *)malloc((size_t)count + 1);
    int64_t *it = (int64_t *)malloc(sizeof(int64_t) * (size_t)(count + 1));
    int rc = -3;
    if (err && syn && succ && it) {
        rc = qsgo_sample_errors(g->n, epsilon, seed, start, count, err);
        if (rc == 0) {
            qsgo_syndromes_of(g, err, count, syn);
            double l0 = log(3.0 * (1.0 - epsilon0) / epsilon0); /* channel.py:48-52 */
            rc = QF(_decode)(g, cfg, l0, syn, count, succ, e_hat, it, NULL, nthreads);
        }
        if (rc == 0) {
            int64_t nf = 0, si = 0;
            for (int64_t b = 0; b < count; ++b) {
                if (fails) fails[b] = !succ[b];
                if (iterations) iterations[b] = it[b];
                nf += !succ[b];
                si += it[b];
            }
            if (counters) {
                counters[0] += count;
                counters[1] += nf;
                counters[2] += si;
                counters[3] += g->E * (si - count);
            }
        }
    }
    free(err); free(syn); free(succ); free(it);
    return rc;
}

#undef QF
