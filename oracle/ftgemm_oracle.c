/*
 * ftgemm_oracle.c -- plain, slow, obviously-correct CPU oracle for the online
 * ABFT GEMM of arXiv 2305.01024 ("Anatomy of High-Performance GEMM with Online
 * Fault Tolerance on GPUs").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path
 * (paper_2305_01024_b200/csrc); neither side includes or links the other.
 *
 * Arithmetic: FP64 throughout (acc_mode FP64), or -- only for pinning the FP32
 * SIMT kernel bit-exactly -- the paper's SGEMM numerics (acc_mode FP32SEQ):
 * every output element accumulated with one correctly-rounded fmaf per k, in
 * ascending k (section 3.1, the step-wise SGEMM whose thread
 * tile accumulates C_t over the k-loop).
 *
 * What is computed, per output tile (rows P_i x cols Q_j, sizes from the plan):
 *   product      P = A B                         PAPER.md:150-164 Eq. (1)-(3)
 *   encode       Ac = e^T A_i, Br = B_j e        Eq. (1) A^c, Eq. (2) B^r
 *   references   R_row = A_i Br,  R_col = Ac B_j (the carried C^r, C^c of Eq. (3))
 *   verify       r_p = sum_q P[p,q] - R_row[p];  c_q = sum_p P[p,q] - R_col[q]
 *                flagged iff !(|r| <= tau)       PAPER.md:166 "exceeds a
 *                                                predetermined threshold"
 *   locate       the single flagged row x single flagged column
 *                                                PAPER.md:317 "relative positions
 *                                                in two checksums"
 *   correct      P[p*,q*] = R_row[p*] - sum_{q != q*} P[p*,q]
 *                                                PAPER.md:317 "offset in the
 *                                                checksums", :505 "subtracting the
 *                                                error magnitude" (R2)
 *   output       C = alpha P + beta C_in, rounded to the output dtype.
 * Fault injection (section 5.3): a bit flip of (or an addend to) the
 * FP32 partial accumulator of one element after the k-block containing k_elem.
 * Threshold (PAPER.md gives no value; reading R1):
 *   tau_row(p) = u (l1 sqrt(K) |R_row[p]| + l2 ||A[p,:]||_2 ||Br||_2)
 *   tau_col(q) = u (l1 sqrt(K) |R_col[q]| + l2 ||Ac||_2 ||B[:,q]||_2)
 * Tiles are independent, so any subset of tiles can be checked by passing the
 * sub-block (the tile-sampled oracle in tests/ relies on this).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_ERR_ARG 1
#define OR_ERR_NOMEM 2

enum { OR_ACC_FP64 = 0, OR_ACC_FP32SEQ = 1 };
enum { OR_OUT_F32 = 0, OR_OUT_BF16 = 1 };
enum { OR_FT_OFF = 0, OR_FT_DETECT = 1, OR_FT_CORRECT = 2, OR_FT_DETECT_ROWS = 3 };
enum { OR_INJ_FLIP = 0, OR_INJ_ADD = 1 };
enum { OR_TGT_ACC = 0, OR_TGT_ROW_REF = 1, OR_TGT_COL_REF = 2 };
enum { OR_EV_CORRECTED = 1, OR_EV_CHECKSUM_ONLY = 2, OR_EV_UNCORRECTABLE = 3, OR_EV_LOCATED = 4, OR_EV_DETECTED = 5 };

typedef struct {
    int64_t row, col, k_elem;
    int32_t bit, mode, target;
    float addend;
} oracle_inject_t;

typedef struct {
    int64_t row, col;
    int32_t tile_m, tile_n, kind, n_rows, n_cols, k_checked;
    double resid_row, resid_col, tau_row, tau_col;
} oracle_event_t;

typedef struct {
    int64_t tiles_checked, tiles_detected, corrected, checksum_only,
            uncorrectable, located, events, dropped;
} oracle_counts_t;

typedef struct {
    int64_t M, N, K;
    double alpha, beta;
    const float *A; int64_t lda;
    const float *B; int64_t ldb;
    const float *Cin; int64_t ldc;          /* may be NULL when beta == 0 */
    int32_t out_dtype; int32_t acc_mode;
    void *Cout;                             /* leading dimension ldc */
    int64_t tile_m, tile_n, bk;
    double u_acc, lambda1, lambda2;
    int32_t ft_level; int32_t n_inj;
    const oracle_inject_t *inj;
    oracle_counts_t *counts;
    oracle_event_t *events; int32_t max_events; int32_t pad0;
    double *P_out;       /* optional M x N, ld N: accumulator after correction */
    double *resid_row;   /* optional M x tiles_n */
    double *resid_col;   /* optional tiles_m x N */
    double *tau_row;     /* optional M x tiles_n */
    double *tau_col;     /* optional tiles_m x N */
    int64_t ks;          /* > 0: online verification every ks of K (run_tile_intervals) */
} oracle_problem_t;

/* ---- scalar helpers -------------------------------------------------------- */

static float flip_bit(float x, int bit) {
    uint32_t u; memcpy(&u, &x, 4); u ^= (1u << bit); memcpy(&x, &u, 4); return x;
}

/* Round a double directly to bfloat16 (round to nearest, ties to even), no
 * intermediate float rounding.  Returns the 16-bit pattern. */
static uint16_t double_to_bf16(double d) {
    if (isnan(d)) return 0x7FC0;
    float f = (float)d;                 /* used only to get sign / exponent range */
    if (isinf(f) && !isinf(d)) {        /* overflow of float => overflow of bf16 */
        return d > 0 ? 0x7F80 : 0xFF80;
    }
    if (isinf(d)) return d > 0 ? 0x7F80 : 0xFF80;
    if (d == 0.0) return signbit(d) ? 0x8000 : 0x0000;
    /* bf16 has 8 significand bits; for normal range scale to find spacing. */
    int e; double m = frexp(fabs(d), &e);       /* |d| = m 2^e, m in [0.5,1) */
    int emin = -125;                             /* smallest normal: 2^-126 = 0.5*2^-125 */
    int q = (e < emin) ? emin : e;               /* subnormals use fixed spacing */
    double spacing = ldexp(1.0, q - 8);          /* ulp for 8 significant bits */
    double t = fabs(d) / spacing;                /* exact (power-of-two scaling) */
    double fl = floor(t), rem = t - fl;
    double r = fl;
    if (rem > 0.5 || (rem == 0.5 && fmod(fl, 2.0) != 0.0)) r = fl + 1.0;
    double v = r * spacing;
    float fv = (float)v;                         /* exact: v has <= 8 significant bits */
    if (isinf(fv)) return signbit(d) ? 0xFF80 : 0x7F80;
    uint32_t u; memcpy(&u, &fv, 4);
    if (signbit(d)) u |= 0x80000000u;
    return (uint16_t)(u >> 16);
}

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

/* ---- encode (Eq. 1, Eq. 2) ------------------------------------------------- */

/* Ac[i*K + k] = sum_{p in P_i} A[p,k]  (column checksum e^T A per M-tile). */
int oracle_encode_col(int64_t M, int64_t K, const float *A, int64_t lda, int64_t tile_m, double *Ac) {
    if (M < 1 || K < 1 || tile_m < 1 || !A || !Ac) return OR_ERR_ARG;
    int64_t tm = cdiv(M, tile_m);
    for (int64_t i = 0; i < tm; ++i) {
        for (int64_t k = 0; k < K; ++k) Ac[i * K + k] = 0.0;
        for (int64_t p = i * tile_m; p < M && p < (i + 1) * tile_m; ++p)
            for (int64_t k = 0; k < K; ++k) Ac[i * K + k] += (double)A[p * lda + k];
    }
    return OR_OK;
}

/* Br[j*K + k] = sum_{q in Q_j} B[k,q]  (row checksum B e per N-tile). */
int oracle_encode_row(int64_t K, int64_t N, const float *B, int64_t ldb, int64_t tile_n, double *Br) {
    if (N < 1 || K < 1 || tile_n < 1 || !B || !Br) return OR_ERR_ARG;
    int64_t tn = cdiv(N, tile_n);
    for (int64_t j = 0; j < tn; ++j)
        for (int64_t k = 0; k < K; ++k) {
            double s = 0.0;
            for (int64_t q = j * tile_n; q < N && q < (j + 1) * tile_n; ++q) s += (double)B[k * ldb + q];
            Br[j * K + k] = s;
        }
    return OR_OK;
}

/* ---- the per-tile algorithm -------------------------------------------------- */

typedef struct { int64_t idx; int64_t keff; } inj_ref_t;

static int cmp_keff(const void *a, const void *b) {
    const inj_ref_t *x = (const inj_ref_t *)a, *y = (const inj_ref_t *)b;
    if (x->keff != y->keff) return x->keff < y->keff ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static int64_t eff_k(const oracle_problem_t *pr, int64_t k_elem) {
    int64_t nkb = cdiv(pr->K, pr->bk);
    int64_t kb = k_elem / pr->bk;
    if (kb < 0) kb = 0;
    if (kb > nkb - 1) kb = nkb - 1;
    int64_t ke = (kb + 1) * pr->bk;
    return ke < pr->K ? ke : pr->K;
}

/* Apply one injection to a partial value x (FP32 view) -> new FP32 value. */
static float inject_value(float x, const oracle_inject_t *in) {
    if (in->mode == OR_INJ_ADD) return x + in->addend;   /* FP32 add, like the accumulator */
    return flip_bit(x, in->bit);
}

static void emit_event_k(const oracle_problem_t *pr, int64_t ti, int64_t tj, int kind,
                         int64_t row, int64_t col, int nr, int nc,
                         double rr, double rc, double tr, double tc, int64_t kchk) {
    oracle_counts_t *ct = pr->counts;
    int64_t slot;
#pragma omp atomic capture
    slot = ct->events++;
    if (pr->events && slot < pr->max_events) {
        oracle_event_t *e = &pr->events[slot];
        e->row = row; e->col = col; e->tile_m = (int32_t)ti; e->tile_n = (int32_t)tj;
        e->kind = kind; e->n_rows = nr; e->n_cols = nc; e->k_checked = (int32_t)kchk;
        e->resid_row = rr; e->resid_col = rc; e->tau_row = tr; e->tau_col = tc;
    } else {
#pragma omp atomic
        ct->dropped++;
    }
}

static void emit_event(const oracle_problem_t *pr, int64_t ti, int64_t tj, int kind,
                       int64_t row, int64_t col, int nr, int nc,
                       double rr, double rc, double tr, double tc) {
    emit_event_k(pr, ti, tj, kind, row, col, nr, nc, rr, rc, tr, tc, pr->K);
}

static int run_tile(const oracle_problem_t *pr, int64_t ti, int64_t tj) {
    const int64_t M = pr->M, N = pr->N, K = pr->K;
    const int64_t r0 = ti * pr->tile_m, c0 = tj * pr->tile_n;
    const int64_t bm = (r0 + pr->tile_m <= M) ? pr->tile_m : M - r0;
    const int64_t bn = (c0 + pr->tile_n <= N) ? pr->tile_n : N - c0;
    const float *A = pr->A, *B = pr->B;
    const int64_t lda = pr->lda, ldb = pr->ldb;
    const int64_t tiles_n = cdiv(N, pr->tile_n);

    double *P = (double *)calloc((size_t)(bm * bn), sizeof(double));
    float *Pf = NULL;
    double *Ac = (double *)calloc((size_t)K, sizeof(double));
    double *Br = (double *)calloc((size_t)K, sizeof(double));
    double *Rr = (double *)calloc((size_t)bm, sizeof(double));
    double *Rc = (double *)calloc((size_t)bn, sizeof(double));
    double *Sr = (double *)calloc((size_t)bm, sizeof(double));
    double *Sc = (double *)calloc((size_t)bn, sizeof(double));
    double *tr = (double *)calloc((size_t)bm, sizeof(double));
    double *tc = (double *)calloc((size_t)bn, sizeof(double));
    inj_ref_t *mine = (inj_ref_t *)calloc((size_t)(pr->n_inj > 0 ? pr->n_inj : 1), sizeof(inj_ref_t));
    if (!P || !Ac || !Br || !Rr || !Rc || !Sr || !Sc || !tr || !tc || !mine) return OR_ERR_NOMEM;

    /* Injections that land in this tile, in (k_eff, list) order. */
    int nm = 0;
    for (int32_t t = 0; t < pr->n_inj; ++t) {
        const oracle_inject_t *in = &pr->inj[t];
        int64_t row = in->row, col = in->col;
        int hit = 0;
        if (in->target == OR_TGT_ACC) hit = row >= r0 && row < r0 + bm && col >= c0 && col < c0 + bn;
        else if (in->target == OR_TGT_ROW_REF) hit = row >= r0 && row < r0 + bm && col >= c0 && col < c0 + bn;
        else if (in->target == OR_TGT_COL_REF) hit = row >= r0 && row < r0 + bm && col >= c0 && col < c0 + bn;
        if (hit) { mine[nm].idx = t; mine[nm].keff = eff_k(pr, in->k_elem); ++nm; }
    }
    qsort(mine, (size_t)nm, sizeof(inj_ref_t), cmp_keff);

    /* Step 1: product P = A_i B_j (Eq. 3, the C block of C^f). */
    if (pr->acc_mode == OR_ACC_FP64) {
        for (int64_t p = 0; p < bm; ++p) {
            double *Pp = P + p * bn;
            for (int64_t k = 0; k < K; ++k) {
                double a = (double)A[(r0 + p) * lda + k];
                const float *Bk = B + k * ldb + c0;
                for (int64_t q = 0; q < bn; ++q) Pp[q] += a * (double)Bk[q];
            }
        }
        /* Step 2: accumulator faults.  The FP32 partial x after
         * the k-block of k_elem is flipped; the difference delta = y - x is
         * carried by the remaining accumulation. */
        for (int t = 0; t < nm; ++t) {
            const oracle_inject_t *in = &pr->inj[mine[t].idx];
            if (in->target != OR_TGT_ACC) continue;
            int64_t p = in->row - r0, q = in->col - c0;
            double s = 0.0;
            for (int64_t k = 0; k < mine[t].keff; ++k) s += (double)A[in->row * lda + k] * (double)B[k * ldb + in->col];
            /* earlier faults on the same element (smaller k_eff) are part of the
             * partial sum: they are P's offset from the fault-free full sum */
            double full = 0.0;
            for (int64_t k = 0; k < K; ++k) full += (double)A[in->row * lda + k] * (double)B[k * ldb + in->col];
            double prior = P[p * bn + q] - full;      /* sum of earlier deltas (0 if none) */
            if (!isfinite(P[p * bn + q])) continue;   /* already non-finite: stays so */
            float x = (float)(s + prior);
            float y = inject_value(x, in);
            if (!isfinite(y)) P[p * bn + q] = (double)y;
            else P[p * bn + q] += (double)y - (double)x;
        }
    } else {
        /* FP32SEQ: fmaf per k, ascending k; faults applied at the exact k-block
         * boundary to the running FP32 accumulator. */
        Pf = (float *)calloc((size_t)(bm * bn), sizeof(float));
        if (!Pf) return OR_ERR_NOMEM;
        int next = 0;
        int64_t kstart = 0;
        while (kstart < K) {
            int64_t kend = K;
            while (next < nm && pr->inj[mine[next].idx].target != OR_TGT_ACC) ++next;
            if (next < nm) kend = mine[next].keff;
            for (int64_t p = 0; p < bm; ++p) {
                float *Pp = Pf + p * bn;
                for (int64_t k = kstart; k < kend; ++k) {
                    float a = A[(r0 + p) * lda + k];
                    const float *Bk = B + k * ldb + c0;
                    for (int64_t q = 0; q < bn; ++q) Pp[q] = fmaf(a, Bk[q], Pp[q]);
                }
            }
            kstart = kend;
            /* apply every ACC injection whose k_eff == kend */
            while (next < nm && mine[next].keff == kend) {
                const oracle_inject_t *in = &pr->inj[mine[next].idx];
                if (in->target == OR_TGT_ACC) {
                    int64_t p = in->row - r0, q = in->col - c0;
                    Pf[p * bn + q] = inject_value(Pf[p * bn + q], in);
                }
                ++next;
            }
        }
        for (int64_t e = 0; e < bm * bn; ++e) P[e] = (double)Pf[e];
    }

    /* Step 3: encode (Eq. 1, Eq. 2). */
    for (int64_t p = 0; p < bm; ++p)
        for (int64_t k = 0; k < K; ++k) Ac[k] += (double)A[(r0 + p) * lda + k];
    for (int64_t k = 0; k < K; ++k) {
        double s = 0.0;
        for (int64_t q = 0; q < bn; ++q) s += (double)B[k * ldb + c0 + q];
        Br[k] = s;
    }
    /* Step 4: carried references C^r = A (B e), C^c = (e^T A) B (Eq. 3). */
    for (int64_t p = 0; p < bm; ++p) {
        double s = 0.0;
        for (int64_t k = 0; k < K; ++k) s += (double)A[(r0 + p) * lda + k] * Br[k];
        Rr[p] = s;
    }
    for (int64_t k = 0; k < K; ++k)
        for (int64_t q = 0; q < bn; ++q) Rc[q] += Ac[k] * (double)B[k * ldb + c0 + q];

    /* Reference faults (targets ROW_REF / COL_REF): same rule applied to the
     * FP32 partial of the reference sum. */
    for (int t = 0; t < nm; ++t) {
        const oracle_inject_t *in = &pr->inj[mine[t].idx];
        if (in->target == OR_TGT_ROW_REF) {
            int64_t p = in->row - r0;
            double s = 0.0;
            for (int64_t k = 0; k < mine[t].keff; ++k) s += (double)A[in->row * lda + k] * Br[k];
            float x = (float)s, y = inject_value(x, in);
            if (!isfinite(y)) Rr[p] = (double)y; else Rr[p] += (double)y - (double)x;
        } else if (in->target == OR_TGT_COL_REF) {
            int64_t q = in->col - c0;
            double s = 0.0;
            for (int64_t k = 0; k < mine[t].keff; ++k) s += Ac[k] * (double)B[k * ldb + in->col];
            float x = (float)s, y = inject_value(x, in);
            if (!isfinite(y)) Rc[q] = (double)y; else Rc[q] += (double)y - (double)x;
        }
    }

    /* Step 5: recomputed sums, residuals and thresholds. */
    for (int64_t p = 0; p < bm; ++p) {
        double s = 0.0;
        for (int64_t q = 0; q < bn; ++q) s += P[p * bn + q];
        Sr[p] = s;
    }
    for (int64_t p = 0; p < bm; ++p)
        for (int64_t q = 0; q < bn; ++q) Sc[q] += P[p * bn + q];

    double nBr = 0.0, nAc = 0.0;
    for (int64_t k = 0; k < K; ++k) { nBr += Br[k] * Br[k]; nAc += Ac[k] * Ac[k]; }
    nBr = sqrt(nBr); nAc = sqrt(nAc);
    const double sqK = sqrt((double)K), u = pr->u_acc, l1 = pr->lambda1, l2 = pr->lambda2;
    for (int64_t p = 0; p < bm; ++p) {
        double na = 0.0;
        for (int64_t k = 0; k < K; ++k) { double a = A[(r0 + p) * lda + k]; na += a * a; }
        tr[p] = u * (l1 * sqK * fabs(Rr[p]) + l2 * sqrt(na) * nBr);
    }
    for (int64_t q = 0; q < bn; ++q) {
        double nb = 0.0;
        for (int64_t k = 0; k < K; ++k) { double b = B[k * ldb + c0 + q]; nb += b * b; }
        tc[q] = u * (l1 * sqK * fabs(Rc[q]) + l2 * nAc * sqrt(nb));
    }

    int nr = 0, nc = 0;
    int64_t pstar = -1, qstar = -1;
    double rstar = 0.0, cstar = 0.0;
    for (int64_t p = 0; p < bm; ++p) {
        double r = Sr[p] - Rr[p];
        if (pr->resid_row) pr->resid_row[(r0 + p) * tiles_n + tj] = r;
        if (pr->tau_row) pr->tau_row[(r0 + p) * tiles_n + tj] = tr[p];
        if (!(fabs(r) <= tr[p])) { if (nr == 0) { pstar = p; rstar = r; } ++nr; }
    }
    for (int64_t q = 0; q < bn; ++q) {
        double c = Sc[q] - Rc[q];
        if (pr->resid_col) pr->resid_col[ti * N + c0 + q] = c;
        if (pr->tau_col) pr->tau_col[ti * N + c0 + q] = tc[q];
        if (!(fabs(c) <= tc[q])) { if (nc == 0) { qstar = q; cstar = c; } ++nc; }
    }

    /* Step 6 (offline, detect-only ABFT, R15): only
     * the row checks count; any flagged row marks the tile for re-computation,
     * C is left as computed. */
    if (pr->ft_level == OR_FT_DETECT_ROWS) {
#pragma omp atomic
        pr->counts->tiles_checked++;
        if (nr > 0) {
#pragma omp atomic
            pr->counts->tiles_detected++;
            emit_event(pr, ti, tj, OR_EV_DETECTED, r0 + pstar, -1, nr, 0, rstar, 0.0, tr[pstar], 0.0);
        }
    }
    /* Step 6: decide (R3-R5) and correct. */
    else if (pr->ft_level != OR_FT_OFF) {
#pragma omp atomic
        pr->counts->tiles_checked++;
        if (nr > 0 || nc > 0) {
#pragma omp atomic
            pr->counts->tiles_detected++;
        }
        double trs = pstar >= 0 ? tr[pstar] : 0.0, tcs = qstar >= 0 ? tc[qstar] : 0.0;
        if (nr == 1 && nc == 1) {
            double big = fabs(rstar) > fabs(cstar) ? fabs(rstar) : fabs(cstar);
            double guard = trs + tcs + 2.0 * u * (double)(bm + bn) * big;
            int consistent = !(fabs(rstar - cstar) > guard);
            if (consistent) {
                if (pr->ft_level == OR_FT_CORRECT) {
                    double s = 0.0;
                    for (int64_t q = 0; q < bn; ++q) if (q != qstar) s += P[pstar * bn + q];
                    P[pstar * bn + qstar] = Rr[pstar] - s;
#pragma omp atomic
                    pr->counts->corrected++;
                    emit_event(pr, ti, tj, OR_EV_CORRECTED, r0 + pstar, c0 + qstar, nr, nc, rstar, cstar, trs, tcs);
                } else {
#pragma omp atomic
                    pr->counts->located++;
                    emit_event(pr, ti, tj, OR_EV_LOCATED, r0 + pstar, c0 + qstar, nr, nc, rstar, cstar, trs, tcs);
                }
            } else {
#pragma omp atomic
                pr->counts->uncorrectable++;
                emit_event(pr, ti, tj, OR_EV_UNCORRECTABLE, r0 + pstar, c0 + qstar, nr, nc, rstar, cstar, trs, tcs);
            }
        } else if ((nr == 1 && nc == 0) || (nr == 0 && nc == 1)) {
#pragma omp atomic
            pr->counts->checksum_only++;
            emit_event(pr, ti, tj, OR_EV_CHECKSUM_ONLY, nr ? r0 + pstar : -1, nc ? c0 + qstar : -1,
                       nr, nc, rstar, cstar, trs, tcs);
        } else if (nr > 0 || nc > 0) {
#pragma omp atomic
            pr->counts->uncorrectable++;
            emit_event(pr, ti, tj, OR_EV_UNCORRECTABLE, nr ? r0 + pstar : -1, nc ? c0 + qstar : -1,
                       nr, nc, rstar, cstar, trs, tcs);
        }
    }

    /* Step 7: C = alpha P + beta C_in, rounded to the output dtype. */
    for (int64_t p = 0; p < bm; ++p)
        for (int64_t q = 0; q < bn; ++q) {
            int64_t g = (r0 + p) * pr->ldc + (c0 + q);
            double cin = (pr->beta != 0.0 && pr->Cin) ? (double)pr->Cin[g] : 0.0;
            if (pr->P_out) pr->P_out[(r0 + p) * N + (c0 + q)] = P[p * bn + q];
            if (pr->acc_mode == OR_ACC_FP32SEQ && pr->out_dtype == OR_OUT_F32) {
                /* SIMT epilogue numerics: fmaf(alpha, acc, beta * C_in) in FP32 */
                float acc = (float)P[p * bn + q];
                float bc = (pr->beta != 0.0) ? (float)pr->beta * (float)cin : 0.0f;
                ((float *)pr->Cout)[g] = fmaf((float)pr->alpha, acc, bc);
            } else {
                double v = pr->alpha * P[p * bn + q] + pr->beta * cin;
                if (pr->out_dtype == OR_OUT_F32) ((float *)pr->Cout)[g] = (float)v;
                else ((uint16_t *)pr->Cout)[g] = double_to_bf16(v);
            }
        }

    free(P); free(Pf); free(Ac); free(Br); free(Rr); free(Rc); free(Sr); free(Sc);
    free(tr); free(tc); free(mine);
    return OR_OK;
}

/* ---- online verification every K_s -----------------
 * Chen's outer-product online ABFT: C^f = sum_s A^c(:,s) B^r(s,:) keeps the
 * checksum relation after every step s, so the tile is verified (and one error
 * corrected) after each K_s-wide step instead of once at the end -- "the online
 * version, which corrects a single error for each step of the outer-product
 * update, can handle multiple errors".  Step by step, FP64:
 *   for each step [k0, k1), k1 = min(K, k0 + ks):
 *     P += A_i[:, k0:k1] B_j[k0:k1, :];  R_row += A_i[:, k0:k1] Br[k0:k1];
 *     R_col += Ac[k0:k1] B_j[k0:k1, :]                (the carried C^r, C^c)
 *     faults whose k-block ends in (k0, k1]: the FP32 view x of the running
 *       value at that k-block is flipped (or offset) and the difference kept
 *     verify with tau from DESIGN.md R1 / R17 (sqrt(k1) in place of sqrt(K),
 *       the full-K norms) -- before the end of K the columns only when a row
 *       is flagged (R20) -- decide and correct as at the end of K;
 *       every step's check counts in tiles_checked; events carry k_checked = k1.
 * Mode FP64 only (the tensor-core paths). */
static int run_tile_intervals(const oracle_problem_t *pr, int64_t ti, int64_t tj) {
    const int64_t M = pr->M, N = pr->N, K = pr->K;
    const int64_t r0 = ti * pr->tile_m, c0 = tj * pr->tile_n;
    const int64_t bm = (r0 + pr->tile_m <= M) ? pr->tile_m : M - r0;
    const int64_t bn = (c0 + pr->tile_n <= N) ? pr->tile_n : N - c0;
    const float *A = pr->A, *B = pr->B;
    const int64_t lda = pr->lda, ldb = pr->ldb;
    double *P = (double *)calloc((size_t)(bm * bn), sizeof(double));
    double *Ac = (double *)calloc((size_t)K, sizeof(double));
    double *Br = (double *)calloc((size_t)K, sizeof(double));
    double *Rr = (double *)calloc((size_t)bm, sizeof(double));
    double *Rc = (double *)calloc((size_t)bn, sizeof(double));
    double *na = (double *)calloc((size_t)bm, sizeof(double));
    double *nb = (double *)calloc((size_t)bn, sizeof(double));
    double *tr = (double *)calloc((size_t)bm, sizeof(double));
    double *tc = (double *)calloc((size_t)bn, sizeof(double));
    double *Sc = (double *)calloc((size_t)bn, sizeof(double));
    if (!P || !Ac || !Br || !Rr || !Rc || !na || !nb || !tr || !tc || !Sc) return OR_ERR_NOMEM;

    /* encode (Eq. 1, 2) and the full-K norms of the threshold (R1) */
    for (int64_t p = 0; p < bm; ++p)
        for (int64_t k = 0; k < K; ++k) {
            double a = (double)A[(r0 + p) * lda + k];
            Ac[k] += a; na[p] += a * a;
        }
    for (int64_t k = 0; k < K; ++k)
        for (int64_t q = 0; q < bn; ++q) {
            double b = (double)B[k * ldb + c0 + q];
            Br[k] += b; nb[q] += b * b;
        }
    double nBr = 0.0, nAc = 0.0;
    for (int64_t k = 0; k < K; ++k) { nBr += Br[k] * Br[k]; nAc += Ac[k] * Ac[k]; }
    nBr = sqrt(nBr); nAc = sqrt(nAc);
    const double u = pr->u_acc, l1 = pr->lambda1, l2 = pr->lambda2;

    for (int64_t k0 = 0; k0 < K; ) {
        const int64_t k1 = (k0 + pr->ks < K) ? k0 + pr->ks : K;
        /* faults of this step, applied in (k_eff, list) order at their k-block:
         * the running value at k_eff = value at k0 + the products in [k0, k_eff) */
        int64_t kdone = k0;
        for (;;) {
            int64_t knext = k1 + 1; int32_t first = -1;
            for (int32_t t = 0; t < pr->n_inj; ++t) {
                const oracle_inject_t *in = &pr->inj[t];
                if (in->row < r0 || in->row >= r0 + bm || in->col < c0 || in->col >= c0 + bn) continue;
                int64_t ke = eff_k(pr, in->k_elem);
                if (ke > kdone && ke <= k1 && ke < knext) { knext = ke; first = t; }
            }
            if (first < 0) break;
            /* advance every running sum to knext */
            for (int64_t p = 0; p < bm; ++p)
                for (int64_t k = kdone; k < knext; ++k) {
                    double a = (double)A[(r0 + p) * lda + k];
                    for (int64_t q = 0; q < bn; ++q) P[p * bn + q] += a * (double)B[k * ldb + c0 + q];
                    Rr[p] += a * Br[k];
                }
            for (int64_t k = kdone; k < knext; ++k)
                for (int64_t q = 0; q < bn; ++q) Rc[q] += Ac[k] * (double)B[k * ldb + c0 + q];
            kdone = knext;
            for (int32_t t = first; t < pr->n_inj; ++t) {       /* every fault at knext, list order */
                const oracle_inject_t *in = &pr->inj[t];
                if (in->row < r0 || in->row >= r0 + bm || in->col < c0 || in->col >= c0 + bn) continue;
                if (eff_k(pr, in->k_elem) != knext) continue;
                double *v = in->target == OR_TGT_ROW_REF ? &Rr[in->row - r0]
                          : in->target == OR_TGT_COL_REF ? &Rc[in->col - c0]
                          : &P[(in->row - r0) * bn + (in->col - c0)];
                if (!isfinite(*v)) continue;
                float x = (float)*v, y = inject_value(x, in);
                if (!isfinite(y)) *v = (double)y; else *v += (double)y - (double)x;
            }
        }
        for (int64_t p = 0; p < bm; ++p)
            for (int64_t k = kdone; k < k1; ++k) {
                double a = (double)A[(r0 + p) * lda + k];
                for (int64_t q = 0; q < bn; ++q) P[p * bn + q] += a * (double)B[k * ldb + c0 + q];
                Rr[p] += a * Br[k];
            }
        for (int64_t k = kdone; k < k1; ++k)
            for (int64_t q = 0; q < bn; ++q) Rc[q] += Ac[k] * (double)B[k * ldb + c0 + q];

        /* verify this step: the rows first (R20) -- a
         * corrupted element of C always moves its row sum, so a step before the
         * end of K whose rows all match is clean for C and its columns are not
         * examined; otherwise (and at the end of K) rows and columns as usual */
        const double sqk = sqrt((double)k1);
        int nr = 0, nc = 0; int64_t pstar = -1, qstar = -1; double rstar = 0.0, cstar = 0.0;
        for (int64_t q = 0; q < bn; ++q) Sc[q] = 0.0;
        for (int64_t p = 0; p < bm; ++p) {
            double s = 0.0;
            for (int64_t q = 0; q < bn; ++q) { s += P[p * bn + q]; Sc[q] += P[p * bn + q]; }
            tr[p] = u * (l1 * sqk * fabs(Rr[p]) + l2 * sqrt(na[p]) * nBr);
            double r = s - Rr[p];
            if (!(fabs(r) <= tr[p])) { if (nr == 0) { pstar = p; rstar = r; } ++nr; }
        }
        if (k1 < K && nr == 0) {
#pragma omp atomic
            pr->counts->tiles_checked++;
            k0 = k1;
            continue;
        }
        for (int64_t q = 0; q < bn; ++q) {
            tc[q] = u * (l1 * sqk * fabs(Rc[q]) + l2 * nAc * sqrt(nb[q]));
            double c = Sc[q] - Rc[q];
            if (!(fabs(c) <= tc[q])) { if (nc == 0) { qstar = q; cstar = c; } ++nc; }
        }
#pragma omp atomic
        pr->counts->tiles_checked++;
        if (nr > 0 || nc > 0) {
#pragma omp atomic
            pr->counts->tiles_detected++;
        }
        double trs = pstar >= 0 ? tr[pstar] : 0.0, tcs = qstar >= 0 ? tc[qstar] : 0.0;
        if (nr == 1 && nc == 1) {
            double big = fabs(rstar) > fabs(cstar) ? fabs(rstar) : fabs(cstar);
            int consistent = !(fabs(rstar - cstar) > trs + tcs + 2.0 * u * (double)(bm + bn) * big);
            if (consistent && pr->ft_level == OR_FT_CORRECT) {
                double s = 0.0;
                for (int64_t q = 0; q < bn; ++q) if (q != qstar) s += P[pstar * bn + q];
                P[pstar * bn + qstar] = Rr[pstar] - s;
#pragma omp atomic
                pr->counts->corrected++;
                emit_event_k(pr, ti, tj, OR_EV_CORRECTED, r0 + pstar, c0 + qstar, nr, nc, rstar, cstar, trs, tcs, k1);
            } else if (consistent) {
#pragma omp atomic
                pr->counts->located++;
                emit_event_k(pr, ti, tj, OR_EV_LOCATED, r0 + pstar, c0 + qstar, nr, nc, rstar, cstar, trs, tcs, k1);
            } else {
#pragma omp atomic
                pr->counts->uncorrectable++;
                emit_event_k(pr, ti, tj, OR_EV_UNCORRECTABLE, r0 + pstar, c0 + qstar, nr, nc, rstar, cstar, trs, tcs, k1);
            }
        } else if ((nr == 1 && nc == 0) || (nr == 0 && nc == 1)) {
#pragma omp atomic
            pr->counts->checksum_only++;
            emit_event_k(pr, ti, tj, OR_EV_CHECKSUM_ONLY, nr ? r0 + pstar : -1, nc ? c0 + qstar : -1,
                         nr, nc, rstar, cstar, trs, tcs, k1);
        } else if (nr > 0 || nc > 0) {
#pragma omp atomic
            pr->counts->uncorrectable++;
            emit_event_k(pr, ti, tj, OR_EV_UNCORRECTABLE, nr ? r0 + pstar : -1, nc ? c0 + qstar : -1,
                         nr, nc, rstar, cstar, trs, tcs, k1);
        }
        k0 = k1;
    }
    /* C = alpha P + beta C_in, rounded to the output dtype */
    for (int64_t p = 0; p < bm; ++p)
        for (int64_t q = 0; q < bn; ++q) {
            int64_t g = (r0 + p) * pr->ldc + (c0 + q);
            double cin = (pr->beta != 0.0 && pr->Cin) ? (double)pr->Cin[g] : 0.0;
            if (pr->P_out) pr->P_out[(r0 + p) * N + (c0 + q)] = P[p * bn + q];
            double v = pr->alpha * P[p * bn + q] + pr->beta * cin;
            if (pr->out_dtype == OR_OUT_F32) ((float *)pr->Cout)[g] = (float)v;
            else ((uint16_t *)pr->Cout)[g] = double_to_bf16(v);
        }
    free(P); free(Ac); free(Br); free(Rr); free(Rc); free(na); free(nb); free(tr); free(tc); free(Sc);
    return OR_OK;
}

int oracle_ftgemm(oracle_problem_t *pr) {
    if (!pr || pr->M < 1 || pr->N < 1 || pr->K < 1 || !pr->A || !pr->B || !pr->Cout ||
        pr->tile_m < 1 || pr->tile_n < 1 || pr->bk < 1 || !pr->counts ||
        pr->lda < pr->K || pr->ldb < pr->N || pr->ldc < pr->N || (pr->beta != 0.0 && !pr->Cin))
        return OR_ERR_ARG;
    memset(pr->counts, 0, sizeof(*pr->counts));
    const int64_t tm = cdiv(pr->M, pr->tile_m), tn = cdiv(pr->N, pr->tile_n);
    int err = OR_OK;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < tm * tn; ++t) {
        int e = (pr->ks > 0 && pr->ft_level != OR_FT_OFF) ? run_tile_intervals(pr, t / tn, t % tn)
                                                            : run_tile(pr, t / tn, t % tn);
        if (e) {
#pragma omp critical
            err = e;
        }
    }
    return err;
}

/* Plain FP64 GEMM, C = alpha A B + beta C_in, for the cpu_baseline timing and
 * for pinning the product alone (no ABFT). */
int oracle_gemm_f64(int64_t M, int64_t N, int64_t K, double alpha, const float *A, int64_t lda,
                    const float *B, int64_t ldb, double beta, const float *Cin, int64_t ldc, double *Cout) {
    if (M < 1 || N < 1 || K < 1) return OR_ERR_ARG;
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < M; ++p) {
        double *row = Cout + p * N;
        for (int64_t q = 0; q < N; ++q) row[q] = 0.0;
        for (int64_t k = 0; k < K; ++k) {
            double a = (double)A[p * lda + k];
            for (int64_t q = 0; q < N; ++q) row[q] += a * (double)B[k * ldb + q];
        }
        for (int64_t q = 0; q < N; ++q)
            row[q] = alpha * row[q] + (beta != 0.0 ? beta * (double)Cin[p * ldc + q] : 0.0);
    }
    return OR_OK;
}

uint16_t oracle_double_to_bf16(double d) { return double_to_bf16(d); }

int oracle_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
