/*
 * ftgemm.h -- C ABI of the B200-native fused online-ABFT GEMM
 * (arXiv 2305.01024, "Anatomy of High-Performance GEMM with Online Fault
 * Tolerance on GPUs").  Library: paper_2305_01024_b200/libftgemm.so.
 *
 *   C = alpha * A * B + beta * C
 *
 * computed with the paper's checksum scheme (section 2.2,
 * Eq. (1)-(3)): a column checksum e^T A of every M-tile and a row checksum B e
 * of every N-tile are encoded (ftgemm_encode), carried through the same
 * mainloop as C (the references C^c = (e^T A) B and C^r = A (B e)), and in the
 * epilogue of every output tile the recomputed row / column sums of the FP32
 * accumulator are compared with them; one corrupted element per tile is
 * located at the intersection of the mismatching row and column and corrected
 * from the row checksum (section 4.2.1, section 5.3),
 * under the paper's single-event-upset fault model (section 4.1).
 *
 * Conventions (all entry points):
 *   - Matrices are ROW-MAJOR: A is M x K (lda >= K), B is K x N (ldb >= N),
 *     C is M x N (ldc >= N).  Leading dimensions are in elements.
 *   - All pointers except those documented as host pointers are DEVICE
 *     pointers owned by the caller.  The library allocates no device memory
 *     and keeps no state between calls other than host-side caches.
 *   - All sizes are int64_t.  Every call is asynchronous on `stream`
 *     (a cudaStream_t passed as void*), except ftgemm_plan (pure host) and
 *     ftgemm_report (synchronises the stream).
 *   - Return value: FTGEMM_OK or an FTGEMM_ERR_* code; argument errors are
 *     detected synchronously before anything is launched; the message is
 *     available from ftgemm_last_error() (thread-local).  Faults that the ABFT
 *     scheme detects are NOT errors: C is written and the report records them.
 *   - There is no CPU fallback: when the device path cannot run the call,
 *     the call fails.
 */
#ifndef FTGEMM_H_
#define FTGEMM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FTGEMM_ABI_VERSION 2

#if defined(__GNUC__)
#define FTGEMM_API __attribute__((visibility("default")))
#else
#define FTGEMM_API
#endif

/* ---- return codes ---------------------------------------------------------- */
#define FTGEMM_OK                 0
#define FTGEMM_ERR_INVALID_VALUE  1   /* null pointer, dim < 1, ld < cols, bad enum, small workspace */
#define FTGEMM_ERR_UNSUPPORTED    2   /* alignment (TMA needs 16-byte bases and row pitches), no sm_100 device */
#define FTGEMM_ERR_CUDA           3   /* a CUDA runtime error (launch or asynchronous kernel fault) */

/* ---- precision variants (north_star item 3) -------------------------------- */
#define FTGEMM_F32_SIMT 0   /* FP32 in/out, FP32 FFMA on CUDA cores; the paper's SGEMM numerics
                               (one fmaf per k, ascending k; section 3.1) */
#define FTGEMM_TF32     1   /* FP32 in/out, tcgen05.mma kind::tf32, FP32 accumulate in TMEM */
#define FTGEMM_BF16     2   /* BF16 in/out, tcgen05.mma kind::f16 (bf16), FP32 accumulate in TMEM */

/* Every `dtype` argument below is a dtype CODE: one of the precision variants
 * above, optionally OR-ed with an explicit tensor-core tile class
 *     FTGEMM_TF32 | FTGEMM_TILE(bn, cta_group),  bn in {128, 256}, cta_group in {1, 2}
 * (check tile 125 x (bn - 4); cta_group 2 = a CTA pair issues one M = 256 MMA).
 * Without a class the plan chooses one from the shape (north_star item 4).  The
 * class travels with every call -- there is no process-wide tile-class state --
 * so ftgemm_encode and ftgemm_run given the same code, M, N, K always derive the
 * same encode layout; plan.dtype returns the fully explicit code of a plan
 * (pass it to encode / run to reproduce exactly that plan, e.g. on every rank
 * of an M-block partition: SURVEY.md 8(e)).  A class on F32_SIMT, an unknown
 * class or other set bits: FTGEMM_ERR_INVALID_VALUE.                          */
#define FTGEMM_TILE(bn, cta_group) ((((bn) / 128) << 8) | ((cta_group) << 12))
#define FTGEMM_DTYPE_MASK 0xff

/* ---- fault-tolerance level -------------------------------------------------- */
#define FTGEMM_FT_OFF     0  /* same tile shape family, checksums compiled out (the overhead baseline) */
#define FTGEMM_FT_DETECT  1  /* verify + locate, report, leave C as computed (detect-only flavour) */
#define FTGEMM_FT_CORRECT 2  /* verify + locate + correct (the paper's online ABFT) */
#define FTGEMM_FT_DETECT_ROWS 3 /* offline (detect-only) ABFT: row checks only, no
                                   column sums, no correction; a flagged tile is reported (EV_DETECTED)
                                   and the caller re-computes (ftgemm_run_offline) */

/* ---- fault injection (section 5.3) ---------------------------- */
#define FTGEMM_INJ_FLIP 0    /* acc bits ^= (1 << bit)            (register bit flip) */
#define FTGEMM_INJ_ADD  1    /* acc += addend                      (the paper's "numerical offset") */
#define FTGEMM_TGT_ACC     0 /* the output accumulator of element (row, col) */
#define FTGEMM_TGT_ROW_REF 1 /* the carried row-checksum reference C^r of row `row` in col's tile */
#define FTGEMM_TGT_COL_REF 2 /* the carried column-checksum reference C^c of column `col` in row's tile */

/* One fault: applied once, to the FP32 accumulator, right after the MMA
 * k-block that contains k_elem has been accumulated (k_elem is rounded UP to
 * the end of its k-block of size plan.bk; values >= K address the last block). */
typedef struct ftgemm_inject {
    int64_t row, col, k_elem;
    int32_t bit;        /* 0..31 for FLIP */
    int32_t mode;       /* FTGEMM_INJ_* */
    int32_t target;     /* FTGEMM_TGT_* */
    float   addend;     /* for FTGEMM_INJ_ADD */
} ftgemm_inject_t;      /* 40 bytes */

/* ---- run with the A-side encode inside the GEMM kernel -----------------------
 * SURVEY 8(f) row 1, the paper's threadblock-level fusion of the checksum
 * encoding into the prefetch stage.  As ftgemm_run, but the
 * column checksum of A (Eq. 1: e^T A per check tile, its exact split into the
 * operand format) and the threshold's row / tile norms are computed inside
 * the GEMM kernel, so enc_ws needs only the B part (ftgemm_encode which = 2).
 * One encoder warp per CTA (and, during the first wave, the epilogue warps)
 * claims (check tile, k-block) items in the order the tile schedule first
 * needs them, reads A from global memory, and publishes each item with a
 * release flag; the split-row loads of every k-block wait for its flag.  Every
 * item is computed once per call (not once per tile column).  The call first
 * clears the item flags in enc_ws (cudaMemsetAsync on `stream`), so enc_ws
 * must not be in use by another call in flight on another stream; the pair
 * (memset, kernel) is CUDA-graph capturable.  The kernel's CTAs wait on each
 * other's flags: the persistent grid (one CTA per SM) must become fully
 * resident, which holds unless other work pins SMs indefinitely.  C is
 * bit-identical to ftgemm_run's (same operands, same k order); the carried
 * references and norms may differ in the last bits (summation order).
 * Tensor-core dtypes, ft_level DETECT, CORRECT or DETECT_ROWS; UNSUPPORTED for
 * F32_SIMT, FT_OFF, batched runs and the online-interval mode.               */
FTGEMM_API int ftgemm_run_fused(int dtype, int64_t M, int64_t N, int64_t K, float alpha,
               const void* A, int64_t lda, const void* B, int64_t ldb,
               float beta, void* C, int64_t ldc, const void* enc_ws, int ft_level,
               const ftgemm_inject_t* inj, int32_t n_inj, void* report_ws, void* stream);

/* ---- online verification every K_s (outer-product online ABFT) ----------------
 * PAPER.md:170-173 (Chen's online scheme: the checksum relation holds after
 * every outer-product step, so "the online version, which corrects a single
 * error for each step ..., can handle multiple errors") with the paper's
 * step K_s.  As ftgemm_run, plus: after every ks of K (ks a
 * positive multiple of plan.bk) the fused kernel verifies the partial
 * accumulator against the partial carried references and corrects in place
 * (TMEM), so up to ceil(K / ks) faults per check tile are corrected.  Each
 * step's check counts in tiles_checked; events carry k_checked.  The step
 * threshold uses sqrt(k_checked) and the full-K norms (R17).  The
 * checks before the end of K are row-first (R20): the column sums
 * are formed only when a row residual is flagged (a fault in C always moves
 * its row), so a column-reference fault is reported by the end-of-K check.
 * ft_level DETECT or CORRECT; tensor-core dtypes (F32_SIMT -> UNSUPPORTED).  */
FTGEMM_API int ftgemm_run_online(int dtype, int64_t M, int64_t N, int64_t K, float alpha,
               const void* A, int64_t lda, const void* B, int64_t ldb,
               float beta, void* C, int64_t ldc, const void* enc_ws, int ft_level, int64_t ks,
               const ftgemm_inject_t* inj, int32_t n_inj, void* report_ws, void* stream);

/* ---- non-fused ABFT baseline (the paper's comparison scheme) -----------------
 * Ding et al. 2011 as the paper benchmarks it:
 * library GEMMs + separate kernels instead of one fused kernel.  C32 = A B by
 * cuBLAS with an FP32 result; the references A (B e) and (e^T A) B by two more
 * cuBLAS GEMMs (BF16: exact 3-term splits of B e and e^T A); faults (inj, same
 * type as ftgemm_run; k_elem is ignored: a library GEMM cannot be entered
 * mid-K, so a fault strikes the FP32 result); then one verification kernel per
 * check tile with the fused path's threshold, decision and correction, and the
 * alpha / beta store.  enc_ws: ftgemm_encode(which = 3 | 4) of A and B (4 =
 * checksums only, no encoded operand).  nf_ws: device workspace of
 * ftgemm_nonfused_workspace() bytes (C32, references, split operands).
 * ft_level FT_OFF = the plain cuBLAS GEMM into C.  dtypes BF16 and F32_SIMT
 * (FP32 SGEMM, no TF32); TF32 -> UNSUPPORTED.  Report as ftgemm_run.        */
FTGEMM_API int ftgemm_nonfused_workspace(int dtype, int64_t M, int64_t N, int64_t K, int64_t* bytes);
FTGEMM_API int ftgemm_run_nonfused(int dtype, int64_t M, int64_t N, int64_t K, float alpha,
               const void* A, int64_t lda, const void* B, int64_t ldb,
               float beta, void* C, int64_t ldc, const void* enc_ws, void* nf_ws, int ft_level,
               const ftgemm_inject_t* inj, int32_t n_inj, void* report_ws, void* stream);

/* ---- offline (detect-only) ABFT with re-computation -------------------------
 * PAPER.md:571-583 (section 5.5, "Online ABFT vs. Offline ABFT"): executions of
 * ftgemm_run at FT_DETECT_ROWS (row checks only, nothing corrected); after
 * each execution the host reads the detection counter (the call synchronises
 * `stream`) and, if a tile was flagged, re-computes the whole product, up to
 * max_runs executions in total.  Fault i strikes execution inj_run[i]
 * (0-based; inj_run may be NULL: every fault strikes execution 0), so faults
 * during re-computation can be modelled.  When beta != 0 the product reads C,
 * which an execution overwrites: c_backup (device, M x N with leading
 * dimension ldc, caller-owned -- the extra memory an offline scheme needs,
 * PAPER.md:173) receives C_in before execution 0 and restores it before each
 * re-execution; it may be NULL when beta == 0.
 * out[0] = executions performed, out[1] = 1 if the last execution passed the
 * row checks (0: max_runs exhausted, C not trusted; the report has the events).
 * Errors: as ftgemm_run, INVALID_VALUE (max_runs < 1, inj_run out of range,
 * beta != 0 without c_backup).                                                */
FTGEMM_API int ftgemm_run_offline(int dtype, int64_t M, int64_t N, int64_t K, float alpha,
               const void* A, int64_t lda, const void* B, int64_t ldb,
               float beta, void* C, int64_t ldc, void* c_backup,
               const void* enc_ws, const ftgemm_inject_t* inj, const int32_t* inj_run,
               int32_t n_inj, int32_t max_runs, void* report_ws, int32_t* out, void* stream);

/* ---- online vs offline cost model --------------------------
 * Pure host function.  tiles = M/m_tb x N/n_tb threadblock (check) tiles,
 * gamma0 = per-tile error probability of one execution.
 *   gamma = 1 - (1 - gamma0)^tiles                     (whole-call error rate)
 *   online_expected_runs  = 1                          (errors corrected on the fly)
 *   offline_expected_runs = (1 - gamma) / (1 - 2 gamma) (the paper's restart series;
 *                           +INFINITY when gamma >= 1/2: the series diverges)
 * Errors: INVALID_VALUE (gamma0 outside [0, 1), tiles < 1, null out).          */
typedef struct ftgemm_cost {
    double gamma0;
    int64_t tiles;
    double gamma;
    double online_expected_runs;
    double offline_expected_runs;
} ftgemm_cost_t;
FTGEMM_API int ftgemm_cost_model(double gamma0, int64_t tiles, ftgemm_cost_t* out);

/* ---- report ------------------------------------------------------------------ */
#define FTGEMM_EV_CORRECTED      1  /* one row + one column flagged, consistent: element corrected */
#define FTGEMM_EV_CHECKSUM_ONLY  2  /* one row only or one column only: the fault hit a reference; C untouched */
#define FTGEMM_EV_UNCORRECTABLE  3  /* >= 2 rows or >= 2 columns, or inconsistent magnitudes; C untouched */
#define FTGEMM_EV_LOCATED        4  /* FT_DETECT: single error located, not corrected */
#define FTGEMM_EV_DETECTED       5  /* FT_DETECT_ROWS: >= 1 row flagged (row = first flagged row, col = -1);
                                       counted in tiles_detected only */

typedef struct ftgemm_event {
    int64_t row, col;            /* global position (p*, q*); -1 when that side had no flag */
    int32_t tile_m, tile_n;      /* check-tile coordinates */
    int32_t kind;                /* FTGEMM_EV_* */
    int32_t n_rows, n_cols;      /* number of flagged rows / columns in the tile */
    int32_t k_checked;           /* K accumulated when the check fired: K for the end-of-K check,
                                    the end of the K_s step in online-interval mode (ftgemm_run_online) */
    float   resid_row, resid_col;/* residual of the first flagged row / column */
    float   tau_row, tau_col;    /* the thresholds they were compared against */
} ftgemm_event_t;                /* 56 bytes */

typedef struct ftgemm_counts {
    int64_t tiles_checked;       /* tiles verified (FT level != OFF) */
    int64_t tiles_detected;      /* tiles with >= 1 flagged row or column */
    int64_t corrected, checksum_only, uncorrectable, located;
    int64_t events;              /* events recorded or dropped */
    int64_t dropped;             /* events that did not fit the ring */
    float   max_resid_ratio;     /* threshold margin telemetry: the largest |residual| / tau over every
                                    residual that was NOT flagged (fused kernels; 0 if none) -- a
                                    fault-free run's distance from a false positive */
    int32_t pad;
} ftgemm_counts_t;                /* 72 bytes */

/* ---- plan --------------------------------------------------------------------
 * The host-side instantiation table (north_star item 4): which compile-time
 * kernel serves (dtype, M, N, K), the check-tile geometry the verification
 * works on, and the workspace sizes.  Pure host function, no device access.  */
typedef struct ftgemm_plan {
    int32_t dtype;               /* the fully explicit dtype code of this plan (tensor-core
                                    dtypes: | FTGEMM_TILE(bn, cta_group)) */
    int32_t shape_class;         /* FTGEMM_SHAPE_* */
    int32_t bm, bn, bk;          /* MMA / CTA tile */
    int32_t check_tile_m;        /* data rows per check tile (FT on)    */
    int32_t check_tile_n;        /* data columns per check tile (FT on) */
    int32_t off_tile_m, off_tile_n; /* data tile with FT_OFF */
    int32_t stages;              /* smem pipeline depth */
    int32_t cta_group;           /* 1, or 2: a CTA pair issues one M = 256 tcgen05.mma (cta_group::2);
                                    each CTA still owns one 128-row (125 + 3) check tile */
    int32_t max_events, max_inject;
    int32_t pad0;
    int64_t tiles_m, tiles_n;    /* check-tile grid with FT on */
    int64_t enc_bytes;           /* size of enc_ws (A part + B part)          */
    int64_t enc_b_offset;        /* byte offset of the B part inside enc_ws   */
    int64_t enc_b_bytes;         /* bytes of the B part (broadcast unit, multi-GPU) */
    int64_t report_bytes;        /* size of report_ws                         */
    float   u_acc, lambda1, lambda2;   /* threshold constants (R1) */
    int32_t pad1;
} ftgemm_plan_t;

#define FTGEMM_SHAPE_SQUARE      0  /* 128 x 256 tcgen05 tile (128 x 128 SIMT) */
#define FTGEMM_SHAPE_SMALL_N     1  /* 128 x 128 tcgen05 tile: narrow N or too few tiles for 148 SMs */

/* Fill *out for a problem.  Errors: INVALID_VALUE (dims < 1, bad dtype code, null out). */
FTGEMM_API int ftgemm_plan(int dtype, int64_t M, int64_t N, int64_t K, ftgemm_plan_t* out);

/* ---- encode (Eq. 1 / Eq. 2) -------------------------
 * which = 1: encode A  ->  per check-tile i: Ac_i[k] = sum_{p in tile rows} A[p,k]
 *                         (FP32), its exact split into three operand-format
 *                         values (hi+mid+lo == Ac_i) for the tensor-core path,
 *                         ||A[p,:]||_2 per row and ||Ac_i||_2.
 * which = 2: encode B  ->  per check-tile j: Br_j[k] = sum_{q in tile cols} B[k,q],
 *                         its split, ||B[:,q]||_2 per column and ||Br_j||_2.
 * which = 3: both.  which | 4: checksums and norms only, without the encoded
 * operand B^r (the non-fused baseline's encode).  Writes only enc_ws (plan.enc_bytes, caller-allocated,
 * 256-byte aligned); A and B are read-only.  The A part and the B part are
 * disjoint ([0, enc_b_offset) and [enc_b_offset, +enc_b_bytes)), so a B
 * encoded on one GPU can be broadcast with B and reused (weights).
 * Asynchronous on stream: which = 3 is one kernel launch (plus two small
 * memsets of the reduction tickets); a following ftgemm_run on the same stream
 * may begin its prologue before the encode finishes (programmatic dependent
 * launch) but reads nothing until it has.
 * Errors: INVALID_VALUE, UNSUPPORTED (misaligned), CUDA.                      */
FTGEMM_API int ftgemm_encode(int dtype, int64_t M, int64_t N, int64_t K,
                  const void* A, int64_t lda, const void* B, int64_t ldb,
                  void* enc_ws, int which, void* stream);

/* Where ftgemm_encode puts its results inside enc_ws (byte offsets from the
 * workspace base), for inspection and tests; pure host function.  FP32 arrays:
 *   ac      [tiles_m][kp]  Ac_i[k]  (Eq. 1), k >= K zero
 *   br      [tiles_n][kp]  Br_j[k]  (Eq. 2)
 *   rownorm [M] ||A[p,:]||_2,  acnorm [tiles_m] ||Ac_i||_2
 *   colnorm [N] ||B[:,q]||_2,  brnorm [tiles_n] ||Br_j||_2
 * and, for the tensor-core dtypes, the encoded operand B^r in the operand type:
 *   bt      [kp][bt_ld], bt_ld = tiles_n * bn: slot j = columns j*bn .. j*bn+bn-1
 *           holds B[k, j*check_tile_n + c] for c < check_tile_n, then the exact
 *           three-term split hi, mid, lo of Br_j[k] (hi + mid + lo == Br_j[k]),
 *           then zero (bt = -1 for F32_SIMT);
 *   y       [tiles_m][kp / bk][3][128 bytes]: row r = split term r (hi, mid, lo)
 *           of Ac_i[kb*bk .. kb*bk+bk) in the operand type, its 16-byte chunks
 *           permuted c -> c ^ ((125 + r) & 7) (the SWIZZLE_128B order of MMA
 *           rows 125..127; y = -1 for F32_SIMT).
 * Errors: INVALID_VALUE (dims < 1, bad dtype, null out).                      */
typedef struct ftgemm_enc_layout {
    int64_t ac, br, bt, rownorm, colnorm, acnorm, brnorm;
    int64_t kp, bt_ld, y;
} ftgemm_enc_layout_t;
FTGEMM_API int ftgemm_encode_layout(int dtype, int64_t M, int64_t N, int64_t K, ftgemm_enc_layout_t* out);

/* ---- run --------------------------------------------------------------------
 * C = alpha A B + beta C with online ABFT at ft_level.  A, B, C are device
 * row-major matrices of the dtype's operand type (float for F32_SIMT/TF32,
 * __nv_bfloat16 for BF16); C is read only when beta != 0.  enc_ws must hold
 * the encode of these A and B (ignored for FT_OFF).  With FT on, the
 * tensor-core dtypes multiply by the copy of B inside enc_ws (the encoded
 * operand B^r of Eq. 2) and do not read B itself: after changing B, encode it
 * again (which = 2) before the next run.  inj is a HOST array of
 * n_inj faults (copied during the call; may be NULL when n_inj == 0;
 * n_inj <= plan.max_inject).  report_ws (plan.report_bytes, device) receives
 * counters and events; it accumulates across calls until ftgemm_report_reset.
 * Faults and their corrections are recorded, never returned as errors.
 * Errors: INVALID_VALUE, UNSUPPORTED (alignment: A, B, C bases 16-byte
 * aligned; lda, ldb, ldc * sizeof(elem) multiples of 16), CUDA.               */
FTGEMM_API int ftgemm_run(int dtype, int64_t M, int64_t N, int64_t K, float alpha,
               const void* A, int64_t lda, const void* B, int64_t ldb,
               float beta, void* C, int64_t ldc,
               const void* enc_ws, int ft_level,
               const ftgemm_inject_t* inj, int32_t n_inj,
               void* report_ws, void* stream);

/* ---- batched runs (cfg4 "tall-skinny batches") ---------------------------------
 * `batch` independent problems of one shape in ONE persistent launch (PAPER.md
 * :450, :501 evaluate irregular and tall-skinny shapes; 32 launches of a
 * 4096 x 128 x 4096 GEMM leave most of the 148 SMs idle).  Problem b reads
 * A + b stride_a, B + b stride_b and writes C + b stride_c (strides in
 * ELEMENTS, multiples of 16 bytes; stride_b may be 0 for a shared B; C problems
 * must not overlap: stride_c >= M ldc), and uses its own encode at
 * enc_ws + b enc_stride (BYTES, a multiple of 256, >= plan.enc_bytes of
 * ftgemm_plan_batched).  Every problem is planned, encoded, verified and
 * corrected exactly as the single-problem call would do it with the batched
 * plan's tile class.  Faults and events use the stacked (batch x M) x N view:
 * inj.row and event.row in [0, batch M), event.tile_m = b tiles_m + ti.
 * Tensor-core dtypes only (F32_SIMT -> UNSUPPORTED); ftgemm_encode_batched's
 * `which` as ftgemm_encode.  ftgemm_plan_batched: the tile-class choice counts
 * all problems' work units (explicit FTGEMM_TILE classes are honoured).
 * Errors: as ftgemm_run / ftgemm_encode, INVALID_VALUE (batch < 1, bad strides). */
FTGEMM_API int ftgemm_plan_batched(int dtype, int64_t batch, int64_t M, int64_t N, int64_t K, ftgemm_plan_t* out);
FTGEMM_API int ftgemm_encode_batched(int dtype, int64_t batch, int64_t M, int64_t N, int64_t K,
               const void* A, int64_t lda, int64_t stride_a, const void* B, int64_t ldb, int64_t stride_b,
               void* enc_ws, int64_t enc_stride, int which, void* stream);
FTGEMM_API int ftgemm_run_batched(int dtype, int64_t batch, int64_t M, int64_t N, int64_t K, float alpha,
               const void* A, int64_t lda, int64_t stride_a, const void* B, int64_t ldb, int64_t stride_b,
               float beta, void* C, int64_t ldc, int64_t stride_c, const void* enc_ws, int64_t enc_stride,
               int ft_level, const ftgemm_inject_t* inj, int32_t n_inj, void* report_ws, void* stream);

/* ---- report ------------------------------------------------------------------
 * Synchronises `stream`, then copies the counters into *counts (host) and up
 * to max_events events into events (host array, may be NULL when
 * max_events == 0).  Surfaces asynchronous kernel faults as FTGEMM_ERR_CUDA.   */
FTGEMM_API int ftgemm_report(const void* report_ws, ftgemm_counts_t* counts,
                  ftgemm_event_t* events, int32_t max_events, void* stream);

/* Zero the counters and the event ring (asynchronous on stream). */
FTGEMM_API int ftgemm_report_reset(void* report_ws, int64_t report_bytes, void* stream);

/* Thread-local message of the last failing call ("" if none). */
FTGEMM_API const char* ftgemm_last_error(void);

/* ABI version (FTGEMM_ABI_VERSION) and the compiled device architecture (1000 = sm_100a). */
FTGEMM_API int ftgemm_version(void);
FTGEMM_API int ftgemm_device_arch(void);

#ifdef __cplusplus
}
#endif
#endif /* FTGEMM_H_ */
