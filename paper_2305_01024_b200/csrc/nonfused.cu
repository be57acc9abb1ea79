// nonfused.cu -- the NON-FUSED ABFT baseline: the scheme
// the paper compares against, "the prior state-of-the-art fault-tolerant GEMM
// implementation first presented by Ding et al. in 2011" (PAPER.md:415,
// :469, :515), rebuilt on B200 from library GEMMs and separate kernels:
//
//   1. encode        ftgemm_encode(which = 3 | 4): Ac, Br and the norms (the
//                    same kernels as the fused path, no encoded operand)
//   2. GEMM          cuBLAS: C32 = A B with FP32 output (the verification must
//                    see the accumulator precision, not the rounded BF16 C)
//   3. references    cuBLAS: R_row = A (B e) and R_col = (e^T A) B (Eq. 3,
//                    PAPER.md:161), BF16 operands as exact 3-term splits
//   4. faults        (optional) applied to the FP32 result before verification
//   5. verify        one CTA per check tile: row / column sums of C32 against
//                    R_row / R_col, the same threshold, decision and row-based
//                    correction as the fused kernel,
//                    then alpha / beta and the store in the output dtype.
//
// Everything the fused kernel keeps on chip (C, the carried references, the
// verification sums) makes a round trip through HBM here: C32 is written by
// the GEMM and read back by the verifier, and A and B are read again by the
// reference GEMMs.  That traffic is what the fused design removes.
#include <cublas_v2.h>

#include <cstdint>
#include <mutex>

#include "common.cuh"

namespace ftg {

// workspace: C32 [M][N] f32 | R_row [M][S*tiles_n] f32 | R_col [S*tiles_m][N] f32
//            | Xs [S*tiles_n][kp] bf16 | Ys [S*tiles_m][kp] bf16       (S = 3 BF16, 1 FP32)
struct NfLayout {
    size_t c32, rrow, rcol, xs, ys, total;
    int S;
};

inline NfLayout nf_layout(const Geometry& g, int64_t M, int64_t N) {
    NfLayout L{};
    L.S = g.dtype == FTGEMM_BF16 ? 3 : 1;
    size_t o = 0;
    L.c32 = o;  o = align256(o + sizeof(float) * (size_t)M * N);
    L.rrow = o; o = align256(o + sizeof(float) * (size_t)M * L.S * g.tiles_n);
    L.rcol = o; o = align256(o + sizeof(float) * (size_t)L.S * g.tiles_m * N);
    L.xs = o;   o = align256(o + (g.dtype == FTGEMM_BF16 ? 2 * (size_t)L.S * g.tiles_n * g.kp : 0));
    L.ys = o;   o = align256(o + (g.dtype == FTGEMM_BF16 ? 2 * (size_t)L.S * g.tiles_m * g.kp : 0));
    L.total = o;
    return L;
}

size_t nonfused_ws_bytes(const Geometry& g, int64_t M, int64_t N) { return nf_layout(g, M, N).total; }

// ---- 3-term BF16 splits of Ac (rows) and Br (rows of the transposed view) ----
__global__ void nf_split_kernel(const float* __restrict__ Ac, const float* __restrict__ Br, int tiles_m, int tiles_n,
                                int kp, uint16_t* __restrict__ Ys, uint16_t* __restrict__ Xs) {
    const int64_t n_a = (int64_t)tiles_m * kp, n = n_a + (int64_t)tiles_n * kp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const bool isa = i < n_a;
        const int64_t j = isa ? i : i - n_a;
        const int64_t t = j / kp, k = j % kp;
        float hi, mid, lo;
        split3<0>(isa ? Ac[j] : Br[j], hi, mid, lo);
        uint16_t* dst = isa ? Ys : Xs;
        dst[(3 * t + 0) * kp + k] = f32_to_bf16_rn(hi);
        dst[(3 * t + 1) * kp + k] = f32_to_bf16_rn(mid);
        dst[(3 * t + 2) * kp + k] = f32_to_bf16_rn(lo);
    }
}

// ---- faults on the FP32 result (the library GEMM cannot be entered mid-K) ----
struct NfInject {
    int64_t row, col;
    int32_t bit, mode, target;
    float addend;
};

__global__ void nf_inject_kernel(const NfInject* __restrict__ f, int n, float* C32, int64_t N, float* rrow, int ldr,
                                 float* rcol, int tile_m, int tile_n, int S) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int i = 0; i < n; ++i) {                 // serial: faults on one element compose in list order
        const NfInject x = f[i];
        float* p;
        if (x.target == FTGEMM_TGT_ROW_REF) p = rrow + x.row * ldr + (int64_t)S * (x.col / tile_n);
        else if (x.target == FTGEMM_TGT_COL_REF) p = rcol + (int64_t)S * (x.row / tile_m) * N + x.col;
        else p = C32 + x.row * N + x.col;
        *p = x.mode == FTGEMM_INJ_ADD ? *p + x.addend : __uint_as_float(__float_as_uint(*p) ^ (1u << (x.bit & 31)));
    }
}

struct NfArgs {
    int M, N, K, tiles_m, tiles_n, bmd, bnd, S, ft_level, out_bf16;
    float alpha, beta;
    const float* C32; const float* rrow; const float* rcol;
    void* C; int64_t ldc;
    const float* rownorm; const float* colnorm; const float* acnorm; const float* brnorm;
    float tau_u, tau_l1, tau_l2, sqrtK;
    ReportDev* rep;
};

__device__ __forceinline__ float nf_block_sum(float x, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += red[i];
    return s;
}

// one CTA (256 threads) per check tile; thread t owns column t of the tile
__global__ void __launch_bounds__(256) nf_verify_kernel(const NfArgs a) {
    __shared__ __align__(16) float buf[32][260];     // 32 rows of the tile
    __shared__ float rsum[128], rres[128], rtau[128], cres[256], ctau[256], red[8];
    __shared__ int sflag[5];
    const int tj = blockIdx.x, ti = blockIdx.y, t = threadIdx.x, w = t >> 5, lane = t & 31;
    const int r0 = ti * a.bmd, c0 = tj * a.bnd;
    const int bm = min(a.bmd, a.M - r0), bn = min(a.bnd, a.N - c0);
    const float* Ct = a.C32 + (int64_t)r0 * a.N + c0;
    int kind = 0, pstar = -1, qstar = -1, nr = 0, nc = 0;
    float corr = 0.0f;
    if (a.ft_level != FTGEMM_FT_OFF) {
        if (t == 0) { sflag[0] = 0; sflag[1] = 0; sflag[2] = 1 << 30; sflag[3] = 1 << 30; }
        float cs = 0.0f;
        for (int ch = 0; ch * 32 < bm; ++ch) {
            const int rows = min(32, bm - ch * 32);
            // stream 32 rows: coalesced along the row, column sums thread-local
#pragma unroll 8
            for (int r = 0; r < 32; ++r) {
                float v = 0.0f;
                if (r < rows && t < bn) v = __ldg(Ct + (int64_t)(ch * 32 + r) * a.N + t);
                buf[r][t] = v;
                cs += v;
            }
            __syncthreads();
            // row sums: warp w reduces rows 4w..4w+3 (8 columns per lane)
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
                const int r = 4 * w + rr;
                const float4 x0 = *reinterpret_cast<const float4*>(&buf[r][lane * 8]);
                const float4 x1 = *reinterpret_cast<const float4*>(&buf[r][lane * 8 + 4]);
                float s = ((x0.x + x0.y) + (x0.z + x0.w)) + ((x1.x + x1.y) + (x1.z + x1.w));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0 && r < rows) rsum[ch * 32 + r] = s;
            }
            __syncthreads();
        }
        // residuals against the references (sum of the S split products)
        if (t < bm) {
            const float* rp = a.rrow + (int64_t)(r0 + t) * (a.S * a.tiles_n) + a.S * tj;
            float ref = 0.0f;
            for (int s = 0; s < a.S; ++s) ref += rp[s];
            const float r = rsum[t] - ref;
            const float tr = a.tau_u * (a.tau_l1 * a.sqrtK * fabsf(ref) + a.tau_l2 * a.rownorm[r0 + t] * a.brnorm[tj]);
            rres[t] = r; rtau[t] = tr;
            if (!(fabsf(r) <= tr)) { atomicAdd(&sflag[0], 1); atomicMin(&sflag[2], t); }
        }
        if (t < bn && a.ft_level != FTGEMM_FT_DETECT_ROWS) {
            const float* cp = a.rcol + (int64_t)a.S * ti * a.N + c0 + t;
            float ref = 0.0f;
            for (int s = 0; s < a.S; ++s) ref += cp[(int64_t)s * a.N];
            const float c = cs - ref;
            const float tc = a.tau_u * (a.tau_l1 * a.sqrtK * fabsf(ref) + a.tau_l2 * a.acnorm[ti] * a.colnorm[c0 + t]);
            cres[t] = c; ctau[t] = tc;
            if (!(fabsf(c) <= tc)) { atomicAdd(&sflag[1], 1); atomicMin(&sflag[3], t); }
        }
        __syncthreads();
        nr = sflag[0]; nc = sflag[1];
        pstar = nr ? sflag[2] : -1;
        qstar = nc ? sflag[3] : -1;
        if (a.ft_level == FTGEMM_FT_DETECT_ROWS) {
            kind = nr ? FTGEMM_EV_DETECTED : 0;
            qstar = -1;
        } else if (nr == 1 && nc == 1) {
            const float rr = rres[pstar], cc = cres[qstar];
            const float big = fmaxf(fabsf(rr), fabsf(cc));
            const float guard = rtau[pstar] + ctau[qstar] + 2.0f * a.tau_u * (float)(bm + bn) * big;
            const bool consistent = !(fabsf(rr - cc) > guard);
            kind = consistent ? (a.ft_level == FTGEMM_FT_CORRECT ? FTGEMM_EV_CORRECTED : FTGEMM_EV_LOCATED)
                              : FTGEMM_EV_UNCORRECTABLE;
        } else if ((nr == 1 && nc == 0) || (nr == 0 && nc == 1)) {
            kind = FTGEMM_EV_CHECKSUM_ONLY;
        } else if (nr || nc) {
            kind = FTGEMM_EV_UNCORRECTABLE;
        }
        if (kind == FTGEMM_EV_CORRECTED) {          // acc[p*,q*] = R_row[p*] - sum_{q != q*} acc[p*,q]
            const float v = (t < bn && t != qstar) ? Ct[(int64_t)pstar * a.N + t] : 0.0f;
            const float sx = nf_block_sum(v, red);
            const float* rp = a.rrow + (int64_t)(r0 + pstar) * (a.S * a.tiles_n) + a.S * tj;
            float ref = 0.0f;
            for (int s = 0; s < a.S; ++s) ref += rp[s];
            corr = ref - sx;
        }
        if (t == 0) {
            unsigned long long* cnt = a.rep->counts;
            atomicAdd(&cnt[CNT_CHECKED], 1ull);
            if (kind) {
                atomicAdd(&cnt[CNT_DETECTED], 1ull);
                const int ci = kind == FTGEMM_EV_CORRECTED ? CNT_CORRECTED
                             : kind == FTGEMM_EV_CHECKSUM_ONLY ? CNT_CHECKSUM_ONLY
                             : kind == FTGEMM_EV_LOCATED ? CNT_LOCATED
                             : kind == FTGEMM_EV_DETECTED ? -1 : CNT_UNCORRECTABLE;
                if (ci >= 0) atomicAdd(&cnt[ci], 1ull);
                const unsigned long long slot = atomicAdd(&cnt[CNT_EVENTS], 1ull);
                if (slot < (unsigned long long)kMaxEvents) {
                    ftgemm_event_t& e = a.rep->events[slot];
                    e.row = pstar >= 0 ? (int64_t)(r0 + pstar) : -1;
                    e.col = qstar >= 0 ? (int64_t)(c0 + qstar) : -1;
                    e.tile_m = ti; e.tile_n = tj; e.kind = kind;
                    e.n_rows = nr; e.n_cols = kind == FTGEMM_EV_DETECTED ? 0 : nc; e.k_checked = a.K;
                    e.resid_row = pstar >= 0 ? rres[pstar] : 0.0f;
                    e.resid_col = qstar >= 0 ? cres[qstar] : 0.0f;
                    e.tau_row = pstar >= 0 ? rtau[pstar] : 0.0f;
                    e.tau_col = qstar >= 0 ? ctau[qstar] : 0.0f;
                } else {
                    atomicAdd(&cnt[CNT_DROPPED], 1ull);
                }
            }
        }
    }
    // alpha / beta and the store (the tile is read again, mostly from L2)
    if (t < bn) {
        for (int p = 0; p < bm; ++p) {
            float v = Ct[(int64_t)p * a.N + t];
            if (kind == FTGEMM_EV_CORRECTED && p == pstar && t == qstar) v = corr;
            const int64_t gi = (int64_t)(r0 + p) * a.ldc + c0 + t;
            if (a.out_bf16) {
                uint16_t* Co = reinterpret_cast<uint16_t*>(a.C);
                const float o = a.beta != 0.0f ? fmaf(a.beta, bf16_to_f32(Co[gi]), a.alpha * v) : a.alpha * v;
                Co[gi] = f32_to_bf16_rn(o);
            } else {
                float* Co = reinterpret_cast<float*>(a.C);
                Co[gi] = fmaf(a.alpha, v, a.beta != 0.0f ? a.beta * Co[gi] : 0.0f);
            }
        }
    }
}

// ---------------------------------------------------------------- host -------
namespace {
std::mutex g_blas_mu;
cublasHandle_t g_blas[64] = {};

cublasHandle_t blas_handle() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_blas_mu);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!g_blas[dev] && cublasCreate(&g_blas[dev]) != CUBLAS_STATUS_SUCCESS) g_blas[dev] = nullptr;
    return g_blas[dev];
}
}  // namespace

// row-major X[r x c] (ld) is column-major X^T: C = A B  <=>  C^T = B^T A^T
static cublasStatus_t gemm_rm(cublasHandle_t h, bool bt_, int64_t M, int64_t N, int64_t K, const void* A,
                              int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc, cudaDataType tin,
                              cudaDataType tout, float beta) {
    // row-major C[M x N] = A[M x K] * op(B); bt_: B is stored as row-major [N x K]
    const float alpha = 1.0f;
    return cublasGemmEx(h, bt_ ? CUBLAS_OP_T : CUBLAS_OP_N, CUBLAS_OP_N, (int)N, (int)M, (int)K, &alpha, B, tin,
                        (int)ldb, A, tin, (int)lda, &beta, C, tout, (int)ldc, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
}

cudaError_t launch_nonfused(const Geometry& g, const EncLayout& E, int64_t M, int64_t N, int64_t K, float alpha,
                            const void* A, int64_t lda, const void* B, int64_t ldb, float beta, void* C, int64_t ldc,
                            const void* enc_ws, void* nf_ws, int ft_level, const NfInject* dinj, int n_inj,
                            ReportDev* rep, float tau_u, float l1, float l2, cudaStream_t st, const char** why) {
    cublasHandle_t h = blas_handle();
    if (!h) { *why = "cublasCreate failed"; return cudaErrorUnknown; }
    if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) { *why = "cublasSetStream failed"; return cudaErrorUnknown; }
    const bool bf = g.dtype == FTGEMM_BF16;
    const cudaDataType tin = bf ? CUDA_R_16BF : CUDA_R_32F;
    if (ft_level == FTGEMM_FT_OFF) {                 // plain library GEMM, straight into C
        const float a1 = alpha, b1 = beta;
        cublasStatus_t s = cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)N, (int)M, (int)K, &a1, B, tin, (int)ldb, A, tin,
                                        (int)lda, &b1, C, tin, (int)ldc, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
        if (s != CUBLAS_STATUS_SUCCESS) { *why = "cublasGemmEx failed"; return cudaErrorUnknown; }
        return cudaGetLastError();
    }
    const NfLayout L = nf_layout(g, M, N);
    char* ws = reinterpret_cast<char*>(nf_ws);
    const char* enc = reinterpret_cast<const char*>(enc_ws);
    float* C32 = reinterpret_cast<float*>(ws + L.c32);
    float* rrow = reinterpret_cast<float*>(ws + L.rrow);
    float* rcol = reinterpret_cast<float*>(ws + L.rcol);
    const float* Ac = reinterpret_cast<const float*>(enc + E.ac);
    const float* Br = reinterpret_cast<const float*>(enc + E.br);
    const int S = L.S, tm = g.tiles_m, tn = g.tiles_n;
    cublasStatus_t s;
    // 2. C32 = A B (FP32 result)
    s = gemm_rm(h, false, M, N, K, A, lda, B, ldb, C32, N, tin, CUDA_R_32F, 0.0f);
    if (s != CUBLAS_STATUS_SUCCESS) { *why = "cublasGemmEx (C) failed"; return cudaErrorUnknown; }
    // 3. references: R_row[M x S tn] = A Xs^T,  R_col[S tm x N] = Ys B
    const void *X = Br, *Y = Ac;
    if (bf) {
        uint16_t* Xs = reinterpret_cast<uint16_t*>(ws + L.xs);
        uint16_t* Ys = reinterpret_cast<uint16_t*>(ws + L.ys);
        nf_split_kernel<<<2 * device_sms(), 256, 0, st>>>(Ac, Br, tm, tn, g.kp, Ys, Xs);
        X = Xs; Y = Ys;
    }
    s = gemm_rm(h, true, M, (int64_t)S * tn, K, A, lda, X, g.kp, rrow, (int64_t)S * tn, tin, CUDA_R_32F, 0.0f);
    if (s != CUBLAS_STATUS_SUCCESS) { *why = "cublasGemmEx (row references) failed"; return cudaErrorUnknown; }
    s = gemm_rm(h, false, (int64_t)S * tm, N, K, Y, g.kp, B, ldb, rcol, N, tin, CUDA_R_32F, 0.0f);
    if (s != CUBLAS_STATUS_SUCCESS) { *why = "cublasGemmEx (column references) failed"; return cudaErrorUnknown; }
    // 4. faults
    if (n_inj > 0) nf_inject_kernel<<<1, 32, 0, st>>>(dinj, n_inj, C32, N, rrow, S * tn, rcol, g.bmd, g.bnd, S);
    // 5. verify + correct + alpha/beta + store
    NfArgs a{};
    a.M = (int)M; a.N = (int)N; a.K = (int)K; a.tiles_m = tm; a.tiles_n = tn; a.bmd = g.bmd; a.bnd = g.bnd;
    a.S = S; a.ft_level = ft_level; a.out_bf16 = bf; a.alpha = alpha; a.beta = beta;
    a.C32 = C32; a.rrow = rrow; a.rcol = rcol; a.C = C; a.ldc = ldc;
    a.rownorm = reinterpret_cast<const float*>(enc + E.rownorm);
    a.colnorm = reinterpret_cast<const float*>(enc + E.colnorm);
    a.acnorm = reinterpret_cast<const float*>(enc + E.acnorm);
    a.brnorm = reinterpret_cast<const float*>(enc + E.brnorm);
    a.tau_u = tau_u; a.tau_l1 = l1; a.tau_l2 = l2; a.sqrtK = sqrtf((float)K);
    a.rep = rep;
    nf_verify_kernel<<<dim3(tn, tm), 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace ftg
