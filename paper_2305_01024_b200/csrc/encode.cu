// encode.cu -- checksum-encode kernels (north_star item 2, "a checksum-encode
// kernel with coalesced, vectorised HBM reads and warp-shuffle reductions").
//
//   encode A (Eq. (1), A^c = [A; e^T A]):  per check tile i
//       Ac_i[k] = sum_{p in tile rows} A[p,k]            (FP32)
//       Ypack_i = exact 3-way split of Ac_i into operand-format values
//                 (hi + mid + lo == Ac_i), pre-swizzled as MMA rows 125..127
//       ||A[p,:]||_2 per row, ||Ac_i||_2 per tile         (threshold, R1)
//   encode B (Eq. (2), B^r = [B, B e]):   per check tile j
//       Br_j[k] = sum_{q in tile cols} B[k,q]            (FP32)
//       Bt_j    = B^r_j = [B_j, split(B_j e), 0], K-major (tensor-core paths)
//       ||B[:,q]||_2 per column, ||Br_j||_2 per tile.
//
// Single streaming passes over each operand (HBM bound), every global access a
// 16-byte (A; TF32 / FP32 B) or 8-byte (BF16 B: 252-column tiles start on
// 8-byte boundaries) vector with several rows in flight per lane; reductions go
// through registers, warp shuffles and shared memory; with both operands,
// one launch (encode_ab_kernel) runs the blocks of both passes.  The
// per-row / per-column norms are reduced across K-chunk blocks by the LAST
// block of each tile (atomic ticket, self-resetting), so no extra launch is
// needed.  TF32 mode sums the values exactly as the tensor core will see them
// (low 13 mantissa bits dropped), so the carried references and the main
// product are built from the same operands.
//
// Measured alternatives (profiles/r1_encode.md): a TMA-fed encode A (one
// 64 KB box per block, column sums from shared memory) ran at 3.2 TB/s against
// 4.0 TB/s for the register-streaming kernel below; for BF16 encode B, a
// shared-memory-staged tile-pair kernel (16-byte cp.async or per-row bulk TMA
// copies, shifted re-reads for the 4-column slot offset) and a shuffle-based
// tile-pair kernel were 2-40 % slower than the 8-byte register kernel.
#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace ftg {

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// sum_{c < n} p[c * stride]: independent loads in flight (the partial-norm
// reductions of the last block sit on the kernel's critical tail)
__device__ __forceinline__ float strided_sum(const float* p, int n, int64_t stride) {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int c = 0;
    for (; c + 4 <= n; c += 4) {
        a0 += p[(int64_t)c * stride];
        a1 += p[(int64_t)(c + 1) * stride];
        a2 += p[(int64_t)(c + 2) * stride];
        a3 += p[(int64_t)(c + 3) * stride];
    }
    for (; c < n; ++c) a0 += p[(int64_t)c * stride];
    return (a0 + a1) + (a2 + a3);
}

// Returns true in every thread of the block that arrives last for ticket[idx];
// that block then sees all partial results of the others.  Resets the ticket.
__device__ __forceinline__ bool last_block(int* ticket, int idx, int nblocks, int* s_flag) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int prev = atomicAdd(&ticket[idx], 1);
        *s_flag = (prev == nblocks - 1);
        if (*s_flag) ticket[idx] = 0;
    }
    __syncthreads();
    const bool last = *s_flag != 0;
    if (last) __threadfence();
    return last;
}

// parameters of the encode passes (one struct per operand, so that one launch
// can carry both: encode_ab_kernel)
struct EncAP {
    const void* A; int64_t lda; int M, K, bmd, kp, bk, nkc;
    float* Ac; uint8_t* Y; float* rn2; float* acn2; int* ticket; float* rownorm; float* acnorm;
    int64_t sA, sE;        // batched encode: bytes between problems (A, encode workspace)
};
struct EncBP {
    const void* B; int64_t ldb; int N, K, bnd, bn, kp, ldt, nkc, rpb;
    float* Br; uint8_t* Bt; float* cn2; float* brn2; int* ticket; float* colnorm; float* brnorm;
    int64_t sB, sE;
};

// the parameters of problem b of a batched encode (every output lives in that
// problem's copy of the encode workspace)
template <class T> __device__ __forceinline__ T* boff(T* p, int64_t bytes) {
    return p ? reinterpret_cast<T*>(reinterpret_cast<char*>(const_cast<std::remove_const_t<T>*>(p)) + bytes) : p;
}
__device__ __forceinline__ EncAP at_batch(const EncAP& P, int b) {
    if (b == 0) return P;
    EncAP Q = P;
    const int64_t e = (int64_t)b * P.sE;
    Q.A = boff(P.A, (int64_t)b * P.sA);
    Q.Ac = boff(P.Ac, e); Q.Y = boff(P.Y, e); Q.rn2 = boff(P.rn2, e); Q.acn2 = boff(P.acn2, e);
    Q.ticket = boff(P.ticket, e); Q.rownorm = boff(P.rownorm, e); Q.acnorm = boff(P.acnorm, e);
    return Q;
}
__device__ __forceinline__ EncBP at_batch(const EncBP& P, int b) {
    if (b == 0) return P;
    EncBP Q = P;
    const int64_t e = (int64_t)b * P.sE;
    Q.B = boff(P.B, (int64_t)b * P.sB);
    Q.Br = boff(P.Br, e); Q.Bt = boff(P.Bt, e); Q.cn2 = boff(P.cn2, e); Q.brn2 = boff(P.brn2, e);
    Q.ticket = boff(P.ticket, e); Q.colnorm = boff(P.colnorm, e); Q.brnorm = boff(P.brnorm, e);
    return Q;
}

// ------------------------------------------ encode A (register streaming) --
// grid (nkc = ceil(kp/KC), tiles_m); block 256.  Same outputs as the TMA-fed
// kernel above, without the shared-memory round trip: warp w streams rows
// w, w+8, ... of check tile ti, every lane one 16-byte vector of the row's
// 512-byte k-chunk (a warp reads one full row per instruction, coalesced), ENC_U
// rows in flight per lane.  Column sums stay in registers (8 BF16 / 4 FP32
// columns per lane) and are reduced across the 8 warps once per block; row sums
// of squares are warp-shuffle reductions.
constexpr int ENC_U = 8;
// batches loaded before the first is reduced (measured: 2 batches at 2 blocks /
// SM 35-40 us against 33 us for 1 batch at 4 blocks / SM, BF16 8192^2 --
// resident warps matter more than loads in flight per warp)
#ifndef ENC_NB
#define ENC_NB 1
#endif
#ifndef ENC_A_MINB
#define ENC_A_MINB 4
#endif
template <int MODE>
__device__ __forceinline__ void encode_a_body(const int kc, const int ti, const EncAP& P) {
    const void* __restrict__ A_ = P.A;
    const int64_t lda = P.lda;
    const int M = P.M, K = P.K, bmd = P.bmd, kp = P.kp, bk = P.bk, nkc = P.nkc;
    float* __restrict__ Ac = P.Ac;
    uint8_t* __restrict__ Y = P.Y;
    float* rn2 = P.rn2;
    float* acn2 = P.acn2;
    int* ticket = P.ticket;
    float* __restrict__ rownorm = P.rownorm;
    float* __restrict__ acnorm = P.acnorm;
    constexpr int ELT = MODE == 0 ? 2 : 4;
    constexpr int KC = 512 / ELT;                       // k per block (512-byte rows)
    constexpr int VPL = 16 / ELT;                       // values per lane
    __shared__ __align__(16) float colp[8][KC];
    __shared__ float red8[8];
    __shared__ int s_flag;
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    const int rbeg = ti * bmd, rows = min(bmd, M - rbeg);
    const int k0 = kc * KC + lane * VPL;
    const bool full = k0 + VPL <= K;
    const bool blk_full = (kc + 1) * KC <= K;
    const int64_t ldb_ = lda * ELT;                     // row pitch (bytes)
    const uint8_t* base = reinterpret_cast<const uint8_t*>(A_) + (int64_t)rbeg * ldb_ + (int64_t)k0 * ELT;
    // ragged K: the lane's elements below K, zeros above (no local arrays)
    auto load_partial = [&](const uint8_t* p) -> uint4 {
        uint32_t wd[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
            if (k0 + i < K) {
                if constexpr (ELT == 2) wd[i >> 1] |= (uint32_t)reinterpret_cast<const uint16_t*>(p)[i] << (16 * (i & 1));
                else wd[i] = reinterpret_cast<const uint32_t*>(p)[i];
            }
        }
        return make_uint4(wd[0], wd[1], wd[2], wd[3]);
    };
    // value pair j of a 16-byte vector as the MMA sees it
    auto pair = [](const uint4& u, int j) -> float2 {
        const uint32_t wd[4] = {u.x, u.y, u.z, u.w};
        if constexpr (MODE == 0) return make_float2(__uint_as_float(wd[j] << 16), __uint_as_float(wd[j] & 0xFFFF0000u));
        else if constexpr (MODE == 1)
            return make_float2(tf32_trunc(__uint_as_float(wd[2 * j])), tf32_trunc(__uint_as_float(wd[2 * j + 1])));
        else return make_float2(__uint_as_float(wd[2 * j]), __uint_as_float(wd[2 * j + 1]));
    };
    float2 col2[VPL / 2];
#pragma unroll
    for (int j = 0; j < VPL / 2; ++j) col2[j] = make_float2(0.0f, 0.0f);
    // the lane that ends up holding row u's sum of squares after the transposed
    // reduction below: bits 4, 3, 2 of the lane index encode u
    const int my_u = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    // one batch: ENC_U rows r0, r0+8, ... of this warp already in registers
    auto process = [&](const uint4 (&raw)[ENC_U], const int r0) {
        float q[ENC_U];
#pragma unroll
        for (int u = 0; u < ENC_U; ++u) {
            float2 q2 = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int j = 0; j < VPL / 2; ++j) {
                const float2 x = pair(raw[u], j);
                col2[j] = __fadd2_rn(col2[j], x);
                q2 = __ffma2_rn(x, x, q2);
            }
            q[u] = q2.x + q2.y;
        }
        // transposed reduction of the 8 rows' squares: 4 + 2 + 1 exchanges halve
        // the set each lane carries, then two plain butterfly steps (9 shuffles
        // for 8 rows instead of 40)
        static_assert(ENC_U == 8, "transposed reduction assumes 8 rows per batch");
        float h4[4], h2[2], h1;
        {
            const bool up = lane & 16;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float send = up ? q[i] : q[i + 4];
                const float keep = up ? q[i + 4] : q[i];
                h4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
            }
        }
        {
            const bool up = lane & 8;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const float send = up ? h4[i] : h4[i + 2];
                const float keep = up ? h4[i + 2] : h4[i];
                h2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
            }
        }
        {
            const bool up = lane & 4;
            const float send = up ? h2[0] : h2[1];
            const float keep = up ? h2[1] : h2[0];
            h1 = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        h1 += __shfl_xor_sync(0xffffffffu, h1, 2);
        h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
        if ((lane & 3) == 0 && r0 + 8 * my_u < rows) rn2[(int64_t)kc * M + rbeg + r0 + 8 * my_u] = h1;
    };
    // ENC_NB batches (ENC_NB * ENC_U rows per warp) loaded before the first is
    // reduced: every row of the block in flight at once (bmd = 125 rows, 8 warps)
    for (int rb = w; rb < rows; rb += 8 * ENC_U * ENC_NB) {
        uint4 rawb[ENC_NB][ENC_U];
#pragma unroll
        for (int b = 0; b < ENC_NB; ++b) {
            const int r0 = rb + 8 * ENC_U * b;
            uint4 (&raw)[ENC_U] = rawb[b];
            if (blk_full) {                                 // block-uniform: the common case, 8 plain loads
#pragma unroll
                for (int u = 0; u < ENC_U; ++u) {
                    const int r = r0 + 8 * u;
                    raw[u] = r < rows ? ldg_stream_v4(base + (int64_t)r * ldb_) : make_uint4(0u, 0u, 0u, 0u);
                }
            } else {
#pragma unroll
                for (int u = 0; u < ENC_U; ++u) {
                    const int r = r0 + 8 * u;
                    const uint8_t* p = base + (int64_t)r * ldb_;
                    raw[u] = make_uint4(0u, 0u, 0u, 0u);
                    if (r < rows) {
                        if (full) raw[u] = ldg_stream_v4(p);
                        else if (k0 < K) raw[u] = load_partial(p);
                    }
                }
            }
        }
#pragma unroll
        for (int b = 0; b < ENC_NB; ++b) process(rawb[b], rb + 8 * ENC_U * b);
    }
    float col[VPL];
#pragma unroll
    for (int j = 0; j < VPL / 2; ++j) { col[2 * j] = col2[j].x; col[2 * j + 1] = col2[j].y; }
#pragma unroll
    for (int i = 0; i < VPL; i += 4)
        *reinterpret_cast<float4*>(&colp[w][lane * VPL + i]) = make_float4(col[i], col[i + 1], col[i + 2], col[i + 3]);
    __syncthreads();
    // Ac, its split rows (pre-swizzled Ypack) and the partial ||Ac||^2
    float s2 = 0.0f;
    for (int c = t; c < KC; c += 256) {
        const int k = kc * KC + c;
        if (k >= kp) break;
        float s = 0.0f;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) s += colp[ww][c];
        if (k >= K) s = 0.0f;
        Ac[(int64_t)ti * kp + k] = s;
        s2 = fmaf(s, s, s2);
        if constexpr (MODE != 2) {
            float hi, mid, lo;
            split3<MODE>(s, hi, mid, lo);
            const int kb = k / bk, kk = k % bk;
            const int chunk = (kk * ELT) >> 4, within = (kk * ELT) & 15;
            uint8_t* yb = Y + ((int64_t)ti * (kp / bk) + kb) * 384;
            const float parts[3] = {hi, mid, lo};
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                const int row = 125 + r;
                uint8_t* dst = yb + r * 128 + ((chunk ^ (row & 7)) << 4) + within;
                if constexpr (MODE == 0) *reinterpret_cast<uint16_t*>(dst) = f32_to_bf16_rn(parts[r]);
                else *reinterpret_cast<float*>(dst) = parts[r];
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) red8[w] = s2;
    __syncthreads();
    if (t == 0) {
        float q = 0.0f;
        for (int i = 0; i < 8; ++i) q += red8[i];
        acn2[(int64_t)ti * nkc + kc] = q;
    }
    if (last_block(ticket, ti, nkc, &s_flag)) {
        for (int p = rbeg + t; p < rbeg + rows; p += 256) rownorm[p] = sqrtf(strided_sum(rn2 + p, nkc, M));
        if (t == 0) acnorm[ti] = sqrtf(strided_sum(acn2 + (int64_t)ti * nkc, nkc, 1));
    }
}

// ----------------------------------------------------- encode B (FP32 SIMT) --
// grid (nkc = ceil(kp/rpb), tiles_n): Br_j (warp per k-row) and column squares.
__device__ __forceinline__ void encode_b_simt_body(const int kc, const int tj, const EncBP& P) {
    const float* __restrict__ B = reinterpret_cast<const float*>(P.B);
    const int64_t ldb = P.ldb;
    const int N = P.N, K = P.K, bnd = P.bnd, kp = P.kp, nkc = P.nkc, rpb = P.rpb;
    float* __restrict__ Br = P.Br;
    float* cn2 = P.cn2;
    float* brn2 = P.brn2;
    int* ticket = P.ticket;
    float* __restrict__ colnorm = P.colnorm;
    float* __restrict__ brnorm = P.brnorm;
    __shared__ float red[8][257];
    __shared__ float red8[8];
    __shared__ int s_flag;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nch = bnd / 4;
    const int c0 = tj * bnd;
    float csq[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) csq[i] = 0.0f;
    float bq = 0.0f;
    for (int r = w; r < rpb; r += 8) {
        const int k = kc * rpb + r;
        if (k >= kp) break;
        float s = 0.0f;
        if (k < K) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int ch = lane + 32 * h;
                const int col = c0 + ch * 4;
                if (ch < nch && col < N) {
                    const float* p = B + (int64_t)k * ldb + col;
                    float v[4];
                    if (N - col >= 4) {
                        const float4 a = __ldg(reinterpret_cast<const float4*>(p));
                        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
                    } else {
#pragma unroll
                        for (int i = 0; i < 4; ++i) v[i] = (col + i < N) ? __ldg(p + i) : 0.0f;
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        s += v[i];
                        csq[h * 4 + i] = fmaf(v[i], v[i], csq[h * 4 + i]);
                    }
                }
            }
        }
        s = warp_sum(s);
        if (lane == 0) Br[(int64_t)tj * kp + k] = s;
        bq = fmaf(s, s, bq);                       // identical in every lane
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int ch = lane + 32 * h;
            if (ch < nch) red[w][ch * 4 + i] = csq[h * 4 + i];
        }
    if (lane == 0) red8[w] = bq;
    __syncthreads();
    for (int t = threadIdx.x; t < bnd; t += 256) {
        const int col = c0 + t;
        if (col < N) {
            float s = 0.0f;
#pragma unroll
            for (int ww = 0; ww < 8; ++ww) s += red[ww][t];
            cn2[(int64_t)kc * N + col] = s;
        }
    }
    if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int i = 0; i < 8; ++i) s += red8[i];
        brn2[(int64_t)tj * nkc + kc] = s;
    }
    if (last_block(ticket, tj, nkc, &s_flag)) {
        for (int t = threadIdx.x; t < bnd; t += 256) {
            const int col = c0 + t;
            if (col < N) colnorm[col] = sqrtf(strided_sum(cn2 + col, nkc, N));
        }
        if (threadIdx.x == 0) brnorm[tj] = sqrtf(strided_sum(brn2 + (int64_t)tj * nkc, nkc, 1));
    }
}

// -------------------------------------------- encode B (tensor-core paths) --
// grid (nkc = ceil(kp/rpb), tiles_n); warp w handles k-rows kc*rpb + w + 8i (rpb: a multiple of 32).
// Per k-row of check tile j the warp streams the bnd data columns (4-element
// chunks: lane l owns chunks l and l+32), reduces B_j e with warp shuffles,
// accumulates column squares in registers, and writes the encoded operand row
//     Bt[k][j*bn : (j+1)*bn] = [B[k, j*bnd : j*bnd+bnd], split(B_j e)[k], 0]
// (B^r of Eq. (2), N-major, every tile slot 16-byte / 128-byte aligned so the
// fused kernel's TMA boxes start on cache-line boundaries).
template <int MODE>
__device__ __forceinline__ void encode_b_tc_body(const int kc, const int tj, const EncBP& P) {
    const void* __restrict__ B_ = P.B;
    const int64_t ldb = P.ldb;
    const int N = P.N, K = P.K, bnd = P.bnd, bn = P.bn, kp = P.kp, ldt = P.ldt, nkc = P.nkc, rpb = P.rpb;
    float* __restrict__ Br = P.Br;
    uint8_t* __restrict__ Bt = P.Bt;
    float* cn2 = P.cn2;
    float* brn2 = P.brn2;
    int* ticket = P.ticket;
    float* __restrict__ colnorm = P.colnorm;
    float* __restrict__ brnorm = P.brnorm;
    constexpr int ELT = MODE == 0 ? 2 : 4;
    using T = typename std::conditional<MODE == 0, uint16_t, float>::type;
    using V = typename std::conditional<MODE == 0, uint2, uint4>::type;     // 4 elements
    constexpr int RB = 4;                                                   // rows per batch
    __shared__ float red[8][257];
    __shared__ float red8[8];
    __shared__ int s_flag;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c0 = tj * bnd;
    const int nch = bnd / 4;                  // data chunks; chunk index nch is the split slot
    float colq[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) colq[i] = 0.0f;
    float2 colq2[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) colq2[i] = make_float2(0.0f, 0.0f);
    float bq = 0.0f;
    auto to_f = [](T x) -> float {
        if constexpr (MODE == 0) return bf16_to_f32(x);
        else return tf32_trunc(x);
    };
#if !defined(FTGEMM_EXP_ENCB_SCALAR)
    // Interior blocks (all rows < K, all 252 columns < N): no per-element
    // guards, pointer increments instead of per-row index arithmetic, and the
    // 4 rows' sums reduced transposed (6 shuffles for 4 rows instead of 20):
    // lanes with bits (4,3) = (b4,b3) end up holding row 2*b4+b3, and lanes
    // 0, 8, 16, 24 write that row's split columns and Br.
    const bool interior = Bt != nullptr && nch == 63 && (kc + 1) * rpb <= K && c0 + bnd <= N;
    if (interior) {
        static_assert(RB == 4, "transposed row reduction assumes 4 rows per batch");
        const int u_me = 2 * ((lane >> 4) & 1) + ((lane >> 3) & 1);
        const bool writer = (lane & 7) == 0;
        const bool h1ok = lane < 31;                     // chunk 32+lane; chunk 63 is the split slot
        const int64_t sstep = 8 * ldb, dstep = (int64_t)8 * ldt * ELT;
        const T* src = reinterpret_cast<const T*>(B_) + (int64_t)(kc * rpb + w) * ldb + c0 + lane * 4;
        uint8_t* dst = Bt + ((int64_t)(kc * rpb + w) * ldt + (int64_t)tj * bn + lane * 4) * ELT;
        V zero;
        if constexpr (MODE == 0) zero = make_uint2(0u, 0u); else zero = make_uint4(0u, 0u, 0u, 0u);
        float bqw = 0.0f;
        for (int r = w; r < rpb; r += 8 * RB) {
            V raw[RB][2];
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                const T* p = src + u * sstep;
                raw[u][0] = __ldg(reinterpret_cast<const V*>(p));
                raw[u][1] = h1ok ? __ldg(reinterpret_cast<const V*>(p + 128)) : zero;
            }
            float q[RB];
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                float2 acc2 = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        float2 x;
                        if constexpr (MODE == 0) {
                            const uint32_t wd = j == 0 ? reinterpret_cast<const uint2&>(raw[u][h]).x
                                                       : reinterpret_cast<const uint2&>(raw[u][h]).y;
                            x = make_float2(__uint_as_float(wd << 16), __uint_as_float(wd & 0xFFFF0000u));
                        } else {
                            const uint4& v = reinterpret_cast<const uint4&>(raw[u][h]);
                            x = j == 0 ? make_float2(tf32_trunc(__uint_as_float(v.x)), tf32_trunc(__uint_as_float(v.y)))
                                       : make_float2(tf32_trunc(__uint_as_float(v.z)), tf32_trunc(__uint_as_float(v.w)));
                        }
                        acc2 = __fadd2_rn(acc2, x);
                        colq2[h * 2 + j] = __ffma2_rn(x, x, colq2[h * 2 + j]);
                    }
                }
                q[u] = acc2.x + acc2.y;
                uint8_t* d = dst + u * dstep;
                *reinterpret_cast<V*>(d) = raw[u][0];
                if (h1ok) *reinterpret_cast<V*>(d + 128 * ELT) = raw[u][1];
            }
            float h2[2], h1;
            {
                const bool up = lane & 16;
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const float send = up ? q[i] : q[i + 2];
                    const float keep = up ? q[i + 2] : q[i];
                    h2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                }
            }
            {
                const bool up = lane & 8;
                const float send = up ? h2[0] : h2[1];
                const float keep = up ? h2[1] : h2[0];
                h1 = keep + __shfl_xor_sync(0xffffffffu, send, 8);
            }
            h1 += __shfl_xor_sync(0xffffffffu, h1, 4);
            h1 += __shfl_xor_sync(0xffffffffu, h1, 2);
            h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
            if (writer) {
                const int k = kc * rpb + r + 8 * u_me;
                uint8_t* sp = Bt + ((int64_t)k * ldt + (int64_t)tj * bn + 4 * nch) * ELT;
                float hi, mid, lo;
                split3<MODE>(h1, hi, mid, lo);
                if constexpr (MODE == 0) {
                    uint2 pk;
                    pk.x = (uint32_t)f32_to_bf16_rn(hi) | ((uint32_t)f32_to_bf16_rn(mid) << 16);
                    pk.y = (uint32_t)f32_to_bf16_rn(lo);
                    *reinterpret_cast<uint2*>(sp) = pk;
                } else {
                    *reinterpret_cast<float4*>(sp) = make_float4(hi, mid, lo, 0.0f);
                }
                Br[(int64_t)tj * kp + k] = h1;
                bqw = fmaf(h1, h1, bqw);
            }
            src += RB * sstep;
            dst += RB * dstep;
        }
        bq = warp_sum(bqw);
    } else
#endif
    for (int r = w; r < rpb; r += 8 * RB) {
        V raw[RB][2];
        float s[RB];
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const int k = kc * rpb + r + 8 * u;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int ch = lane + 32 * h;
                const int col = c0 + ch * 4;
                V x;
                if constexpr (MODE == 0) x = make_uint2(0u, 0u); else x = make_uint4(0u, 0u, 0u, 0u);
                if (k < K && ch < nch && col < N) {
                    const T* p = reinterpret_cast<const T*>(B_) + (int64_t)k * ldb + col;
                    if (N - col >= 4) {
                        x = __ldg(reinterpret_cast<const V*>(p));
                    } else {
                        alignas(16) T e4[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) e4[q] = (col + q < N) ? __ldg(p + q) : T(0);
                        x = *reinterpret_cast<V*>(e4);
                    }
                }
                raw[u][h] = x;
            }
        }
#if defined(FTGEMM_EXP_ENCB_SCALAR)
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            float acc = 0.0f;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const T* e4 = reinterpret_cast<const T*>(&raw[u][h]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float x = to_f(e4[q]);
                    acc += x;
                    colq[h * 4 + q] = fmaf(x, x, colq[h * 4 + q]);
                }
            }
            s[u] = acc;
        }
#else
        // paired FP32 ops (FADD2 / FFMA2): two columns per instruction; BF16
        // pairs unpacked with one shift / one mask per 32-bit word
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            float2 acc2 = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    float2 x;
                    if constexpr (MODE == 0) {
                        const uint32_t wd = j == 0 ? reinterpret_cast<const uint2&>(raw[u][h]).x
                                                   : reinterpret_cast<const uint2&>(raw[u][h]).y;
                        x = make_float2(__uint_as_float(wd << 16), __uint_as_float(wd & 0xFFFF0000u));
                    } else {
                        const uint4& v = reinterpret_cast<const uint4&>(raw[u][h]);
                        x = j == 0 ? make_float2(tf32_trunc(__uint_as_float(v.x)), tf32_trunc(__uint_as_float(v.y)))
                                   : make_float2(tf32_trunc(__uint_as_float(v.z)), tf32_trunc(__uint_as_float(v.w)));
                    }
                    acc2 = __fadd2_rn(acc2, x);
                    colq2[h * 2 + j] = __ffma2_rn(x, x, colq2[h * 2 + j]);
                }
            }
            s[u] = acc2.x + acc2.y;
        }
#endif
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < RB; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const int k = kc * rpb + r + 8 * u;
            if (k >= kp) continue;
            uint8_t* row = Bt + ((int64_t)k * ldt + (int64_t)tj * bn) * ELT;
#pragma unroll
            for (int h = 0; h < 2 && Bt != nullptr; ++h) {     // Bt == nullptr: checksums only
                const int ch = lane + 32 * h;
                if (ch < nch) {
                    *reinterpret_cast<V*>(row + ch * 4 * ELT) = raw[u][h];
                } else if (ch == nch) {               // the split of B_j e, then a zero column
                    float hi, mid, lo;
                    split3<MODE>(s[u], hi, mid, lo);
                    if constexpr (MODE == 0) {
                        uint2 pk;
                        pk.x = (uint32_t)f32_to_bf16_rn(hi) | ((uint32_t)f32_to_bf16_rn(mid) << 16);
                        pk.y = (uint32_t)f32_to_bf16_rn(lo);
                        *reinterpret_cast<uint2*>(row + ch * 4 * ELT) = pk;
                    } else {
                        *reinterpret_cast<float4*>(row + ch * 4 * ELT) = make_float4(hi, mid, lo, 0.0f);
                    }
                }
            }
            if (lane == 0) Br[(int64_t)tj * kp + k] = s[u];
            bq = fmaf(s[u], s[u], bq);
        }
    }
#if !defined(FTGEMM_EXP_ENCB_SCALAR)
#pragma unroll
    for (int i = 0; i < 4; ++i) { colq[2 * i] = colq2[i].x; colq[2 * i + 1] = colq2[i].y; }
#endif
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int ch = lane + 32 * h;
            if (ch < nch) red[w][ch * 4 + q] = colq[h * 4 + q];
        }
    if (lane == 0) red8[w] = bq;
    __syncthreads();
    for (int t = threadIdx.x; t < bnd; t += 256) {
        const int col = c0 + t;
        if (col < N) {
            float q = 0.0f;
#pragma unroll
            for (int ww = 0; ww < 8; ++ww) q += red[ww][t];
            cn2[(int64_t)kc * N + col] = q;
        }
    }
    if (threadIdx.x == 0) {
        float q = 0.0f;
        for (int i = 0; i < 8; ++i) q += red8[i];
        brn2[(int64_t)tj * nkc + kc] = q;
    }
    if (last_block(ticket, tj, nkc, &s_flag)) {
        for (int t = threadIdx.x; t < bnd; t += 256) {
            const int col = c0 + t;
            if (col < N) colnorm[col] = sqrtf(strided_sum(cn2 + col, nkc, N));
        }
        if (threadIdx.x == 0) brnorm[tj] = sqrtf(strided_sum(brn2 + (int64_t)tj * nkc, nkc, 1));
    }
}

// ---------------------------------------------------------------- kernels ---
// grid (nkc, tiles) per operand; encode_ab_kernel runs both operands in one
// 1-D launch (the B blocks first: they carry more bytes each), so a step's
// encode is one kernel on the caller's stream -- no side stream, no fork / join
// events -- and releases the fused GEMM (programmatic dependent launch) as soon
// as every block has started.
template <int MODE>
__global__ void __launch_bounds__(256, ENC_A_MINB) encode_a_kernel(const EncAP P) {
    griddep_launch_dependents();
    encode_a_body<MODE>(blockIdx.x, blockIdx.y, at_batch(P, blockIdx.z));
}
template <int MODE>
__global__ void __launch_bounds__(256) encode_b_tc_kernel(const EncBP P) {
    griddep_launch_dependents();
    encode_b_tc_body<MODE>(blockIdx.x, blockIdx.y, at_batch(P, blockIdx.z));
}
__global__ void __launch_bounds__(256) encode_b_simt_kernel(const EncBP P) {
    griddep_launch_dependents();
    encode_b_simt_body(blockIdx.x, blockIdx.y, at_batch(P, blockIdx.z));
}
template <int MODE>
__global__ void __launch_bounds__(256, 4) encode_ab_kernel(const EncAP PA, const EncBP PB, const int nblk_b) {
    griddep_launch_dependents();
    const int i = blockIdx.x;
    if (i < nblk_b) {
        const EncBP pb = at_batch(PB, blockIdx.y);
        if constexpr (MODE == 2) encode_b_simt_body(i % pb.nkc, i / pb.nkc, pb);
        else encode_b_tc_body<MODE>(i % pb.nkc, i / pb.nkc, pb);
    } else {
        const int j = i - nblk_b;
        const EncAP pa = at_batch(PA, blockIdx.y);
        encode_a_body<MODE>(j % pa.nkc, j / pa.nkc, pa);
    }
}

// ---------------------------------------------------------------- launch ---

cudaError_t launch_encode(const Geometry& g, const EncLayout& L, int64_t M, int64_t N, int64_t K,
                          const void* A, int64_t lda, const void* B, int64_t ldb, void* enc, int which,
                          cudaStream_t st, int batch, int64_t sA, int64_t sB, int64_t sE) {
    char* base = reinterpret_cast<char*>(enc);
    const int mode = g.dtype == FTGEMM_BF16 ? 0 : (g.dtype == FTGEMM_TF32 ? 1 : 2);
    auto F = [&](size_t off) { return reinterpret_cast<float*>(base + off); };
    cudaError_t e;
    EncAP pa{};
    EncBP pb{};
    if (which & 2) {
        // tickets of the last-block norm reduction (self-resetting; zeroed here
        // because enc_ws is caller memory of unknown content)
        if ((e = cudaMemset2DAsync(base + L.cnt_b, (size_t)(batch > 1 ? sE : (int64_t)sizeof(int) * g.tiles_n), 0, sizeof(int) * (size_t)g.tiles_n,
                                   (size_t)batch, st)) != cudaSuccess) return e;
        uint8_t* Bt = (mode == 2 || (which & 4)) ? nullptr : reinterpret_cast<uint8_t*>(base + L.bt);   // 4: no encoded operand
        pb = EncBP{B, ldb, (int)N, (int)K, g.bnd, g.bn, g.kp, g.tiles_n * g.bn, g.nkc_b, g.enc_b_rows,
                   F(L.br), Bt, F(L.cn2), F(L.brn2), reinterpret_cast<int*>(base + L.cnt_b), F(L.colnorm), F(L.brnorm),
                   sB, sE};
    }
    if (which & 1) {
        if ((e = cudaMemset2DAsync(base + L.cnt_a, (size_t)(batch > 1 ? sE : (int64_t)sizeof(int) * g.tiles_m), 0, sizeof(int) * (size_t)g.tiles_m,
                                   (size_t)batch, st)) != cudaSuccess) return e;
        pa = EncAP{A, lda, (int)M, (int)K, g.bmd, g.kp, g.bk, g.nkc_a, F(L.ac), reinterpret_cast<uint8_t*>(base + L.y),
                   F(L.rn2), F(L.acn2), reinterpret_cast<int*>(base + L.cnt_a), F(L.rownorm), F(L.acnorm), sA, sE};
    }
    if ((which & 3) == 3) {                      // both operands: one launch
        const int nb = g.nkc_b * g.tiles_n, na = g.nkc_a * g.tiles_m;
#define ENC_AB(MD) encode_ab_kernel<MD><<<dim3(nb + na, batch), 256, 0, st>>>(pa, pb, nb)
        if (mode == 0) ENC_AB(0); else if (mode == 1) ENC_AB(1); else ENC_AB(2);
#undef ENC_AB
        return cudaGetLastError();
    }
    if (which & 2) {
        dim3 grid(g.nkc_b, g.tiles_n, batch);
        if (mode == 2) encode_b_simt_kernel<<<grid, 256, 0, st>>>(pb);
        else if (mode == 0) encode_b_tc_kernel<0><<<grid, 256, 0, st>>>(pb);
        else encode_b_tc_kernel<1><<<grid, 256, 0, st>>>(pb);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (which & 1) {
        dim3 grid(g.nkc_a, g.tiles_m, batch);
        if (mode == 0) encode_a_kernel<0><<<grid, 256, 0, st>>>(pa);
        else if (mode == 1) encode_a_kernel<1><<<grid, 256, 0, st>>>(pa);
        else encode_a_kernel<2><<<grid, 256, 0, st>>>(pa);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace ftg
