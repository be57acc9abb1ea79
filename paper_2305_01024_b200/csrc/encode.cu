// encode.cu -- checksum-encode kernels (north_star item 2, "a checksum-encode
// kernel with coalesced, vectorised HBM reads and warp-shuffle reductions").
//
//   encode A (Eq. (1), A^c = [A; e^T A]):  per check tile i
//       Ac_i[k] = sum_{p in tile rows} A[p,k]            (FP32)
//       Y_i     = exact 3-way split of Ac_i into operand-format values
//                 (hi + mid + lo == Ac_i), appended to the MMA's A tile as
//                 rows 125..127 by the fused kernel
//       ||A[p,:]||_2 per row, ||Ac_i||_2 per tile         (threshold, R1)
//   encode B (Eq. (2), B^r = [B, B e]):   per check tile j
//       Br_j[k] = sum_{q in tile cols} B[k,q], split X_j (appended as columns
//       BN-4..BN-2 of the MMA's B tile), ||B[:,q]||_2, ||Br_j||_2.
//
// Both are single streaming passes over the operand (HBM bound); the only
// other traffic is the small outputs.  TF32 mode sums the values exactly as the
// tensor core will see them (low 13 mantissa bits dropped), so that the
// carried references and the main product are built from the same operands.
#include <cstdint>
#include <type_traits>

#include "common.cuh"

namespace ftg {

__device__ __forceinline__ void load8_bf16(const uint16_t* p, int valid, float (&v)[8]) {
    if (valid >= 8) {
        uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
        uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[2 * i] = __uint_as_float(w[i] << 16);
            v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = (i < valid) ? bf16_to_f32(__ldg(p + i)) : 0.0f;
    }
}
__device__ __forceinline__ void load8_f32(const float* p, int valid, float (&v)[8]) {
    if (valid >= 8) {
        float4 a = __ldg(reinterpret_cast<const float4*>(p));
        float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = (i < valid) ? __ldg(p + i) : 0.0f;
    }
}
__device__ __forceinline__ void load4_bf16(const uint16_t* p, int valid, float (&v)[4]) {
    if (valid >= 4) {
        uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
        v[0] = __uint_as_float(u.x << 16); v[1] = __uint_as_float(u.x & 0xFFFF0000u);
        v[2] = __uint_as_float(u.y << 16); v[3] = __uint_as_float(u.y & 0xFFFF0000u);
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = (i < valid) ? bf16_to_f32(__ldg(p + i)) : 0.0f;
    }
}
__device__ __forceinline__ void load4_f32(const float* p, int valid, float (&v)[4]) {
    if (valid >= 4) {
        float4 a = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = (i < valid) ? __ldg(p + i) : 0.0f;
    }
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Exact three-term split of an FP32 value into operand-format values.
// kind 0 = BF16 (round-to-nearest-even per term), 1 = TF32 (truncation).
template <int KIND>
__device__ __forceinline__ void split3(float s, float& hi, float& mid, float& lo) {
    if constexpr (KIND == 0) {
        hi = bf16_to_f32(f32_to_bf16_rn(s));
        float r1 = s - hi;
        mid = bf16_to_f32(f32_to_bf16_rn(r1));
        lo = bf16_to_f32(f32_to_bf16_rn(r1 - mid));
    } else {
        hi = tf32_trunc(s);
        float r1 = s - hi;
        mid = tf32_trunc(r1);
        lo = r1 - mid;
    }
}

// MODE: 0 = BF16 operands, 1 = TF32 (FP32 storage, truncated), 2 = FP32 SIMT (no split)
template <int MODE>
__global__ void __launch_bounds__(256) encode_a_kernel(const void* __restrict__ A_, int64_t lda, int M, int K,
                                                       int bmd, int kp, int bk, float* __restrict__ Ac,
                                                       void* __restrict__ Y_, float* __restrict__ rn2) {
    __shared__ float red[8][257];
    const int kc = blockIdx.x, ti = blockIdx.y;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k0 = kc * 256 + lane * 8;
    const int valid = K - k0;             // elements of this lane's 8 inside K
    float ac[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) ac[i] = 0.0f;
    const int rbeg = ti * bmd;
    const int rend = min(M, rbeg + bmd);
    for (int row = rbeg + w; row < rend; row += 8) {
        float v[8];
        if (valid > 0) {
            if constexpr (MODE == 0) load8_bf16(reinterpret_cast<const uint16_t*>(A_) + (int64_t)row * lda + k0, valid, v);
            else load8_f32(reinterpret_cast<const float*>(A_) + (int64_t)row * lda + k0, valid, v);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = 0.0f;
        }
        float sq = 0.0f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float x = (MODE == 1) ? tf32_trunc(v[i]) : v[i];
            ac[i] += x;
            sq = fmaf(x, x, sq);
        }
        sq = warp_sum(sq);
        if (lane == 0) rn2[(int64_t)kc * M + row] = sq;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) red[w][lane * 8 + i] = ac[i];
    __syncthreads();
    const int t = threadIdx.x;
    const int k = kc * 256 + t;
    if (k < kp) {
        float s = 0.0f;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) s += red[ww][t];
        if (k >= K) s = 0.0f;
        Ac[(int64_t)ti * kp + k] = s;
        if constexpr (MODE != 2) {
            float hi, mid, lo;
            split3<MODE>(s, hi, mid, lo);
            // Ypack[tile][k-block][r][128 bytes]: split row r lands in MMA row
            // 125 + r of the A tile, whose 16-byte chunks are stored in the
            // SWIZZLE_128B order (chunk c at c ^ (row & 7)) so the fused kernel
            // can bulk-copy the 384 bytes straight into shared memory.
            constexpr int ELT = MODE == 0 ? 2 : 4;
            const int kb = k / bk, kk = k % bk;
            const int chunk = (kk * ELT) >> 4, within = (kk * ELT) & 15;
            uint8_t* yb = reinterpret_cast<uint8_t*>(Y_) + ((int64_t)ti * (kp / bk) + kb) * 384;
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
}

// FP32 SIMT path: B e per tile, column sums of squares (no operand copy).
// Each warp reduces whole k-rows of one check tile j along its bnd columns
// (4-element chunks, lane l owns chunks l and l+32).
__global__ void __launch_bounds__(256) encode_b_simt_kernel(const float* __restrict__ B, int64_t ldb, int N, int K,
                                                            int bnd, int kp, float* __restrict__ Br,
                                                            float* __restrict__ cn2) {
    __shared__ float red[8][257];
    const int kc = blockIdx.x, tj = blockIdx.y;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nch = bnd / 4;
    const int c0 = tj * bnd;
    float csq[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) csq[i] = 0.0f;
    for (int r = w; r < 256; r += 8) {
        const int k = kc * 256 + r;
        if (k >= kp) break;
        float s = 0.0f;
        if (k < K) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int ch = lane + 32 * h;
                if (ch < nch) {
                    const int col = c0 + ch * 4;
                    float v[4] = {0.f, 0.f, 0.f, 0.f};
                    if (N - col > 0) load4_f32(B + (int64_t)k * ldb + col, N - col, v);
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
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int ch = lane + 32 * h;
            if (ch < nch) red[w][ch * 4 + i] = csq[h * 4 + i];
        }
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
}

// Tensor-core paths: one block per (k-block of KC = one 128-byte row of K,
// check tile j).  Stages B[k0:k0+KC, c0:c0+bnd] in shared memory (row stride
// 257 elements: conflict-free transpose), reduces B_j e per k-row (warp
// shuffles), the column sums of squares, and writes the encoded operand
// B^r_j = [B_j, split(B_j e), 0] transposed (K-major, bn rows of KC) with
// coalesced 128-byte row stores.
template <int MODE>
__global__ void __launch_bounds__(256) encode_b_tc_kernel(const void* __restrict__ B_, int64_t ldb, int N, int K,
                                                          int bnd, int bn, int kp, float* __restrict__ Br,
                                                          void* __restrict__ Bt_, float* __restrict__ cn2) {
    constexpr int ELT = MODE == 0 ? 2 : 4;
    constexpr int KC = 128 / ELT;
    constexpr int S = 257;
    using T = typename std::conditional<MODE == 0, uint16_t, float>::type;
    __shared__ T sb[KC * S];
    __shared__ float br_s[KC];
    const int kc = blockIdx.x, tj = blockIdx.y;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k0 = kc * KC, c0 = tj * bnd;
    const int nch = bnd / 4;
    // ---- load (coalesced 4-element chunks) ----
    for (int idx = threadIdx.x; idx < KC * nch; idx += 256) {
        const int kk = idx / nch, ch = idx - kk * nch;
        const int k = k0 + kk, col = c0 + ch * 4;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (k < K && col < N) {
            if constexpr (MODE == 0) load4_bf16(reinterpret_cast<const uint16_t*>(B_) + (int64_t)k * ldb + col, N - col, v);
            else load4_f32(reinterpret_cast<const float*>(B_) + (int64_t)k * ldb + col, N - col, v);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if constexpr (MODE == 0) sb[kk * S + ch * 4 + i] = f32_to_bf16_rn(v[i]);   // exact (bf16 values)
            else sb[kk * S + ch * 4 + i] = tf32_trunc(v[i]);
        }
    }
    __syncthreads();
    auto val = [&](int kk, int n) -> float {
        if constexpr (MODE == 0) return bf16_to_f32(sb[kk * S + n]);
        else return sb[kk * S + n];
    };
    // ---- B_j e per k-row ----
    for (int kk = w; kk < KC; kk += 8) {
        float s = 0.0f;
        for (int n = lane; n < bnd; n += 32) s += val(kk, n);
        s = warp_sum(s);
        if (lane == 0) {
            br_s[kk] = s;
            Br[(int64_t)tj * kp + k0 + kk] = s;
        }
    }
    // ---- column sums of squares (partial over this k-block) ----
    for (int n = threadIdx.x; n < bnd; n += 256) {
        float q = 0.0f;
        for (int kk = 0; kk < KC; ++kk) { const float x = val(kk, n); q = fmaf(x, x, q); }
        if (c0 + n < N) cn2[(int64_t)kc * N + c0 + n] = q;
    }
    __syncthreads();
    // ---- write B^r rows (K-major) ----
    for (int n = w; n < bn; n += 8) {
        uint8_t* dst = reinterpret_cast<uint8_t*>(Bt_) + (((int64_t)tj * bn + n) * kp + k0) * ELT;
        if constexpr (MODE == 0) {
            uint32_t pk;
            const int kk = 2 * lane;
            if (n < bnd) {
                pk = (uint32_t)sb[kk * S + n] | ((uint32_t)sb[(kk + 1) * S + n] << 16);
            } else if (n < bnd + 3) {
                float p0[3], p1[3];
                split3<0>(br_s[kk], p0[0], p0[1], p0[2]);
                split3<0>(br_s[kk + 1], p1[0], p1[1], p1[2]);
                const int r = n - bnd;
                pk = (uint32_t)f32_to_bf16_rn(p0[r]) | ((uint32_t)f32_to_bf16_rn(p1[r]) << 16);
            } else {
                pk = 0u;
            }
            reinterpret_cast<uint32_t*>(dst)[lane] = pk;
        } else {
            const int kk = lane;
            float v;
            if (n < bnd) {
                v = sb[kk * S + n];
            } else if (n < bnd + 3) {
                float p[3];
                split3<1>(br_s[kk], p[0], p[1], p[2]);
                v = p[n - bnd];
            } else {
                v = 0.0f;
            }
            reinterpret_cast<float*>(dst)[lane] = v;
        }
    }
}

// norms: rownorm[p] = sqrt(sum_c rn2[c][p]); acnorm[i] = ||Ac_i||_2.
__global__ void __launch_bounds__(256) finalize_kernel(int n_vec, int nkc, const float* __restrict__ part,
                                                       float* __restrict__ vecnorm, int ntiles, int kp,
                                                       const float* __restrict__ sums, float* __restrict__ tilenorm) {
    const int nvb = (n_vec + 255) / 256;
    if ((int)blockIdx.x < nvb) {
        const int i = blockIdx.x * 256 + threadIdx.x;
        if (i < n_vec) {
            float s = 0.0f;
            for (int c = 0; c < nkc; ++c) s += part[(int64_t)c * n_vec + i];
            vecnorm[i] = sqrtf(s);
        }
        return;
    }
    const int t = blockIdx.x - nvb;
    if (t >= ntiles) return;
    __shared__ float red[8];
    float s = 0.0f;
    for (int k = threadIdx.x; k < kp; k += 256) {
        float x = sums[(int64_t)t * kp + k];
        s = fmaf(x, x, s);
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        float tot = 0.0f;
        for (int i = 0; i < 8; ++i) tot += red[i];
        tilenorm[t] = sqrtf(tot);
    }
}

// ---------------------------------------------------------------- launch ---
cudaError_t launch_encode(const Geometry& g, const EncLayout& L, int64_t M, int64_t N, int64_t K,
                          const void* A, int64_t lda, const void* B, int64_t ldb, void* enc, int which,
                          cudaStream_t st) {
    char* base = reinterpret_cast<char*>(enc);
    const int mode = g.dtype == FTGEMM_BF16 ? 0 : (g.dtype == FTGEMM_TF32 ? 1 : 2);
    if (which & 1) {
        dim3 grid(g.nkc_a, g.tiles_m);
        float* Ac = reinterpret_cast<float*>(base + L.ac);
        void* Y = base + L.y;
        float* rn2 = reinterpret_cast<float*>(base + L.rn2);
        if (mode == 0) encode_a_kernel<0><<<grid, 256, 0, st>>>(A, lda, (int)M, (int)K, g.bmd, g.kp, g.bk, Ac, Y, rn2);
        else if (mode == 1) encode_a_kernel<1><<<grid, 256, 0, st>>>(A, lda, (int)M, (int)K, g.bmd, g.kp, g.bk, Ac, Y, rn2);
        else encode_a_kernel<2><<<grid, 256, 0, st>>>(A, lda, (int)M, (int)K, g.bmd, g.kp, g.bk, Ac, Y, rn2);
        const int nb = (int)((M + 255) / 256) + g.tiles_m;
        finalize_kernel<<<nb, 256, 0, st>>>((int)M, g.nkc_a, rn2, reinterpret_cast<float*>(base + L.rownorm),
                                            g.tiles_m, g.kp, Ac, reinterpret_cast<float*>(base + L.acnorm));
    }
    if (which & 2) {
        float* Br = reinterpret_cast<float*>(base + L.br);
        float* cn2 = reinterpret_cast<float*>(base + L.cn2);
        if (mode == 2) {
            dim3 grid(g.nkc_b, g.tiles_n);
            encode_b_simt_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(B), ldb, (int)N, (int)K, g.bnd,
                                                       g.kp, Br, cn2);
        } else {
            dim3 grid(g.nkc_b, g.tiles_n);
            void* Bt = base + L.bt;
            if (mode == 0) encode_b_tc_kernel<0><<<grid, 256, 0, st>>>(B, ldb, (int)N, (int)K, g.bnd, g.bn, g.kp, Br, Bt, cn2);
            else encode_b_tc_kernel<1><<<grid, 256, 0, st>>>(B, ldb, (int)N, (int)K, g.bnd, g.bn, g.kp, Br, Bt, cn2);
        }
        const int nb = (int)((N + 255) / 256) + g.tiles_n;
        finalize_kernel<<<nb, 256, 0, st>>>((int)N, g.nkc_b, cn2, reinterpret_cast<float*>(base + L.colnorm),
                                            g.tiles_n, g.kp, Br, reinterpret_cast<float*>(base + L.brnorm));
    }
    return cudaGetLastError();
}

}  // namespace ftg
