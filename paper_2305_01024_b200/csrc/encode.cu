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
                                                       int bmd, int kp, float* __restrict__ Ac,
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
            if constexpr (MODE == 0) {
                uint16_t* Y = reinterpret_cast<uint16_t*>(Y_);
                Y[((int64_t)ti * 3 + 0) * kp + k] = f32_to_bf16_rn(hi);
                Y[((int64_t)ti * 3 + 1) * kp + k] = f32_to_bf16_rn(mid);
                Y[((int64_t)ti * 3 + 2) * kp + k] = f32_to_bf16_rn(lo);
            } else {
                float* Y = reinterpret_cast<float*>(Y_);
                Y[((int64_t)ti * 3 + 0) * kp + k] = hi;
                Y[((int64_t)ti * 3 + 1) * kp + k] = mid;
                Y[((int64_t)ti * 3 + 2) * kp + k] = lo;
            }
        }
    }
}

// Each warp reduces whole k-rows of one check tile j along its bnd columns
// (4-element chunks, lane l owns chunks l and l+32); column sums of squares
// are accumulated per lane and reduced over the 8 warps through shared memory.
template <int MODE>
__global__ void __launch_bounds__(256) encode_b_kernel(const void* __restrict__ B_, int64_t ldb, int N, int K,
                                                       int bnd, int kp, float* __restrict__ Br,
                                                       void* __restrict__ X_, float* __restrict__ cn2) {
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
                    const int valid = N - col;
                    float v[4] = {0.f, 0.f, 0.f, 0.f};
                    if (valid > 0) {
                        if constexpr (MODE == 0) load4_bf16(reinterpret_cast<const uint16_t*>(B_) + (int64_t)k * ldb + col, valid, v);
                        else load4_f32(reinterpret_cast<const float*>(B_) + (int64_t)k * ldb + col, valid, v);
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        float x = (MODE == 1) ? tf32_trunc(v[i]) : v[i];
                        s += x;
                        csq[h * 4 + i] = fmaf(x, x, csq[h * 4 + i]);
                    }
                }
            }
        }
        s = warp_sum(s);
        if (lane == 0) {
            Br[(int64_t)tj * kp + k] = s;
            if constexpr (MODE != 2) {
                float hi, mid, lo;
                split3<MODE>(s, hi, mid, lo);
                if constexpr (MODE == 0) {
                    uint16_t* X = reinterpret_cast<uint16_t*>(X_) + ((int64_t)tj * kp + k) * 4;
                    uint2 pk;
                    pk.x = (uint32_t)f32_to_bf16_rn(hi) | ((uint32_t)f32_to_bf16_rn(mid) << 16);
                    pk.y = (uint32_t)f32_to_bf16_rn(lo);
                    *reinterpret_cast<uint2*>(X) = pk;
                } else {
                    float* X = reinterpret_cast<float*>(X_) + ((int64_t)tj * kp + k) * 4;
                    *reinterpret_cast<float4*>(X) = make_float4(hi, mid, lo, 0.0f);
                }
            }
        }
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
        dim3 grid(g.nkc, g.tiles_m);
        float* Ac = reinterpret_cast<float*>(base + L.ac);
        void* Y = base + L.y;
        float* rn2 = reinterpret_cast<float*>(base + L.rn2);
        if (mode == 0) encode_a_kernel<0><<<grid, 256, 0, st>>>(A, lda, (int)M, (int)K, g.bmd, g.kp, Ac, Y, rn2);
        else if (mode == 1) encode_a_kernel<1><<<grid, 256, 0, st>>>(A, lda, (int)M, (int)K, g.bmd, g.kp, Ac, Y, rn2);
        else encode_a_kernel<2><<<grid, 256, 0, st>>>(A, lda, (int)M, (int)K, g.bmd, g.kp, Ac, Y, rn2);
        const int nb = (int)((M + 255) / 256) + g.tiles_m;
        finalize_kernel<<<nb, 256, 0, st>>>((int)M, g.nkc, rn2, reinterpret_cast<float*>(base + L.rownorm),
                                            g.tiles_m, g.kp, Ac, reinterpret_cast<float*>(base + L.acnorm));
    }
    if (which & 2) {
        dim3 grid(g.nkc, g.tiles_n);
        float* Br = reinterpret_cast<float*>(base + L.br);
        void* X = base + L.x;
        float* cn2 = reinterpret_cast<float*>(base + L.cn2);
        if (mode == 0) encode_b_kernel<0><<<grid, 256, 0, st>>>(B, ldb, (int)N, (int)K, g.bnd, g.kp, Br, X, cn2);
        else if (mode == 1) encode_b_kernel<1><<<grid, 256, 0, st>>>(B, ldb, (int)N, (int)K, g.bnd, g.kp, Br, X, cn2);
        else encode_b_kernel<2><<<grid, 256, 0, st>>>(B, ldb, (int)N, (int)K, g.bnd, g.kp, Br, X, cn2);
        const int nb = (int)((N + 255) / 256) + g.tiles_n;
        finalize_kernel<<<nb, 256, 0, st>>>((int)N, g.nkc, cn2, reinterpret_cast<float*>(base + L.colnorm),
                                            g.tiles_n, g.kp, Br, reinterpret_cast<float*>(base + L.brnorm));
    }
    return cudaGetLastError();
}

}  // namespace ftg
