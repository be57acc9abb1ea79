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
// Single streaming passes over each operand (HBM bound): loads are 8- or
// 16-byte vectors, issued in unrolled batches before use (memory-level
// parallelism), reductions go through warp shuffles and shared memory.  The
// per-row / per-column norms are reduced across K-chunk blocks by the LAST
// block of each tile (atomic ticket, self-resetting), so no extra launch is
// needed.  TF32 mode sums the values exactly as the tensor core will see them
// (low 13 mantissa bits dropped), so the carried references and the main
// product are built from the same operands.
#include <cstdint>
#include <type_traits>

#include "common.cuh"

namespace ftg {

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// sum over the 256 threads of a block (result valid in every thread)
__device__ __forceinline__ float block_sum256(float x, float* red8) {
    x = warp_sum(x);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red8[threadIdx.x >> 5] = x;
    __syncthreads();
    float t = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red8[i];
    return t;
}

// 8 consecutive operand values of a row starting at p (valid = elements inside K)
template <int MODE>
__device__ __forceinline__ void load8(const void* base, int64_t off, int valid, float (&v)[8]) {
    if constexpr (MODE == 0) {
        const uint16_t* p = reinterpret_cast<const uint16_t*>(base) + off;
        if (valid >= 8) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                v[2 * i] = __uint_as_float(w[i] << 16);
                v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = (i < valid) ? bf16_to_f32(__ldg(p + i)) : 0.0f;
        }
    } else {
        const float* p = reinterpret_cast<const float*>(base) + off;
        if (valid >= 8) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(p));
            const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = (i < valid) ? __ldg(p + i) : 0.0f;
        }
        if constexpr (MODE == 1) {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = tf32_trunc(v[i]);
        }
    }
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

// ---------------------------------------------------------------- encode A --
// grid (nkc = ceil(kp/256), tiles_m); block 256 = 8 warps.  Lane l owns k in
// [kc*256 + 8l, +8); warp w sums rows w, w+8, ... of the tile (4 rows per batch).
// MODE: 0 = BF16, 1 = TF32 (FP32 storage, truncated), 2 = FP32 SIMT (no split).
template <int MODE>
__global__ void __launch_bounds__(256) encode_a_kernel(const void* __restrict__ A, int64_t lda, int M, int K,
                                                       int bmd, int kp, int bk, int nkc, float* __restrict__ Ac,
                                                       uint8_t* __restrict__ Y, float* rn2, float* acn2, int* ticket,
                                                       float* __restrict__ rownorm, float* __restrict__ acnorm) {
    __shared__ float red[8][257];
    __shared__ float red8[8];
    __shared__ int s_flag;
    const int kc = blockIdx.x, ti = blockIdx.y;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k0 = kc * 256 + lane * 8;
    const int valid = K - k0;
    float ac[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) ac[i] = 0.0f;
    const int rbeg = ti * bmd;
    const int rend = min(M, rbeg + bmd);
    // rows w, w+8, ... of the tile; RB rows per batch so that RB independent
    // 16-byte loads per lane are in flight (BF16 keeps them packed until use)
    constexpr int RB = MODE == 0 ? 8 : 4;
    for (int row = rbeg + w; row < rend; row += 8 * RB) {
        float sq[RB];
        if constexpr (MODE == 0) {
            uint4 raw[RB];
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                const int r = row + 8 * u;
                raw[u] = make_uint4(0u, 0u, 0u, 0u);
                if (r < rend && valid >= 8) {
                    raw[u] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(A) + (int64_t)r * lda + k0));
                } else if (r < rend && valid > 0) {
                    float v[8];
                    load8<0>(A, (int64_t)r * lda + k0, valid, v);
                    uint32_t pk[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        pk[i] = (__float_as_uint(v[2 * i]) >> 16) | (__float_as_uint(v[2 * i + 1]) & 0xFFFF0000u);
                    raw[u] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
            }
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                const uint32_t wd[4] = {raw[u].x, raw[u].y, raw[u].z, raw[u].w};
                float q = 0.0f;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float lo = __uint_as_float(wd[i] << 16), hi = __uint_as_float(wd[i] & 0xFFFF0000u);
                    ac[2 * i] += lo;
                    ac[2 * i + 1] += hi;
                    q = fmaf(lo, lo, q);
                    q = fmaf(hi, hi, q);
                }
                sq[u] = q;
            }
        } else {
            float v[RB][8];
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                const int r = row + 8 * u;
                if (r < rend && valid > 0) load8<MODE>(A, (int64_t)r * lda + k0, valid, v[u]);
                else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[u][i] = 0.0f;
                }
            }
#pragma unroll
            for (int u = 0; u < RB; ++u) {
                float q = 0.0f;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    ac[i] += v[u][i];
                    q = fmaf(v[u][i], v[u][i], q);
                }
                sq[u] = q;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < RB; ++u) sq[u] += __shfl_xor_sync(0xffffffffu, sq[u], o);
        if (lane == 0) {
#pragma unroll
            for (int u = 0; u < RB; ++u)
                if (row + 8 * u < rend) rn2[(int64_t)kc * M + row + 8 * u] = sq[u];
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) red[w][lane * 8 + i] = ac[i];
    __syncthreads();
    const int t = threadIdx.x;
    const int k = kc * 256 + t;
    float s = 0.0f;
    if (k < kp) {
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
            // bulk-copies the 384 bytes straight into shared memory.
            constexpr int ELT = MODE == 0 ? 2 : 4;
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
    const float s2 = block_sum256(s * s, red8);
    if (t == 0) acn2[(int64_t)ti * nkc + kc] = s2;
    if (last_block(ticket, ti, nkc, &s_flag)) {
        for (int p = rbeg + t; p < rend; p += 256) rownorm[p] = sqrtf(strided_sum(rn2 + p, nkc, M));
        if (t == 0) acnorm[ti] = sqrtf(strided_sum(acn2 + (int64_t)ti * nkc, nkc, 1));
    }
}

// ----------------------------------------------------- encode B (FP32 SIMT) --
// grid (nkc = ceil(kp/256), tiles_n): Br_j (warp per k-row) and column squares.
__global__ void __launch_bounds__(256) encode_b_simt_kernel(const float* __restrict__ B, int64_t ldb, int N, int K,
                                                            int bnd, int kp, int nkc, float* __restrict__ Br,
                                                            float* cn2, float* brn2, int* ticket,
                                                            float* __restrict__ colnorm, float* __restrict__ brnorm) {
    __shared__ float red[8][257];
    __shared__ float red8[8];
    __shared__ int s_flag;
    const int kc = blockIdx.x, tj = blockIdx.y;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nch = bnd / 4;
    const int c0 = tj * bnd;
    float csq[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) csq[i] = 0.0f;
    float bq = 0.0f;
    for (int r = w; r < 256; r += 8) {
        const int k = kc * 256 + r;
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
// grid (nkc = ceil(kp/256), tiles_n); warp w handles k-rows kc*256 + w + 8i.
// Per k-row of check tile j the warp streams the bnd data columns (4-element
// chunks: lane l owns chunks l and l+32), reduces B_j e with warp shuffles,
// accumulates column squares in registers, and writes the encoded operand row
//     Bt[k][j*bn : (j+1)*bn] = [B[k, j*bnd : j*bnd+bnd], split(B_j e)[k], 0]
// (B^r of Eq. (2), N-major, every tile slot 16-byte / 128-byte aligned so the
// fused kernel's TMA boxes start on cache-line boundaries).
template <int MODE>
__global__ void __launch_bounds__(256) encode_b_tc_kernel(const void* __restrict__ B_, int64_t ldb, int N, int K,
                                                          int bnd, int bn, int kp, int ldt, int nkc,
                                                          float* __restrict__ Br, uint8_t* __restrict__ Bt,
                                                          float* cn2, float* brn2, int* ticket,
                                                          float* __restrict__ colnorm, float* __restrict__ brnorm) {
    constexpr int ELT = MODE == 0 ? 2 : 4;
    using T = typename std::conditional<MODE == 0, uint16_t, float>::type;
    using V = typename std::conditional<MODE == 0, uint2, uint4>::type;     // 4 elements
    constexpr int RB = 4;                                                   // rows per batch
    __shared__ float red[8][257];
    __shared__ float red8[8];
    __shared__ int s_flag;
    const int kc = blockIdx.x, tj = blockIdx.y;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c0 = tj * bnd;
    const int nch = bnd / 4;                  // data chunks; chunk index nch is the split slot
    float colq[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) colq[i] = 0.0f;
    float bq = 0.0f;
    auto to_f = [](T x) -> float {
        if constexpr (MODE == 0) return bf16_to_f32(x);
        else return tf32_trunc(x);
    };
    for (int r = w; r < 256; r += 8 * RB) {
        V raw[RB][2];
        float s[RB];
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const int k = kc * 256 + r + 8 * u;
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
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < RB; ++u) s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
#pragma unroll
        for (int u = 0; u < RB; ++u) {
            const int k = kc * 256 + r + 8 * u;
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

// ---------------------------------------------------------------- launch ---
cudaError_t launch_encode(const Geometry& g, const EncLayout& L, int64_t M, int64_t N, int64_t K,
                          const void* A, int64_t lda, const void* B, int64_t ldb, void* enc, int which,
                          cudaStream_t st) {
    char* base = reinterpret_cast<char*>(enc);
    const int mode = g.dtype == FTGEMM_BF16 ? 0 : (g.dtype == FTGEMM_TF32 ? 1 : 2);
    auto F = [&](size_t off) { return reinterpret_cast<float*>(base + off); };
    if (which & 1) {
        cudaError_t e = cudaMemsetAsync(base + L.cnt_a, 0, sizeof(int) * (size_t)g.tiles_m, st);
        if (e != cudaSuccess) return e;
        dim3 grid(g.nkc_a, g.tiles_m);
        uint8_t* Y = reinterpret_cast<uint8_t*>(base + L.y);
        int* tk = reinterpret_cast<int*>(base + L.cnt_a);
#define ENC_A(MD) encode_a_kernel<MD><<<grid, 256, 0, st>>>(A, lda, (int)M, (int)K, g.bmd, g.kp, g.bk, g.nkc_a, \
            F(L.ac), Y, F(L.rn2), F(L.acn2), tk, F(L.rownorm), F(L.acnorm))
        if (mode == 0) ENC_A(0); else if (mode == 1) ENC_A(1); else ENC_A(2);
#undef ENC_A
    }
    if (which & 2) {
        cudaError_t e = cudaMemsetAsync(base + L.cnt_b, 0, sizeof(int) * (size_t)g.tiles_n, st);
        if (e != cudaSuccess) return e;
        int* tk = reinterpret_cast<int*>(base + L.cnt_b);
        dim3 grid(g.nkc_b, g.tiles_n);
        if (mode == 2) {
            encode_b_simt_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(B), ldb, (int)N, (int)K, g.bnd,
                                                       g.kp, g.nkc_b, F(L.br), F(L.cn2), F(L.brn2), tk,
                                                       F(L.colnorm), F(L.brnorm));
        } else {
            uint8_t* Bt = (which & 4) ? nullptr : reinterpret_cast<uint8_t*>(base + L.bt);   // 4: no encoded operand
#define ENC_B(MD) encode_b_tc_kernel<MD><<<grid, 256, 0, st>>>(B, ldb, (int)N, (int)K, g.bnd, g.bn, g.kp, \
            g.tiles_n * g.bn, g.nkc_b, F(L.br), Bt, F(L.cn2), F(L.brn2), tk, F(L.colnorm), F(L.brnorm))
            if (mode == 0) ENC_B(0); else ENC_B(1);
#undef ENC_B
        }
    }
    return cudaGetLastError();
}

}  // namespace ftg
