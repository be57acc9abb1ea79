// simt_gemm.cu -- exact-semantics FP32 SIMT fused ABFT SGEMM (north_star item 3).
//
// The paper's threadblock-level FT-SGEMM (section 4.2.3) on
// CUDA cores, with the paper's SGEMM structure (section 3.1 and
// the "huge" row of Table 1: m_tb = n_tb = 128, k_tb = 8,
// 8 x 8 outputs per thread, 256 threads, double-buffered shared memory).
// Every output is accumulated with one fmaf per k in ascending k, so a clean
// element is bit-identical to the oracle's FP32SEQ mode.
//
// Checksums (Eq. (3)): the encoded e^T A_i and B_j e (from the
// encode kernel) are staged with each k-block next to A_tb and B_tb -- the
// paper fuses their loads with the prefetch -- and carried by
// the CTA through the same k-loop:
//     threads 0..127  : C^r_ref[p] += A_tb[p,k] * (B_j e)[k]     (row p = tid)
//     threads 128..255: C^c_ref[q] += (e^T A_i)[k] * B_tb[k,q]   (col q = tid-128)
// i.e. 2 x 128 x 8 extra FMAs per 128 x 128 x 8 k-block (1.6 %).  After the
// k-loop the tile's row and column sums are reduced (shuffles + shared memory),
// compared with the references, and a single error is located and corrected
// from the row checksum.
#include <cstdint>

#include "common.cuh"
#include "ptx.cuh"

namespace ftg {

#ifndef FTGEMM_SIMT_SK
#define FTGEMM_SIMT_SK 32
#endif
constexpr int SB = 128, SK = FTGEMM_SIMT_SK;       // tile, k-block (plan.bk)
#ifndef FTGEMM_SIMT_NST
#define FTGEMM_SIMT_NST (SK == 8 ? 4 : 3)
#endif
constexpr int NST = FTGEMM_SIMT_NST;                // smem pipeline stages
// A tile rows padded by 4 floats: the row-reference FMAs read A[p][k] with one
// thread per row, which at a 64-byte row pitch hit 2 banks (16-way conflicts);
// at 80 bytes the 16-byte reads of 8 lanes cover all 32 banks
constexpr int SKP_FT = SK + 4;
constexpr int STAGE_FLOATS = SB * SKP_FT + SK * SB + 2 * SK;     // sized for the padded (FT) layout
constexpr int SIMT_DSMEM = NST * STAGE_FLOATS * 4;  // dynamic smem: the stage ring

__device__ __forceinline__ int simt_inj_lower(const DevInject* inj, int n, int t) {
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (inj[mid].tile < t) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ float simt_fault(float x, const DevInject& f) {
    if (f.mode == FTGEMM_INJ_ADD) return x + f.addend;
    return __uint_as_float(__float_as_uint(x) ^ (1u << (f.bit & 31)));
}

#ifndef FTGEMM_SIMT_AK
#define FTGEMM_SIMT_AK 4     // k per A-fragment load (4: 16-byte loads, 2: 8-byte loads)
#endif
#ifndef FTGEMM_SIMT_MINB
#define FTGEMM_SIMT_MINB 2
#endif
template <bool FT>
__global__ void __launch_bounds__(256, FTGEMM_SIMT_MINB) simt_ftgemm_kernel(const SimtArgs a) {
    // stage ring (dynamic smem): A tile row-major (k contiguous), B tile, and
    // e^T A_i, B_j e for the k-block
    extern __shared__ __align__(16) float simt_dsmem[];
    constexpr int SKP = FT ? SKP_FT : SK;            // FT off: unpadded rows (measured 2.5 % faster)
    float (*As)[SB][SKP] = reinterpret_cast<float (*)[SB][SKP]>(simt_dsmem);
    float (*Bs)[SK][SB] = reinterpret_cast<float (*)[SK][SB]>(simt_dsmem + NST * SB * SKP);
    float (*acs)[SK] = reinterpret_cast<float (*)[SK]>(simt_dsmem + NST * SB * SKP + NST * SK * SB);
    float (*brs)[SK] = reinterpret_cast<float (*)[SK]>(simt_dsmem + NST * SB * SKP + NST * SK * SB + NST * SK);
    __shared__ float red_col[8][SB];                   // column partial sums per warp
    __shared__ float srow_s[SB], rref_s[SB], cref_s[SB], rres[SB], rtau[SB], cres[SB], ctau[SB];
    __shared__ int sflag[6];
    __shared__ DevInject sinj[8];
    __shared__ int s_ninj;

    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    // tile raster: group 8 M-tiles for L2 reuse
    int ti, tj;
    {
        const int t = blockIdx.x;
        constexpr int G = 8;
        const int per = G * a.tiles_n;
        const int grp = t / per, first = grp * G;
        const int gsz = min(G, a.tiles_m - first);
        const int loc = t - grp * per;
        ti = first + loc % gsz;
        tj = loc / gsz;
    }
    const int tile = ti * a.tiles_n + tj;
    const int r0 = ti * SB, c0 = tj * SB;
    const int bm = min(SB, a.M - r0), bn = min(SB, a.N - c0);

    // faults of this tile (at most 8 handled per tile; the host enforces it)
    if (FT && tid == 0) {
        int n = 0;
        if (a.n_inj > 0) {
            const int lo = simt_inj_lower(a.inj, a.n_inj, tile);
            const int hi = simt_inj_lower(a.inj, a.n_inj, tile + 1);
            for (int i = lo; i < hi && n < 8; ++i) sinj[n++] = a.inj[i];
        }
        s_ninj = n;
    }

    // global -> shared copies of one k-block (16-byte cp.async, NST-stage ring,
    // out-of-range elements zero-filled), issued NST-1 k-blocks ahead.
    // Interior tiles (whole 128 x 128 tile inside C, K a multiple of SK) take a
    // guard-free path over per-thread source pointers computed once: the
    // per-k-block index arithmetic of the general path ran on the FMA pipe
    // beside the FFMA2 stream and spilled registers.
    const bool interior = r0 + SB <= a.M && c0 + SB <= a.N && a.K % SK == 0;
    const float* pa0 = a.A + (int64_t)(r0 + tid / (SK / 4)) * a.lda + (tid % (SK / 4)) * 4;
    const float* pb0 = a.B + (int64_t)(tid >> 5) * a.ldb + c0 + (tid & 31) * 4;
    constexpr int A_ROWS_PER_U = 256 / (SK / 4);        // A rows covered by one 256-thread pass
    const int64_t a_ustep = (int64_t)A_ROWS_PER_U * a.lda, b_ustep = (int64_t)8 * a.ldb;
    const uint32_t sa0 = (uint32_t)__cvta_generic_to_shared(&As[0][tid / (SK / 4)][(tid % (SK / 4)) * 4]);
    const uint32_t sb0 = (uint32_t)__cvta_generic_to_shared(&Bs[0][tid >> 5][(tid & 31) * 4]);
    auto issue = [&](int kb, int s) {
        const int k0 = kb * SK;
        if (interior) {
            const float* pa = pa0 + k0;
            const float* pb = pb0 + (int64_t)k0 * a.ldb;
#pragma unroll
            for (int u = 0; u < SK / 8; ++u) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                             :: "r"(sa0 + (uint32_t)(s * SB * SKP + u * A_ROWS_PER_U * SKP) * 4u), "l"(pa + u * a_ustep)
                             : "memory");
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                             :: "r"(sb0 + (uint32_t)(s * SK * SB + u * 8 * SB) * 4u), "l"(pb + u * b_ustep)
                             : "memory");
            }
            if (FT) {
                if (tid < SK) cp_async4(&acs[s][tid], a.Ac + (int64_t)ti * a.kp + k0 + tid, 4);
                else if (tid < 2 * SK) cp_async4(&brs[s][tid - SK], a.Br + (int64_t)tj * a.kp + k0 + tid - SK, 4);
            }
            return;
        }
#pragma unroll
        for (int u = 0; u < SK / 8; ++u) {                  // A: 128 rows x SK k, 16-byte chunks
            const int L = tid + 256 * u;
            const int a_row = L / (SK / 4), a_k = (L % (SK / 4)) * 4;
            const int gr = r0 + a_row, gk = k0 + a_k;
            const int na = gr < a.M ? max(0, min(4, a.K - gk)) : 0;
            cp_async16(&As[s][a_row][a_k], a.A + (int64_t)min(gr, a.M - 1) * a.lda + (na ? gk : 0), 4 * na);
        }
#pragma unroll
        for (int u = 0; u < SK / 8; ++u) {                  // B: SK k x 128 cols
            const int L = tid + 256 * u;
            const int b_k = L >> 5, b_col = (L & 31) * 4;
            const int bk = k0 + b_k, gc = c0 + b_col;
            const int nv = bk < a.K ? max(0, min(4, a.N - gc)) : 0;
            cp_async16(&Bs[s][b_k][b_col], a.B + (int64_t)min(bk, a.K - 1) * a.ldb + (nv ? gc : 0), 4 * nv);
        }
        if (FT) {
            if (tid < SK) cp_async4(&acs[s][tid], a.Ac + (int64_t)ti * a.kp + k0 + tid, 4);
            else if (tid < 2 * SK) cp_async4(&brs[s][tid - SK], a.Br + (int64_t)tj * a.kp + k0 + tid - SK, 4);
        }
    };

    // 8 x 8 accumulators as column pairs: one FFMA2 (two independent,
    // individually rounded fmaf -- the same arithmetic as fmaf per element)
    // updates two outputs of a row per issue slot
    float2 acc2[8][4];
#define ACC(i, j) (((j) & 1) ? acc2[i][(j) >> 1].y : acc2[i][(j) >> 1].x)
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc2[i][j] = make_float2(0.0f, 0.0f);
    float ref = 0.0f;   // row ref (tid < 128) or col ref (tid >= 128)

#pragma unroll
    for (int s = 0; s < NST - 1; ++s) {
        if (s < a.num_kb) issue(s, s);
        cp_async_commit();
    }
    __syncthreads();                                   // s_ninj / sinj visible
    int ninj = FT ? s_ninj : 0;
    int next_inj = 0;

    for (int kb = 0; kb < a.num_kb; ++kb) {
        const int buf = kb % NST;
        cp_async_wait<NST - 2>();                      // this thread's copies of k-block kb landed
        __syncthreads();                               // everyone's, and stage (kb-1) % NST is free
        if (kb + NST - 1 < a.num_kb) issue(kb + NST - 1, (kb + NST - 1) % NST);
        cp_async_commit();
        // two halves of 4 k: the thread's 8 rows x 4 k of A (one 16-byte load
        // per row), then per k the 8 columns of B; every output still sees
        // one fmaf per k in ascending k
#if FTGEMM_SIMT_AK == 4
#pragma unroll
        for (int kh = 0; kh < SK; kh += 4) {
            float4 ar[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                ar[i] = *reinterpret_cast<const float4*>(&As[buf][(i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4)][kh]);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kh + k][tx * 4]);
                const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kh + k][64 + tx * 4]);
                const float2 bf2[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                       make_float2(b1.z, b1.w)};
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float av = k == 0 ? ar[i].x : k == 1 ? ar[i].y : k == 2 ? ar[i].z : ar[i].w;
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc2[i][j] = __ffma2_rn(make_float2(av, av), bf2[j], acc2[i][j]);
                }
            }
        }
#else
        // 2 k per A fragment load (8-byte loads): 16 fragment registers instead
        // of 32, so the 8 x 8 accumulators, both fragments and the copy
        // pointers fit the 128-register budget of 2 CTAs per SM without spills
#pragma unroll
        for (int kh = 0; kh < SK; kh += 2) {
            float2 ar[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                ar[i] = *reinterpret_cast<const float2*>(&As[buf][(i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4)][kh]);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kh + k][tx * 4]);
                const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kh + k][64 + tx * 4]);
                const float2 bf2[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                       make_float2(b1.z, b1.w)};
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float av = k == 0 ? ar[i].x : ar[i].y;
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc2[i][j] = __ffma2_rn(make_float2(av, av), bf2[j], acc2[i][j]);
                }
            }
        }
#endif
        if (FT) {
            // carried references, ascending k, once per k-block (one branch per
            // warp); the row side reads A[p][k] from the padded rows (80-byte
            // pitch: conflict-free 16-byte reads).  Measured: a branch-free form
            // (per-thread operand pointers) was 3 % slower.
            if (tid < SB) {
#pragma unroll
                for (int k = 0; k < SK; ++k) ref = fmaf(As[buf][tid][k], brs[buf][k], ref);
            } else {
#pragma unroll
                for (int k = 0; k < SK; ++k) ref = fmaf(acs[buf][k], Bs[buf][k][tid - SB], ref);
            }
        }
        // fault injection after this k-block, warp-uniform check
        if (FT) {
            while (next_inj < ninj && sinj[next_inj].kb == kb) {
                const DevInject f = sinj[next_inj];
                if (f.target == FTGEMM_TGT_ACC) {
                    const int pi = f.p, qj = f.q;
                    const int ii = (pi & 64) ? 4 + ((pi - 64) - ty * 4) : (pi - ty * 4);
                    const int jj = (qj & 64) ? 4 + ((qj - 64) - tx * 4) : (qj - tx * 4);
                    const bool own_r = ((pi & 63) >> 2) == ty, own_c = ((qj & 63) >> 2) == tx;
                    if (own_r && own_c) {
#pragma unroll
                        for (int i = 0; i < 8; ++i)
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                if (i == ii && j == jj) ACC(i, j) = simt_fault(ACC(i, j), f);
                    }
                } else if (f.target == FTGEMM_TGT_ROW_REF) {
                    if (tid == f.p) ref = simt_fault(ref, f);
                } else {
                    if (tid == SB + f.q) ref = simt_fault(ref, f);
                }
                ++next_inj;
            }
        }
    }
    cp_async_wait<0>();
    __syncthreads();

    int kind = 0, pstar = -1, qstar = -1;
    if (FT) {
        // ---- verification ----
        if (tid == 0) { sflag[0] = 0; sflag[1] = 0; sflag[2] = 1 << 30; sflag[3] = 1 << 30; sflag[5] = 0; }
        float rs[8], cs[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float s = 0.0f;
#pragma unroll
            for (int j = 0; j < 8; ++j) s += ACC(i, j);
            rs[i] = s;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float s = 0.0f;
#pragma unroll
            for (int i = 0; i < 8; ++i) s += ACC(i, j);
            cs[j] = s;
        }
        // rows: reduce across the 16 tx of the same ty (same warp, lanes xor 1..8)
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], o);
        // cols: reduce ty pairs inside the warp (xor 16), then across 8 warps via smem
#pragma unroll
        for (int j = 0; j < 8; ++j) cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], 16);
        const int wid = tid >> 5;
        if (tx == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) srow_s[(i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4)] = rs[i];
        }
        if ((tid & 31) < 16) {
#pragma unroll
            for (int j = 0; j < 8; ++j) red_col[wid][(j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4)] = cs[j];
        }
        if (tid < SB) rref_s[tid] = ref; else cref_s[tid - SB] = ref;
        __syncthreads();
        unsigned margin = 0u;        // largest |r| / tau among unflagged residuals (telemetry)
        if (tid < SB) {
            const int p = tid;
            if (p < bm) {
                const float rr = ref;
                const float r = srow_s[p] - rr;
                const float tr = a.tau_u * (a.tau_l1 * a.sqrtK * fabsf(rr) +
                                            a.tau_l2 * __ldg(a.rownorm + r0 + p) * __ldg(a.brnorm + tj));
                rres[p] = r; rtau[p] = tr;
                if (!(fabsf(r) <= tr)) { atomicAdd(&sflag[0], 1); atomicMin(&sflag[2], p); }
                else if (tr > 0.0f) margin = __float_as_uint(fabsf(r) / tr);
            }
        } else {
            const int q = tid - SB;
            if (q < bn) {
                float sc = 0.0f;
#pragma unroll
                for (int w = 0; w < 8; ++w) sc += red_col[w][q];
                const float rc = ref;
                const float c = sc - rc;
                const float tc = a.tau_u * (a.tau_l1 * a.sqrtK * fabsf(rc) +
                                            a.tau_l2 * __ldg(a.acnorm + ti) * __ldg(a.colnorm + c0 + q));
                cres[q] = c; ctau[q] = tc;
                if (!(fabsf(c) <= tc)) { atomicAdd(&sflag[1], 1); atomicMin(&sflag[3], q); }
                else if (tc > 0.0f) margin = __float_as_uint(fabsf(c) / tc);
            }
        }
        margin = __reduce_max_sync(0xffffffffu, margin);
        if ((tid & 31) == 0 && margin) atomicMax(reinterpret_cast<unsigned*>(&sflag[5]), margin);
        __syncthreads();
        if (tid == 0 && sflag[5]) atomicMax(&a.rep->max_ratio_bits, (unsigned)sflag[5]);
        const int nr = sflag[0], nc = sflag[1];
        pstar = nr ? sflag[2] : -1;
        qstar = nc ? sflag[3] : -1;
        if (a.ft_level == FTGEMM_FT_DETECT_ROWS) {          // offline ABFT: rows only
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
        if (kind == FTGEMM_EV_CORRECTED) {
            // exclusive row sum of p*, reconstruct acc[p*, q*] = ref_row - sum_{q != q*}
            const bool own_r = ((pstar & 63) >> 2) == ty;
            const int ii = (pstar & 64) ? 4 + ((pstar - 64) - ty * 4) : (pstar - ty * 4);
            float part = 0.0f;
            if (own_r) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (i == ii) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int q = (j < 4) ? tx * 4 + j : 64 + tx * 4 + j - 4;
                            if (q != qstar) part += ACC(i, j);
                        }
                    }
            }
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            const bool own_c = ((qstar & 63) >> 2) == tx;
            const int jj = (qstar & 64) ? 4 + ((qstar - 64) - tx * 4) : (qstar - tx * 4);
            if (own_r && own_c) {
                const float val = rref_s[pstar] - part;
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (i == ii && j == jj) ACC(i, j) = val;
            }
        }
        if (tid == 0) {
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

    // ---- epilogue: C = fmaf(alpha, acc, beta * C_in) ----
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int p = (i < 4) ? ty * 4 + i : 64 + ty * 4 + i - 4;
        const int gr = r0 + p;
        if (p >= bm) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int q = h * 64 + tx * 4;
            const int gc = c0 + q;
            float* Cp = a.C + (int64_t)gr * a.ldc + gc;
            float o[4];
            if (q + 3 < bn) {
                float4 cin = make_float4(0.f, 0.f, 0.f, 0.f);
                if (a.beta != 0.0f) cin = *reinterpret_cast<const float4*>(Cp);
                const float ci[4] = {cin.x, cin.y, cin.z, cin.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) o[j] = fmaf(a.alpha, ACC(i, h * 4 + j), a.beta != 0.0f ? a.beta * ci[j] : 0.0f);
                *reinterpret_cast<float4*>(Cp) = make_float4(o[0], o[1], o[2], o[3]);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (q + j < bn) Cp[j] = fmaf(a.alpha, ACC(i, h * 4 + j), a.beta != 0.0f ? a.beta * Cp[j] : 0.0f);
            }
        }
    }
}

cudaError_t launch_simt(bool ft, const SimtArgs& a, cudaStream_t st) {
    static PerDeviceOnce attr;
    cudaError_t e = attr.run([] {
        cudaError_t r = cudaFuncSetAttribute(simt_ftgemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SIMT_DSMEM);
        if (r == cudaSuccess)
            r = cudaFuncSetAttribute(simt_ftgemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SIMT_DSMEM);
        return r;
    });
    if (e != cudaSuccess) return e;
    const int grid = a.tiles_m * a.tiles_n;
    if (ft) simt_ftgemm_kernel<true><<<grid, 256, SIMT_DSMEM, st>>>(a);
    else simt_ftgemm_kernel<false><<<grid, 256, SIMT_DSMEM, st>>>(a);
    return cudaGetLastError();
}

int simt_bk() { return SK; }

}  // namespace ftg
