// tc_gemm.cu -- fused online-ABFT GEMM on the 5th-generation tensor cores
// (tcgen05 / TMEM / TMA) for sm_100a, BF16 and TF32 operands, FP32 accumulate.
//
// The paper's threadblock-level fused ABFT (section 4.2.3,
// Fig. tb_abft) re-derived for tcgen05: instead of carrying e^T A B and A B e in
// registers next to a SIMT outer product, the encoded operands of Eq. (1)/(2)
// are fed to the tensor core as part of the MMA tiles, so the
// single tensor-core mainloop that computes C also computes the carried
// references of Eq. (3):
//
//     A tile (128 x BK, K-major)   rows 0..124  = A_i           (TMA, 125-row box)
//                                  rows 125..127 = split(e^T A_i) (bulk copy of the
//                                                 pre-swizzled encode output)
//     B tile (BK x BN, N-major)    = B^r_j = [B_j, split(B_j e), 0] materialised by
//                                    the encode kernel in BN-wide, 128-byte
//                                    aligned slots (cols 0..BN-5 = B_j)
//     D = A_tile B_tile in TMEM   = [[ C_ij , C^r_ij (3 partial cols) ],
//                                    [ C^c_ij (3 partial rows), unused ]]
//
// so the check tile is 125 x (BN-4) and verification needs no extra MMA.
// With FT off the same kernel family reads A and the row-major B directly
// (B N-major, 128 x BN data tiles).  Warp roles (one CTA per SM, persistent;
// E = 4 x epilogue warpgroups = 8 with FT, 4 without):
//   warps 0..E-1  epilogue: TMEM -> registers; row sums (thread = row), column
//                 sums (warp transpose-reduce + smem), residuals vs thresholds,
//                 locate, correct, alpha/beta, store; they
//                 also service mid-mainloop fault injections
//   warp E        TMEM allocator; in-kernel A encode (ftgemm_run_fused)
//   warp E+1      Y producer (split rows of e^T A; waits for the in-kernel
//                 encode's item flags)
//   warp E+2      TMA producer
//   warp E+3      MMA issuer (one thread: tcgen05.mma, tcgen05.commit)
// (FTGEMM_ROLES_HI=0 restores the earlier layout: producer 0, MMA 1, epilogue 4..)
// The accumulator is double-buffered in TMEM (2 x BN columns), so the epilogue
// of tile t (verification included) overlaps the mainloop of tile t+1.
#include <cstdint>
#include <cstdio>
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace ftg {

// epilogue warpgroups: 2 = one warpgroup per TMEM accumulator buffer, so the
// epilogues (verification included) of two consecutive tiles run concurrently
// (FT on); FT off keeps one and spends the staging memory on a deeper ring
#ifndef FTGEMM_ROLES_HI
#define FTGEMM_ROLES_HI 1
#endif
#ifndef FTGEMM_EPI_WG
#define FTGEMM_EPI_WG 2
#endif
#ifndef FTGEMM_MAX_STAGES
#define FTGEMM_MAX_STAGES 8    // (development: cap the smem ring depth)
#endif

// EPI_: epilogue warpgroups with FT on, one TMEM accumulator buffer each (2 by
// default; 3 for the small-K BN = 128 instantiation, where the verification
// pass bounds the kernel and a third tile in flight hides its latency)
template <bool kTF32, int BN_, bool FT, int CG_ = 1, int EPI_ = FTGEMM_EPI_WG>
struct TcCfg {
    static constexpr int CG = CG_;                 // 1: one CTA per MMA; 2: CTA pair (M = 256)
    static constexpr int BM = 128;
    static constexpr int BN = BN_;
    static constexpr int ELT = kTF32 ? 4 : 2;
    static constexpr int BK = 128 / ELT;           // one 128-byte swizzle row of K
    static constexpr int UK = 32 / ELT;            // K per tcgen05.mma
    static constexpr int BOXN = 128 / ELT;         // B columns per TMA box
    static constexpr int NBOX = BN / BOXN;
    static constexpr int A_BYTES = BM * 128;
    static constexpr int B_BOX_BYTES = BK * 128;
    static constexpr int B_BYTES = (NBOX / CG) * B_BOX_BYTES;   // this CTA's share of the B tile
    static constexpr int Y_BYTES = 384;            // 3 split rows x 128 bytes
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int EPI_WG = FT ? EPI_ : 1;
    static constexpr int NACC = EPI_WG > 2 ? EPI_WG : 2;   // TMEM accumulator buffers
    static_assert(NACC * BN_ <= 512, "accumulator buffers must fit the 512 TMEM columns");
    static constexpr int THREADS = 128 + 128 * EPI_WG;
    static constexpr int STG_BYTES = 4 * 2 * 4096;     // per epilogue warpgroup (see below)
    static constexpr int EPI_BYTES = EPI_WG * STG_BYTES;
    static constexpr int MISC_BYTES = 2048;            // barriers, TMEM address, in-kernel-encode norms
    static_assert((4 * 8 + 4 * NACC + 4 * EPI_WG) * 8 + 16 + (2 * 128 + 2) * 4 <= MISC_BYTES, "misc shared memory");
    static constexpr int STAGE_FIT = (227 * 1024 - 1024 - MISC_BYTES - EPI_BYTES) / (A_BYTES + B_BYTES);
    static constexpr int STAGES = STAGE_FIT < FTGEMM_MAX_STAGES ? STAGE_FIT : FTGEMM_MAX_STAGES;
    static constexpr int BMD = FT ? BM - 3 : BM;   // data rows of a check tile
    static constexpr int BND = FT ? BN - 4 : BN;   // data cols of a check tile
    static constexpr int TMEM_COLS = NACC * BN <= 256 ? 256 : 512;   // tcgen05.alloc: a power of two
    static constexpr int NCHUNK = BN / 32;
    // epilogue shared memory: per-warp double-buffered 32 x 128-byte SWIZZLE_128B
    // staging for the TMA stores; the verification arrays (column partial sums,
    // reference rows, residuals, thresholds) alias the staging area (pass 1 runs
    // only after the previous tile's stores have read it)
    static constexpr int VER_BYTES = (4 * BN + 3 * BN + 2 * BN + 2 * BM) * 4 + 64;
    static_assert(VER_BYTES <= 12288, "verification arrays must fit below the transpose buffers");
    static_assert(12288 + 4 * 32 * 36 * 4 <= STG_BYTES, "transpose buffers must fit in the staging area");
    static constexpr int GW = kTF32 ? 32 : 64;     // output columns per 128-byte store box
    static constexpr int NG = (BND + GW - 1) / GW; // store groups per tile
    static constexpr int LAST = BND - GW;          // start of the last group (overlaps the previous one by BND % GW)
    static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + MISC_BYTES;
};

// Tile schedule: groups of G consecutive M-tiles are swept across all N-tiles
// (M-tile fastest), so concurrently running tiles share A rows and B^r slots in
// L2.  G comes from the host (tc_group(), also used to key fault lists).
__device__ __forceinline__ void tile_coords(int t, const TcArgs& a, int& ti, int& tj) {
    const int per_group = a.group * a.tiles_n;
    const int grp = (int)a.fd_pg.div((uint32_t)t);
    const int first = grp * a.group;
    const bool full = a.units_m - first >= a.group;          // every group but a ragged last one
    const int gsz = full ? a.group : a.units_m - first;
    const int loc = t - grp * per_group;
    const int q = (int)(full ? a.fd_g.div((uint32_t)loc) : a.fd_gt.div((uint32_t)loc));
    ti = first + (loc - q * gsz);
    tj = q;
}

// first index of inj[] with tile >= t (inj sorted by tile, then kb)
__device__ __forceinline__ int inj_lower(const DevInject* inj, int n, int t) {
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (inj[mid].tile < t) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ float transpose_reduce32(float (&w)[32], uint32_t lane) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
            float send = upper ? w[i] : w[i + off];
            float keep = upper ? w[i + off] : w[i];
            w[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return w[0];
}

__device__ __forceinline__ uint32_t apply_fault(uint32_t bits, const DevInject& f) {
    if (f.mode == FTGEMM_INJ_ADD) return __float_as_uint(__uint_as_float(bits) + f.addend);
    return bits ^ (1u << (f.bit & 31));
}

#if defined(FTGEMM_EXP_FA_TRACE)
// timing experiment: globaltimer stamps into a debug buffer (ftgemm_debug_trace)
__device__ unsigned long long g_fa_trace[1 << 17];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// -DFTGEMM_DEBUG_CHECKS: device-side bounds assertions on the in-kernel encode's
// item, flag and norm indices (a stand-in for compute-sanitizer memcheck, which
// is closed on the GPU pool; tests/test_gpu_parity.py runs under such a build)
#if defined(FTGEMM_DEBUG_CHECKS)
#define FTG_CHECK(cond) do { if (!(cond)) { printf("FTG_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); __trap(); } } while (0)
#else
#define FTG_CHECK(cond) do { } while (0)
#endif

// item index (claim order) -> (check tile, k-block): the order in which the
// persistent schedule first needs them -- schedule group by schedule group,
// k-block by k-block, the group's check tiles fastest
__device__ __forceinline__ void enc_item_coords(int it, const TcArgs& a, int cg, int& ti, int& kb) {
    const int tpg = a.group * cg;
    const int per_group = tpg * a.num_kb;
    const int grp = it / per_group;
    const int first = grp * tpg;
    const int tg = min(tpg, a.tiles_m - first);
    const int rem = it - grp * per_group;
    kb = rem / tg;
    ti = first + (rem - kb * tg);
    FTG_CHECK(it >= 0 && ti >= 0 && ti < a.tiles_m && kb >= 0 && kb < a.num_kb && tg > 0);
}

// One item of the in-kernel A encode (one warp): check tile ti (125 rows of A),
// k-block kb (128 bytes of every row).  Lane = (row group rg = lane / 8, 16-byte
// chunk c = lane % 8); the lane loads rows rg, rg + 4, ..., rg + 124 -- all 32
// loads in flight at once (one memory round trip per item).
//   split rows 125..127 of the MMA A tile: the exact 3-term split of
//       e^T A_i [kb * BK .. +BK) (Eq. 1), pre-swizzled, into Y
//   frn2[ti][row][kb]: this k-block's sum of squares of every row (R1)
//   facn2[ti][kb]:     this k-block's sum of (e^T A_i)^2
// then a release flag.  Rows >= M and columns >= K are zeros, as the TMA loads.
template <bool kTF32>
__device__ __forceinline__ void encode_a_item(const TcArgs& a, const int ti, const int kb, const uint32_t lane) {
    constexpr int ELT = kTF32 ? 4 : 2, EPC = 16 / ELT, BK = 128 / ELT, BMD = 125;
    const int rg = (int)(lane >> 3), c = (int)(lane & 7);
    const int r0 = ti * BMD, bm = min(BMD, a.M - r0);
    const int k0 = kb * BK + c * EPC;
    const int64_t pitch = a.lda * ELT;
    FTG_CHECK(bm > 0 && bm <= BMD && kb < a.num_kb && a.nkb4 >= a.num_kb && (a.nkb4 & 3) == 0);
    const uint8_t* base = reinterpret_cast<const uint8_t*>(a.A) + ((int64_t)r0 * a.lda + k0) * ELT;
    const bool kfull = k0 + EPC <= a.K;
#if defined(FTGEMM_EXP_FA_TRACE)
    if (lane == 0) g_fa_trace[20480 + ti * a.num_kb + kb] = gtimer();
#endif
    uint4 v[32];
    if (kfull && rg + 4 * 31 < bm) {                     // every row present, whole chunk below K
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = ldg_stream_v4(base + (int64_t)(rg + 4 * i) * pitch);
    } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            const int r = rg + 4 * i;
            v[i] = make_uint4(0u, 0u, 0u, 0u);
            if (r < bm && k0 < a.K) {
                const uint8_t* p = base + (int64_t)r * pitch;
                if (kfull) {
                    v[i] = ldg_stream_v4(p);
                } else {
                    uint32_t wd[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                    for (int e = 0; e < EPC; ++e) {
                        if (k0 + e < a.K) {
                            if constexpr (ELT == 2) wd[e >> 1] |= (uint32_t)reinterpret_cast<const uint16_t*>(p)[e] << (16 * (e & 1));
                            else wd[e] = reinterpret_cast<const uint32_t*>(p)[e];
                        }
                    }
                    v[i] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
                }
            }
        }
    }
#if defined(FTGEMM_EXP_FA_TRACE)
    {
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) x ^= v[i].x ^ v[i].w;
        x = __reduce_xor_sync(0xffffffffu, x);
        if (lane == 0) g_fa_trace[60000 + ti * a.num_kb + kb] = gtimer() + (x == 0x12345678u);
    }
#endif
    float2 cs2[EPC / 2];
#pragma unroll
    for (int j = 0; j < EPC / 2; ++j) cs2[j] = make_float2(0.0f, 0.0f);
    float* rn2 = a.frn2 + (int64_t)ti * 128 * a.nkb4 + kb;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        float q[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const uint4 u = v[16 * b + i];
            const uint32_t wd[4] = {u.x, u.y, u.z, u.w};
            float2 q2 = make_float2(0.0f, 0.0f);
#pragma unroll
            for (int j = 0; j < EPC / 2; ++j) {
                float2 x;
                if constexpr (kTF32) x = make_float2(tf32_trunc(__uint_as_float(wd[2 * j])), tf32_trunc(__uint_as_float(wd[2 * j + 1])));
                else x = make_float2(__uint_as_float(wd[j] << 16), __uint_as_float(wd[j] & 0xFFFF0000u));
                cs2[j] = __fadd2_rn(cs2[j], x);
                q2 = __ffma2_rn(x, x, q2);
            }
            q[i] = q2.x + q2.y;
        }
        // row sums of squares across the 8 chunk lanes, transposed: the lane with
        // chunk c ends up holding rows i = 2c, 2c + 1 of this half (14 shuffles)
        float h8[8], h4[4], h2[2];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const bool up = c & 4;
            const float send = up ? q[i] : q[i + 8], keep = up ? q[i + 8] : q[i];
            h8[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const bool up = c & 2;
            const float send = up ? h8[i] : h8[i + 4], keep = up ? h8[i + 4] : h8[i];
            h4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const bool up = c & 1;
            const float send = up ? h4[i] : h4[i + 2], keep = up ? h4[i + 2] : h4[i];
            h2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) rn2[(int64_t)(rg + 4 * (16 * b + 2 * c + j)) * a.nkb4] = h2[j];
    }
    // column sums across the 4 row groups
    float cs[EPC];
#pragma unroll
    for (int j = 0; j < EPC / 2; ++j) { cs[2 * j] = cs2[j].x; cs[2 * j + 1] = cs2[j].y; }
#pragma unroll
    for (int j = 0; j < EPC; ++j) {
        cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], 8);
        cs[j] += __shfl_xor_sync(0xffffffffu, cs[j], 16);
    }
    float asq = 0.0f;
    if (rg == 0) {
        uint32_t pk[3][4];
#pragma unroll
        for (int j = 0; j < EPC; ++j) {
            const float sv = cs[j];
            asq = fmaf(sv, sv, asq);
            float hi, mid, lo;
            split3<kTF32 ? 1 : 0>(sv, hi, mid, lo);
            const float parts[3] = {hi, mid, lo};
#pragma unroll
            for (int r3 = 0; r3 < 3; ++r3) {
                if constexpr (kTF32) pk[r3][j] = __float_as_uint(parts[r3]);
                else if (j & 1) pk[r3][j >> 1] |= (uint32_t)f32_to_bf16_rn(parts[r3]) << 16;
                else pk[r3][j >> 1] = (uint32_t)f32_to_bf16_rn(parts[r3]);
            }
        }
        uint8_t* yb = reinterpret_cast<uint8_t*>(const_cast<void*>(a.Y)) + ((int64_t)ti * a.num_kb + kb) * 384;
#pragma unroll
        for (int r3 = 0; r3 < 3; ++r3) {
            const int row = BMD + r3;
            *reinterpret_cast<uint4*>(yb + r3 * 128 + ((c ^ (row & 7)) << 4)) = make_uint4(pk[r3][0], pk[r3][1], pk[r3][2], pk[r3][3]);
        }
    }
    asq += __shfl_xor_sync(0xffffffffu, asq, 1);
    asq += __shfl_xor_sync(0xffffffffu, asq, 2);
    asq += __shfl_xor_sync(0xffffffffu, asq, 4);
    if (lane == 0) a.facn2[(int64_t)ti * a.nkb4 + kb] = asq;
    // publish: every lane's writes (the Y rows are read by TMA -- the async
    // proxy -- on other SMs), then one release flag (cumulative over the
    // warp's writes ordered before it by the warp barrier)
#if defined(FTGEMM_EXP_FA_TRACE)
    __syncwarp();
    if (lane == 0) g_fa_trace[80000 + ti * a.num_kb + kb] = gtimer();
#endif
    fence_proxy_async_global();
    __syncwarp();
#if defined(FTGEMM_EXP_FA_TRACE)
    if (lane == 0) g_fa_trace[100000 + ti * a.num_kb + kb] = gtimer();
#endif
    if (lane == 0) st_release_u32(a.fflag + (int64_t)ti * a.num_kb + kb, 1u);
#if defined(FTGEMM_EXP_FA_TRACE)
    if (lane == 0) {
        g_fa_trace[4096 + ti * a.num_kb + kb] = gtimer();
    }
#endif
    __syncwarp();
}

#ifndef FTGEMM_FA_LEAD
#define FTGEMM_FA_LEAD 4           // waves of units the in-kernel A encode may run ahead of the MMA warps
#endif
// Claim the next item of the in-kernel A encode (warp-uniform result; an
// index >= the item count means every item is claimed).
__device__ __forceinline__ uint32_t enc_claim(const TcArgs& a, uint32_t lane) {
    uint32_t it = 0;
    if (lane == 0) it = atomicAdd(a.fflag + (int64_t)a.tiles_m * a.num_kb, 1u);
    return __shfl_sync(0xffffffffu, it, 0);
}

// EXT: the extended modes compiled in -- 1: the in-kernel A encode
// (ftgemm_run_fused), 2: the row-first K_s checks of the online mode -- each
// in its own instantiation (their code raised the register pressure of the
// plain path's epilogue into spills)
template <bool kTF32, int BN, bool FT, int CG, int EPI, int EXT>
__global__ void __launch_bounds__(TcCfg<kTF32, BN, FT, CG, EPI>::THREADS, 1)
tc_ftgemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC29,
                 const __grid_constant__ CUtensorMap tmY, const TcArgs a) {
    using Cfg = TcCfg<kTF32, BN, FT, CG, EPI>;
    constexpr int S = Cfg::STAGES;
    constexpr int NACC = Cfg::NACC;
    constexpr int kEpiWG = Cfg::EPI_WG;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte aligned base (SWIZZLE_128B atoms); pointer arithmetic on the
    // __shared__ array keeps the shared address space visible to the compiler
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* stage_base = smem;
    uint8_t* const stg0 = smem + S * Cfg::STAGE_BYTES;                        // [kEpiWG][4][2][4096] (1024-aligned)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES + Cfg::EPI_BYTES);
    uint64_t* full = bars;              // [S]  stage landed (TMA + bulk bytes)
    uint64_t* empty = bars + S;         // [S]  producer may refill
    uint64_t* tm_full = bars + 2 * S;   // [NACC]  accumulator complete
    uint64_t* tm_empty = tm_full + NACC;   // [NACC]
    uint64_t* inj_req = tm_empty + NACC;   // [NACC]  mid-mainloop hand-off, per accumulator buffer
    uint64_t* inj_done = inj_req + NACC;   // [NACC]
    uint64_t* cbar = inj_done + NACC;   // [4 kEpiWG]  C_in tile loads (beta != 0), one per epilogue warp
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(cbar + 4 * kEpiWG);
    // row-first K_s checks (online mode): per epilogue warpgroup two slots of
    // {row flagged, max |r|/tau}, alternating between consecutive checks
    int* rf_slots = reinterpret_cast<int*>(tmem_holder + 4);                // [kEpiWG][2][2]

    const int warp = threadIdx.x >> 5;
    // Warp roles.  The SM sub-partition scheduler favours the highest warp id
    // among eligible warps, and the single MMA-issuing thread is latency
    // critical, so the control warps take the highest ids (MMA issuer = the last
    // warp, TMA producer = the one before) and the epilogue warps (whose TMEM
    // lane quadrant is warp % 4) the lowest.
    constexpr int kEpiWarps = 4 * kEpiWG;
#if FTGEMM_ROLES_HI
    constexpr int W_EPI0 = 0, W_ALLOC = kEpiWarps, W_ENC0 = kEpiWarps, W_PROD = kEpiWarps + 2, W_MMA = kEpiWarps + 3;
#else
    constexpr int W_PROD = 0, W_MMA = 1, W_ALLOC = 2, W_ENC0 = 2, W_EPI0 = 4;
#endif
    const uint32_t lane = lane_id();
    // CTA pair: rank 0 is the MMA leader; each CTA owns 128 of the 256 MMA rows
    // (one check tile) and half of the B tile's columns
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    const bool leader = rank == 0;
    const int cluster_id = blockIdx.x / CG, num_clusters = gridDim.x / CG;

#if defined(FTGEMM_EXP_FA_TRACE)
    if (threadIdx.x == 0) g_fa_trace[40000 + blockIdx.x] = gtimer();
#endif
    if (warp == W_PROD && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmC);
        tma_prefetch_desc(&tmC29);
        if constexpr (FT) tma_prefetch_desc(&tmY);
        // FT with the Y-producer warp: the TMA producer and the Y producer arrive
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], (FT && a.y_warp) ? 2 : 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < NACC; ++b) {
            mbar_init(&tm_full[b], 1);
            mbar_init(&tm_empty[b], 4 * CG);     // every epilogue warp of the pair
            mbar_init(&inj_req[b], 1);
            mbar_init(&inj_done[b], CG);
        }
        for (int w = 0; w < 4 * kEpiWG; ++w) mbar_init(&cbar[w], 1);
        for (int i = 0; i < 4 * kEpiWG; ++i) rf_slots[i] = 0;
        fence_barrier_init();
    }
    if (warp == W_ALLOC) tmem_alloc<Cfg::TMEM_COLS, CG>(tmem_holder);
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    griddep_wait();                     // the encode (or any earlier kernel) has completed
    const uint32_t tmem_base = *tmem_holder;

    if (warp == W_PROD) {
        // ------------------------------------------------ TMA producer ----
        if (lane == 0) {
            int s = 0; uint32_t ph = 0;
            // FT: A box of 125 data rows + the 384-byte pre-swizzled split rows into
            // rows 125..127 (TMA, no swizzle); B^r.  FT off: 128-row A box and the
            // row-major B.  B is N-major in BOXN-column boxes; with a CTA pair each
            // CTA loads half of the tile's columns.  All bytes of a stage (both CTAs)
            // are counted on the leader's full barrier.
            const bool b3d = a.b3d != 0;                 // B tile in one 3-D TMA request
            // (FT: the split rows of e^T A come from the Y-producer warp, which
            // arrives on the same full barrier with their bytes)
            const bool yself = FT && !a.y_warp;          // short K: this thread loads them too
            const uint32_t bytes_cta = !FT ? (Cfg::A_BYTES + Cfg::B_BYTES)
                                     : (Cfg::BMD * 128 + Cfg::B_BYTES + (yself ? Cfg::Y_BYTES : 0));
            for (int u = cluster_id; u < a.num_units; u += num_clusters) {
                // batched launches: unit u = problem bb's unit ul (problems back to back)
                const int bb = (int)a.fd_upb.div((uint32_t)u), ul = u - bb * a.units_pb;
                int tmu, tj;
                tile_coords(ul, a, tmu, tj);
                const int ti = tmu * CG + (int)rank;
                const int row0 = ti * Cfg::BMD;
                const int colb = tj * BN + (int)rank * (BN / CG);
                for (int kb = 0; kb < a.num_kb; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[s], CG * bytes_cta);
                    uint8_t* sa = stage_base + s * Cfg::STAGE_BYTES;
                    uint8_t* sb = sa + Cfg::A_BYTES;
                    if constexpr (CG == 1) {
                        tma_load_3d(sa, &tmA, &full[s], kb * Cfg::BK, row0, bb);
                        if (yself) tma_load_3d(sa + Cfg::BMD * 128, &tmY, &full[s], 0, ti * a.num_kb + kb, bb);
                        if (b3d) {
                            tma_load_4d(sb, &tmB, &full[s], 0, kb * Cfg::BK, colb / Cfg::BOXN, bb);
                        } else {
#pragma unroll
                            for (int b = 0; b < Cfg::NBOX; ++b)
                                tma_load_3d(sb + b * Cfg::B_BOX_BYTES, &tmB, &full[s], colb + b * Cfg::BOXN, kb * Cfg::BK, bb);
                        }
                    } else {
                        const uint32_t mb = smem_u32(&full[s]) & kPeerBitMask;
                        tma_load_3d_pair(sa, &tmA, mb, kb * Cfg::BK, row0, bb);
                        if (yself) tma_load_3d_pair(sa + Cfg::BMD * 128, &tmY, mb, 0, ti * a.num_kb + kb, bb);
                        if (b3d) {
                            tma_load_4d_pair(sb, &tmB, mb, 0, kb * Cfg::BK, colb / Cfg::BOXN, bb);
                        } else {
#pragma unroll
                            for (int b = 0; b < Cfg::NBOX / CG; ++b)
                                tma_load_3d_pair(sb + b * Cfg::B_BOX_BYTES, &tmB, mb, colb + b * Cfg::BOXN, kb * Cfg::BK, bb);
                        }
                    }
                    if (++s == S) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == W_MMA) {
        // ------------------------------------------------- MMA issuer -----
        if (lane == 0 && leader) {
            constexpr uint32_t idesc = instr_desc(kTF32, Cfg::BM * CG, BN, false, true);
            constexpr uint16_t pair = (1u << CG) - 1;
            auto commit = [&](uint64_t* bar) {
                if constexpr (CG == 2) umma_commit_pair(bar, pair); else umma_commit(bar);
            };
            int s = 0; uint32_t ph = 0;
            uint32_t injph = 0;                         // hand-off phase bit per accumulator buffer
            const int ks_kb = a.ks_kb, nkb = a.num_kb;
            int lt = 0;
            for (int t = cluster_id; t < a.num_units; t += num_clusters, ++lt) {
                const int acc = lt % NACC;
                const uint32_t accph = (uint32_t)(lt / NACC) & 1u;
                mbar_wait(&tm_empty[acc], accph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                int ii = 0, ie = 0;
                if (FT && a.n_inj > 0) {
                    ii = inj_lower(a.inj, a.n_inj, t);
                    ie = inj_lower(a.inj, a.n_inj, t + 1);
                }
                // next k-block that needs a mid-mainloop hand-off (a fault, or the
                // end of a K_s step); the hot loop tests only kb == evt -- the MMA
                // issue loop is latency-critical (measured: per-k-block flag and
                // modulo tests here cost 9 % of the tensor pipe at 8192^3)
                auto next_event = [&](int after) -> int {
                    int e = ii < ie ? a.inj[ii].kb : 0x7fffffff;
                    if (ks_kb > 0) {
                        const int c = ((after + 1) / ks_kb + 1) * ks_kb - 1;
                        if (c < nkb - 1 && c < e) e = c;
                    }
                    return e;
                };
                int evt = FT ? next_event(-1) : 0x7fffffff;
                // in-kernel encode: publish the schedule's progress (the encoder
                // warps stay a few waves ahead of it, not a whole operand: running
                // ahead through A evicted the GEMM's L2 working set)
                if constexpr (FT && EXT == 1) {
                    if (a.fuse_a) atomicMax(a.fflag + (int64_t)a.tiles_m * nkb + 1, (uint32_t)t);
                }
#if defined(FTGEMM_EXP_FA_TRACE)
                if (t < 2048) g_fa_trace[2 * t] = gtimer();
#endif
                // one k-block: wait for the stage, issue its MMAs, release the stage
                auto kblock = [&](int kb) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(stage_base + s * Cfg::STAGE_BYTES);
                    const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < Cfg::BK / Cfg::UK; ++kk) {
                        const uint64_t ad = smem_desc_sw128(sa + kk * 32, 16, 1024);
                        // B is N-major: bf16 -> SW128 (8-row atoms), tf32 -> SW128_BASE32B (4-row atoms)
                        const uint64_t bd = kTF32 ? smem_desc_sw128<1>(sb + kk * Cfg::UK * 128, Cfg::B_BOX_BYTES, 512)
                                                  : smem_desc_sw128<2>(sb + kk * Cfg::UK * 128, Cfg::B_BOX_BYTES, 1024);
                        umma<kTF32, CG>(d, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
                    }
                    commit(&empty[s]);
                    if (++s == S) { s = 0; ph ^= 1; }
                };
                // hand the accumulator to the epilogue warps (of both CTAs) for the
                // fault(s) of k-block kb and / or the check closing a K_s step
                auto handoff = [&](int kb) {
                    commit(&inj_req[acc]);
                    mbar_wait(&inj_done[acc], (injph >> acc) & 1u);
                    injph ^= 1u << acc;
                    tc_fence_after();
                    while (ii < ie && a.inj[ii].kb == kb) ++ii;
                    evt = next_event(kb);
                };
                {
                    // lean runs of k-blocks between hand-offs: no per-k-block tests in
                    // the issue loop (a tile with a fault pays only its hand-offs)
                    int kb = 0;
                    for (;;) {
                        const int end = evt < nkb ? evt + 1 : nkb;
                        for (; kb < end; ++kb) kblock(kb);
                        if (kb >= nkb && !(evt < nkb)) break;
                        handoff(kb - 1);
                        if (kb >= nkb) break;
                    }
                }
                commit(&tm_full[acc]);
#if defined(FTGEMM_EXP_FA_TRACE)
                if (t < 2048) g_fa_trace[2 * t + 1] = gtimer();
#endif
            }
        }
        __syncwarp();
    } else if (warp == W_ENC0 || warp == W_ENC0 + 1) {
        if (FT && a.y_warp && warp == W_ENC0 + 1) {
            // ---------------------------------------------- Y producer -------
            // The 384-byte split rows of e^T A (rows 125..127 of every stage's A
            // tile) from their own warp: a third TMA per stage on the main
            // producer thread made its issue rate the limiter (BF16 8192^3 FT run
            // -2.8 %).  Short K (<= 4 k-blocks, separate encode): the producer
            // loads them itself.  With the in-kernel encode (a.fuse_a) the warp
            // first waits for the item flags of the k-blocks it loads (32 flags
            // per poll, one L2 round trip per 32 k-blocks).
            int s = 0; uint32_t ph = 0;
            for (int u = cluster_id; u < a.num_units; u += num_clusters) {
                const int bb = (int)a.fd_upb.div((uint32_t)u), ul = u - bb * a.units_pb;
                int tmu, tj;
                tile_coords(ul, a, tmu, tj);
                const int ti = tmu * CG + (int)rank;
#if defined(FTGEMM_EXP_FA_NOWAIT) || defined(FTGEMM_EXP_FA_NOENC)
                int ready = a.num_kb;                                      // timing experiment: no waits
#else
                int ready = (EXT == 1 && a.fuse_a && ti < a.tiles_m) ? 0 : a.num_kb;   // k-blocks known published
#endif
                for (int kb = 0; kb < a.num_kb; ++kb) {
                    if (kb >= ready) {
                        const uint32_t* fl = a.fflag + (int64_t)ti * a.num_kb;
                        FTG_CHECK(ti >= 0 && ti < a.tiles_m && kb < a.num_kb);
                        for (;;) {
                            const int k = kb + (int)lane;
                            const bool ok = k >= a.num_kb || ld_acquire_u32(fl + k) != 0u;
                            const uint32_t bad = __ballot_sync(0xffffffffu, !ok);
                            const int n = bad ? __ffs(bad) - 1 : 32;
                            if (n > 0) { ready = kb + n; break; }
                            __nanosleep(400);
                        }
                        __syncwarp();
                        fence_proxy_async_global();      // the TMA below reads what the flags published
                    }
                    if (lane == 0) {
                        mbar_wait(&empty[s], ph ^ 1);
                        if (leader) mbar_arrive_expect_tx(&full[s], CG * Cfg::Y_BYTES);
                        uint8_t* sy = stage_base + s * Cfg::STAGE_BYTES + Cfg::BMD * 128;
                        if constexpr (CG == 1) {
                            tma_load_3d(sy, &tmY, &full[s], 0, ti * a.num_kb + kb, bb);
                        } else {
                            tma_load_3d_pair(sy, &tmY, smem_u32(&full[s]) & kPeerBitMask, 0, ti * a.num_kb + kb, bb);
                        }
                    }
                    __syncwarp();
                    if (++s == S) { s = 0; ph ^= 1; }
                }
            }
        } else if (FT && EXT == 1 && a.fuse_a && warp == W_ENC0) {
            // ------------------------------------- in-kernel encode of A -------
            // (the paper fuses the checksum encoding into the
            // prefetch stage.)  Items (check tile, k-block) are
            // claimed from one counter, in the order the persistent schedule
            // first needs them, by this warp of every CTA (and by the epilogue
            // warps while their first accumulator is not ready); each is
            // computed once (not once per tile column) from global memory, off
            // the tensor core's shared-memory path, and published with a
            // release flag.
#if defined(FTGEMM_EXP_FA_NOENC)
            const uint32_t total = 0;
#else
            const uint32_t total = (uint32_t)(a.tiles_m * a.num_kb);
#endif
            for (uint32_t it = enc_claim(a, lane); it < total; it = enc_claim(a, lane)) {
                int ti, kb;
                enc_item_coords((int)it, a, CG, ti, kb);
                // the item's schedule group starts at unit first_unit: wait until the
                // MMA warps are within FTGEMM_FA_LEAD waves of it
                const uint32_t first_unit = (uint32_t)((ti / (a.group * CG)) * a.group * a.tiles_n);
                const uint32_t lead = (uint32_t)(FTGEMM_FA_LEAD * num_clusters);
                if (first_unit > lead) {
                    const uint32_t* prog = a.fflag + (int64_t)a.tiles_m * a.num_kb + 1;
                    for (;;) {
                        uint32_t p = lane == 0 ? ld_relaxed_u32(prog) : 0u;
                        if (__shfl_sync(0xffffffffu, p, 0) + lead >= first_unit) break;
                        __nanosleep(2000);
                    }
                }
                encode_a_item<kTF32>(a, ti, kb, lane);
            }
        }
    } else if (warp >= W_EPI0 && warp < W_EPI0 + kEpiWarps) {
        // ----------------------------------------------------- epilogue -----
        const int wg = (warp - W_EPI0) >> 2;          // epilogue warpgroup (owns accumulator buffer wg when kEpiWG > 1)
        const int ew = (warp - W_EPI0) & 3;           // TMEM lane quadrant
        const int rloc = ew * 32 + (int)lane;    // row of the 128-row tile
        const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
        const int et = threadIdx.x - 32 * W_EPI0 - 128 * wg;   // 0..127
        const uint32_t ebar = 1 + wg;            // named barrier of this warpgroup
        uint32_t injph = 0, cph = 0, gcount = 0;   // injph: hand-off phase bit per buffer; gcount: store groups of this warp
        uint64_t* cbw = &cbar[4 * wg + ew];
        uint8_t* stg = stg0 + wg * Cfg::STG_BYTES;
        float* colsum = reinterpret_cast<float*>(stg);                            // [4][BN] (aliases staging)
        float* refrow = colsum + 4 * BN;                          // [3][BN] split rows of C^c
        float* cres = refrow + 3 * BN;                            // [BN]
        float* ctau = cres + BN;                                  // [BN]
        float* rres = ctau + BN;                                  // [BM]
        float* rtau = rres + Cfg::BM;                             // [BM]
        int* sflag = reinterpret_cast<int*>(rtau + Cfg::BM);      // nr, nc, p*, q*, corr

        unsigned long long n_checked = 0;
        int lt = 0;
        bool enc_help = true;                    // in-kernel encode: epilogue warps help on their first tile
        uint32_t rf_parity = 0;                  // row-first check slots (online mode)
        // arrival on a barrier of the MMA leader (remote for the peer CTA)
        auto arrive_leader = [&](uint64_t* bar) {
            if (CG == 1 || leader) mbar_arrive(bar);
            else mbar_arrive_cluster(mapa_shared(smem_u32(bar), 0));
        };
        for (int t = cluster_id; t < a.num_units; t += num_clusters, ++lt) {
            const int bb = (int)a.fd_upb.div((uint32_t)t);     // problem of a batched launch
            int tmu, tj;
            tile_coords(t - bb * a.units_pb, a, tmu, tj);
            const int ti = tmu * CG + (int)rank;
            const int r0 = ti * Cfg::BMD, c0 = tj * Cfg::BND;
            const bool has_rows = r0 < a.M;                    // the pair's second tile may lie beyond M
            const int bm = min(Cfg::BMD, a.M - r0), bn = min(Cfg::BND, a.N - c0);
            constexpr int doff = 0;                            // data col q <-> MMA col q
            constexpr int xoff = BN - 4;                       // row-reference split columns
            const int acc = lt % NACC;
            if (kEpiWG > 1 && acc != wg) continue;             // another warpgroup's tile
            const uint32_t accph = (uint32_t)(lt / NACC) & 1u;
            const uint32_t tb = tmem_base + acc * BN;
            // norms for this tile's thresholds, fetched before the accumulator is ready
            float nrow = 0.f, nbr = 0.f, nac = 0.f, ncol[2] = {0.f, 0.f};
            if (FT && has_rows) {
                const int64_t eo = (int64_t)bb * a.enc_bs;     // this problem's encode (floats)
                if (!a.fuse_a) {
                    if (rloc < bm) nrow = __ldg(a.rownorm + eo + r0 + rloc);
                    nac = __ldg(a.acnorm + eo + ti);
                }
                nbr = __ldg(a.brnorm + eo + tj);
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if (et + 128 * h < bn) ncol[h] = __ldg(a.colnorm + eo + c0 + et + 128 * h);
            }

            // Verification of the accumulator in TMEM:
            // row sums, column sums, residuals against the carried references,
            // threshold (sqrtk = sqrt of the K accumulated so far), decision and
            // the corrected value (applied by the caller).  Called once at the
            // end of K, and after every K_s step in online-interval mode.
            auto verify = [&](float sqrtk, int kchk, int& kind, int& pstar, int& qstar, float& corr, bool rows_first) {
                kind = 0; pstar = -1; qstar = -1; corr = 0.0f;
#if !defined(FTGEMM_EXP_ONLINE_FULL)
                if constexpr (EXT == 2) if (rows_first) {
                    // Row checks first (the K_s checks of the online mode, DESIGN.md
                    // R20): any corrupted element of C moves its row sum, so when
                    // every row matches its reference the tile is clean for C and
                    // the column pass (the shared-memory transposes, most of the
                    // verification time) is skipped; a flagged row runs the full
                    // row + column verification below.  The flags live in their own
                    // slots (not the staging area: no wait for earlier stores), two
                    // per warpgroup used alternately, so one barrier per check
                    // suffices: the slot of the next check is cleared here, before
                    // the hand-off's barrier that precedes that check.
                    int* rf = rf_slots + 4 * wg + 2 * (rf_parity & 1);
                    int* rf_next = rf_slots + 4 * wg + 2 * ((rf_parity + 1) & 1);
                    ++rf_parity;
                    float2 rs2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
                    float rr = 0.0f;
#pragma unroll
                    for (int c = 0; c < Cfg::NCHUNK; ++c) {
                        float v[32];
                        tmem_ld32(tb + lane_off + c * 32, v);
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (c * 32 + 2 * i < Cfg::BND)
                                rs2[i & 1] = __fadd2_rn(rs2[i & 1], make_float2(v[2 * i], v[2 * i + 1]));
                        if (c + 1 == Cfg::NCHUNK) rr = (v[28] + v[29]) + v[30];
                    }
                    const float sr = (rs2[0].x + rs2[0].y) + (rs2[1].x + rs2[1].y);
                    unsigned margin = 0u;
                    if (rloc < bm) {
                        const float r = sr - rr;
                        const float tr = a.tau_u * (a.tau_l1 * sqrtk * fabsf(rr) + a.tau_l2 * nrow * nbr);
                        if (!(fabsf(r) <= tr)) rf[0] = 1;
                        else if (tr > 0.0f) margin = __float_as_uint(fabsf(r) / tr);
                    }
                    margin = __reduce_max_sync(0xffffffffu, margin);
                    if (lane == 0 && margin) atomicMax(reinterpret_cast<unsigned*>(&rf[1]), margin);
                    named_bar_sync(ebar, 128);
                    const bool any = rf[0] != 0;
                    if (et == 0) {
                        rf_next[0] = 0; rf_next[1] = 0;
                        if (!any) {
                            ++n_checked;
                            if (rf[1]) atomicMax(&a.rep->max_ratio_bits, (unsigned)rf[1]);
                        }
                    }
                    if (!any) return;
                }
#endif
                // ---- pass 1: row sums, row refs, column partial sums ----
                // previous tile's stores have read the staging area (aliased below) and
                // every reader of sflag / residual arrays is done
                if (lane == 0) bulk_wait_read0();
                named_bar_sync(ebar, 128);
                if (et == 0) { sflag[0] = 0; sflag[1] = 0; sflag[2] = 1 << 30; sflag[3] = 1 << 30; sflag[5] = 0; }
                const bool rvalid = rloc < bm;
                const bool isref = rloc >= Cfg::BMD;      // lanes 29..31 of warp 3: split rows of e^T A B
                const bool all_rows = ew < 3 && bm >= (ew + 1) * 32;   // warp-uniform: no row of this warp masked
                float* tbuf = reinterpret_cast<float*>(stg + 12288) + ew * (32 * 36);   // 32 x 36 transpose buffer
                float srow = 0.0f, rref = 0.0f;
                {
                    // 64 columns per TMEM load; row sums in 2 independent chains of
                    // paired FP32 adds (FADD2; BND is even, so no pair straddles the
                    // data / reference boundary)
                    float2 rs2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
                    const bool w3 = ew == 3;
                    const bool rows_only = a.ft_level == FTGEMM_FT_DETECT_ROWS;   // offline ABFT: no column sums
                    if constexpr (CG == 1 && kEpiWG <= 2) {
                    // (one CTA per MMA: the small-K classes, where the epilogue bounds the
                    // kernel; measured -3 % at 16384^2 x 128.  The CTA-pair instantiation
                    // keeps the single-buffer form below: the extra live registers spill
                    // there and cost 0.9 % at 8192^3.)
                    // 32-column chunks, double-buffered: the TMEM load of chunk
                    // c+1 is in flight while chunk c is summed and transposed
                    uint32_t rb[2][32];
                    __syncwarp();
                    tmem_ld32_issue(tb + lane_off, rb[0]);
                    tmem_ld32_wait(rb[0]);
#pragma unroll
                    for (int c = 0; c < Cfg::NCHUNK; ++c) {
                        uint32_t (&cur)[32] = rb[c & 1];
                        if (c + 1 < Cfg::NCHUNK) {
                            __syncwarp();
                            tmem_ld32_issue(tb + lane_off + (c + 1) * 32, rb[(c + 1) & 1]);
                        }
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (c * 32 + 2 * i < Cfg::BND)
                                rs2[i & 1] = __fadd2_rn(rs2[i & 1], make_float2(__uint_as_float(cur[2 * i]),
                                                                                __uint_as_float(cur[2 * i + 1])));
                        if (c + 1 == Cfg::NCHUNK)
                            rref = (__uint_as_float(cur[28]) + __uint_as_float(cur[29])) + __uint_as_float(cur[30]);
                        if (!rows_only) {
                            // column partial sums over this warp's 32 rows: transpose
                            // through shared memory (row-major writes, 16-byte column
                            // reads).  Warp 3's lanes 29..31 are the split rows of
                            // e^T A B: they pass through the transpose unmasked and
                            // come out as the column references.
                            if (all_rows) {
#pragma unroll
                                for (int i = 0; i < 32; ++i) tbuf[i * 36 + lane] = __uint_as_float(cur[i]);
                            } else {
#pragma unroll
                                for (int i = 0; i < 32; ++i)
                                    tbuf[i * 36 + lane] = (rvalid || isref) ? __uint_as_float(cur[i]) : 0.0f;
                            }
                            __syncwarp();
                            float2 s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
#pragma unroll
                            for (int r4 = 0; r4 < 7; ++r4) {
                                const float4 x = *reinterpret_cast<const float4*>(tbuf + lane * 36 + 4 * r4);
                                s01 = __fadd2_rn(s01, make_float2(x.x, x.y));
                                s23 = __fadd2_rn(s23, make_float2(x.z, x.w));
                            }
                            const float4 x = *reinterpret_cast<const float4*>(tbuf + lane * 36 + 28);
                            if (w3) {
                                s01.x += x.x;
                                refrow[0 * BN + c * 32 + lane] = x.y;
                                refrow[1 * BN + c * 32 + lane] = x.z;
                                refrow[2 * BN + c * 32 + lane] = x.w;
                            } else {
                                s01 = __fadd2_rn(s01, make_float2(x.x, x.y));
                                s23 = __fadd2_rn(s23, make_float2(x.z, x.w));
                            }
                            colsum[ew * BN + c * 32 + lane] = (s01.x + s01.y) + (s23.x + s23.y);
                            __syncwarp();
                        }
                        if (c + 1 < Cfg::NCHUNK) tmem_ld32_wait(rb[(c + 1) & 1]);
                    }
                    } else {
#pragma unroll
                    for (int c2 = 0; c2 < Cfg::NCHUNK; c2 += 2) {
                        float v[64];
                        tmem_ld64(tb + lane_off + c2 * 32, v);
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (c2 * 32 + 2 * i < Cfg::BND)
                                rs2[i & 1] = __fadd2_rn(rs2[i & 1], make_float2(v[2 * i], v[2 * i + 1]));
                        if (c2 + 2 == Cfg::NCHUNK) rref = (v[60] + v[61]) + v[62];
#pragma unroll
                        for (int h = 0; h < 2 && !rows_only; ++h) {
                            const int c = c2 + h;
                            // column partial sums over this warp's 32 rows: transpose
                            // through shared memory (row-major writes, 16-byte column
                            // reads).  Warp 3's lanes 29..31 are the split rows of
                            // e^T A B: they pass through the transpose unmasked and
                            // come out as the column references.
                            if (all_rows) {
#pragma unroll
                                for (int i = 0; i < 32; ++i) tbuf[i * 36 + lane] = v[32 * h + i];
                            } else {
#pragma unroll
                                for (int i = 0; i < 32; ++i) tbuf[i * 36 + lane] = (rvalid || isref) ? v[32 * h + i] : 0.0f;
                            }
                            __syncwarp();
                            float2 s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
#pragma unroll
                            for (int r4 = 0; r4 < 7; ++r4) {
                                const float4 x = *reinterpret_cast<const float4*>(tbuf + lane * 36 + 4 * r4);
                                s01 = __fadd2_rn(s01, make_float2(x.x, x.y));
                                s23 = __fadd2_rn(s23, make_float2(x.z, x.w));
                            }
                            const float4 x = *reinterpret_cast<const float4*>(tbuf + lane * 36 + 28);
                            if (w3) {
                                s01.x += x.x;
                                refrow[0 * BN + c * 32 + lane] = x.y;
                                refrow[1 * BN + c * 32 + lane] = x.z;
                                refrow[2 * BN + c * 32 + lane] = x.w;
                            } else {
                                s01 = __fadd2_rn(s01, make_float2(x.x, x.y));
                                s23 = __fadd2_rn(s23, make_float2(x.z, x.w));
                            }
                            colsum[ew * BN + c * 32 + lane] = (s01.x + s01.y) + (s23.x + s23.y);
                            __syncwarp();
                        }
                    }
                    }
                    srow = (rs2[0].x + rs2[0].y) + (rs2[1].x + rs2[1].y);
                }
                named_bar_sync(ebar, 128);
                // ---- row residuals ----
                // (threshold margin telemetry: the largest |r| / tau among the
                // unflagged residuals, one shared atomic per warp)
                unsigned margin = 0u;
                if (rvalid) {
                    const float r = srow - rref;
                    const float tr = a.tau_u * (a.tau_l1 * sqrtk * fabsf(rref) + a.tau_l2 * nrow * nbr);
                    rres[rloc] = r; rtau[rloc] = tr;
                    if (!(fabsf(r) <= tr)) { atomicAdd(&sflag[0], 1); atomicMin(&sflag[2], rloc); }
                    else if (tr > 0.0f) margin = __float_as_uint(fabsf(r) / tr);
                }
                // ---- column residuals ----
#pragma unroll
                for (int h = 0; h < 2 && a.ft_level != FTGEMM_FT_DETECT_ROWS; ++h) {
                    const int col = et + 128 * h;
                    if (col < bn && col < BN) {
                        const float sc = (colsum[col] + colsum[BN + col]) + (colsum[2 * BN + col] + colsum[3 * BN + col]);
                        const float rc = (refrow[col] + refrow[BN + col]) + refrow[2 * BN + col];
                        const float c = sc - rc;
                        const float tc = a.tau_u * (a.tau_l1 * sqrtk * fabsf(rc) + a.tau_l2 * nac * ncol[h]);
                        cres[col] = c; ctau[col] = tc;
                        if (!(fabsf(c) <= tc)) { atomicAdd(&sflag[1], 1); atomicMin(&sflag[3], col); }
                        else if (tc > 0.0f) margin = max(margin, __float_as_uint(fabsf(c) / tc));
                    }
                }
                margin = __reduce_max_sync(0xffffffffu, margin);
                if (lane == 0 && margin) atomicMax(reinterpret_cast<unsigned*>(&sflag[5]), margin);
                named_bar_sync(ebar, 128);
                // ---- decide (R3-R5) ----
                const int nr = sflag[0], nc = sflag[1];
                pstar = nr ? sflag[2] : -1;
                qstar = nc ? sflag[3] : -1;
                if (a.ft_level == FTGEMM_FT_DETECT_ROWS) {       // offline ABFT: rows only
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
                    // reconstruct from the row checksum, excluding the bad element
                    if ((pstar >> 5) == ew) {
                        float sx = 0.0f;
#pragma unroll 1
                        for (int c = 0; c < Cfg::NCHUNK; ++c) {
                            float v[32];
                            tmem_ld32(tb + lane_off + c * 32, v);
#pragma unroll
                            for (int i = 0; i < 32; ++i) {
                                const int mcol = c * 32 + i;
                                if (mcol >= doff && mcol < doff + Cfg::BND && mcol != qstar + doff) sx += v[i];
                            }
                        }
                        if (rloc == pstar) sflag[4] = __float_as_int(rref - sx);
                    }
                    named_bar_sync(ebar, 128);
                    corr = __int_as_float(sflag[4]);
                }
                if (et == 0) {
                    ++n_checked;
                    if (sflag[5]) atomicMax(&a.rep->max_ratio_bits, (unsigned)sflag[5]);
                    if (kind) {
                        unsigned long long* cnt = a.rep->counts;
                        atomicAdd(&cnt[CNT_DETECTED], 1ull);
                        const int ci = kind == FTGEMM_EV_CORRECTED ? CNT_CORRECTED
                                     : kind == FTGEMM_EV_CHECKSUM_ONLY ? CNT_CHECKSUM_ONLY
                                     : kind == FTGEMM_EV_LOCATED ? CNT_LOCATED
                                     : kind == FTGEMM_EV_DETECTED ? -1 : CNT_UNCORRECTABLE;
                        if (ci >= 0) atomicAdd(&cnt[ci], 1ull);
                        const unsigned long long slot = atomicAdd(&cnt[CNT_EVENTS], 1ull);
                        if (slot < (unsigned long long)kMaxEvents) {
                            ftgemm_event_t& e = a.rep->events[slot];
                            // batched: rows / tile rows of the stacked (batch x M) x N view
                            e.row = pstar >= 0 ? (int64_t)bb * a.M + r0 + pstar : -1;
                            e.col = qstar >= 0 ? (int64_t)(c0 + qstar) : -1;
                            e.tile_m = bb * a.tiles_m + ti; e.tile_n = tj; e.kind = kind;
                            e.n_rows = nr; e.n_cols = kind == FTGEMM_EV_DETECTED ? 0 : nc; e.k_checked = kchk;
                            e.resid_row = pstar >= 0 ? rres[pstar] : 0.0f;
                            e.resid_col = qstar >= 0 ? cres[qstar] : 0.0f;
                            e.tau_row = pstar >= 0 ? rtau[pstar] : 0.0f;
                            e.tau_col = qstar >= 0 ? ctau[qstar] : 0.0f;
                        } else {
                            atomicAdd(&cnt[CNT_DROPPED], 1ull);
                        }
                    }
                }
                // the verification arrays alias the staging buffers that pass 2 writes
                named_bar_sync(ebar, 128);
            };

            // ---- in-kernel encode of A: while this warpgroup's first
            // accumulator is not ready (the first wave, whose tiles need the
            // items first), its warps claim items too -- unless the tile has a
            // mid-mainloop hand-off to service.  (Helping on every tile was
            // measured 7 % slower: an item in flight delays the epilogue.) ----
            if constexpr (FT && EXT == 1) {
                if (a.fuse_a && enc_help) {
                    enc_help = false;
                    const bool handoffs = a.n_inj > 0 && inj_lower(a.inj, a.n_inj, t) != inj_lower(a.inj, a.n_inj, t + 1);
#if defined(FTGEMM_EXP_FA_NOHELP) || defined(FTGEMM_EXP_FA_NOENC)
                    if (false) {
#else
                    if (!handoffs) {
#endif
                        const uint32_t total = (uint32_t)(a.tiles_m * a.num_kb);
                        for (;;) {
                            uint32_t ready = lane == 0 ? (uint32_t)mbar_test_wait(&tm_full[acc], accph) : 0u;
                            if (__shfl_sync(0xffffffffu, ready, 0)) break;
                            // only items of the first schedule group (needed now)
                            uint32_t nxt = lane == 0 ? ld_relaxed_u32(a.fflag + (int64_t)a.tiles_m * a.num_kb) : 0u;
                            nxt = __shfl_sync(0xffffffffu, nxt, 0);
                            if (nxt >= (uint32_t)(min(a.group * CG, a.tiles_m) * a.num_kb)) break;
                            const uint32_t it = enc_claim(a, lane);
                            if (it >= total) break;
                            int eti, ekb;
                            enc_item_coords((int)it, a, CG, eti, ekb);
                            encode_a_item<kTF32>(a, eti, ekb, lane);
                        }
                    }
                }
            }

            // ---- mid-mainloop hand-offs: fault injection and, in
            // online-interval mode, verification after every K_s step
            // with the correction written back to TMEM ----
            if (FT && (a.n_inj > 0 || a.ks_kb > 0)) {
                int ii = a.n_inj > 0 ? inj_lower(a.inj, a.n_inj, t) : 0;
                const int ie = a.n_inj > 0 ? inj_lower(a.inj, a.n_inj, t + 1) : 0;
                int next_chk = a.ks_kb > 0 ? a.ks_kb - 1 : 0x7fffffff;     // k-block closing the next step
                for (;;) {
                    const int kb_f = ii < ie ? a.inj[ii].kb : 0x7fffffff;
                    const int kb_c = next_chk < a.num_kb - 1 ? next_chk : 0x7fffffff;
                    const int kb = min(kb_f, kb_c);
                    if (kb == 0x7fffffff) break;
                    mbar_wait(&inj_req[acc], (injph >> acc) & 1u);
                    injph ^= 1u << acc;
                    tc_fence_after();
                    for (; ii < ie && a.inj[ii].kb == kb; ++ii) {
                        const DevInject f = a.inj[ii];
                        if ((f.target >> 8) != (int)rank) continue;   // fault in the other CTA's check tile
                        const int tgt = f.target & 0xff;
                        int trow, tcol;
                        if (tgt == FTGEMM_TGT_ROW_REF) { trow = f.p; tcol = xoff; }
                        else if (tgt == FTGEMM_TGT_COL_REF) { trow = Cfg::BMD; tcol = f.q + doff; }
                        else { trow = f.p; tcol = f.q + doff; }
                        if ((trow >> 5) == ew) {
                            const uint32_t addr = tb + lane_off + (uint32_t)tcol;
                            uint32_t v = tmem_ld1(addr);
                            if ((int)lane == (trow & 31)) v = apply_fault(v, f);
                            tmem_st1(addr, v);
                        }
                    }
                    if (kb == kb_c) {
                        next_chk += a.ks_kb;
                        if (has_rows) {
                            tc_fence_before();
                            named_bar_sync(ebar, 128);             // faults of this k-block are in TMEM
                            tc_fence_after();
                            const int kdone = min(a.K, (kb + 1) * Cfg::BK);
                            int k2 = 0, p2 = -1, q2 = -1;
                            float c2 = 0.0f;
                            verify(sqrtf((float)kdone), kdone, k2, p2, q2, c2, true);
                            if (k2 == FTGEMM_EV_CORRECTED && (p2 >> 5) == ew) {
                                const uint32_t addr = tb + lane_off + (uint32_t)(q2 + doff);
                                uint32_t v = tmem_ld1(addr);
                                if (rloc == p2) v = __float_as_uint(c2);
                                tmem_st1(addr, v);
                            }
                        }
                    }
                    tc_fence_before();
                    named_bar_sync(ebar, 128);
                    if (et == 0) arrive_leader(&inj_done[acc]);
                }
            }

            mbar_wait(&tm_full[acc], accph);
            tc_fence_after();
            if (!has_rows) {                                   // padding half of the last pair row
                __syncwarp();
                if (lane == 0) arrive_leader(&tm_empty[acc]);
                continue;
            }

            if (FT && EXT == 1 && a.fuse_a && has_rows) {
                // norms of the in-kernel encode.  The accumulator is complete, so
                // every k-block item of this check tile was published (the Y
                // warps waited for each flag before loading its split rows): one
                // acquiring pass over the flags (no polling while the items are
                // being written -- polls of every epilogue warp slowed the flag
                // stores), then the per-k-block partials summed in k order
                // (thread = row; 16-byte loads)
                const uint32_t* fl = a.fflag + (int64_t)ti * a.num_kb;
                FTG_CHECK(ti >= 0 && ti < a.tiles_m && rloc >= 0 && rloc < 128);
#if defined(FTGEMM_EXP_FA_NOWAIT) || defined(FTGEMM_EXP_FA_NOENC)
                for (int k0 = a.num_kb; k0 < a.num_kb; k0 += 32) {
#else
                for (int k0 = 0; k0 < a.num_kb; k0 += 32) {
#endif
                    for (;;) {
                        const int k = k0 + (int)lane;
                        const bool ok = k >= a.num_kb || ld_acquire_u32(fl + k) != 0u;
                        if (__all_sync(0xffffffffu, ok)) break;
                        __nanosleep(500);
                    }
                }
                __syncwarp();
                const float* pr = a.frn2 + ((int64_t)ti * 128 + rloc) * a.nkb4;
                const float* pa = a.facn2 + (int64_t)ti * a.nkb4;
                float sr = 0.0f, sa = 0.0f;
#pragma unroll 8
                for (int k = 0; k < a.num_kb; k += 4) {
                    const float4 x = ld_cg_f4(pr + k), y = ld_cg_f4(pa + k);   // padding k-blocks: never read past num_kb
                    sr += x.x; sa += y.x;
                    if (k + 1 < a.num_kb) { sr += x.y; sa += y.y; }
                    if (k + 2 < a.num_kb) { sr += x.z; sa += y.z; }
                    if (k + 3 < a.num_kb) { sr += x.w; sa += y.w; }
                }
                nrow = sqrtf(sr);
                nac = sqrtf(sa);
            }
            int kind = 0, pstar = -1, qstar = -1;
            float corr = 0.0f;
#ifndef FTGEMM_EXP_NO_VERIFY
            if (FT) verify(a.sqrtK, a.K, kind, pstar, qstar, corr, false);
#endif

            // ---- pass 2: alpha/beta, SWIZZLE_128B staging, TMA stores ----
            // Output in groups of GW columns (one 128-byte box row per thread).
            // TMA box starts must be 16-byte aligned: BF16 check tiles (252
            // columns) start at 0 or 4 mod 8, so the groups of odd tiles are
            // shifted by 4 columns and the 4 columns left over (0..3 or
            // 248..251) are written with one 8-byte store per row.  The last
            // group ends at the tile's last data column and overlaps the
            // previous one by OVL columns (identical values).  FT: warp 3 stores
            // 29 rows (96..124).
            const bool do_corr = FT && kind == FTGEMM_EV_CORRECTED && (pstar >> 5) == ew;   // warp-uniform
            const int qs = (rloc == pstar) ? qstar : -1000;
            const CUtensorMap* cmap = (FT && ew == 3) ? &tmC29 : &tmC;
            const int par = (FT && !kTF32) ? (tj & 1) : 0;
            constexpr int GW = Cfg::GW, NG = Cfg::NG;
            constexpr int OVL = FT ? (kTF32 ? 4 : 8) : 0;
            auto group_start = [&](int g) -> int {
                if constexpr (!FT) return g * GW;
                else if constexpr (kTF32) return (g == NG - 1) ? Cfg::BND - GW : g * GW;
                else return (g == NG - 1) ? (Cfg::BND - GW - 4 * (1 - par)) : (g * GW + 4 * par);
            };
            const int trow = ew * 32 + (int)lane;            // row of this thread inside the tile
            const bool row_ok = trow < bm;
#if defined(FTGEMM_EXP_NO_PASS2)
            // timing experiment: no TMEM reads / stores after the verification
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_leader(&tm_empty[acc]);
            if (true) continue;
#endif
            if constexpr (FT && !kTF32) {
                // leftover 4 columns (tile cols 0..3 for odd tiles, BND-4..BND-1 for even ones)
                const int lo = par ? 0 : Cfg::BND - 4;
                float v[32];
                tmem_ld32(tb + lane_off + (lo & ~31), v);
                float x[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) x[i] = par ? v[i] : v[((Cfg::BND - 4) & 31) + i];
                if (do_corr) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) x[i] = (qs == lo + i) ? corr : x[i];
                }
                if (row_ok && lo < bn) {
                    uint16_t* Cp = reinterpret_cast<uint16_t*>(a.C) + (int64_t)bb * a.c_bs + (int64_t)(r0 + trow) * a.ldc + c0 + lo;
                    float o4[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        o4[i] = a.beta != 0.0f && lo + i < bn ? fmaf(a.beta, bf16_to_f32(Cp[i]), a.alpha * x[i]) : a.alpha * x[i];
                    if (lo + 4 <= bn) {
                        uint2 pk;
                        pk.x = (uint32_t)f32_to_bf16_rn(o4[0]) | ((uint32_t)f32_to_bf16_rn(o4[1]) << 16);
                        pk.y = (uint32_t)f32_to_bf16_rn(o4[2]) | ((uint32_t)f32_to_bf16_rn(o4[3]) << 16);
#if !defined(FTGEMM_EXP_NO_STORE)
                        *reinterpret_cast<uint2*>(Cp) = pk;
#endif
                    } else {
#pragma unroll
                        for (int i = 0; i < 4; ++i) if (lo + i < bn) Cp[i] = f32_to_bf16_rn(o4[i]);
                    }
                }
            }
            float carry[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) carry[i] = 0.0f;
#pragma unroll 1
            for (int g = 0; g < NG; ++g) {
                const int cs = group_start(g);
                float o[GW];
                {
                    // gather TMEM columns [cs, cs + GW) (cs mod 32 in {0, 4, 24, 28})
                    const uint32_t base = tb + lane_off + (uint32_t)(cs & ~31);
                    auto gather = [&](auto shc) {
                        constexpr int SH = decltype(shc)::value;
                        constexpr int NL = (SH + GW + 31) / 32;
#pragma unroll
                        for (int h = 0; h < NL; ++h) {
                            float v[32];
                            tmem_ld32(base + 32 * h, v);
#pragma unroll
                            for (int i = 0; i < 32; ++i) {
                                const int idx = 32 * h + i - SH;
                                if (idx >= 0 && idx < GW) o[idx] = v[i];
                            }
                        }
                    };
                    const int sh = cs & 31;
                    if (sh == 0) gather(std::integral_constant<int, 0>{});
                    else if (sh == 4) gather(std::integral_constant<int, 4>{});
                    else if (sh == 24) gather(std::integral_constant<int, 24>{});
                    else gather(std::integral_constant<int, 28>{});
                }
                if (g == NG - 1) {                         // last TMEM read of this accumulator
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) arrive_leader(&tm_empty[acc]);
                }
                if (do_corr) {
                    const int qq = qs - cs;
#pragma unroll
                    for (int i = 0; i < GW; ++i) o[i] = (i == qq) ? corr : o[i];
                }
                // double-buffered staging: the buffer is free once the store issued
                // two groups ago has read it
                uint8_t* sbuf = stg + ew * 8192 + (gcount & 1) * 4096;
                ++gcount;
                if (lane == 0) bulk_wait_read1();
                __syncwarp();
                const int gcol = c0 + cs, grow = r0 + ew * 32;
                if (a.beta != 0.0f) {
                    if (lane == 0) {
                        mbar_arrive_expect_tx(cbw, (FT && ew == 3 ? 29 : 32) * 128);
                        tma_load_3d(sbuf, cmap, cbw, gcol, grow, bb);
                    }
                    mbar_wait(cbw, cph);
                    cph ^= 1;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const uint4 u = ld_shared_v4(sbuf + lane * 128 + ((j ^ (lane & 7)) << 4));
                        const uint32_t wd[4] = {u.x, u.y, u.z, u.w};
                        if constexpr (kTF32) {
#pragma unroll
                            for (int q = 0; q < 4; ++q) o[4 * j + q] = fmaf(a.beta, __uint_as_float(wd[q]), a.alpha * o[4 * j + q]);
                        } else {
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                o[8 * j + 2 * q] = fmaf(a.beta, __uint_as_float(wd[q] << 16), a.alpha * o[8 * j + 2 * q]);
                                o[8 * j + 2 * q + 1] = fmaf(a.beta, __uint_as_float(wd[q] & 0xFFFF0000u), a.alpha * o[8 * j + 2 * q + 1]);
                            }
                        }
                    }
                    if constexpr (OVL > 0) {
                        // overlap columns were already updated in memory: reuse the values computed then
                        if (g == NG - 1) {
#pragma unroll
                            for (int i = 0; i < OVL; ++i) o[i] = carry[i];
                        }
#pragma unroll
                        for (int i = 0; i < OVL; ++i) carry[i] = o[GW - OVL + i];
                    }
                } else if (a.alpha != 1.0f) {
#pragma unroll
                    for (int i = 0; i < GW; ++i) o[i] *= a.alpha;
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    uint32_t pk[4];
                    if constexpr (kTF32) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) pk[q] = __float_as_uint(o[4 * j + q]);
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q) pk[q] = pack_bf16x2(o[8 * j + 2 * q], o[8 * j + 2 * q + 1]);
                    }
                    st_shared_v4(sbuf + lane * 128 + ((j ^ (lane & 7)) << 4), pk[0], pk[1], pk[2], pk[3]);
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
#if !defined(FTGEMM_EXP_NO_STORE)
                    tma_store_3d(cmap, sbuf, gcol, grow, bb);
#endif
                    bulk_commit();
                }
            }
        }
        if (lane == 0) bulk_wait0();
        if (FT && et == 0 && n_checked) atomicAdd(&a.rep->counts[CNT_CHECKED], n_checked);
    }

#if defined(FTGEMM_EXP_FA_TRACE)
    if (threadIdx.x == 0) g_fa_trace[41000 + blockIdx.x] = gtimer();
#endif
    tc_fence_before();
    // a CTA pair stays resident until both are done (remote arrivals, pair MMA into the peer's TMEM)
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    if (warp == W_ALLOC) {
        tc_fence_after();
        tmem_dealloc<Cfg::TMEM_COLS, CG>(tmem_base);
    }
}

// ---------------------------------------------------------------- launch ---
template <bool kTF32, int BN, bool FT, int CG, int EPI = FTGEMM_EPI_WG, int EXT = 0>
cudaError_t launch_tc_t(const CUtensorMap& mA, const CUtensorMap& mB, const CUtensorMap& mC, const CUtensorMap& mC29,
                        const CUtensorMap& mY, const TcArgs& a, cudaStream_t st) {
    using Cfg = TcCfg<kTF32, BN, FT, CG, EPI>;
    auto kern = tc_ftgemm_kernel<kTF32, BN, FT, CG, EPI, EXT>;
    static PerDeviceOnce smem_attr;
    cudaError_t e = smem_attr.run([&] {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    });
    if (e != cudaSuccess) return e;
    // persistent: one CTA (pair) per SM (pair of SMs)
    const int slots = device_sms() / CG;
    const int clusters = a.num_units < slots ? a.num_units : slots;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(clusters * CG, 1, 1);
    cfg.blockDim = dim3(Cfg::THREADS, 1, 1);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // programmatic dependent launch: the prologue (barrier init, TMEM
    // allocation, descriptor prefetch) overlaps the tail of the encode kernel
    // before it; every thread waits (griddepcontrol.wait) before reading anything
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, mA, mB, mC, mC29, mY, a);
}

cudaError_t launch_tc(bool tf32, int bn, bool ft, int cg, int epi, int ext, const CUtensorMap& mA,
                      const CUtensorMap& mB, const CUtensorMap& mC, const CUtensorMap& mC29, const CUtensorMap& mY,
                      const TcArgs& a, cudaStream_t st) {
#define L_(T, B, F) (cg == 2 ? launch_tc_t<T, B, F, 2>(mA, mB, mC, mC29, mY, a, st) \
                             : launch_tc_t<T, B, F, 1>(mA, mB, mC, mC29, mY, a, st))
#define LX_(T, B, X) (cg == 2 ? launch_tc_t<T, B, true, 2, FTGEMM_EPI_WG, X>(mA, mB, mC, mC29, mY, a, st) \
                             : launch_tc_t<T, B, true, 1, FTGEMM_EPI_WG, X>(mA, mB, mC, mC29, mY, a, st))
    // the extended modes (1: in-kernel A encode, 2: online K_s checks): FT on, their own instantiations
    if (ext == 1 && ft) {
        if (tf32) return bn == 256 ? LX_(true, 256, 1) : LX_(true, 128, 1);
        return bn == 256 ? LX_(false, 256, 1) : LX_(false, 128, 1);
    }
    if (ext == 2 && ft) {
        if (tf32) return bn == 256 ? LX_(true, 256, 2) : LX_(true, 128, 2);
        return bn == 256 ? LX_(false, 256, 2) : LX_(false, 128, 2);
    }
    // small-K narrow tiles with FT: three epilogue warpgroups (one CTA per MMA)
    if (ft && tf32 && bn == 128 && epi == 3 && cg == 1)
        return launch_tc_t<true, 128, true, 1, 3>(mA, mB, mC, mC29, mY, a, st);
    if (tf32) {
        if (bn == 256) return ft ? L_(true, 256, true) : L_(true, 256, false);
        return ft ? L_(true, 128, true) : L_(true, 128, false);
    }
    if (bn == 256) return ft ? L_(false, 256, true) : L_(false, 256, false);
    return ft ? L_(false, 128, true) : L_(false, 128, false);
#undef L_
#undef LX_
}

}  // namespace ftg

#if defined(FTGEMM_EXP_FA_TRACE)
extern "C" __attribute__((visibility("default"))) int ftgemm_debug_trace(void* host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, ftg::g_fa_trace, bytes < sizeof(ftg::g_fa_trace) ? bytes : sizeof(ftg::g_fa_trace));
}
#endif
