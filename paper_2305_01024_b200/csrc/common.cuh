// common.cuh -- device-side data layouts shared by the encode, fused-GEMM and
// host API translation units of libftgemm (never by the oracle).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdlib>
#include <mutex>

#include "../../include/ftgemm.h"

namespace ftg {

constexpr int kNumSMsB200 = 148;
constexpr int kMaxEvents = 4096;
constexpr int kMaxInject = 65536;
constexpr int kEncBRows = 256;     // k-rows of B per encode-B block
constexpr int kMaxDevices = 64;    // per-device one-time state (kernel attributes, device checks)

// Development / tuning knobs are compile-time only (-D...): the product path
// reads no environment variables.
#ifndef FTGEMM_B3D
#define FTGEMM_B3D 1               // B tile in one 3-D TMA request per stage
#endif
#ifndef FTGEMM_GROUP
#define FTGEMM_GROUP 16            // M-tiles per schedule group of the tensor-core kernel
#endif

// ---- report workspace (device) --------------------------------------------
struct DevInject {        // one fault, resolved to (check tile, k-block, in-tile position)
    int32_t tile, kb, p, q;
    int32_t bit, mode, target;
    float addend;
};
static_assert(sizeof(DevInject) == 32, "DevInject layout");

struct ReportDev {
    unsigned long long counts[8];     // order of ftgemm_counts_t
    unsigned int max_ratio_bits;      // max |residual| / tau over unflagged residuals (FP32 bits; >= 0)
    unsigned int pad32;
    unsigned long long pad[7];
    ftgemm_event_t events[kMaxEvents];
};
enum { CNT_CHECKED = 0, CNT_DETECTED, CNT_CORRECTED, CNT_CHECKSUM_ONLY, CNT_UNCORRECTABLE,
       CNT_LOCATED, CNT_EVENTS, CNT_DROPPED };

inline size_t report_bytes() { return sizeof(ReportDev) + (size_t)kMaxInject * sizeof(DevInject); }
inline size_t report_inject_offset() { return sizeof(ReportDev); }

// ---- division by a launch constant (host-computed multiplier) ---------------
// q = floor(n / d) = umul64hi(n, ceil(2^64 / d)) for 0 <= n < 2^32, d >= 2 (the
// error n (m - 2^64/d) / 2^64 < 2^-32 cannot carry past an integer); d == 1 is
// passed through.  Replaces the per-tile 32-bit divisions of the persistent
// tile scheduler (a few IMADs instead of ~25 instructions each).
struct FastDiv {
    uint64_t m;
    uint32_t d;
    static FastDiv make(uint32_t d_) {
        FastDiv f;
        f.d = d_ ? d_ : 1u;
        f.m = f.d > 1 ? (~0ull / f.d) + 1ull : 0ull;
        return f;
    }
#ifdef __CUDACC__
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return d == 1u ? n : (uint32_t)__umul64hi((uint64_t)n, m);
    }
#endif
};

// ---- kernel arguments (plain data, passed by value) ------------------------
struct TcArgs {
    int M, N, K, num_kb;
    int tiles_m, tiles_n, num_tiles;
    int units_m, num_units;   // work units: CG check tiles stacked in M (CG = CTAs per MMA); all problems
    int units_pb;             // units per problem (batched launches: num_units = batch x units_pb)
    int64_t enc_bs;           // encode-workspace stride between problems, in floats
    int64_t c_bs;             // C stride between problems, in elements
    int group;            // M-units per schedule group (tile_coords)
    FastDiv fd_upb, fd_pg, fd_g, fd_gt;   // units_pb, group x tiles_n, group, last (ragged) group size
    int ft_level;
    int ks_kb;            // > 0: verify after every ks_kb k-blocks too (online-interval mode)
    int fuse_a;           // 1: the A-side encode (split e^T A rows, row / tile norms) runs in the kernel
    // in-kernel encode of A (fuse_a): encoder warps stream A from global
    // memory, one claimed (check tile, k-block) item at a time, in the order
    // the tile schedule first needs them, and publish each item with a flag
    const void* A; int64_t lda;
    uint32_t* fflag;      // [tiles_m][num_kb]: 1 = item written; then the item claim counter (zeroed before every launch)
    float* frn2;          // [tiles_m][128][nkb4]: per-k-block partial row sums of squares
    float* facn2;         // [tiles_m][nkb4]: per-k-block partial sums of (e^T A)^2
    int nkb4;             // num_kb rounded up to 4
    int b3d;              // 1: tmB is the 3-D (column slice, k, column block) view of B / B^r
    int y_warp;           // FT: 1 = the split rows of e^T A are loaded by their own warp
    float alpha, beta;
    void* C; int64_t ldc;
    const void* Y; int kp;
    const float* rownorm; const float* colnorm; const float* acnorm; const float* brnorm;
    float tau_u, tau_l1, tau_l2, sqrtK;
    ReportDev* rep;
    const DevInject* inj; int n_inj;
};

struct SimtArgs {
    int M, N, K, num_kb;
    int tiles_m, tiles_n, ft_level;
    float alpha, beta;
    const float* A; int64_t lda;
    const float* B; int64_t ldb;
    float* C; int64_t ldc;
    const float* Ac; const float* Br; int kp;
    const float* rownorm; const float* colnorm; const float* acnorm; const float* brnorm;
    float tau_u, tau_l1, tau_l2, sqrtK;
    ReportDev* rep;
    const DevInject* inj; int n_inj;
};

// M-tiles per schedule group of the tensor-core kernel: about FTGEMM_GROUP,
// split evenly so that no group is ragged
inline int tc_group(int units_m, int cg) {
    const int g0 = FTGEMM_GROUP / cg > 0 ? FTGEMM_GROUP / cg : 1;
    const int ng = units_m / g0 > 0 ? (units_m + g0 / 2) / g0 : 1;
    return (units_m + ng - 1) / ng;
}

// ---- tile geometry of a plan ---------------------------------------------
struct Geometry {
    int dtype;            // FTGEMM_*
    int bm, bn, bk;       // CTA / MMA tile
    int bmd, bnd;         // data rows / cols per check tile (FT on)
    int tiles_m, tiles_n; // check-tile grid (FT on)
    int kp;               // K padded to bk
    int nkb;              // kp / bk (MMA k-blocks)
    int nkc_a;            // K chunks of the A-encode partial row norms (256 wide)
    int nkc_b;            // K chunks of the B-encode partial column norms
    int enc_b_rows;       // k-rows per encode-B block (nkc_b = ceil(kp / enc_b_rows))
    int elt;              // operand element bytes
    int tc;               // 1 for the tensor-core paths (split operands, B^r)
};

// Encode workspace layout (byte offsets; each region 256-byte aligned).
//   A part: Ac (FP32 e^T A per tile), Ypack (tensor-core paths: the 3 split rows
//           of e^T A per (tile, k-block), 3 x 128 bytes, already in the smem
//           SWIZZLE_128B order of MMA rows 125..127), row norms, tile norms.
//   B part: Br (FP32 B e per tile), Bt (tensor-core paths: the encoded operand
//           B^r = [B_j, B_j e] of PAPER.md Eq. (2), N-major, kp rows of
//           tiles_n * bn: tile j's slot holds columns 0..bnd-1 of B_j, then
//           split(B_j e) (3 columns) and a zero column), column norms, tile norms.
//   In-kernel A encode (ftgemm_run_fused, tensor-core paths): item flags and
//           the per-k-block partial norms the encoder warps publish.
struct EncLayout {
    size_t ac, y, rownorm, acnorm, rn2, acn2, cnt_a;     // A part
    size_t fflag, frn2, facn2;                           // A part, in-kernel encode
    size_t b_off;                                        // start of the B part
    size_t br, bt, colnorm, brnorm, cn2, brn2, cnt_b;    // absolute offsets
    size_t a_bytes, b_bytes, total;
};

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

inline EncLayout enc_layout(const Geometry& g, int64_t M, int64_t N) {
    EncLayout L{};
    size_t o = 0;
    L.ac = o;      o = align256(o + sizeof(float) * (size_t)g.tiles_m * g.kp);
    L.y = o;       o = align256(o + (g.tc ? (size_t)g.tiles_m * g.nkb * 384 : 0));
    L.rownorm = o; o = align256(o + sizeof(float) * (size_t)M);
    L.acnorm = o;  o = align256(o + sizeof(float) * (size_t)g.tiles_m);
    L.rn2 = o;     o = align256(o + sizeof(float) * (size_t)g.nkc_a * M);
    L.acn2 = o;    o = align256(o + sizeof(float) * (size_t)g.nkc_a * g.tiles_m);
    L.cnt_a = o;   o = align256(o + sizeof(int) * (size_t)g.tiles_m);
    const size_t nkb4 = g.tc ? (size_t)((g.nkb + 3) & ~3) : 0;
    L.fflag = o;   o = align256(o + (g.tc ? sizeof(uint32_t) * ((size_t)g.tiles_m * g.nkb + 2) : 0));   // + claim, publish counters
    L.frn2 = o;    o = align256(o + sizeof(float) * (size_t)g.tiles_m * 128 * nkb4);
    L.facn2 = o;   o = align256(o + sizeof(float) * (size_t)g.tiles_m * nkb4);
    L.a_bytes = o;
    L.b_off = o;
    L.br = o;      o = align256(o + sizeof(float) * (size_t)g.tiles_n * g.kp);
    L.bt = o;      o = align256(o + (g.tc ? (size_t)g.elt * g.tiles_n * g.bn * g.kp : 0));
    L.colnorm = o; o = align256(o + sizeof(float) * (size_t)N);
    L.brnorm = o;  o = align256(o + sizeof(float) * (size_t)g.tiles_n);
    L.cn2 = o;     o = align256(o + sizeof(float) * (size_t)g.nkc_b * N);
    L.brn2 = o;    o = align256(o + sizeof(float) * (size_t)g.nkc_b * g.tiles_n);
    L.cnt_b = o;   o = align256(o + sizeof(int) * (size_t)g.tiles_n);
    L.b_bytes = o - L.b_off;
    L.total = o;
    return L;
}

// cudaFuncSetAttribute is a per-device setting: apply it once per (kernel,
// device), thread-safely.  One instance per kernel (a function-local static).
struct PerDeviceOnce {
    std::mutex mu;
    bool done[kMaxDevices] = {};
    template <class Fn>
    cudaError_t run(Fn fn) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
        std::lock_guard<std::mutex> lk(mu);
        if (done[dev]) return cudaSuccess;
        e = fn();
        if (e == cudaSuccess) done[dev] = true;
        return e;
    }
};

// SMs of the current device (cached per device); the launch grids use it, the
// plan's pure-host cost model assumes a full B200 (kNumSMsB200)
inline int device_sms() {
    static std::mutex mu;
    static int sms[kMaxDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return kNumSMsB200;
    std::lock_guard<std::mutex> lk(mu);
    if (!sms[dev] && cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        sms[dev] = kNumSMsB200;
    }
    return sms[dev];
}

// ---- operand conversions ---------------------------------------------------
// TF32 operand semantics of tcgen05.mma kind::tf32 on FP32 bit patterns:
// the low 13 mantissa bits are ignored (truncation).  Pinned on the device by
// tests/test_gpu_parity.py::test_tf32_operand_semantics.
__device__ __forceinline__ float tf32_trunc(float x) {
    return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
__device__ __forceinline__ float bf16_to_f32(uint16_t h) { return __uint_as_float((uint32_t)h << 16); }
__device__ __forceinline__ uint16_t f32_to_bf16_rn(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
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

// packed bf16x2 word -> (low, high) as FP32 (exact)
__device__ __forceinline__ float2 bf16x2_to_f2(uint32_t w) {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}

// two floats -> packed bf16x2 (RNE), low half = a (one cvt.rn.bf16x2.f32)
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}

}  // namespace ftg
