// api.cu -- the C ABI of libftgemm (include/ftgemm.h): plan table, argument
// validation, TMA descriptor construction, fault-list preparation and kernel
// dispatch.  Host code only; the arithmetic is in encode.cu / tc_gemm.cu /
// simt_gemm.cu.  No CPU fallback exists: anything the device path cannot run is
// rejected with an error code.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <atomic>
#include <cmath>
#include <limits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace ftg {
cudaError_t launch_encode(const Geometry& g, const EncLayout& L, int64_t M, int64_t N, int64_t K,
                          const void* A, int64_t lda, const void* B, int64_t ldb, void* enc, int which,
                          cudaStream_t st, int batch, int64_t sA, int64_t sB, int64_t sE);
}  // namespace ftg

namespace ftg {
cudaError_t launch_tc(bool tf32, int bn, bool ft, int cg, int epi, int ext, const CUtensorMap& mA,
                      const CUtensorMap& mB, const CUtensorMap& mC, const CUtensorMap& mC29, const CUtensorMap& mY,
                      const TcArgs& a, cudaStream_t st);
cudaError_t launch_simt(bool ft, const SimtArgs& a, cudaStream_t st);
int simt_bk();
struct NfInject {
    int64_t row, col;
    int32_t bit, mode, target;
    float addend;
};
size_t nonfused_ws_bytes(const Geometry& g, int64_t M, int64_t N);
cudaError_t launch_nonfused(const Geometry& g, const EncLayout& E, int64_t M, int64_t N, int64_t K, float alpha,
                            const void* A, int64_t lda, const void* B, int64_t ldb, float beta, void* C, int64_t ldc,
                            const void* enc_ws, void* nf_ws, int ft_level, const NfInject* dinj, int n_inj,
                            ReportDev* rep, float tau_u, float l1, float l2, cudaStream_t st, const char** why);
}  // namespace ftg

using namespace ftg;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}
int fail_cuda(cudaError_t e, const char* where) {
    return fail(FTGEMM_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}


bool valid_dtype(int d) { return d == FTGEMM_F32_SIMT || d == FTGEMM_TF32 || d == FTGEMM_BF16; }

// A dtype code is the precision variant (low byte) optionally OR-ed with an
// explicit tensor-core tile class FTGEMM_TILE(bn, cta_group) (include/ftgemm.h).
// The class is part of every call's arguments -- there is no ambient state --
// so an encode and a run given the same code always derive the same layout.
struct Code { int dtype, bn, cg; };
bool parse_code(int code, Code* c) {
    c->dtype = code & FTGEMM_DTYPE_MASK;
    const int tb = (code >> 8) & 0xf, tcg = (code >> 12) & 0xf;
    if (!valid_dtype(c->dtype) || (code & ~0xffff) != 0 || tb > 2 || tcg > 2 || (tb == 0) != (tcg == 0)) return false;
    if (c->dtype == FTGEMM_F32_SIMT && tb) return false;       // the SIMT kernel has one tile class
    c->bn = tb * 128; c->cg = tcg;
    return true;
}

// The shape-class table (north_star item 4): compile-time instantiations
// chosen per problem shape.  `code` must have passed parse_code.
void fill_plan(int code, int64_t M, int64_t N, int64_t K, ftgemm_plan_t* p, int64_t batch = 1) {
    Code cc;
    parse_code(code, &cc);
    const int dtype = cc.dtype;
    std::memset(p, 0, sizeof(*p));
    p->dtype = dtype;
    p->max_events = kMaxEvents;
    p->max_inject = kMaxInject;
    if (dtype == FTGEMM_F32_SIMT) {
        p->shape_class = FTGEMM_SHAPE_SQUARE;
        p->bm = 128; p->bn = 128; p->bk = simt_bk();
        p->check_tile_m = 128; p->check_tile_n = 128;
        p->off_tile_m = 128; p->off_tile_n = 128;
        p->stages = simt_bk() == 8 ? 4 : 3; p->cta_group = 1;
        p->u_acc = std::ldexp(1.0f, -24); p->lambda1 = 16.0f; p->lambda2 = 32.0f;
    } else {
        const int bk = dtype == FTGEMM_TF32 ? 32 : 64;
        const int64_t tiles256 = ((M + 124) / 125) * ((N + 251) / 252);
        // skinny operands (cfg4): one check tile across the narrow dimension, so
        // the long operand streams through each SM once -- N <= 252: one
        // 252-column tile; M <= 250: a CTA pair (2 x 125 rows) per unit
        const bool skinny_n = N <= 252;
        const bool skinny_m = M <= 250 && !skinny_n;
        const int64_t tiles_m125 = (M + 124) / 125;
        bool small = !skinny_n && !skinny_m && (tiles256 * batch < 2 * kNumSMsB200 || N <= 512);
        // CTA pairs (cta_group::2, M = 256 per MMA) halve the B tile each SM
        // loads; they lose on K = 128 shapes (epilogue-bound) and skinny M
        int cg = (!small && ((tiles_m125 >= 4 && (K >= 2048 || (dtype == FTGEMM_TF32 && K >= 1024))) ||
                             (skinny_m && K >= 1024))) ? 2 : 1;
        // small K is epilogue-bound: TF32 K <= 128 runs fastest on the narrow
        // tile (one CTA per MMA), measured 7-10 % over BN = 256 (profiles/r1d_tile_classes.md)
        if (!skinny_n && !skinny_m && dtype == FTGEMM_TF32 && K <= 128) { small = true; cg = 1; }
        // the cost model from K = 1024 (BF16) / 512 (TF32: twice the MMA time per k)
        if (!skinny_n && !skinny_m && K >= (dtype == FTGEMM_TF32 ? 512 : 1024)) {
            // Mainloop-bound shapes: wave-quantised cost model over the four tile
            // classes, time = ceil(units / concurrent units) x (per-wave time of
            // the class at K = 8192, measured on B200: profiles/r1d_tile_classes.md)
            struct Cls { int bn, cg; double c_bf16, c_tf32; };
            const Cls cls[4] = {{256, 2, 54.5, 108.7}, {256, 1, 68.7, 140.2}, {128, 1, 48.0, 98.8}, {128, 2, 49.8, 102.9}};
            double best = 1e300;
            for (const Cls& c : cls) {
                const int64_t tn = (N + c.bn - 5) / (c.bn - 4);
                const int64_t units = ((tiles_m125 + c.cg - 1) / c.cg) * tn * batch;
                const int64_t slots = kNumSMsB200 / c.cg;
                const double t = (double)((units + slots - 1) / slots) * (dtype == FTGEMM_TF32 ? c.c_tf32 : c.c_bf16);
                if (t < best * (1.0 - 1e-9)) { best = t; small = c.bn == 128; cg = c.cg; }
            }
        }
        int bn = small ? 128 : 256;
        // an explicit class in the code wins over every rule above (multi-GPU
        // ranks pass the full problem's class, tests force each class)
        if (cc.bn) { bn = cc.bn; cg = cc.cg; }
        p->dtype = dtype | FTGEMM_TILE(bn, cg);      // the fully explicit code of this plan
        p->shape_class = bn == 128 ? FTGEMM_SHAPE_SMALL_N : FTGEMM_SHAPE_SQUARE;
        p->bm = 128; p->bn = bn; p->bk = bk;
        p->check_tile_m = 125; p->check_tile_n = bn - 4;
        p->off_tile_m = 128; p->off_tile_n = bn;
        p->cta_group = cg;
        const int elt = dtype == FTGEMM_TF32 ? 4 : 2;
        const int stage = 128 * 128 + (bn / cg) * bk * elt;
        p->stages = std::min(8, (196 * 1024) / stage);
        p->u_acc = std::ldexp(1.0f, -23); p->lambda1 = 8.0f; p->lambda2 = 16.0f;
    }
    p->tiles_m = (M + p->check_tile_m - 1) / p->check_tile_m;
    p->tiles_n = (N + p->check_tile_n - 1) / p->check_tile_n;
}

Geometry geometry(const ftgemm_plan_t& p, int64_t K) {
    Geometry g{};
    g.dtype = p.dtype & FTGEMM_DTYPE_MASK;
    g.bm = p.bm; g.bn = p.bn; g.bk = p.bk;
    g.bmd = p.check_tile_m; g.bnd = p.check_tile_n;
    g.tiles_m = (int)p.tiles_m; g.tiles_n = (int)p.tiles_n;
    g.kp = (int)(((K + p.bk - 1) / p.bk) * p.bk);
    g.nkb = g.kp / p.bk;
    g.elt = g.dtype == FTGEMM_BF16 ? 2 : 4;
    g.tc = p.dtype != FTGEMM_F32_SIMT;
    g.nkc_a = (g.kp + 512 / g.elt - 1) / (512 / g.elt);   // encode-A k chunks (512-byte rows)
    // encode B: 256 k-rows per block (measured best or equal against 64 / 128
    // for every profiled shape, profiles/r1_encode.md)
    g.enc_b_rows = kEncBRows;
    g.nkc_b = (g.kp + g.enc_b_rows - 1) / g.enc_b_rows;
    return g;
}

// 1 if the CURRENT device is an sm_100 part (cached per device ordinal)
int check_device() {
    static std::mutex mu;
    static signed char cached[kMaxDevices];
    static bool init = false;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) { cudaGetLastError(); return 0; }
    std::lock_guard<std::mutex> lk(mu);
    if (!init) { std::memset(cached, -1, sizeof(cached)); init = true; }
    if (cached[dev] >= 0) return cached[dev];
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return cached[dev] = (major == 10 && minor == 0) ? 1 : 0;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// Every map carries a trailing batch dimension (size `batch`, stride
// `batch_bytes`; 1 and any valid stride for a single problem), so one kernel
// instantiation serves single and batched launches (ftgemm_run_batched).
struct Batch {
    uint64_t n = 1, bytes = 0;
};
uint64_t batch_stride(const Batch& bt, uint64_t fallback) {
    // a size-1 dimension still needs a legal stride (a multiple of 16 below 2^40)
    if (bt.n > 1) return bt.bytes;
    const uint64_t s = (fallback + 15) & ~(uint64_t)15;
    return s > 0 && s < (1ull << 40) ? s : 16;
}

int make_map(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
             uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
             CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B, Batch bt = Batch{}) {
    auto enc = tensor_map_encoder();
    if (!enc) return fail(FTGEMM_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {inner, outer, bt.n};
    cuuint64_t strides[2] = {row_bytes, batch_stride(bt, row_bytes * outer)};
    cuuint32_t box[3] = {box_inner, box_outer, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FTGEMM_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return FTGEMM_OK;
}

// 3-D view of a row-major [rows][cols] operand as (128-byte column slice,
// row, column block): one box covers nblk consecutive column blocks of bk rows,
// landing as nblk stacked [bk][128 B] SWIZZLE_128B atoms -- the smem layout of
// the N-major B tile (cols must be a multiple of the slice width)
int make_map_3d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t slice, uint64_t rows,
                uint64_t nblocks, uint64_t row_bytes, uint32_t box_rows, uint32_t box_blocks, CUtensorMapSwizzle sw,
                Batch bt = Batch{}) {
    auto enc = tensor_map_encoder();
    if (!enc) return fail(FTGEMM_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
    const uint64_t elt = (dt == CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) ? 2 : 4;
    cuuint64_t dims[4] = {slice, rows, nblocks, bt.n};
    cuuint64_t strides[3] = {row_bytes, slice * elt, batch_stride(bt, row_bytes * rows)};
    cuuint32_t box[4] = {(cuuint32_t)slice, box_rows, box_blocks, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, dt, 4, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FTGEMM_ERR_UNSUPPORTED, "cuTensorMapEncodeTiled (3-D) failed (%d)", (int)r);
    return FTGEMM_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int check_dims(int code, int64_t M, int64_t N, int64_t K) {
    Code cc;
    if (!parse_code(code, &cc))
        return fail(FTGEMM_ERR_INVALID_VALUE, "bad dtype code 0x%x (dtype | FTGEMM_TILE(128|256, 1|2), tensor-core dtypes only)", code);
    if (M < 1 || N < 1 || K < 1) return fail(FTGEMM_ERR_INVALID_VALUE, "dims must be >= 1 (M=%lld N=%lld K=%lld)",
                                             (long long)M, (long long)N, (long long)K);
    if (M >= (1ll << 31) || N >= (1ll << 31) || K >= (1ll << 31))
        return fail(FTGEMM_ERR_UNSUPPORTED, "dims must be < 2^31");
    return FTGEMM_OK;
}

// schedule key of a check tile (the order the kernel walks work units in; a
// unit is cta_group check tiles stacked in M, one per CTA of the pair)
int tile_key(const ftgemm_plan_t& p, int ti, int tj) {
    if ((p.dtype & FTGEMM_DTYPE_MASK) == FTGEMM_F32_SIMT) return ti * (int)p.tiles_n + tj;
    const int cg = p.cta_group;
    const int units_m = ((int)p.tiles_m + cg - 1) / cg, tu = ti / cg;
    const int G = tc_group(units_m, cg);
    const int grp = tu / G, first = grp * G;
    const int gsz = std::min<int>(G, units_m - first);
    return grp * G * (int)p.tiles_n + tj * gsz + (tu - first);
}

}  // namespace

extern "C" {

int ftgemm_version(void) { return FTGEMM_ABI_VERSION; }

int ftgemm_device_arch(void) { return 1000; }
const char* ftgemm_last_error(void) { return g_err.c_str(); }

int ftgemm_plan(int code, int64_t M, int64_t N, int64_t K, ftgemm_plan_t* out) {
    if (!out) return fail(FTGEMM_ERR_INVALID_VALUE, "null plan pointer");
    int e = check_dims(code, M, N, K);
    if (e) return e;
    fill_plan(code, M, N, K, out);
    const Geometry g = geometry(*out, K);
    const EncLayout L = enc_layout(g, M, N);
    out->enc_bytes = (int64_t)L.total;
    out->enc_b_offset = (int64_t)L.b_off;
    out->enc_b_bytes = (int64_t)L.b_bytes;
    out->report_bytes = (int64_t)report_bytes();
    g_err.clear();
    return FTGEMM_OK;
}

int ftgemm_encode_layout(int code, int64_t M, int64_t N, int64_t K, ftgemm_enc_layout_t* out) {
    if (!out) return fail(FTGEMM_ERR_INVALID_VALUE, "null layout pointer");
    int e = check_dims(code, M, N, K);
    if (e) return e;
    ftgemm_plan_t p;
    fill_plan(code, M, N, K, &p);
    const Geometry g = geometry(p, K);
    const EncLayout L = enc_layout(g, M, N);
    out->ac = (int64_t)L.ac; out->br = (int64_t)L.br; out->bt = g.tc ? (int64_t)L.bt : -1;
    out->rownorm = (int64_t)L.rownorm; out->colnorm = (int64_t)L.colnorm;
    out->acnorm = (int64_t)L.acnorm; out->brnorm = (int64_t)L.brnorm;
    out->kp = g.kp; out->bt_ld = (int64_t)g.tiles_n * g.bn;
    out->y = g.tc ? (int64_t)L.y : -1;
    g_err.clear();
    return FTGEMM_OK;
}

static int encode_impl(int code, int64_t batch, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                       int64_t sA, const void* B, int64_t ldb, int64_t sB, void* enc_ws, int64_t enc_stride, int which,
                       void* stream) {
    int e = check_dims(code, M, N, K);
    if (e) return e;
    const int dtype = code & FTGEMM_DTYPE_MASK;
    if ((which & 3) == 0 || which > 7) return fail(FTGEMM_ERR_INVALID_VALUE, "which must be 1, 2 or 3 (| 4)");
    if (!enc_ws) return fail(FTGEMM_ERR_INVALID_VALUE, "null enc_ws");
    if ((which & 1) && (!A || lda < K)) return fail(FTGEMM_ERR_INVALID_VALUE, "bad A / lda");
    if ((which & 2) && (!B || ldb < N)) return fail(FTGEMM_ERR_INVALID_VALUE, "bad B / ldb");
    if (batch < 1 || batch >= 65536) return fail(FTGEMM_ERR_INVALID_VALUE, "batch must be in [1, 65536)");
    if (batch > 1 && dtype == FTGEMM_F32_SIMT) return fail(FTGEMM_ERR_UNSUPPORTED, "batched: tensor-core dtypes");
    if (sA < 0 || sB < 0) return fail(FTGEMM_ERR_INVALID_VALUE, "negative batch stride");
    const int elt = dtype == FTGEMM_BF16 ? 2 : 4;
    if ((which & 1) && (!aligned16(A) || (lda * elt) % 16 || (sA * elt) % 16)) return fail(FTGEMM_ERR_UNSUPPORTED, "A must be 16-byte aligned with 16-byte row pitch");
    if ((which & 2) && (!aligned16(B) || (ldb * elt) % 16 || (sB * elt) % 16)) return fail(FTGEMM_ERR_UNSUPPORTED, "B must be 16-byte aligned with 16-byte row pitch");
    if ((reinterpret_cast<uintptr_t>(enc_ws) & 255) != 0) return fail(FTGEMM_ERR_INVALID_VALUE, "enc_ws must be 256-byte aligned");
    if (!check_device()) return fail(FTGEMM_ERR_UNSUPPORTED, "no sm_100 (B200) device");
    ftgemm_plan_t p;
    fill_plan(code, M, N, K, &p, batch);
    const Geometry g = geometry(p, K);
    const EncLayout L = enc_layout(g, M, N);
    if (batch > 1 && (enc_stride < (int64_t)L.total || enc_stride % 256))
        return fail(FTGEMM_ERR_INVALID_VALUE, "enc_stride must be >= plan.enc_bytes and a multiple of 256");
    cudaError_t ce = launch_encode(g, L, M, N, K, A, lda, B, ldb, enc_ws, which, (cudaStream_t)stream, (int)batch,
                                   sA * elt, sB * elt, batch > 1 ? enc_stride : (int64_t)L.total);
    if (ce != cudaSuccess) return fail_cuda(ce, "encode launch");
    g_err.clear();
    return FTGEMM_OK;
}

// batched launches (ftgemm_run_batched): problem b's operands at A + b sA,
// B + b sB, C + b sC (elements), its encode at enc_ws + b enc_stride (bytes)
struct BatchArgs {
    int64_t n = 1, sA = 0, sB = 0, sC = 0, enc_stride = 0;
};

static int run_impl(int code, int64_t M, int64_t N, int64_t K, float alpha, const void* A, int64_t lda,
                    const void* B, int64_t ldb, float beta, void* C, int64_t ldc, const void* enc_ws, int ft_level,
                    int64_t ks, int fuse_a, const ftgemm_inject_t* inj, int32_t n_inj, void* report_ws, void* stream,
                    const BatchArgs& bt = BatchArgs{}) {
    int e = check_dims(code, M, N, K);
    if (e) return e;
    const int dtype = code & FTGEMM_DTYPE_MASK;
    if (bt.n < 1 || bt.n >= (1 << 20)) return fail(FTGEMM_ERR_INVALID_VALUE, "batch must be in [1, 2^20)");
    if (bt.n > 1 && (dtype == FTGEMM_F32_SIMT || ks > 0 || fuse_a))
        return fail(FTGEMM_ERR_UNSUPPORTED, "batched runs: tensor-core dtypes, end-of-K verification, separate encode");
    if (bt.sA < 0 || bt.sB < 0 || bt.sC < 0 || bt.enc_stride < 0)
        return fail(FTGEMM_ERR_INVALID_VALUE, "negative batch stride");
    if (ks < 0) return fail(FTGEMM_ERR_INVALID_VALUE, "ks must be >= 0");
    if (ks > 0 && dtype == FTGEMM_F32_SIMT) return fail(FTGEMM_ERR_UNSUPPORTED, "online-interval mode: tensor-core dtypes");
    if (ks > 0 && (ft_level == FTGEMM_FT_OFF || ft_level == FTGEMM_FT_DETECT_ROWS))
        return fail(FTGEMM_ERR_INVALID_VALUE, "online-interval mode needs ft_level DETECT or CORRECT");
    if (fuse_a && (dtype == FTGEMM_F32_SIMT || ks > 0 || ft_level == FTGEMM_FT_OFF))
        return fail(FTGEMM_ERR_UNSUPPORTED, "in-kernel encode: tensor-core dtypes, FT on, end-of-K verification");
    if (!A || !B || !C) return fail(FTGEMM_ERR_INVALID_VALUE, "null A, B or C");
    if (lda < K || ldb < N || ldc < N) return fail(FTGEMM_ERR_INVALID_VALUE, "leading dimension too small");
    if (ft_level < FTGEMM_FT_OFF || ft_level > FTGEMM_FT_DETECT_ROWS) return fail(FTGEMM_ERR_INVALID_VALUE, "bad ft_level");
    if (n_inj < 0 || n_inj > kMaxInject || (n_inj > 0 && !inj)) return fail(FTGEMM_ERR_INVALID_VALUE, "bad injection list");
    if (ft_level == FTGEMM_FT_OFF && n_inj > 0) return fail(FTGEMM_ERR_INVALID_VALUE, "fault injection needs ft_level DETECT or CORRECT");
    if (ft_level != FTGEMM_FT_OFF && (!enc_ws || !report_ws)) return fail(FTGEMM_ERR_INVALID_VALUE, "FT needs enc_ws and report_ws");
    if (!std::isfinite(alpha) || !std::isfinite(beta)) return fail(FTGEMM_ERR_INVALID_VALUE, "alpha/beta must be finite");
    const int elt = dtype == FTGEMM_BF16 ? 2 : 4;
    if (!aligned16(A) || !aligned16(B) || !aligned16(C) || (lda * elt) % 16 || (ldb * elt) % 16 || (ldc * elt) % 16)
        return fail(FTGEMM_ERR_UNSUPPORTED, "A, B, C must be 16-byte aligned with 16-byte row pitches");
    if (bt.n > 1 && ((bt.sA * elt) % 16 || (bt.sB * elt) % 16 || (bt.sC * elt) % 16))
        return fail(FTGEMM_ERR_UNSUPPORTED, "batch strides must be multiples of 16 bytes");
    if (bt.n > 1 && bt.sC < M * ldc) return fail(FTGEMM_ERR_INVALID_VALUE, "C problems overlap (stride_c < M * ldc)");
    if (!check_device()) return fail(FTGEMM_ERR_UNSUPPORTED, "no sm_100 (B200) device");

    ftgemm_plan_t p;
    fill_plan(code, M, N, K, &p, bt.n);
    if (ks > 0 && ks % p.bk) return fail(FTGEMM_ERR_INVALID_VALUE, "ks must be a multiple of plan.bk (%d)", p.bk);
    const bool ft = ft_level != FTGEMM_FT_OFF;
    const Geometry g = geometry(p, K);
    const EncLayout L = enc_layout(g, M, N);
    const int64_t enc_stride = bt.n > 1 ? bt.enc_stride : (int64_t)L.total;
    if (ft && bt.n > 1 && (enc_stride < (int64_t)L.total || enc_stride % 256))
        return fail(FTGEMM_ERR_INVALID_VALUE, "enc_stride must be >= plan.enc_bytes and a multiple of 256");
    const int64_t units_m_h = (p.tiles_m + p.cta_group - 1) / p.cta_group;     // tensor-core units per problem
    const int64_t units_pb = dtype == FTGEMM_F32_SIMT ? 0 : units_m_h * p.tiles_n;
    if (units_pb * bt.n >= (1ll << 31)) return fail(FTGEMM_ERR_UNSUPPORTED, "too many tiles in one launch");
    cudaStream_t st = (cudaStream_t)stream;
    const int num_kb = (int)((K + p.bk - 1) / p.bk);

    // ---- faults: resolve to (tile key, k-block, in-tile position), sort ----
    const DevInject* dinj = nullptr;
    if (n_inj > 0) {
        std::vector<DevInject> v((size_t)n_inj);
        std::vector<int> per_tile;
        for (int i = 0; i < n_inj; ++i) {
            const ftgemm_inject_t& f = inj[i];
            // batched: rows of the stacked (batch x M) x N view
            if (f.row < 0 || f.row >= M * bt.n || f.col < 0 || f.col >= N || f.k_elem < 0 ||
                f.bit < 0 || f.bit > 31 || f.mode < 0 || f.mode > 1 || f.target < 0 || f.target > 2)
                return fail(FTGEMM_ERR_INVALID_VALUE, "injection %d out of range", i);
            const int64_t pb = f.row / M, row = f.row - pb * M;
            const int ti = (int)(row / p.check_tile_m), tj = (int)(f.col / p.check_tile_n);
            DevInject d;
            d.tile = (int)(pb * units_pb) + tile_key(p, ti, tj);
            d.kb = (int)std::min<int64_t>(f.k_elem / p.bk, num_kb - 1);
            d.p = (int)(row - (int64_t)ti * p.check_tile_m);
            d.q = (int)(f.col - (int64_t)tj * p.check_tile_n);
            d.bit = f.bit; d.mode = f.mode; d.addend = f.addend;
            // CTA of the pair that owns the tile in bits 8+ (the epilogue filters on it)
            d.target = f.target | (dtype == FTGEMM_F32_SIMT ? 0 : (ti % p.cta_group) << 8);
            v[i] = d;
        }
        std::stable_sort(v.begin(), v.end(), [](const DevInject& x, const DevInject& y) {
            return x.tile != y.tile ? x.tile < y.tile : x.kb < y.kb;
        });
        if (dtype == FTGEMM_F32_SIMT) {
            int run = 1;
            for (int i = 1; i < n_inj; ++i) {
                run = v[i].tile == v[i - 1].tile ? run + 1 : 1;
                if (run > 8) return fail(FTGEMM_ERR_INVALID_VALUE, "at most 8 faults per SIMT tile");
            }
        }
        char* dst = reinterpret_cast<char*>(report_ws) + report_inject_offset();
        cudaError_t ce = cudaMemcpyAsync(dst, v.data(), sizeof(DevInject) * v.size(), cudaMemcpyHostToDevice, st);
        if (ce != cudaSuccess) return fail_cuda(ce, "fault-list upload");
        dinj = reinterpret_cast<const DevInject*>(dst);
    }

    const char* enc = reinterpret_cast<const char*>(enc_ws);
    const float tau_u = p.u_acc, l1 = p.lambda1, l2 = p.lambda2, sqk = std::sqrt((float)K);
    cudaError_t ce;
    if (dtype == FTGEMM_F32_SIMT) {
        SimtArgs a{};
        a.M = (int)M; a.N = (int)N; a.K = (int)K; a.num_kb = num_kb;
        a.tiles_m = (int)p.tiles_m; a.tiles_n = (int)p.tiles_n; a.ft_level = ft_level;
        a.alpha = alpha; a.beta = beta;
        a.A = (const float*)A; a.lda = lda; a.B = (const float*)B; a.ldb = ldb; a.C = (float*)C; a.ldc = ldc;
        if (ft) {
            a.Ac = (const float*)(enc + L.ac); a.Br = (const float*)(enc + L.br); a.kp = g.kp;
            a.rownorm = (const float*)(enc + L.rownorm); a.colnorm = (const float*)(enc + L.colnorm);
            a.acnorm = (const float*)(enc + L.acnorm); a.brnorm = (const float*)(enc + L.brnorm);
        }
        a.tau_u = tau_u; a.tau_l1 = l1; a.tau_l2 = l2; a.sqrtK = sqk;
        a.rep = (ReportDev*)report_ws; a.inj = dinj; a.n_inj = n_inj;
        ce = launch_simt(ft, a, st);
    } else {
        const bool tf32 = dtype == FTGEMM_TF32;
        const CUtensorMapDataType dt = tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        const int bmd = ft ? p.check_tile_m : p.off_tile_m;
        const int bnd = ft ? p.check_tile_n : p.off_tile_n;
        const uint32_t boxn = 128 / elt;
        CUtensorMap mA, mB;
        if ((e = make_map(&mA, dt, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda * elt, (uint32_t)p.bk, (uint32_t)bmd,
                          CU_TENSOR_MAP_SWIZZLE_128B, Batch{(uint64_t)bt.n, (uint64_t)(bt.sA * elt)}))) return e;
        const Batch benc{(uint64_t)bt.n, (uint64_t)enc_stride};
        // B (N-major, 128-byte column slices): one 3-D request per stage when the
        // column count is a whole number of slices (B^r always is), else one
        // 2-D box per slice
        const CUtensorMapSwizzle bsw = tf32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
        const uint32_t nbox_cta = (uint32_t)(p.bn / boxn / p.cta_group);
        bool b3d = FTGEMM_B3D != 0;
#if defined(FTGEMM_EXP_B_DIRECT)
        if (false) {
#else
        if (ft) {
#endif
            // the encoded operand B^r (N-major, kp rows of tiles_n * bn) from the encode workspace
            const uint64_t ldt = (uint64_t)g.tiles_n * p.bn;
            if (b3d) e = make_map_3d(&mB, dt, enc + L.bt, boxn, (uint64_t)g.kp, ldt / boxn, ldt * elt, (uint32_t)p.bk,
                                     nbox_cta, bsw, benc);
            else e = make_map(&mB, dt, enc + L.bt, ldt, (uint64_t)g.kp, ldt * elt, boxn, (uint32_t)p.bk, bsw, benc);
            if (e) return e;
        } else {
            b3d = b3d && (N % boxn) == 0;
            const Batch bb{(uint64_t)bt.n, (uint64_t)(bt.sB * elt)};
            if (b3d) e = make_map_3d(&mB, dt, B, boxn, (uint64_t)K, (uint64_t)N / boxn, (uint64_t)ldb * elt,
                                     (uint32_t)p.bk, nbox_cta, bsw, bb);
            else e = make_map(&mB, dt, B, (uint64_t)N, (uint64_t)K, (uint64_t)ldb * elt, boxn, (uint32_t)p.bk, bsw, bb);
            if (e) return e;
        }
        // C: 128-byte rows of output per thread, 32-row boxes (29 rows for the
        // last epilogue warp of a 125-row check tile)
        CUtensorMap mC, mC29;
        const CUtensorMapDataType dc = tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        const Batch bc{(uint64_t)bt.n, (uint64_t)(bt.sC * elt)};
        if ((e = make_map(&mC, dc, C, (uint64_t)N, (uint64_t)M, (uint64_t)ldc * elt, boxn, 32, CU_TENSOR_MAP_SWIZZLE_128B,
                          bc))) return e;
        if ((e = make_map(&mC29, dc, C, (uint64_t)N, (uint64_t)M, (uint64_t)ldc * elt, boxn, ft ? 29 : 32,
                          CU_TENSOR_MAP_SWIZZLE_128B, bc))) return e;
        TcArgs a{};
        a.M = (int)M; a.N = (int)N; a.K = (int)K; a.num_kb = num_kb;
        a.tiles_m = (int)((M + bmd - 1) / bmd); a.tiles_n = (int)((N + bnd - 1) / bnd);
        a.num_tiles = a.tiles_m * a.tiles_n;
        a.units_m = (a.tiles_m + p.cta_group - 1) / p.cta_group;
        a.units_pb = a.units_m * a.tiles_n;
        a.num_units = (int)(a.units_pb * bt.n);
        a.enc_bs = enc_stride / 4;
        a.c_bs = bt.sC;
        a.group = tc_group(a.units_m, p.cta_group);
        a.fd_upb = FastDiv::make((uint32_t)a.units_pb);
        a.fd_pg = FastDiv::make((uint32_t)(a.group * a.tiles_n));
        a.fd_g = FastDiv::make((uint32_t)a.group);
        a.fd_gt = FastDiv::make((uint32_t)(a.units_m % a.group ? a.units_m % a.group : a.group));
        a.ft_level = ft_level; a.alpha = alpha; a.beta = beta; a.C = C; a.ldc = ldc;
        a.ks_kb = ks > 0 ? (int)std::min<int64_t>(ks / p.bk, num_kb) : 0;
        a.fuse_a = fuse_a;
        a.y_warp = (num_kb > 4 || fuse_a) ? 1 : 0;     // the in-kernel encode's flag waits live in the Y warp
        a.b3d = b3d ? 1 : 0;
        if (ft) {
            a.Y = enc + L.y; a.kp = g.kp;
            a.rownorm = (const float*)(enc + L.rownorm); a.colnorm = (const float*)(enc + L.colnorm);
            a.acnorm = (const float*)(enc + L.acnorm); a.brnorm = (const float*)(enc + L.brnorm);
        }
        if (fuse_a) {
            // the encoder warps' item flags start cleared on every launch (so a
            // replayed or aborted launch never sees stale items)
            a.A = A; a.lda = lda;
            a.fflag = (uint32_t*)(enc + L.fflag);
            a.frn2 = (float*)(enc + L.frn2);
            a.facn2 = (float*)(enc + L.facn2);
            a.nkb4 = (g.nkb + 3) & ~3;
            if ((ce = cudaMemsetAsync(a.fflag, 0, sizeof(uint32_t) * ((size_t)g.tiles_m * g.nkb + 2), st)) != cudaSuccess)
                return fail_cuda(ce, "in-kernel encode flags");
        }
        a.tau_u = tau_u; a.tau_l1 = l1; a.tau_l2 = l2; a.sqrtK = sqk;
        a.rep = (ReportDev*)report_ws; a.inj = dinj; a.n_inj = n_inj;
        // pre-swizzled split rows of A^c: one 384-byte row per (check tile, k-block)
        CUtensorMap mY{};
        if (ft && (e = make_map(&mY, CU_TENSOR_MAP_DATA_TYPE_UINT32, enc + L.y, 96, (uint64_t)g.tiles_m * g.nkb, 384,
                                96, 1, CU_TENSOR_MAP_SWIZZLE_NONE, benc))) return e;
        // small K (<= 4 k-blocks): the verification pass bounds the kernel; the
        // narrow one-CTA TF32 tile then runs three epilogue warpgroups (three tiles
        // in flight; 16384^2 x 128: 0.367 -> 0.334 ms).  The BF16 epilogue spills
        // at the 128 registers three warpgroups allow and measured slower.
        const int ext = fuse_a ? 1 : (ks > 0 ? 2 : 0);   // the extended-mode instantiations
        const int epi = (ft && tf32 && p.bn == 128 && p.cta_group == 1 && num_kb <= 4 && !ext) ? 3 : 2;
        ce = launch_tc(tf32, p.bn, ft, p.cta_group, epi, ext, mA, mB, mC, mC29, mY, a, st);
    }
    if (ce != cudaSuccess) return fail_cuda(ce, "kernel launch");
    g_err.clear();
    return FTGEMM_OK;
}

int ftgemm_encode(int code, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B,
                  int64_t ldb, void* enc_ws, int which, void* stream) {
    return encode_impl(code, 1, M, N, K, A, lda, 0, B, ldb, 0, enc_ws, 0, which, stream);
}

int ftgemm_encode_batched(int code, int64_t batch, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                          int64_t stride_a, const void* B, int64_t ldb, int64_t stride_b, void* enc_ws,
                          int64_t enc_stride, int which, void* stream) {
    return encode_impl(code, batch, M, N, K, A, lda, stride_a, B, ldb, stride_b, enc_ws, enc_stride, which, stream);
}

int ftgemm_plan_batched(int code, int64_t batch, int64_t M, int64_t N, int64_t K, ftgemm_plan_t* out) {
    if (!out) return fail(FTGEMM_ERR_INVALID_VALUE, "null plan pointer");
    int e = check_dims(code, M, N, K);
    if (e) return e;
    if (batch < 1) return fail(FTGEMM_ERR_INVALID_VALUE, "batch must be >= 1");
    fill_plan(code, M, N, K, out, batch);
    const Geometry g = geometry(*out, K);
    const EncLayout L = enc_layout(g, M, N);
    out->enc_bytes = (int64_t)L.total;
    out->enc_b_offset = (int64_t)L.b_off;
    out->enc_b_bytes = (int64_t)L.b_bytes;
    out->report_bytes = (int64_t)report_bytes();
    g_err.clear();
    return FTGEMM_OK;
}

int ftgemm_run_batched(int code, int64_t batch, int64_t M, int64_t N, int64_t K, float alpha, const void* A,
                       int64_t lda, int64_t stride_a, const void* B, int64_t ldb, int64_t stride_b, float beta, void* C,
                       int64_t ldc, int64_t stride_c, const void* enc_ws, int64_t enc_stride, int ft_level,
                       const ftgemm_inject_t* inj, int32_t n_inj, void* report_ws, void* stream) {
    BatchArgs bt;
    bt.n = batch; bt.sA = stride_a; bt.sB = stride_b; bt.sC = stride_c; bt.enc_stride = enc_stride;
    return run_impl(code, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, enc_ws, ft_level, 0, 0, inj, n_inj, report_ws,
                    stream, bt);
}

int ftgemm_run(int dtype, int64_t M, int64_t N, int64_t K, float alpha, const void* A, int64_t lda,
               const void* B, int64_t ldb, float beta, void* C, int64_t ldc, const void* enc_ws, int ft_level,
               const ftgemm_inject_t* inj, int32_t n_inj, void* report_ws, void* stream) {
    return run_impl(dtype, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, enc_ws, ft_level, 0, 0, inj, n_inj, report_ws,
                    stream);
}

int ftgemm_run_fused(int dtype, int64_t M, int64_t N, int64_t K, float alpha, const void* A, int64_t lda,
                     const void* B, int64_t ldb, float beta, void* C, int64_t ldc, const void* enc_ws, int ft_level,
                     const ftgemm_inject_t* inj, int32_t n_inj, void* report_ws, void* stream) {
    return run_impl(dtype, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, enc_ws, ft_level, 0, 1, inj, n_inj, report_ws,
                    stream);
}

int ftgemm_run_online(int dtype, int64_t M, int64_t N, int64_t K, float alpha, const void* A, int64_t lda,
                      const void* B, int64_t ldb, float beta, void* C, int64_t ldc, const void* enc_ws, int ft_level,
                      int64_t ks, const ftgemm_inject_t* inj, int32_t n_inj, void* report_ws, void* stream) {
    if (ks < 1) return fail(FTGEMM_ERR_INVALID_VALUE, "ks must be >= 1");
    return run_impl(dtype, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, enc_ws, ft_level, ks, 0, inj, n_inj, report_ws,
                    stream);
}

int ftgemm_nonfused_workspace(int code, int64_t M, int64_t N, int64_t K, int64_t* bytes) {
    int e = check_dims(code, M, N, K);
    if (e) return e;
    const int dtype = code & FTGEMM_DTYPE_MASK;
    if (!bytes) return fail(FTGEMM_ERR_INVALID_VALUE, "null bytes");
    if (dtype == FTGEMM_TF32) return fail(FTGEMM_ERR_UNSUPPORTED, "non-fused baseline: BF16 and F32_SIMT only");
    ftgemm_plan_t p;
    fill_plan(code, M, N, K, &p);
    *bytes = (int64_t)nonfused_ws_bytes(geometry(p, K), M, N);
    g_err.clear();
    return FTGEMM_OK;
}

int ftgemm_run_nonfused(int code, int64_t M, int64_t N, int64_t K, float alpha, const void* A, int64_t lda,
                        const void* B, int64_t ldb, float beta, void* C, int64_t ldc, const void* enc_ws,
                        void* nf_ws, int ft_level, const ftgemm_inject_t* inj, int32_t n_inj, void* report_ws,
                        void* stream) {
    int e = check_dims(code, M, N, K);
    if (e) return e;
    const int dtype = code & FTGEMM_DTYPE_MASK;
    if (dtype == FTGEMM_TF32) return fail(FTGEMM_ERR_UNSUPPORTED, "non-fused baseline: BF16 and F32_SIMT only");
    if (!A || !B || !C) return fail(FTGEMM_ERR_INVALID_VALUE, "null A, B or C");
    if (lda < K || ldb < N || ldc < N) return fail(FTGEMM_ERR_INVALID_VALUE, "leading dimension too small");
    if (ft_level < FTGEMM_FT_OFF || ft_level > FTGEMM_FT_DETECT_ROWS) return fail(FTGEMM_ERR_INVALID_VALUE, "bad ft_level");
    if (n_inj < 0 || n_inj > kMaxInject || (n_inj > 0 && !inj)) return fail(FTGEMM_ERR_INVALID_VALUE, "bad injection list");
    if (ft_level == FTGEMM_FT_OFF && n_inj > 0) return fail(FTGEMM_ERR_INVALID_VALUE, "fault injection needs FT on");
    if (ft_level != FTGEMM_FT_OFF && (!enc_ws || !nf_ws || !report_ws))
        return fail(FTGEMM_ERR_INVALID_VALUE, "FT needs enc_ws, nf_ws and report_ws");
    if (!std::isfinite(alpha) || !std::isfinite(beta)) return fail(FTGEMM_ERR_INVALID_VALUE, "alpha/beta must be finite");
    const int elt = dtype == FTGEMM_BF16 ? 2 : 4;
    if (!aligned16(A) || !aligned16(B) || !aligned16(C) || (lda * elt) % 16 || (ldb * elt) % 16 || (ldc * elt) % 16)
        return fail(FTGEMM_ERR_UNSUPPORTED, "A, B, C must be 16-byte aligned with 16-byte row pitches");
    if (!check_device()) return fail(FTGEMM_ERR_UNSUPPORTED, "no sm_100 (B200) device");
    ftgemm_plan_t p;
    fill_plan(code, M, N, K, &p);
    const Geometry g = geometry(p, K);
    const EncLayout L = enc_layout(g, M, N);
    cudaStream_t st = (cudaStream_t)stream;
    const NfInject* dinj = nullptr;
    if (n_inj > 0) {
        std::vector<NfInject> v((size_t)n_inj);
        for (int i = 0; i < n_inj; ++i) {
            const ftgemm_inject_t& f = inj[i];
            if (f.row < 0 || f.row >= M || f.col < 0 || f.col >= N || f.bit < 0 || f.bit > 31 || f.mode < 0 ||
                f.mode > 1 || f.target < 0 || f.target > 2)
                return fail(FTGEMM_ERR_INVALID_VALUE, "injection %d out of range", i);
            v[i] = NfInject{f.row, f.col, f.bit, f.mode, f.target, f.addend};
        }
        char* dst = reinterpret_cast<char*>(report_ws) + report_inject_offset();
        cudaError_t ce = cudaMemcpyAsync(dst, v.data(), sizeof(NfInject) * v.size(), cudaMemcpyHostToDevice, st);
        if (ce != cudaSuccess) return fail_cuda(ce, "fault-list upload");
        dinj = reinterpret_cast<const NfInject*>(dst);
    }
    const char* why = "kernel launch";
    cudaError_t ce = launch_nonfused(g, L, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, enc_ws, nf_ws, ft_level, dinj,
                                     n_inj, reinterpret_cast<ReportDev*>(report_ws), p.u_acc, p.lambda1, p.lambda2, st,
                                     &why);
    if (ce != cudaSuccess) return fail_cuda(ce, why);
    g_err.clear();
    return FTGEMM_OK;
}

int ftgemm_run_offline(int dtype, int64_t M, int64_t N, int64_t K, float alpha, const void* A, int64_t lda,
                       const void* B, int64_t ldb, float beta, void* C, int64_t ldc, void* c_backup,
                       const void* enc_ws, const ftgemm_inject_t* inj, const int32_t* inj_run, int32_t n_inj,
                       int32_t max_runs, void* report_ws, int32_t* out, void* stream) {
    if (!out) return fail(FTGEMM_ERR_INVALID_VALUE, "null out");
    if (max_runs < 1) return fail(FTGEMM_ERR_INVALID_VALUE, "max_runs must be >= 1");
    if (n_inj < 0 || (n_inj > 0 && !inj)) return fail(FTGEMM_ERR_INVALID_VALUE, "bad injection list");
    if (beta != 0.0f && !c_backup) return fail(FTGEMM_ERR_INVALID_VALUE, "beta != 0 needs c_backup");
    if (!report_ws) return fail(FTGEMM_ERR_INVALID_VALUE, "null report_ws");
    if (inj_run)
        for (int i = 0; i < n_inj; ++i)
            if (inj_run[i] < 0 || inj_run[i] >= max_runs) return fail(FTGEMM_ERR_INVALID_VALUE, "inj_run[%d] out of range", i);
    cudaStream_t st = (cudaStream_t)stream;
    const int elt = (dtype & FTGEMM_DTYPE_MASK) == FTGEMM_BF16 ? 2 : 4;
    const size_t pitch = (size_t)ldc * elt, width = (size_t)N * elt;
    cudaError_t ce;
    if (beta != 0.0f && (ce = cudaMemcpy2DAsync(c_backup, pitch, C, pitch, width, (size_t)M, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        return fail_cuda(ce, "C_in backup");
    const unsigned long long* dcnt = reinterpret_cast<const ReportDev*>(report_ws)->counts;
    unsigned long long det0 = 0, det = 0;
    if ((ce = cudaMemcpyAsync(&det0, dcnt + CNT_DETECTED, sizeof(det0), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (ce = cudaStreamSynchronize(st)) != cudaSuccess)
        return fail_cuda(ce, "report read");
    std::vector<ftgemm_inject_t> mine;
    int runs = 0, clean = 0;
    for (int r = 0; r < max_runs && !clean; ++r) {
        if (r > 0 && beta != 0.0f &&
            (ce = cudaMemcpy2DAsync(C, pitch, c_backup, pitch, width, (size_t)M, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
            return fail_cuda(ce, "C_in restore");
        mine.clear();
        for (int i = 0; i < n_inj; ++i)
            if ((inj_run ? inj_run[i] : 0) == r) mine.push_back(inj[i]);
        int e = ftgemm_run(dtype, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, enc_ws, FTGEMM_FT_DETECT_ROWS,
                           mine.empty() ? nullptr : mine.data(), (int32_t)mine.size(), report_ws, stream);
        if (e) return e;
        ++runs;
        // the restart decision needs this execution's verdict
        if ((ce = cudaMemcpyAsync(&det, dcnt + CNT_DETECTED, sizeof(det), cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
            (ce = cudaStreamSynchronize(st)) != cudaSuccess)
            return fail_cuda(ce, "report read");
        clean = det == det0;
        det0 = det;
    }
    out[0] = runs;
    out[1] = clean;
    g_err.clear();
    return FTGEMM_OK;
}

int ftgemm_cost_model(double gamma0, int64_t tiles, ftgemm_cost_t* out) {
    if (!out) return fail(FTGEMM_ERR_INVALID_VALUE, "null out");
    if (!(gamma0 >= 0.0 && gamma0 < 1.0) || tiles < 1) return fail(FTGEMM_ERR_INVALID_VALUE, "need 0 <= gamma0 < 1, tiles >= 1");
    out->gamma0 = gamma0;
    out->tiles = tiles;
    // gamma = 1 - (1 - gamma0)^tiles, via log1p/expm1 for small gamma0
    out->gamma = -std::expm1((double)tiles * std::log1p(-gamma0));
    out->online_expected_runs = 1.0;
    out->offline_expected_runs = out->gamma < 0.5 ? (1.0 - out->gamma) / (1.0 - 2.0 * out->gamma)
                                                  : std::numeric_limits<double>::infinity();
    g_err.clear();
    return FTGEMM_OK;
}

int ftgemm_report(const void* report_ws, ftgemm_counts_t* counts, ftgemm_event_t* events, int32_t max_events,
                  void* stream) {
    if (!report_ws || !counts || max_events < 0 || (max_events > 0 && !events))
        return fail(FTGEMM_ERR_INVALID_VALUE, "bad report arguments");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) return fail_cuda(ce, "stream (asynchronous kernel fault)");
    unsigned long long c[8];
    ce = cudaMemcpy(c, report_ws, sizeof(c), cudaMemcpyDeviceToHost);
    if (ce != cudaSuccess) return fail_cuda(ce, "report copy");
    counts->tiles_checked = (int64_t)c[CNT_CHECKED];
    counts->tiles_detected = (int64_t)c[CNT_DETECTED];
    counts->corrected = (int64_t)c[CNT_CORRECTED];
    counts->checksum_only = (int64_t)c[CNT_CHECKSUM_ONLY];
    counts->uncorrectable = (int64_t)c[CNT_UNCORRECTABLE];
    counts->located = (int64_t)c[CNT_LOCATED];
    counts->events = (int64_t)c[CNT_EVENTS];
    counts->dropped = (int64_t)c[CNT_DROPPED];
    unsigned int mr = 0;
    ce = cudaMemcpy(&mr, reinterpret_cast<const char*>(report_ws) + offsetof(ReportDev, max_ratio_bits), sizeof(mr),
                    cudaMemcpyDeviceToHost);
    if (ce != cudaSuccess) return fail_cuda(ce, "report copy");
    std::memcpy(&counts->max_resid_ratio, &mr, sizeof(float));
    counts->pad = 0;
    const int64_t stored = std::min<int64_t>(counts->events, kMaxEvents);
    const int64_t n = std::min<int64_t>(stored, max_events);
    if (n > 0) {
        ce = cudaMemcpy(events, reinterpret_cast<const char*>(report_ws) + offsetof(ReportDev, events),
                        sizeof(ftgemm_event_t) * (size_t)n, cudaMemcpyDeviceToHost);
        if (ce != cudaSuccess) return fail_cuda(ce, "event copy");
    }
    g_err.clear();
    return FTGEMM_OK;
}

int ftgemm_report_reset(void* report_ws, int64_t report_bytes_, void* stream) {
    if (!report_ws || report_bytes_ < (int64_t)sizeof(ReportDev)) return fail(FTGEMM_ERR_INVALID_VALUE, "bad report workspace");
    cudaError_t ce = cudaMemsetAsync(report_ws, 0, sizeof(ReportDev), (cudaStream_t)stream);
    if (ce != cudaSuccess) return fail_cuda(ce, "report reset");
    g_err.clear();
    return FTGEMM_OK;
}

}  // extern "C"
