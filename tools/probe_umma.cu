// Standalone probe of tcgen05.mma operand layouts (tf32 / bf16), no TMA.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../paper_2305_01024_b200/csrc/ptx.cuh"
using namespace ftg;

// VAR 0: bf16, B MN-major SW128.  1: tf32, B K-major SW128.  2: tf32, B MN-major SW128_32B.
// 3: tf32 B MN-major SW128 (16B).
template <int VAR>
__global__ void probe(const float* A, const float* B, float* D) {
    constexpr bool TF = VAR != 0;
    constexpr int ELT = TF ? 4 : 2;
    constexpr int KT = 128 / ELT;       // K of the tile (one 128B row)
    constexpr int UK = 32 / ELT;
    constexpr int N = 128;
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = sm;                 // 128 x KT
    uint8_t* sB = sm + 16384;         // N x KT
    __shared__ uint64_t bar;
    __shared__ uint32_t tholder;
    const int tid = threadIdx.x;
    // fill A (K-major SW128)
    for (int idx = tid; idx < 128 * KT; idx += blockDim.x) {
        int m = idx / KT, k = idx % KT;
        int byte = k * ELT;
        int off = m * 128 + (((byte >> 4) ^ (m & 7)) << 4) + (byte & 15);
        float v = A[m * KT + k];
        if (TF) *(float*)(sA + off) = v; else *(__nv_bfloat16*)(sA + off) = __float2bfloat16(v);
    }
    for (int idx = tid; idx < N * KT; idx += blockDim.x) {
        int n = idx / KT, k = idx % KT;
        float v = B[k * N + n];
        int off;
        if (VAR == 1) {          // K-major: rows n
            int byte = k * ELT;
            off = n * 128 + (((byte >> 4) ^ (n & 7)) << 4) + (byte & 15);
        } else {
            const int per = 128 / ELT;  // cols per box
            int b = n / per, nn = n % per, byte = nn * ELT;
            int boxbytes = KT * 128;
            if (VAR == 2) off = b * boxbytes + k * 128 + (((byte >> 5) ^ (k & 3)) << 5) + (byte & 31);
            else off = b * boxbytes + k * 128 + (((byte >> 4) ^ (k & 7)) << 4) + (byte & 15);
        }
        if (TF) *(float*)(sB + off) = v; else *(__nv_bfloat16*)(sB + off) = __float2bfloat16(v);
    }
    if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (tid < 32) tmem_alloc<128>(&tholder);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t tb = tholder;
    if (tid < 32) {
        if (elect_one()) {
            uint32_t idesc = instr_desc(TF, 128, N, false, VAR != 1);
            for (int kk = 0; kk < KT / UK; ++kk) {
                uint64_t ad = smem_desc_sw128<2>(smem_u32(sA) + kk * 32, 16, 1024);
                uint64_t bd;
                if (VAR == 1) bd = smem_desc_sw128<2>(smem_u32(sB) + kk * 32, 16, 1024);
                else if (VAR == 2) bd = smem_desc_sw128<1>(smem_u32(sB) + kk * UK * 128, KT * 128, 512);
                else bd = smem_desc_sw128<2>(smem_u32(sB) + kk * UK * 128, KT * 128, 1024);
                umma<TF>(tb, ad, bd, idesc, kk > 0);
            }
            umma_commit(&bar);
        }
        __syncwarp();
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int w = tid >> 5, lane = tid & 31;
    for (int c = 0; c < N / 32; ++c) {
        float v[32];
        tmem_ld32(tb + ((uint32_t)(w * 32) << 16) + c * 32, v);
        for (int i = 0; i < 32; ++i) D[(w * 32 + lane) * N + c * 32 + i] = v[i];
    }
    tc_fence_before();
    __syncthreads();
    if (tid < 32) { tc_fence_after(); tmem_dealloc<128>(tb); }
}

template <int VAR>
void run(const char* name) {
    constexpr bool TF = VAR != 0;
    const int KT = TF ? 32 : 64, N = 128;
    std::vector<float> A(128 * KT), B(KT * N), D(128 * N), R(128 * N);
    for (int i = 0; i < 128 * KT; ++i) A[i] = (float)((i * 7 + 3) % 9 - 4);
    for (int i = 0; i < KT * N; ++i) B[i] = (float)((i * 5 + 1) % 9 - 4);
    if (TF) { A[0] = 1.0f + ldexpf(1, -11) + ldexpf(1, -12); for (int k = 1; k < KT; ++k) A[k] = 0; B[0] = 1.0f; for (int k = 1; k < KT; ++k) B[k * N] = 0; }
    for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) { double s = 0; for (int k = 0; k < KT; ++k) s += (double)A[m * KT + k] * B[k * N + n]; R[m * N + n] = (float)s; }
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0xFF, D.size() * 4);
    cudaFuncSetAttribute(probe<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    probe<VAR><<<1, 128, 40000>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double mx = 0; int bad = 0;
    for (int i = 1; i < 128 * N; ++i) { double d = fabs(D[i] - R[i]); if (d > mx) mx = d; if (d > 1e-3) ++bad; }
    printf("%-28s err=%s maxabs(excl[0,0])=%g bad=%d D[0,0]=%.10g ref=%.10g D[1,1]=%g ref=%g\n", name, cudaGetErrorString(e), mx, bad,
           D[0], R[0], D[N + 1], R[N + 1]);
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
}

int main() {
    run<0>("bf16 B MN SW128");
    run<1>("tf32 B K SW128");
    run<2>("tf32 B MN SW128_32B");
    run<3>("tf32 B MN SW128");
    return 0;
}
