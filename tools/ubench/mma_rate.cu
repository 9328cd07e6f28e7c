// Microbenchmark: tcgen05.mma issue/throughput for the operand shapes the attention
// kernels use (SS vs TS, N = 32/64/128/256), one CTA per SM, back-to-back MMAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2602_02108_b200/csrc mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace oomb;

template <int N, bool TS, int LDST = 0>
__global__ void __launch_bounds__(256, 1) k_mma(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&tbase);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = tbase;
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    const uint64_t da = make_sdesc_sw128(a, 16, 1024), db = make_sdesc_sw128(b, 16, 1024);
    constexpr uint32_t idesc = make_idesc_bf16(128, N, 0, 0);
    unsigned long long t0 = clock64();
    if (warp == 0) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                if (TS) umma_ts_w(tmem + 256, tmem + ks * 8, db + ks * 2, idesc, 1);
                else umma_ss_w(tmem + 256, da + ks * 2, db + ks * 2, idesc, 1);
            }
        }
        umma_commit_w(&bar);
        mbar_wait(&bar, 0);
    } else if (LDST && warp >= 4) {
        // interference: tcgen05.ld / st of 32 columns in a loop on this warp's lane quarter
        const uint32_t lo = static_cast<uint32_t>((warp & 3) * 32) << 16;
        uint32_t v[32];
        for (int it = 0; it < iters * (LDST == 2 ? 4 : 1); ++it) {
            tmem_ld32(tmem + 64 + lo, v);
            tmem_wait_ld();
            uint32_t w[16];
            for (int u = 0; u < 16; ++u) w[u] = v[u] + v[u + 16];
            tmem_st16(tmem + 64 + lo, w);
            tmem_wait_st();
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N, bool TS, int LDST = 0>
void run(int sms) {
    unsigned long long* d; cudaMalloc(&d, sms * 8);
    auto k = k_mma<N, TS, LDST>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int iters = 2000;
    k<<<sms, 256, 160 * 1024>>>(10, d);
    k<<<sms, 256, 160 * 1024>>>(iters, d);
    cudaDeviceSynchronize();
    unsigned long long h[256]; cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < sms; ++i) mx = mx > h[i] ? mx : h[i];
    const double fma = 128.0 * N * 16;
    const double clk = mx / (iters * 8.0);
    printf("ldst=%d %s N=%3d:", LDST, TS ? "TS" : "SS", N); printf(" %6.1f clk/MMA  -> %6.0f FMA/clk/SM (%.0f%% of 4096)  err=%s\n", TS ? "TS" : "SS", N, clk, fma / clk,
           fma / clk / 4096 * 100, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}


// The dK/dV kernel's per-half MMA mix: 8 x (N=32) into S, 8 x (N=32) into dP, 2 x (N=128) into
// dV, 2 x (N=128) into dK, repeated; expected 16*16.5 + 4*64 = 520 clk per group without bubbles.
template <int MODE>
__global__ void __launch_bounds__(128, 1) k_mix(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&tbase);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = tbase;
    const uint32_t b = smem_u32(smem + 65536);
    const uint64_t db = make_sdesc_sw128(b, 16, 1024);
    const uint64_t dbmn = make_sdesc_sw128(b, 8192, 1024);
    constexpr uint32_t id32 = make_idesc_bf16(128, 32, 0, 0);
    constexpr uint32_t id128 = make_idesc_bf16(128, 128, 0, 1);
    unsigned long long t0 = clock64();
    if (warp == 0) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) umma_ts_w(tmem + 128, tmem + ks * 8, db + ks * 2, id32, ks);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) umma_ts_w(tmem + 192, tmem + 64 + ks * 8, db + ks * 2, id32, ks);
            if (MODE >= 1) {
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) umma_ts_w(tmem + 256, tmem + 128 + ks * 8, dbmn + ks * 128, id128, 1);
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) umma_ts_w(tmem + 384, tmem + 192 + ks * 8, dbmn + ks * 128, id128, 1);
            }
            if (MODE == 2) umma_commit_w(&bar);  // a commit per group (as the kernel does)
        }
        umma_commit_w(&bar);
        mbar_wait(&bar, MODE == 2 ? (iters & 1) : 0);
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}
template <int MODE>
void run_mix(int sms) {
    unsigned long long* d; cudaMalloc(&d, sms * 8);
    auto k = k_mix<MODE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int iters = 1000;
    k<<<sms, 128, 160 * 1024>>>(10, d);
    k<<<sms, 128, 160 * 1024>>>(iters, d);
    cudaDeviceSynchronize();
    unsigned long long h[256]; cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < sms; ++i) mx = mx > h[i] ? mx : h[i];
    printf("mix mode %d: %.1f clk per group (ideal %d)  err=%s\n", MODE, mx / iters, MODE ? 520 : 264,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

// Round trip: issue G MMAs (TS, N=128), commit to an mbarrier, wait for it, repeat; the excess
// over G*64 clk per group is the drain + commit + wake-up latency a dependency costs.
template <int G>
__global__ void __launch_bounds__(128, 1) k_rt(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&tbase);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = tbase;
    const uint64_t db = make_sdesc_sw128(smem_u32(smem + 65536), 16, 1024);
    constexpr uint32_t id = make_idesc_bf16(128, 128, 0, 0);
    unsigned long long t0 = clock64();
    if (warp == 0) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < G; ++k) umma_ts_w(tmem + 256, tmem + (k & 7) * 8, db + (k & 7) * 2, id, 1);
            umma_commit_w(&bar);
            mbar_wait(&bar, it & 1);
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}
template <int G>
void run_rt(int sms) {
    unsigned long long* d; cudaMalloc(&d, sms * 8);
    auto k = k_rt<G>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int iters = 2000;
    k<<<sms, 128, 160 * 1024>>>(10, d);
    k<<<sms, 128, 160 * 1024>>>(iters, d);
    cudaDeviceSynchronize();
    unsigned long long h[256]; cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < sms; ++i) mx = mx > h[i] ? mx : h[i];
    printf("round trip G=%2d: %.0f clk per group (compute %d) -> overhead %.0f clk\n", G, mx / iters, G * 64,
           mx / iters - G * 64);
    cudaFree(d);
}

// Forward-like contention: warp 1 issues S-like TS MMAs (N=128, A = cols [0,64), D = cols
// [64,192)) in groups of 8 with a commit per group; warps 4..11 continuously tcgen05.ld 2 x 32
// columns of [192,320), do 64 ex2 each, and tcgen05.st 2 x 16 columns back (softmax-like).
template <int SM_WORK>
__global__ void __launch_bounds__(384, 1) k_contend(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    __shared__ volatile int done;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); done = 0; }
    if (warp == 0) tmem_alloc<512>(&tbase);
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = tbase;
    const uint64_t db = make_sdesc_sw128(smem_u32(smem + 65536), 16, 1024);
    constexpr uint32_t id = make_idesc_bf16(128, 128, 0, 0);
    unsigned long long t0 = clock64();
    if (warp == 1) {
        const unsigned long long m0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 8; ++k) umma_ts_w(tmem + 64, tmem + k * 8, db + k * 2, id, k);
            umma_commit_w(&bar);
        }
        mbar_wait(&bar, (iters - 1) & 1);
        const unsigned long long m1 = clock64();
        if (lane_id() == 0) { done = 1; out[blockIdx.x] = m1 - m0; }
    } else if (warp >= 4 && SM_WORK) {
        const uint32_t lo = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t base = tmem + 192 + ((warp - 4) >> 2) * 64 + lo;
        float acc = 0.f;
        while (!done) {
            uint32_t a[32], b[32];
            tmem_ld32(base, a);
            tmem_ld32(base + 32, b);
            tmem_wait_ld();
            uint32_t pk[16], pk2[16];
            for (int u = 0; u < 16; ++u) {
                const float e0 = ex2(__uint_as_float(a[2 * u]) * 0.001f - 1.f), e1 = ex2(__uint_as_float(a[2 * u + 1]) * 0.001f - 1.f);
                const float e2 = ex2(__uint_as_float(b[2 * u]) * 0.001f - 1.f), e3 = ex2(__uint_as_float(b[2 * u + 1]) * 0.001f - 1.f);
                acc += e0 + e1 + e2 + e3;
                pk[u] = pack_bf16(e0, e1);
                pk2[u] = pack_bf16(e2, e3);
            }
            tmem_st16(base, pk);
            tmem_st16(base + 16, pk2);
            tmem_wait_st();
        }
        if (acc == 12345.f) out[0] = 1;
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    (void)t1; (void)t0;
    tc_fence_before(); __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}
template <int SM_WORK>
void run_contend(int sms) {
    unsigned long long* d; cudaMalloc(&d, sms * 8);
    auto k = k_contend<SM_WORK>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int iters = 2000;
    k<<<sms, 384, 160 * 1024>>>(10, d);
    printf("launch: %s\n", cudaGetErrorString(cudaGetLastError()));
    k<<<sms, 384, 160 * 1024>>>(iters, d);
    printf("sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    unsigned long long h[256]; cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < sms; ++i) mx = mx > h[i] ? mx : h[i];
    printf("contend softmax_work=%d: %.0f clk per 8-MMA group (ideal 512) h0=%llu err=%s\n", SM_WORK, mx / iters, h[0],
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    int sms = 148;
    run<32, false>(sms); run<64, false>(sms); run<128, false>(sms);
    run<32, true>(sms); run<64, true>(sms); run<128, true>(sms);
    run<32, true, 1>(sms); run<128, true, 1>(sms); run<32, true, 2>(sms); run<128, true, 2>(sms);
    run_mix<0>(sms); run_mix<1>(sms); run_mix<2>(sms);
    run_rt<1>(sms); run_rt<4>(sms); run_rt<8>(sms); run_rt<16>(sms);
    run_contend<0>(sms); run_contend<1>(sms);
    return 0;
}
