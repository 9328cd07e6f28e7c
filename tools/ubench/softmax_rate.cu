// Microbenchmark: the softmax inner loop of the attention kernels in isolation, per SM.
// Each thread owns one TMEM lane (query / key row); per iteration it loads 32 fp32 columns
// (tcgen05.ld 32x32b.x32 + wait::ld), computes p = exp2(s * c - m) for each, adds them to a row
// sum, packs pairs to bf16 and stores 16 packed columns (tcgen05.st 32x32b.x16) back. Variants drop
// one ingredient at a time, so the difference says what bounds the loop. One CTA per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2602_02108_b200/csrc softmax_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace oomb;

// V: 0 full, 1 no MUFU (FMA instead), 2 no TMEM store, 3 no TMEM load (registers), 4 no pack/store
template <int V>
__global__ void k(int iters, float* out, long long* clk) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) tmem_alloc<512>(&tbase);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // warps w and w + 4k share lane quarter w % 4; each warpgroup k uses its own 64-column window
    const uint32_t taddr = tbase + ((static_cast<uint32_t>(warp & 3) * 32) << 16) + ((warp >> 2) & 7) * 64;
    float rs = 0.f, m = 1.f + lane * 1e-3f;
    uint32_t sv[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) sv[i] = __float_as_uint(-0.5f + i * 1e-3f);
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (V != 3) {
            tmem_ld32(taddr, sv);
            tmem_wait_ld();
        }
        uint32_t pk[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const float x0 = fmaf(__uint_as_float(sv[2 * u]), 0.125f, -m);
            const float x1 = fmaf(__uint_as_float(sv[2 * u + 1]), 0.125f, -m);
            float e0, e1;
            if (V == 1) {
                e0 = fmaf(x0, 0.5f, 1.f);
                e1 = fmaf(x1, 0.5f, 1.f);
            } else if (V == 5) {
                e0 = ex2(x0);
                e1 = (u & 1) ? ex2_lean(x1) : ex2(x1);
            } else if (V == 6) {
                e0 = ex2(x0);
                e1 = ex2_lean(x1);
            } else if (V == 7) {
                e0 = (u & 1) ? ex2_lean(x0) : ex2(x0);
                e1 = ex2_lean(x1);
            } else if ((V == 9 && (u & 3) == 3) || (V == 10 && (u & 1))) {
                const float2 e = ex2_lean2(make_float2(x0, x1));
                e0 = e.x;
                e1 = e.y;
            } else {
                e0 = ex2(x0);
                e1 = ex2(x1);
            }
            rs += e0 + e1;
            pk[u] = pack_bf16(e0, e1);
        }
        if (V == 3) {
#pragma unroll
            for (int i = 0; i < 16; ++i) sv[i] = sv[i + 16] ^ pk[i];
        }
        if (V != 2 && V != 4) tmem_st16(taddr + 32, pk);
        if (V == 4) m += __uint_as_float(pk[it & 15]) * 1e-30f;
    }
    if (V != 2 && V != 4) tmem_wait_st();
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = rs + m;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tbase);
}

int main() {
    float* out;
    long long* clk;
    cudaMalloc(&out, 148 * 1024 * sizeof(float));
    cudaMalloc(&clk, 148 * sizeof(long long));
    const char* nm[] = {"full (ld32, 32 FFMA+ex2, pack, st16)", "no MUFU (FMA instead of ex2)", "no TMEM store",
                        "no TMEM load (registers)", "no pack / store", "1 in 4 exp2 on FMA (lean)",
                        "1 in 2 exp2 on FMA (lean)", "3 in 4 exp2 on FMA (lean)", "", "1 in 4 on FMA, packed pairs",
                        "1 in 2 on FMA, packed pairs"};
    const int iters = 4096;
    for (int w : {4, 8, 16}) {
        for (int v = 0; v < 11; ++v) {
            if (v == 8) continue;
            if (v == 0) k<0><<<148, w * 32>>>(iters, out, clk);
            if (v == 1) k<1><<<148, w * 32>>>(iters, out, clk);
            if (v == 2) k<2><<<148, w * 32>>>(iters, out, clk);
            if (v == 3) k<3><<<148, w * 32>>>(iters, out, clk);
            if (v == 4) k<4><<<148, w * 32>>>(iters, out, clk);
            if (v == 5) k<5><<<148, w * 32>>>(iters, out, clk);
            if (v == 6) k<6><<<148, w * 32>>>(iters, out, clk);
            if (v == 7) k<7><<<148, w * 32>>>(iters, out, clk);
            if (v == 9) k<9><<<148, w * 32>>>(iters, out, clk);
            if (v == 10) k<10><<<148, w * 32>>>(iters, out, clk);
            long long c = 0;
            cudaMemcpy(&c, clk, sizeof(c), cudaMemcpyDeviceToHost);
            // elements per SM per clock: w warps x 32 lanes x 32 elements per iteration
            printf("warps %2d  %-40s %6.1f elements/clk/SM\n", w, nm[v], double(w) * 32 * 32 * iters / double(c));
        }
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
