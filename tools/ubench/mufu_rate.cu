// MUFU.EX2 / FFMA / FFMA2 issue rates per SM on this GPU: one CTA per SM, W warps, each thread
// runs N independent chains. Prints SM clocks per warp-instruction for each op.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f - 1.f;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            if (OP == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0fBF000000;" : "+f"(a[i]));
            if (OP == 2) {
                unsigned long long v = *reinterpret_cast<unsigned long long*>(&a[i & 6]);
                asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v));
                *reinterpret_cast<unsigned long long*>(&a[i & 6]) = v;
            }
            if (OP == 4) {  // F2FP.BF16.F32.PACK_AB alone
                unsigned int h;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(h) : "f"(a[i]));
                a[i] = __uint_as_float(h) + 1e-30f;
            }
            if (OP == 5) {  // one ex2 and one bf16x2 pack per element, independent chains
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
                unsigned int h;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(h) : "f"(a[(i + 4) & 7]));
                a[(i + 4) & 7] = __uint_as_float(h ^ 0x1u);
            }
            if (OP == 3) {
                unsigned int h;
                asm volatile("cvt.rn.f16x2.f32 %0, %1, %1;" : "=r"(h) : "f"(a[i]));
                asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h));
                a[i] = __uint_as_float(h);
            }
        }
    }
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0)
        printf("op %d warps %d: %.2f clk per warp-instr per SM\n", OP, blockDim.x / 32,
               double(t1 - t0) / (double(iters) * 8 * (blockDim.x / 32)));
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 1024 * sizeof(float));
    for (int w : {4, 8, 16}) {
        k<0><<<148, w * 32>>>(out, 4096);
        k<1><<<148, w * 32>>>(out, 4096);
        k<2><<<148, w * 32>>>(out, 4096);
        k<3><<<148, w * 32>>>(out, 4096);
        k<4><<<148, w * 32>>>(out, 4096);
        k<5><<<148, w * 32>>>(out, 4096);
        cudaDeviceSynchronize();
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
