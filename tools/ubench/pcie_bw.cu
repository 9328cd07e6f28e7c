// Host<->device copy throughput on the box: one large copy per direction, both directions at
// once, and runs of page-sized copies (one cudaMemcpyAsync per page-sized copy, as the offload engine
// issues them).
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                    \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess) {                                                 \
            std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            return 1;                                                            \
        }                                                                        \
    } while (0)

int main() {
    const size_t big = size_t(1) << 30;
    void *h = nullptr, *h2 = nullptr, *d = nullptr, *d2 = nullptr;
    CK(cudaHostAlloc(&h, big, cudaHostAllocDefault));
    CK(cudaHostAlloc(&h2, big, cudaHostAllocDefault));
    CK(cudaMalloc(&d, big));
    CK(cudaMalloc(&d2, big));
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t a, b, c, e;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventCreate(&c));
    CK(cudaEventCreate(&e));
    auto gbps = [](size_t bytes, float ms) { return bytes / (ms * 1e-3) / 1e9; };
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(a, s1));
        CK(cudaMemcpyAsync(d, h, big, cudaMemcpyHostToDevice, s1));
        CK(cudaEventRecord(b, s1));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        if (rep) std::printf("H2D 1 GiB: %.1f GB/s\n", gbps(big, ms));
        CK(cudaEventRecord(a, s1));
        CK(cudaMemcpyAsync(h, d, big, cudaMemcpyDeviceToHost, s1));
        CK(cudaEventRecord(b, s1));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        if (rep) std::printf("D2H 1 GiB: %.1f GB/s\n", gbps(big, ms));
        CK(cudaEventRecord(a, s1));
        CK(cudaStreamWaitEvent(s2, a, 0));
        CK(cudaMemcpyAsync(d, h, big, cudaMemcpyHostToDevice, s1));
        CK(cudaMemcpyAsync(h2, d2, big, cudaMemcpyDeviceToHost, s2));
        CK(cudaEventRecord(b, s1));
        CK(cudaEventRecord(c, s2));
        CK(cudaEventSynchronize(b));
        CK(cudaEventSynchronize(c));
        float m2 = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        CK(cudaEventElapsedTime(&m2, a, c));
        if (rep) std::printf("both at once: H2D %.1f GB/s, D2H %.1f GB/s\n", gbps(big, ms), gbps(big, m2));
    }
    // page batches: n pages of K, V (128 KB) + dK, dV (256 KB) into scattered slots
    for (int pages : {16, 70, 256}) {
        for (int both = 0; both < 2; ++both) {
            std::vector<void*> dst, src, dst2, src2;
            std::vector<size_t> sz;
            for (int p = 0; p < pages; ++p) {
                const size_t slot = (size_t(p) * 37) % 1024;  // scattered device slots
                const size_t sizes[4] = {131072, 131072, 262144, 262144};
                size_t off = 0;
                for (int j = 0; j < 4; ++j) {
                    dst.push_back(static_cast<char*>(d) + slot * 786432 + off);
                    src.push_back(static_cast<char*>(h) + size_t(p) * 786432 + off);
                    dst2.push_back(static_cast<char*>(h2) + size_t(p) * 786432 + off);
                    src2.push_back(static_cast<char*>(d2) + slot * 786432 + off);
                    sz.push_back(sizes[j]);
                    off += sizes[j];
                }
            }
            float best = 1e9, best2 = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                CK(cudaEventRecord(a, s1));
                CK(cudaStreamWaitEvent(s2, a, 0));
                for (size_t j = 0; j < sz.size(); ++j) {
                    CK(cudaMemcpyAsync(dst[j], src[j], sz[j], cudaMemcpyHostToDevice, s1));
                    if (both) CK(cudaMemcpyAsync(dst2[j], src2[j], sz[j], cudaMemcpyDeviceToHost, s2));
                }
                CK(cudaEventRecord(b, s1));
                CK(cudaEventRecord(c, s2));
                CK(cudaEventSynchronize(b));
                CK(cudaEventSynchronize(c));
                float m2 = 0;
                CK(cudaEventElapsedTime(&ms, a, b));
                CK(cudaEventElapsedTime(&m2, a, c));
                best = ms < best ? ms : best;
                best2 = m2 < best2 ? m2 : best2;
            }
            const size_t bytes = size_t(pages) * 786432;
            if (both)
                std::printf("batch %3d pages (%zu copies) both directions: H2D %.1f GB/s (%.3f ms), D2H %.1f GB/s\n",
                            pages, sz.size(), gbps(bytes, best), best, gbps(bytes, best2));
            else
                std::printf("batch %3d pages (%zu copies) H2D: %.1f GB/s (%.3f ms)\n", pages, sz.size(),
                            gbps(bytes, best), best);
        }
    }
    return 0;
}
