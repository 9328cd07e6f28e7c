// SPDX-License-Identifier: Apache-2.0
//
// SIMT kernels of the hot path: page append + K_avg, page mean keys,
// gather / scatter-add of page data, lazy gradient-page initialisation,
// exact page scoring (vote), top-k page selection, and the SIMT paged
// attention forward / backward used for fp32 mode (the 1e-5 parity mode) and
// for shapes the tcgen05 kernels do not cover.
//
// Pool layout (device, per slot): K, V  [Hkv][P][hd] (pool dtype);
// gradient pool dK, dV [Hkv][P][hd] fp32. Page tables map logical page ->
// slot per layer (d_kvslot / d_gslot, -1 = none).

#include <cstdlib>
#include <cub/block/block_scan.cuh>

#include "oomb_internal.h"
#include "ptx.cuh"

namespace oomb {

std::atomic<int64_t> g_kernel_launches{0};

void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(OOMB_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
    count_launch();
}

template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// fp64 pools (OOMB_F64: the reference's Real = double) store and accumulate in double; fp32 and
// bf16 pools accumulate in float. to_f / from_f of double exist only for the RoPE helpers, which the
// host never runs on an fp64 pool.
template <>
__device__ __forceinline__ float to_f<double>(double x) { return static_cast<float>(x); }
template <>
__device__ __forceinline__ double from_f<double>(float x) { return x; }
template <typename T>
struct AccOf {
    using type = float;
};
template <>
struct AccOf<double> {
    using type = double;
};
template <typename T>
using acc_t = typename AccOf<T>::type;
template <typename A, typename T>
__device__ __forceinline__ A to_a(T x) { return static_cast<A>(x); }
template <>
__device__ __forceinline__ float to_a<float, __nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T, typename A>
__device__ __forceinline__ T from_a(A x) { return static_cast<T>(x); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_a<__nv_bfloat16, float>(float x) { return __float2bfloat16_rn(x); }
__device__ __forceinline__ float exp_a(float x) { return expf(x); }
__device__ __forceinline__ double exp_a(double x) { return exp(x); }
__device__ __forceinline__ float log_a(float x) { return logf(x); }
__device__ __forceinline__ double log_a(double x) { return log(x); }
__device__ __forceinline__ float max_a(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double max_a(double a, double b) { return fmax(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
template <typename A>
struct Stat {  // score_pages row statistics: max and 1 / sum
    A m, il;
};
template <typename A>
__device__ __forceinline__ A scale_of(const AttnGeom& g);
template <>
__device__ __forceinline__ float scale_of<float>(const AttnGeom& g) { return g.scale; }
template <>
__device__ __forceinline__ double scale_of<double>(const AttnGeom& g) { return g.scale64; }

template <typename A>
__device__ __forceinline__ A warp_sum(A v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <typename A>
__device__ __forceinline__ A warp_max(A v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max_a(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ int valid_in_page(int64_t filled, int pid, int P) {
    int64_t v = filled - static_cast<int64_t>(pid) * P;
    return static_cast<int>(v < 0 ? 0 : (v > P ? P : v));
}

// ===========================================================================
// append_chunk + K_avg  (paged_kv.hpp:73-108)
// One thread per (page touched, h, d): copies the page's new rows in order and
// accumulates kavg_sum in append order -> bit-identical fp32 sums.
// ===========================================================================
// RoPE of one element (ops.hpp:192-225): row at absolute position pos, element d of a head;
// angle = pos * base^(-2i/d) in double (inv_freq precomputed on the host with the reference's
// std::pow), cos / sin in double rounded to Real, then the rotation in Real with no contraction.
template <typename T>
__device__ __forceinline__ float rope_elem(const T* __restrict__ row, int d, double pos, const double* inv_freq) {
    const int i = d >> 1;
    const double ang = pos * inv_freq[i];
    const float c = static_cast<float>(cos(ang)), s = static_cast<float>(sin(ang));
    const float x0 = to_f(row[2 * i]), x1 = to_f(row[2 * i + 1]);
    return (d & 1) ? __fadd_rn(__fmul_rn(x0, s), __fmul_rn(x1, c)) : __fsub_rn(__fmul_rn(x0, c), __fmul_rn(x1, s));
}

template <typename T>
__global__ void append_kernel(const T* __restrict__ k, const T* __restrict__ v, int64_t rows, int64_t filled,
                              int P, int Hkv, int hd, int first_page, NewSlots ns, int32_t* __restrict__ kvslot,
                              T* __restrict__ kpool, T* __restrict__ vpool, acc_t<T>* __restrict__ ksum,
                              int32_t* __restrict__ kcnt, int* err, const double* __restrict__ rope_inv_freq,
                              __nv_bfloat16* __restrict__ planes, int64_t plane_stride) {
    const int re = Hkv * hd;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int pg = first_page + blockIdx.y;
    if (blockIdx.x == 0 && blockIdx.y == 0) {
        for (int i = threadIdx.x; i < ns.n; i += blockDim.x) kvslot[ns.first_page + i] = ns.slot[i];
    }
    if (e >= re) return;
    const bool is_new = pg >= ns.first_page && pg < ns.first_page + ns.n;
    const int slot = is_new ? ns.slot[pg - ns.first_page] : kvslot[pg];
    const int h = e / hd, d = e - (e / hd) * hd;
    const int64_t s0 = max(filled, static_cast<int64_t>(pg) * P);
    const int64_t s1 = min(filled + rows, static_cast<int64_t>(pg + 1) * P);
    acc_t<T> sum = is_new ? acc_t<T>(0) : ksum[static_cast<int64_t>(pg) * re + e];
    // a REMOTE page (another page-range shard stores it) only gets its K_avg sums; a page with no
    // slot at all is not resident (the host checks the tail page first): flag it, write nothing
    const bool store = slot >= 0;
    if (slot == -1 && e == 0) atomicOr(err, DERR_NOT_RESIDENT);
    // rows in batches of 16: all loads of a batch are issued before its stores and the
    // in-order (append order, paged_kv.hpp:98-104) fp32 sum, so 32 loads are in flight per thread
    constexpr int kB = 16;
    const size_t dst0 = ((static_cast<size_t>(store ? slot : 0) * Hkv + h) * P) * hd + d;
    for (int64_t sb = s0; sb < s1; sb += kB) {
        T kb[kB], vb[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            if (sb + u < s1) {
                const int64_t r = sb + u - filled;
                // fused RoPE (chunk_trainer.hpp:424-432): K is rotated at its absolute position
                // on the way into the page, never written back un-rotated
                kb[u] = rope_inv_freq ? from_f<T>(rope_elem(k + r * re + h * hd, d, static_cast<double>(sb + u),
                                                            rope_inv_freq))
                                      : k[r * re + e];
                vb[u] = v[r * re + e];
            }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            if (sb + u < s1) {
                const int off = static_cast<int>(sb + u - static_cast<int64_t>(pg) * P);
                if (store) {
                    kpool[dst0 + static_cast<size_t>(off) * hd] = kb[u];
                    vpool[dst0 + static_cast<size_t>(off) * hd] = vb[u];
                }
                sum = add_rn(sum, to_a<acc_t<T>>(kb[u]));
            }
        }
    }
    ksum[static_cast<int64_t>(pg) * re + e] = sum;
    if (e == 0) kcnt[pg] = (is_new ? 0 : kcnt[pg]) + static_cast<int>(s1 - s0);
    if (planes) {
        // the tcgen05 scorer's hi / lo bf16 planes of K_avg = sum * (1/count) (paged_kv.hpp:177-180),
        // [2][Hkv][plane_stride][hd]: kept current here, so scoring never re-splits completed pages
        const int cnt = static_cast<int>(s1 - static_cast<int64_t>(pg) * P);  // rows the page holds now
        const float kav = __fmul_rn(static_cast<float>(sum), __fdiv_rn(1.0f, static_cast<float>(cnt)));
        const __nv_bfloat16 hi = __float2bfloat16_rn(kav);
        const size_t at = (static_cast<size_t>(h) * plane_stride + pg) * hd + d;
        planes[at] = hi;
        planes[at + static_cast<size_t>(Hkv) * plane_stride * hd] = __float2bfloat16_rn(kav - __bfloat162float(hi));
    }
}

// Staged variant (no RoPE, 64-column slices, 16-byte aligned K / V): a CTA owns one page touched
// and 64 columns of its [Hkv x hd] row. All rows of a 64-row segment are loaded at once with
// 16-byte vectors (copied to the page as they arrive, K also into shared memory), then one thread
// per column adds the segment's K rows in append order: the same add_rn sequence as append_kernel,
// so the sums are bit-identical, with one load latency per segment instead of one per row batch.
constexpr int kAppCols = 64, kAppRows = 64, kAppThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kAppThreads)
    append_staged_kernel(const T* __restrict__ k, const T* __restrict__ v, int64_t rows, int64_t filled, int P,
                         int Hkv, int hd, int first_page, NewSlots ns, int32_t* __restrict__ kvslot,
                         T* __restrict__ kpool, T* __restrict__ vpool, acc_t<T>* __restrict__ ksum,
                         int32_t* __restrict__ kcnt, int* err, __nv_bfloat16* __restrict__ planes,
                         int64_t plane_stride) {
    constexpr int VE = 16 / sizeof(T);   // elements per 16-byte vector
    constexpr int VPR = kAppCols / VE;   // vectors per 64-column row slice
    __shared__ __align__(16) T sk[kAppRows][kAppCols];
    const int re = Hkv * hd;
    const int c0 = blockIdx.x * kAppCols;
    const int h = c0 / hd, d0 = c0 - h * hd;
    const int pg = first_page + blockIdx.y;
    const int tid = threadIdx.x;
    if (blockIdx.x == 0 && blockIdx.y == 0)
        for (int i = tid; i < ns.n; i += blockDim.x) kvslot[ns.first_page + i] = ns.slot[i];
    const bool is_new = pg >= ns.first_page && pg < ns.first_page + ns.n;
    const int slot = is_new ? ns.slot[pg - ns.first_page] : kvslot[pg];
    const int64_t s0 = max(filled, static_cast<int64_t>(pg) * P);
    const int64_t s1 = min(filled + rows, static_cast<int64_t>(pg + 1) * P);
    const bool store = slot >= 0;  // REMOTE pages get only their sums; -1: not resident (flagged)
    if (slot == -1 && tid == 0 && blockIdx.x == 0) atomicOr(err, DERR_NOT_RESIDENT);
    acc_t<T> sum = acc_t<T>(0);
    if (tid < kAppCols && !is_new) sum = ksum[static_cast<int64_t>(pg) * re + c0 + tid];
    const size_t dst0 = ((static_cast<size_t>(store ? slot : 0) * Hkv + h) * P) * hd + d0;
    for (int64_t sb = s0; sb < s1; sb += kAppRows) {
        const int n = static_cast<int>(min(static_cast<int64_t>(kAppRows), s1 - sb));
        for (int idx = tid; idx < n * VPR; idx += kAppThreads) {
            const int u = idx / VPR, j = idx - (idx / VPR) * VPR;
            const int64_t r = sb + u - filled;
            const uint4 kv = *reinterpret_cast<const uint4*>(k + r * re + c0 + j * VE);
            const uint4 vv = *reinterpret_cast<const uint4*>(v + r * re + c0 + j * VE);
            if (store) {
                const size_t off = dst0 + static_cast<size_t>(sb + u - static_cast<int64_t>(pg) * P) * hd + j * VE;
                *reinterpret_cast<uint4*>(kpool + off) = kv;
                *reinterpret_cast<uint4*>(vpool + off) = vv;
            }
            *reinterpret_cast<uint4*>(&sk[u][j * VE]) = kv;
        }
        __syncthreads();
        if (tid < kAppCols)
            for (int u = 0; u < n; ++u) sum = add_rn(sum, to_a<acc_t<T>>(sk[u][tid]));
        __syncthreads();
    }
    if (tid < kAppCols) {
        ksum[static_cast<int64_t>(pg) * re + c0 + tid] = sum;
        if (planes) {  // as append_kernel: the scorer's hi / lo bf16 planes of K_avg
            const int cnt = static_cast<int>(s1 - static_cast<int64_t>(pg) * P);
            const float kav = __fmul_rn(static_cast<float>(sum), __fdiv_rn(1.0f, static_cast<float>(cnt)));
            const __nv_bfloat16 hi = __float2bfloat16_rn(kav);
            const size_t at = (static_cast<size_t>(h) * plane_stride + pg) * hd + d0 + tid;
            planes[at] = hi;
            planes[at + static_cast<size_t>(Hkv) * plane_stride * hd] = __float2bfloat16_rn(kav - __bfloat162float(hi));
        }
    }
    if (blockIdx.x == 0 && tid == 0) kcnt[pg] = (is_new ? 0 : kcnt[pg]) + static_cast<int>(s1 - s0);
}

void launch_append(int dtype, const void* k, const void* v, int64_t rows, int64_t filled_before, int P, int Hkv,
                   int hd, int first_page, int n_pages_touched, const NewSlots& ns, int32_t* d_kvslot_layer,
                   void* kpool, void* vpool, void* kavg_sum_layer, int32_t* kavg_cnt_layer, int* d_err,
                   cudaStream_t st, const double* rope_inv_freq, void* kavg_planes_layer, int64_t plane_stride) {
    if (rows <= 0 || n_pages_touched <= 0) return;
    __nv_bfloat16* planes = static_cast<__nv_bfloat16*>(kavg_planes_layer);
    ProfScope prof_(PK_APPEND, st);
    const int re = Hkv * hd;
    const bool aligned = ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
    if (!rope_inv_freq && hd % kAppCols == 0 && aligned && !std::getenv("OOMB_APPEND_UNSTAGED")) {
        const dim3 sg(re / kAppCols, n_pages_touched);
        if (dtype == OOMB_BF16)
            append_staged_kernel<__nv_bfloat16><<<sg, kAppThreads, 0, st>>>(
                static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v), rows, filled_before, P,
                Hkv, hd, first_page, ns, d_kvslot_layer, static_cast<__nv_bfloat16*>(kpool),
                static_cast<__nv_bfloat16*>(vpool), static_cast<float*>(kavg_sum_layer), kavg_cnt_layer, d_err, planes,
                plane_stride);
        else if (dtype == OOMB_F64)
            append_staged_kernel<double><<<sg, kAppThreads, 0, st>>>(
                static_cast<const double*>(k), static_cast<const double*>(v), rows, filled_before, P, Hkv, hd,
                first_page, ns, d_kvslot_layer, static_cast<double*>(kpool), static_cast<double*>(vpool),
                static_cast<double*>(kavg_sum_layer), kavg_cnt_layer, d_err, nullptr, 0);
        else
            append_staged_kernel<float><<<sg, kAppThreads, 0, st>>>(
                static_cast<const float*>(k), static_cast<const float*>(v), rows, filled_before, P, Hkv, hd,
                first_page, ns, d_kvslot_layer, static_cast<float*>(kpool), static_cast<float*>(vpool),
                static_cast<float*>(kavg_sum_layer), kavg_cnt_layer, d_err, nullptr, 0);
        check_launch("append_staged_kernel");
        return;
    }
    dim3 grid((re + 127) / 128, n_pages_touched);
    if (dtype == OOMB_BF16)
        append_kernel<__nv_bfloat16><<<grid, 128, 0, st>>>(
            static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v), rows, filled_before, P, Hkv,
            hd, first_page, ns, d_kvslot_layer, static_cast<__nv_bfloat16*>(kpool), static_cast<__nv_bfloat16*>(vpool),
            static_cast<float*>(kavg_sum_layer), kavg_cnt_layer, d_err, rope_inv_freq, planes, plane_stride);
    else if (dtype == OOMB_F64)
        append_kernel<double><<<grid, 128, 0, st>>>(static_cast<const double*>(k), static_cast<const double*>(v), rows,
                                                    filled_before, P, Hkv, hd, first_page, ns, d_kvslot_layer,
                                                    static_cast<double*>(kpool), static_cast<double*>(vpool),
                                                    static_cast<double*>(kavg_sum_layer), kavg_cnt_layer, d_err,
                                                    nullptr, nullptr, 0);
    else
        append_kernel<float><<<grid, 128, 0, st>>>(static_cast<const float*>(k), static_cast<const float*>(v), rows,
                                                   filled_before, P, Hkv, hd, first_page, ns, d_kvslot_layer,
                                                   static_cast<float*>(kpool), static_cast<float*>(vpool),
                                                   static_cast<float*>(kavg_sum_layer), kavg_cnt_layer, d_err,
                                                   rope_inv_freq, nullptr, 0);
    check_launch("append_kernel");
}

// ===========================================================================
// Page-range shard sub-selection: keep the ids a shard owns (id % stride == rank), list order
// kept. One CTA walks the query pages in order, compacting 1,024 ids per pass with warp ballots.
// ===========================================================================
__global__ void __launch_bounds__(1024) filter_owned_kernel(const int32_t* __restrict__ src_off,
                                                            const int32_t* __restrict__ src_ids, int m, int stride,
                                                            int rank, int32_t* __restrict__ dst_off,
                                                            int32_t* __restrict__ dst_ids) {
    __shared__ int warp_base[33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int out = 0;
    for (int qp = 0; qp < m; ++qp) {
        if (threadIdx.x == 0) dst_off[qp] = out;
        const int b = src_off[qp], e = src_off[qp + 1];
        for (int base = b; base < e; base += blockDim.x) {
            const int i = base + threadIdx.x;
            int id = 0;
            bool keep = false;
            if (i < e) {
                id = src_ids[i];
                keep = id % stride == rank;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) warp_base[warp] = __popc(bal);
            __syncthreads();
            if (threadIdx.x == 0) {
                int acc = 0;
                for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
                    const int c = warp_base[w];
                    warp_base[w] = acc;
                    acc += c;
                }
                warp_base[32] = acc;
            }
            __syncthreads();
            if (keep) dst_ids[out + warp_base[warp] + __popc(bal & ((1u << lane) - 1u))] = id;
            out += warp_base[32];
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) dst_off[m] = out;
}

void launch_filter_owned(const int32_t* src_off, const int32_t* src_ids, int m, int stride, int rank,
                         int32_t* dst_off, int32_t* dst_ids, cudaStream_t st) {
    ProfScope prof_(PK_OTHER, st);
    filter_owned_kernel<<<1, 1024, 0, st>>>(src_off, src_ids, m, stride, rank, dst_off, dst_ids);
    check_launch("filter_owned_kernel");
}

// ===========================================================================
// page_mean_keys (paged_kv.hpp:170-183): sum * (1/count), IEEE ops.
// ===========================================================================
template <typename A>
__global__ void mean_keys_kernel(const A* __restrict__ sum, const int32_t* __restrict__ cnt, int n, int re,
                                 A* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(n) * re) return;
    const int p = static_cast<int>(i / re);
    const A inv = div_rn(A(1), static_cast<A>(cnt[p]));
    out[i] = mul_rn(sum[i], inv);
}

void launch_mean_keys(const void* kavg_sum_layer, const int32_t* kavg_cnt_layer, int n, int row_elems, void* out,
                      cudaStream_t st, bool f64) {
    if (n <= 0) return;
    ProfScope prof_(PK_OTHER, st);
    const int64_t tot = static_cast<int64_t>(n) * row_elems;
    const unsigned blocks = static_cast<unsigned>((tot + 255) / 256);
    if (f64)
        mean_keys_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(kavg_sum_layer), kavg_cnt_layer, n,
                                                         row_elems, static_cast<double*>(out));
    else
        mean_keys_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(kavg_sum_layer), kavg_cnt_layer, n,
                                                        row_elems, static_cast<float*>(out));
    check_launch("mean_keys_kernel");
}

// ===========================================================================
// gather_pages / gather_grad_pages (paged_kv.hpp:118-130, 314-347)
// Output in the reference layout [n*P][Hkv][hd]; unfilled slots zero + masked.
// ===========================================================================
template <typename T, typename TO>
__global__ void gather_kernel(const int32_t* __restrict__ ids, int n, const int32_t* __restrict__ slotmap,
                              const T* __restrict__ pk, const T* __restrict__ pv, int64_t filled, int P, int Hkv,
                              int hd, int grads, TO* __restrict__ ko, TO* __restrict__ vo, uint8_t* __restrict__ valid,
                              int* err) {
    const int re = Hkv * hd;
    const int64_t total = static_cast<int64_t>(n) * P * re;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx / (static_cast<int64_t>(P) * re));
        const int rem = static_cast<int>(idx - static_cast<int64_t>(i) * P * re);
        const int s = rem / re, e = rem - (rem / re) * re;
        const int h = e / hd, d = e - (e / hd) * hd;
        const int pid = ids[i];
        const int vs = valid_in_page(filled, pid, P);
        const int slot = slotmap[pid];
        acc_t<TO> kv = 0, vv = 0;
        if (slot < 0) {
            if (!grads) atomicOr(err, DERR_NOT_RESIDENT);
        } else if (s < vs) {
            const size_t src = ((static_cast<size_t>(slot) * Hkv + h) * P + s) * hd + d;
            kv = to_a<acc_t<TO>>(pk[src]);
            vv = to_a<acc_t<TO>>(pv[src]);
        }
        ko[idx] = from_a<TO>(kv);
        vo[idx] = from_a<TO>(vv);
        if (e == 0) valid[static_cast<int64_t>(i) * P + s] = s < vs ? 1 : 0;
    }
}

void launch_gather(int dtype, int grads, const int32_t* d_ids, int n, const int32_t* d_slot_layer, const void* pk,
                   const void* pv, int64_t filled, int P, int Hkv, int hd, void* k_out, void* v_out,
                   uint8_t* valid_out, int* d_err, cudaStream_t st) {
    if (n <= 0) return;
    ProfScope prof_(PK_GATHER, st);
    const int64_t total = static_cast<int64_t>(n) * P * Hkv * hd;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 32));
    if (dtype == OOMB_F64) {  // K/V and gradient pages are both double
        gather_kernel<double, double><<<blocks, 256, 0, st>>>(d_ids, n, d_slot_layer, static_cast<const double*>(pk),
                                                              static_cast<const double*>(pv), filled, P, Hkv, hd, grads,
                                                              static_cast<double*>(k_out), static_cast<double*>(v_out),
                                                              valid_out, d_err);
    } else if (grads) {
        gather_kernel<float, float><<<blocks, 256, 0, st>>>(d_ids, n, d_slot_layer, static_cast<const float*>(pk),
                                                            static_cast<const float*>(pv), filled, P, Hkv, hd, 1,
                                                            static_cast<float*>(k_out), static_cast<float*>(v_out),
                                                            valid_out, d_err);
    } else if (dtype == OOMB_BF16) {
        gather_kernel<__nv_bfloat16, __nv_bfloat16><<<blocks, 256, 0, st>>>(
            d_ids, n, d_slot_layer, static_cast<const __nv_bfloat16*>(pk), static_cast<const __nv_bfloat16*>(pv),
            filled, P, Hkv, hd, 0, static_cast<__nv_bfloat16*>(k_out), static_cast<__nv_bfloat16*>(v_out), valid_out,
            d_err);
    } else {
        gather_kernel<float, float><<<blocks, 256, 0, st>>>(d_ids, n, d_slot_layer, static_cast<const float*>(pk),
                                                            static_cast<const float*>(pv), filled, P, Hkv, hd, 0,
                                                            static_cast<float*>(k_out), static_cast<float*>(v_out),
                                                            valid_out, d_err);
    }
    check_launch("gather_kernel");
}

// ===========================================================================
// scatter_add_grads (paged_kv.hpp:135-164): valid slots only, in place. One thread per element
// offset of a page walks the id list in order, so a page listed twice receives its additions in
// list order (no atomics: deterministic, the reference's order).
// ===========================================================================
template <typename A>
__global__ void scatter_kernel(const int32_t* __restrict__ ids, int n, const int32_t* __restrict__ gslot,
                               A* __restrict__ gk, A* __restrict__ gv, const A* __restrict__ dk,
                               const A* __restrict__ dv, int64_t filled, int P, int Hkv, int hd, int* err) {
    const int re = Hkv * hd;
    const int64_t per_page = static_cast<int64_t>(P) * re;
    for (int64_t off = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; off < per_page;
         off += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int s = static_cast<int>(off / re), e = static_cast<int>(off - static_cast<int64_t>(s) * re);
        const int h = e / hd, d = e - h * hd;
        for (int i = 0; i < n; ++i) {
            const int pid = ids[i];
            if (s >= valid_in_page(filled, pid, P)) continue;
            const int g = gslot[pid];
            if (g < 0) {
                atomicOr(err, DERR_NOT_RESIDENT);
                continue;
            }
            const size_t dst = ((static_cast<size_t>(g) * Hkv + h) * P + s) * hd + d;
            const int64_t src = static_cast<int64_t>(i) * per_page + off;
            gk[dst] += dk[src];
            gv[dst] += dv[src];
        }
    }
}

void launch_scatter(const int32_t* d_ids, int n, const int32_t* d_gslot_layer, void* gk, void* gv,
                    const void* dk, const void* dv, int64_t filled, int P, int Hkv, int hd, int* d_err,
                    cudaStream_t st, bool f64) {
    if (n <= 0) return;
    ProfScope prof_(PK_GATHER, st);
    const int64_t per_page = static_cast<int64_t>(P) * Hkv * hd;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((per_page + 255) / 256, 148 * 32));
    if (f64)
        scatter_kernel<double><<<blocks, 256, 0, st>>>(d_ids, n, d_gslot_layer, static_cast<double*>(gk),
                                                       static_cast<double*>(gv), static_cast<const double*>(dk),
                                                       static_cast<const double*>(dv), filled, P, Hkv, hd, d_err);
    else
        scatter_kernel<float><<<blocks, 256, 0, st>>>(d_ids, n, d_gslot_layer, static_cast<float*>(gk),
                                                      static_cast<float*>(gv), static_cast<const float*>(dk),
                                                      static_cast<const float*>(dv), filled, P, Hkv, hd, d_err);
    check_launch("scatter_kernel");
}

// dM_i read-back (chunk_trainer.hpp:575-587): dk/dv (reference layout) += grad pages.
template <typename A>
__global__ void accumulate_grads_kernel(const int32_t* __restrict__ ids, int n, const int32_t* __restrict__ gslot,
                                        const A* __restrict__ gk, const A* __restrict__ gv, int64_t filled,
                                        int P, int Hkv, int hd, A* __restrict__ dk, A* __restrict__ dv, int first) {
    const int re = Hkv * hd;  // ids == null: the pages are first, first + 1, ... (a chunk's own pages)
    const int64_t total = static_cast<int64_t>(n) * P * re;
    for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx / (static_cast<int64_t>(P) * re));
        const int rem = static_cast<int>(idx - static_cast<int64_t>(i) * P * re);
        const int s = rem / re, e = rem - (rem / re) * re;
        const int h = e / hd, d = e - (e / hd) * hd;
        const int pid = ids ? ids[i] : first + i;
        const int g = gslot[pid];
        if (g < 0 || s >= valid_in_page(filled, pid, P)) continue;
        const size_t src = ((static_cast<size_t>(g) * Hkv + h) * P + s) * hd + d;
        dk[idx] += gk[src];
        dv[idx] += gv[src];
    }
}

// The reverse projection epilogue (chunk_trainer.hpp:575-592): dM_i read-back
// then rope_backward of dK in one pass: dk <- rope^-1(dk + grad_k(own pages)), dv += grad_v. One
// rotation pair per thread, the same fp32 operations in the same order as the two separate steps.
__global__ void accumulate_grads_rope_kernel(const int32_t* __restrict__ ids, int n, const int32_t* __restrict__ gslot,
                                             const float* __restrict__ gk, const float* __restrict__ gv,
                                             int64_t filled, int P, int Hkv, int hd, int64_t pos0,
                                             const double* __restrict__ inv_freq, float* __restrict__ dk,
                                             float* __restrict__ dv) {
    const int re = Hkv * hd;
    const int64_t pairs = static_cast<int64_t>(n) * P * re / 2;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < pairs;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t idx = q * 2;
        const int i = static_cast<int>(idx / (static_cast<int64_t>(P) * re));
        const int rem = static_cast<int>(idx - static_cast<int64_t>(i) * P * re);
        const int s = rem / re, e = rem - (rem / re) * re;
        const int h = e / hd, d = e - (e / hd) * hd;
        const int pid = ids[i];
        const int g = gslot[pid];
        float k2[2] = {dk[idx], dk[idx + 1]};
        if (g >= 0 && s < valid_in_page(filled, pid, P)) {
            const size_t src = ((static_cast<size_t>(g) * Hkv + h) * P + s) * hd + d;
            k2[0] += gk[src];
            k2[1] += gk[src + 1];
            dv[idx] += gv[src];
            dv[idx + 1] += gv[src + 1];
        }
        // rope_elem (ops.hpp:192-225) at position -(pos0 + row): angle and trig in double, rotation in fp32
        const double ang = -static_cast<double>(pos0 + static_cast<int64_t>(i) * P + s) * inv_freq[d >> 1];
        const float c = static_cast<float>(cos(ang)), sn = static_cast<float>(sin(ang));
        dk[idx] = __fsub_rn(__fmul_rn(k2[0], c), __fmul_rn(k2[1], sn));
        dk[idx + 1] = __fadd_rn(__fmul_rn(k2[0], sn), __fmul_rn(k2[1], c));
    }
}

void launch_accumulate_grads(const int32_t* d_ids, int n, const int32_t* d_gslot_layer, const void* gk_v,
                             const void* gv_v, int64_t filled, int P, int Hkv, int hd, void* dk_v, void* dv_v,
                             cudaStream_t st, int64_t rope_pos0, const double* rope_inv_freq, bool f64, int first) {
    const float* gk = static_cast<const float*>(gk_v);
    const float* gv = static_cast<const float*>(gv_v);
    float* dk = static_cast<float*>(dk_v);
    float* dv = static_cast<float*>(dv_v);
    if (n <= 0) return;
    ProfScope prof_(PK_GATHER, st);
    const int64_t total = static_cast<int64_t>(n) * P * Hkv * hd;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16));
    if (rope_inv_freq) {
        accumulate_grads_rope_kernel<<<blocks, 256, 0, st>>>(d_ids, n, d_gslot_layer, gk, gv, filled, P, Hkv, hd,
                                                             rope_pos0, rope_inv_freq, dk, dv);
        check_launch("accumulate_grads_rope_kernel");
        return;
    }
    if (f64)
        accumulate_grads_kernel<double><<<blocks, 256, 0, st>>>(d_ids, n, d_gslot_layer, static_cast<const double*>(gk_v),
                                                                static_cast<const double*>(gv_v), filled, P, Hkv, hd,
                                                                static_cast<double*>(dk_v), static_cast<double*>(dv_v), first);
    else
        accumulate_grads_kernel<float><<<blocks, 256, 0, st>>>(d_ids, n, d_gslot_layer, gk, gv, filled, P, Hkv, hd, dk,
                                                               dv, first);
    check_launch("accumulate_grads_kernel");
}

// Lazy gradient pages: publish slot + zero (paged_kv.hpp:148-153).
__global__ void grad_init_kernel(const int32_t* __restrict__ pages, const int32_t* __restrict__ slots, int n,
                                 int32_t* __restrict__ gslot, float* __restrict__ gk, float* __restrict__ gv,
                                 int64_t page_words) {  // page size in 4-byte words (fp64 pages: 2 per element)
    const int i = blockIdx.y;
    if (i >= n) return;
    const int64_t base = static_cast<int64_t>(slots[i]) * page_words;
    float* pk = gk + base;
    float* pv = gv + base;
    const int64_t n4 = (page_words % 4 == 0 && base % 4 == 0) ? page_words / 4 : 0;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n4;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        reinterpret_cast<float4*>(pk)[j] = z;
        reinterpret_cast<float4*>(pv)[j] = z;
    }
    for (int64_t j = 4 * n4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < page_words;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        pk[j] = 0.f;
        pv[j] = 0.f;
    }
    if (pages != nullptr && blockIdx.x == 0 && threadIdx.x == 0) gslot[pages[i]] = slots[i];
}

void launch_grad_init(const int32_t* d_pages, const int32_t* d_slots, int n, int32_t* d_gslot_layer, void* gk,
                      void* gv, int64_t page_elems, cudaStream_t st, int elem_bytes) {
    if (n <= 0) return;
    ProfScope prof_(PK_GRAD_INIT, st);
    const int64_t words = page_elems * (elem_bytes / 4);
    dim3 grid(static_cast<unsigned>(std::min<int64_t>((words / 4 + 255) / 256 + 1, 16)), n);
    grad_init_kernel<<<grid, 256, 0, st>>>(d_pages, d_slots, n, d_gslot_layer, static_cast<float*>(gk),
                                           static_cast<float*>(gv), words);
    check_launch("grad_init_kernel");
}

void launch_zero_slots(const int32_t* d_slots, int n, void* gk, void* gv, int64_t page_elems, cudaStream_t st,
                       int elem_bytes) {
    launch_grad_init(nullptr, d_slots, n, nullptr, gk, gv, page_elems, st, elem_bytes);
}

// ===========================================================================
// score_pages (attention.hpp:32-67), exact SIMT form.
// Pass 1: per (token, head) row max and 1/sum over candidates (warp per row).
// Pass 2: per (query page, candidate) thread, sum over tokens asc then heads asc
//         — the reference's accumulation order for the vote.
// Dot products use the reference's sequential order with no FMA contraction.
// ===========================================================================
template <typename T>
__device__ __forceinline__ acc_t<T> dot_seq(const T* __restrict__ q, const acc_t<T>* __restrict__ k, int hd) {
    using A = acc_t<T>;
    A dot = A(0);
    for (int j = 0; j < hd; ++j) dot = add_rn(dot, mul_rn(to_a<A>(q[j]), k[j]));
    return dot;
}

template <typename T>
__global__ void score_stats_kernel(const T* __restrict__ q, int64_t tokens, int Hq, int hd,
                                   const acc_t<T>* __restrict__ kavg, int64_t n, int Hkv, acc_t<T> scale,
                                   Stat<acc_t<T>>* __restrict__ stats) {
    using A = acc_t<T>;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= tokens * Hq) return;
    const int h = static_cast<int>(row % Hq);
    const int kvh = h / (Hq / Hkv);
    const T* qv = q + row * hd;
    A mx = -INFINITY;
    for (int64_t p = lane; p < n; p += 32) {
        const A raw = mul_rn(dot_seq(qv, kavg + (p * Hkv + kvh) * hd, hd), scale);
        mx = max_a(mx, raw);
    }
    mx = warp_max(mx);
    A sum = A(0);
    for (int64_t p = lane; p < n; p += 32) {
        const A raw = mul_rn(dot_seq(qv, kavg + (p * Hkv + kvh) * hd, hd), scale);
        sum += exp_a(raw - mx);
    }
    sum = warp_sum(sum);
    if (lane == 0) stats[row] = Stat<A>{mx, div_rn(A(1), sum)};
}

template <typename T>
__global__ void score_vote_kernel(const T* __restrict__ q, int64_t tokens, int Hq, int hd,
                                  const acc_t<T>* __restrict__ kavg, int64_t n, int Hkv, int P, acc_t<T> scale,
                                  const Stat<acc_t<T>>* __restrict__ stats, acc_t<T>* __restrict__ vote, int h0, int h1) {
    using A = acc_t<T>;
    extern __shared__ __align__(16) unsigned char qs_raw[];
    A* qs = reinterpret_cast<A*>(qs_raw);  // [hd]
    const int qp = blockIdx.y;
    const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int group = Hq / Hkv;
    A acc = A(0);
    const int64_t t0 = static_cast<int64_t>(qp) * P;
    const int64_t t1 = min(tokens, t0 + P);
    for (int64_t t = t0; t < t1; ++t) {
        for (int h = h0; h < h1; ++h) {
            __syncthreads();
            for (int j = threadIdx.x; j < hd; j += blockDim.x) qs[j] = to_a<A>(q[(t * Hq + h) * hd + j]);
            __syncthreads();
            if (p < n) {
                const A* kv = kavg + (p * Hkv + h / group) * hd;
                A dot = A(0);
                for (int j = 0; j < hd; ++j) dot = add_rn(dot, mul_rn(qs[j], kv[j]));
                const Stat<A> st = stats[t * Hq + h];
                acc = add_rn(acc, mul_rn(exp_a(mul_rn(dot, scale) - st.m), st.il));
            }
        }
    }
    if (p < n) vote[static_cast<int64_t>(qp) * n + p] = acc;
}

void launch_score_simt(int dtype, const void* q, int64_t tokens, int Hq, int hd, const void* k_avg, int64_t n,
                       int Hkv, int P, float scale, double scale64, void* vote, void* stats_scratch, cudaStream_t st,
                       bool partial_only) {
    ProfScope prof_(PK_SCORE, st);
    const int64_t rows = tokens * Hq;
    const int m = static_cast<int>((tokens + P - 1) / P);
    dim3 g1(static_cast<unsigned>((rows + 7) / 8));
    dim3 g2(static_cast<unsigned>((n + 127) / 128), m);
    auto run = [&](auto tag, auto sc) {
        using T = decltype(tag);
        using A = acc_t<T>;
        auto qq = static_cast<const T*>(q);
        auto ka = static_cast<const A*>(k_avg);
        auto stats = static_cast<Stat<A>*>(stats_scratch);
        auto vo = static_cast<A*>(vote);
        score_stats_kernel<T><<<g1, 256, 0, st>>>(qq, tokens, Hq, hd, ka, n, Hkv, static_cast<A>(sc), stats);
        check_launch("score_stats_kernel");
        for (int g = 0; g < (partial_only ? Hkv : 1); ++g)
            score_vote_kernel<T><<<g2, 128, hd * sizeof(A), st>>>(
                qq, tokens, Hq, hd, ka, n, Hkv, P, static_cast<A>(sc), stats, vo + (partial_only ? g * m * n : 0),
                partial_only ? g * (Hq / Hkv) : 0, partial_only ? (g + 1) * (Hq / Hkv) : Hq);
        check_launch("score_vote_kernel");
    };
    if (dtype == OOMB_BF16) run(__nv_bfloat16{}, scale);
    else if (dtype == OOMB_F64) run(double{}, scale64);
    else run(float{}, scale);
}

// ===========================================================================
// select_topk_row (attention.hpp:71-96): per row, the k largest scores with ties
// to the lower id, emitted ascending. One CTA per row: 4-pass MSB radix select of
// the k-th largest order-preserving key, then id-ordered compaction in which the
// threshold-equal elements are admitted lowest-id first. Exact and deterministic.
// ===========================================================================
__device__ __forceinline__ uint32_t order_key(float f) {
    uint32_t u = __float_as_uint(f);
    if (f == 0.f) u = 0u;  // the reference compares doubles: -0 == +0 (tie -> id order)
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ unsigned long long order_key(double f) {  // fp64 pools: 8 radix passes
    unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(f));
    if (f == 0.0) u = 0ull;
    return (u >> 63) ? ~u : (u | (1ull << 63));
}

constexpr int kTopkThreads = 1024;

template <typename V>
__global__ void __launch_bounds__(kTopkThreads) topk_kernel(const V* __restrict__ vote, int m, int n, int k,
                                                            int32_t* __restrict__ off, int32_t* __restrict__ ids) {
    using K = decltype(order_key(V(0)));
    constexpr int kPasses = static_cast<int>(sizeof(K));
    using Scan = cub::BlockScan<int, kTopkThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ uint32_t hist[256];
    __shared__ K s_prefix, s_mask;
    __shared__ int s_remaining;
    const int row = blockIdx.x;
    const int tid = threadIdx.x;
    const int kk = k < n ? k : n;
    if (tid == 0) {
        off[row] = row * kk;
        if (row == m - 1) off[m] = m * kk;
    }
    int32_t* out = ids + static_cast<int64_t>(row) * kk;
    const V* s = vote + static_cast<int64_t>(row) * n;
    if (kk == n) {
        for (int i = tid; i < n; i += kTopkThreads) out[i] = i;
        return;
    }
    if (kk == 0) return;
    if (tid == 0) {
        s_prefix = 0;
        s_mask = 0;
        s_remaining = kk;
    }
    for (int pass = 0; pass < kPasses; ++pass) {
        const int shift = 8 * (kPasses - 1 - pass);
        if (tid < 256) hist[tid] = 0;
        __syncthreads();
        const K prefix = s_prefix, mask = s_mask;
        for (int i = tid; i < n; i += kTopkThreads) {
            const K key = order_key(s[i]);
            if ((key & mask) == prefix) atomicAdd(&hist[static_cast<uint32_t>(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid == 0) {
            int rem = s_remaining;
            uint32_t cum = 0;
            int chosen = 0;
            for (int b = 255; b >= 0; --b) {
                if (cum + hist[b] >= static_cast<uint32_t>(rem)) {
                    chosen = b;
                    rem -= static_cast<int>(cum);
                    break;
                }
                cum += hist[b];
            }
            s_remaining = rem;
            s_prefix = prefix | (static_cast<K>(chosen) << shift);
            s_mask = mask | (static_cast<K>(255u) << shift);
        }
        __syncthreads();
    }
    const K thr = s_prefix;
    const int take_eq = s_remaining;  // threshold-equal elements to admit, lowest ids first
    const int ipt = (n + kTopkThreads - 1) / kTopkThreads;
    const int i0 = min(n, tid * ipt), i1 = min(n, i0 + ipt);
    int n_eq = 0;
    for (int i = i0; i < i1; ++i) n_eq += order_key(s[i]) == thr;
    int eq_before;
    Scan(scan_tmp).ExclusiveSum(n_eq, eq_before);
    __syncthreads();
    int n_sel = 0;
    {
        int r = eq_before;
        for (int i = i0; i < i1; ++i) {
            const K key = order_key(s[i]);
            if (key > thr) ++n_sel;
            else if (key == thr) n_sel += (r++ < take_eq);
        }
    }
    int pos;
    Scan(scan_tmp).ExclusiveSum(n_sel, pos);
    int r = eq_before;
    for (int i = i0; i < i1; ++i) {
        const K key = order_key(s[i]);
        bool take = key > thr;
        if (key == thr) take = (r++ < take_eq);
        if (take) out[pos++] = i;
    }
}

void launch_topk(const void* vote, int m, int n, int k, int32_t* sel_off, int32_t* sel_ids, cudaStream_t st,
                 bool f64) {
    if (m <= 0) return;
    ProfScope prof_(PK_TOPK, st);
    if (f64) topk_kernel<double><<<m, kTopkThreads, 0, st>>>(static_cast<const double*>(vote), m, n, k, sel_off, sel_ids);
    else topk_kernel<float><<<m, kTopkThreads, 0, st>>>(static_cast<const float*>(vote), m, n, k, sel_off, sel_ids);
    check_launch("topk_kernel");
}

// select_all / select_recent broadcast to m query pages: ids first..first+count-1.
__global__ void fill_csr_kernel(int32_t* off, int32_t* ids, int m, int first, int count) {
    const int qp = blockIdx.x;
    if (threadIdx.x == 0) {
        off[qp] = qp * count;
        if (qp == m - 1) off[m] = m * count;
    }
    for (int i = threadIdx.x; i < count; i += blockDim.x) ids[static_cast<int64_t>(qp) * count + i] = first + i;
}

void launch_fill_csr_all(int32_t* off, int32_t* ids, int m, int first, int count, cudaStream_t st) {
    if (m <= 0) return;
    ProfScope prof_(PK_OTHER, st);
    fill_csr_kernel<<<m, 256, 0, st>>>(off, ids, m, first, count);
    check_launch("fill_csr_kernel");
}

// ===========================================================================
// SIMT paged attention (attention.hpp:156-293): one warp per (token, q-head).
// Forward = the reference's OnlineRow over past valid slots in list order, then
// the chunk's causal prefix. Backward rebuilds p from the saved lse and D from
// the saved O; dK/dV go to the fp32 gradient pool / dk_cur, dv_cur by atomics.
// ===========================================================================
constexpr int kMaxLaneElems = 8;  // hd <= 256

template <typename T>
__global__ void attn_fwd_simt_kernel(AttnGeom g, const T* __restrict__ q, const int32_t* __restrict__ sel_off,
                                     const int32_t* __restrict__ sel_ids, const int32_t* __restrict__ kvslot,
                                     const T* __restrict__ kpool, const T* __restrict__ vpool,
                                     const T* __restrict__ k_cur, const T* __restrict__ v_cur, T* __restrict__ out,
                                     acc_t<T>* __restrict__ lse, int* err) {
    using A = acc_t<T>;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= static_cast<int64_t>(g.C) * g.Hq) return;
    const int t = static_cast<int>(row / g.Hq), h = static_cast<int>(row % g.Hq);
    const int kvh = h / g.group, qp = t / g.P, hd = g.hd;
    const int nd = (hd + 31) / 32;
    A qv[kMaxLaneElems], acc[kMaxLaneElems];
#pragma unroll
    for (int i = 0; i < kMaxLaneElems; ++i) {
        const int d = lane + 32 * i;
        qv[i] = (i < nd && d < hd) ? to_a<A>(q[row * hd + d]) : A(0);
        acc[i] = A(0);
    }
    A m = -INFINITY, l = A(0);
    auto visit = [&](const T* kr, const T* vr) {
        A part = A(0);
#pragma unroll
        for (int i = 0; i < kMaxLaneElems; ++i) {
            const int d = lane + 32 * i;
            if (i < nd && d < hd) part += qv[i] * to_a<A>(kr[d]);
        }
        const A logit = warp_sum(part) * scale_of<A>(g);
        if (logit > m) {
            const A corr = (l == A(0)) ? A(0) : exp_a(m - logit);
#pragma unroll
            for (int i = 0; i < kMaxLaneElems; ++i) acc[i] *= corr;
            l *= corr;
            m = logit;
        }
        const A w = exp_a(logit - m);
        l += w;
#pragma unroll
        for (int i = 0; i < kMaxLaneElems; ++i) {
            const int d = lane + 32 * i;
            if (i < nd && d < hd) acc[i] += w * to_a<A>(vr[d]);
        }
    };
    for (int idx = sel_off[qp]; idx < sel_off[qp + 1]; ++idx) {
        const int pid = sel_ids[idx];
        if (pid < 0 || pid >= g.max_pages || static_cast<int64_t>(pid) * g.P >= g.filled) {
            if (lane == 0) atomicOr(err, DERR_BAD_ID);
            continue;
        }
        const int slot = kvslot[pid];
        if (slot < 0) {
            if (lane == 0) atomicOr(err, DERR_NOT_RESIDENT);
            continue;
        }
        const int vs = valid_in_page(g.filled, pid, g.P);
        const size_t base = (static_cast<size_t>(slot) * g.Hkv + kvh) * g.P * hd;
        for (int s = 0; s < vs; ++s) visit(kpool + base + static_cast<size_t>(s) * hd, vpool + base + static_cast<size_t>(s) * hd);
    }
    if (g.chunk_keys) {
        for (int s = 0; s <= t; ++s) {
            const size_t o = (static_cast<size_t>(s) * g.Hkv + kvh) * hd;
            visit(k_cur + o, v_cur + o);
        }
    }
    const A inv = l > A(0) ? A(1) / l : A(0);  // a shard that attended no key: O = 0, lse = -inf
#pragma unroll
    for (int i = 0; i < kMaxLaneElems; ++i) {
        const int d = lane + 32 * i;
        if (i < nd && d < hd) out[row * hd + d] = from_a<T>(acc[i] * inv);
    }
    if (lane == 0) lse[row] = l > A(0) ? m + log_a(l) : -INFINITY;
}

template <typename T>
__global__ void attn_bwd_simt_kernel(AttnGeom g, const T* __restrict__ dout, const T* __restrict__ q,
                                     const int32_t* __restrict__ sel_off, const int32_t* __restrict__ sel_ids,
                                     const int32_t* __restrict__ kvslot, const int32_t* __restrict__ gslot,
                                     const T* __restrict__ kpool, const T* __restrict__ vpool, acc_t<T>* __restrict__ gk,
                                     acc_t<T>* __restrict__ gv, const T* __restrict__ k_cur, const T* __restrict__ v_cur,
                                     const T* __restrict__ o, const acc_t<T>* __restrict__ lse, acc_t<T>* __restrict__ dq,
                                     acc_t<T>* __restrict__ d_rows, int* err) {
    using A = acc_t<T>;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= static_cast<int64_t>(g.C) * g.Hq) return;
    const int t = static_cast<int>(row / g.Hq), h = static_cast<int>(row % g.Hq);
    const int kvh = h / g.group, qp = t / g.P, hd = g.hd;
    const int nd = (hd + 31) / 32;
    A qv[kMaxLaneElems], dov[kMaxLaneElems], dqa[kMaxLaneElems];
    A dpart = A(0);
#pragma unroll
    for (int i = 0; i < kMaxLaneElems; ++i) {
        const int d = lane + 32 * i;
        const bool ok = i < nd && d < hd;
        qv[i] = ok ? to_a<A>(q[row * hd + d]) : A(0);
        dov[i] = ok ? to_a<A>(dout[row * hd + d]) : A(0);
        dpart += ok ? dov[i] * to_a<A>(o[row * hd + d]) : A(0);
        dqa[i] = A(0);
    }
    const A D = warp_sum(dpart);
    if (lane == 0) d_rows[row] = D;
    const A L = lse[row];
    auto visit = [&](const T* kr, const T* vr) {
        A p1 = A(0), p2 = A(0);
#pragma unroll
        for (int i = 0; i < kMaxLaneElems; ++i) {
            const int d = lane + 32 * i;
            if (i < nd && d < hd) {
                p1 += qv[i] * to_a<A>(kr[d]);
                p2 += dov[i] * to_a<A>(vr[d]);
            }
        }
        const A dot = warp_sum(p1);
        const A dpv = warp_sum(p2);
        const A p = exp_a(dot * scale_of<A>(g) - L);
        const A dlogit = p * (dpv - D) * scale_of<A>(g);
#pragma unroll
        for (int i = 0; i < kMaxLaneElems; ++i) {
            const int d = lane + 32 * i;
            if (i < nd && d < hd) {
                dqa[i] += dlogit * to_a<A>(kr[d]);
            }
        }
    };
    for (int idx = sel_off[qp]; idx < sel_off[qp + 1]; ++idx) {
        const int pid = sel_ids[idx];
        if (pid < 0 || pid >= g.max_pages || static_cast<int64_t>(pid) * g.P >= g.filled) {
            if (lane == 0) atomicOr(err, DERR_BAD_ID);
            continue;
        }
        const int slot = kvslot[pid], gs = gslot[pid];
        if (slot < 0 || gs < 0) {
            if (lane == 0) atomicOr(err, DERR_NOT_RESIDENT);
            continue;
        }
        const int vs = valid_in_page(g.filled, pid, g.P);
        const size_t base = (static_cast<size_t>(slot) * g.Hkv + kvh) * g.P * hd;
        for (int s = 0; s < vs; ++s) {
            const size_t so = static_cast<size_t>(s) * hd;
            visit(kpool + base + so, vpool + base + so);
        }
    }
    if (g.chunk_keys) {
        for (int s = 0; s <= t; ++s) {
            const size_t so = (static_cast<size_t>(s) * g.Hkv + kvh) * hd;
            visit(k_cur + so, v_cur + so);
        }
    }
#pragma unroll
    for (int i = 0; i < kMaxLaneElems; ++i) {
        const int d = lane + 32 * i;
        if (i < nd && d < hd) dq[row * hd + d] = dqa[i];
    }
}

// dK / dV, key-major and deterministic: one warp per (key row, kv head) sums its contributions in
// the reference's order (attention.hpp:239-290): query pages ascending, then rows, then the group's
// heads. A past page's sum is flushed into its gradient page once per query page that selected it
// (scatter_add_grads per query page, :288-290); the chunk's own keys sum over every row t >= s
// into dk_cur / dv_cur. Single writer per element: no atomics. grid.x = past pages (then the
// chunk's own key blocks of P rows), grid.y = kv head, grid.z = groups of 4 keys (one per warp).
template <typename T>
__global__ void attn_bwd_kv_simt_kernel(AttnGeom g, const T* __restrict__ dout, const T* __restrict__ q,
                                        const int32_t* __restrict__ sel_off, const int32_t* __restrict__ sel_ids,
                                        const int32_t* __restrict__ kvslot, const int32_t* __restrict__ gslot,
                                        const T* __restrict__ kpool, const T* __restrict__ vpool,
                                        acc_t<T>* __restrict__ gk, acc_t<T>* __restrict__ gv, const T* __restrict__ k_cur,
                                        const T* __restrict__ v_cur, const acc_t<T>* __restrict__ lse,
                                        const acc_t<T>* __restrict__ d_rows, acc_t<T>* __restrict__ dk_cur,
                                        acc_t<T>* __restrict__ dv_cur, int n_past_pages) {
    using A = acc_t<T>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int kvh = blockIdx.y, hd = g.hd, nd = (hd + 31) / 32;
    const bool past = static_cast<int>(blockIdx.x) < n_past_pages;
    const int pid = past ? static_cast<int>(blockIdx.x) : -1;
    const int blk = past ? 0 : static_cast<int>(blockIdx.x) - n_past_pages;  // chunk key block
    if (!past && !g.chunk_keys) return;
    int slot = -1, gs = -1, n_keys = g.P;
    if (past) {
        slot = kvslot[pid];
        gs = gslot[pid];
        if (slot < 0 || gs < 0) return;  // never selected (the query kernel flags selected non-resident pages)
        n_keys = valid_in_page(g.filled, pid, g.P);
    } else {
        n_keys = min(g.P, g.C - blk * g.P);
    }
    for (int s = static_cast<int>(blockIdx.z) * nw + warp; s < n_keys; s += nw * static_cast<int>(gridDim.z)) {
        const T* kr;
        const T* vr;
        A* dkr;
        A* dvr;
        int key_t = 0;  // chunk keys: the key's row
        if (past) {
            const size_t off = ((static_cast<size_t>(slot) * g.Hkv + kvh) * g.P + s) * hd;
            const size_t goff = ((static_cast<size_t>(gs) * g.Hkv + kvh) * g.P + s) * hd;
            kr = kpool + off;
            vr = vpool + off;
            dkr = gk + goff;
            dvr = gv + goff;
        } else {
            key_t = blk * g.P + s;
            const size_t off = (static_cast<size_t>(key_t) * g.Hkv + kvh) * hd;
            kr = k_cur + off;
            vr = v_cur + off;
            dkr = dk_cur + off;
            dvr = dv_cur + off;
        }
        A kv[kMaxLaneElems], vv[kMaxLaneElems], ak[kMaxLaneElems], av[kMaxLaneElems];
#pragma unroll
        for (int i = 0; i < kMaxLaneElems; ++i) {
            const int d = lane + 32 * i;
            const bool ok = i < nd && d < hd;
            kv[i] = ok ? to_a<A>(kr[d]) : A(0);
            vv[i] = ok ? to_a<A>(vr[d]) : A(0);
            ak[i] = av[i] = A(0);
        }
        auto rows = [&](int t0, int t1) {  // rows t0..t1-1, the group's heads: accumulate in order
            for (int t = t0; t < t1; ++t)
                for (int j = 0; j < g.group; ++j) {
                    const int64_t row = static_cast<int64_t>(t) * g.Hq + kvh * g.group + j;
                    A p1 = A(0), p2 = A(0), qv[kMaxLaneElems], dv2[kMaxLaneElems];
#pragma unroll
                    for (int i = 0; i < kMaxLaneElems; ++i) {
                        const int d = lane + 32 * i;
                        const bool ok = i < nd && d < hd;
                        qv[i] = ok ? to_a<A>(q[row * hd + d]) : A(0);
                        dv2[i] = ok ? to_a<A>(dout[row * hd + d]) : A(0);
                        p1 += qv[i] * kv[i];
                        p2 += dv2[i] * vv[i];
                    }
                    const A dot = warp_sum(p1);
                    const A dpv = warp_sum(p2);
                    const A p = exp_a(dot * scale_of<A>(g) - lse[row]);
                    const A dlogit = p * (dpv - d_rows[row]) * scale_of<A>(g);
#pragma unroll
                    for (int i = 0; i < kMaxLaneElems; ++i) {
                        ak[i] += dlogit * qv[i];
                        av[i] += p * dv2[i];
                    }
                }
        };
        if (past) {
            for (int qp = 0; qp < g.m; ++qp) {
                bool sel = false;
                for (int idx = sel_off[qp]; idx < sel_off[qp + 1] && !sel; ++idx) sel = sel_ids[idx] == pid;
                if (!sel) continue;
                rows(qp * g.P, min(g.C, (qp + 1) * g.P));
#pragma unroll
                for (int i = 0; i < kMaxLaneElems; ++i) {  // this query page's scatter_add
                    const int d = lane + 32 * i;
                    if (i < nd && d < hd) {
                        dkr[d] += ak[i];
                        dvr[d] += av[i];
                    }
                    ak[i] = av[i] = A(0);
                }
            }
        } else {
            rows(key_t, g.C);
#pragma unroll
            for (int i = 0; i < kMaxLaneElems; ++i) {
                const int d = lane + 32 * i;
                if (i < nd && d < hd) {
                    dkr[d] = ak[i];
                    dvr[d] = av[i];
                }
            }
        }
    }
}

void launch_attn_fwd_simt(int dtype, const AttnGeom& g, const void* q, const int32_t* sel_off, const int32_t* sel_ids,
                          const int32_t* d_kvslot_layer, const void* kpool, const void* vpool, const void* k_cur,
                          const void* v_cur, void* out, void* lse, int* d_err, cudaStream_t st) {
    ProfScope prof_(PK_FWD, st);
    const int64_t rows = static_cast<int64_t>(g.C) * g.Hq;
    const unsigned blocks = static_cast<unsigned>((rows + 3) / 4);
    auto run = [&](auto tag) {
        using T = decltype(tag);
        attn_fwd_simt_kernel<T><<<blocks, 128, 0, st>>>(g, static_cast<const T*>(q), sel_off, sel_ids, d_kvslot_layer,
                                                        static_cast<const T*>(kpool), static_cast<const T*>(vpool),
                                                        static_cast<const T*>(k_cur), static_cast<const T*>(v_cur),
                                                        static_cast<T*>(out), static_cast<acc_t<T>*>(lse), d_err);
    };
    if (dtype == OOMB_BF16) run(__nv_bfloat16{});
    else if (dtype == OOMB_F64) run(double{});
    else run(float{});
    check_launch("attn_fwd_simt_kernel");
}

void launch_attn_bwd_simt(int dtype, const AttnGeom& g, const void* dout, const void* q, const int32_t* sel_off,
                          const int32_t* sel_ids, const int32_t* d_kvslot_layer, const int32_t* d_gslot_layer,
                          const void* kpool, const void* vpool, void* gkpool, void* gvpool, const void* k_cur,
                          const void* v_cur, const void* out, const void* lse, void* dq, void* dk_cur,
                          void* dv_cur, int* d_err, cudaStream_t st, int n_past_pages) {
    ProfScope prof_(PK_BWD_SIMT, st);
    const int64_t rows = static_cast<int64_t>(g.C) * g.Hq;
    const unsigned blocks = static_cast<unsigned>((rows + 3) / 4);
    void* d_rows = nullptr;
    OOMB_CUDA(cudaMallocAsync(&d_rows, std::max<int64_t>(rows, 1) * sizeof(double), st));
    const dim3 kv_grid(static_cast<unsigned>(n_past_pages + (g.C + g.P - 1) / g.P), g.Hkv,
                       static_cast<unsigned>((g.P + 3) / 4));
    auto run = [&](auto zero) {
        using T = decltype(zero);
        using A = acc_t<T>;
        attn_bwd_simt_kernel<T><<<blocks, 128, 0, st>>>(
            g, static_cast<const T*>(dout), static_cast<const T*>(q), sel_off, sel_ids, d_kvslot_layer, d_gslot_layer,
            static_cast<const T*>(kpool), static_cast<const T*>(vpool), static_cast<A*>(gkpool), static_cast<A*>(gvpool),
            static_cast<const T*>(k_cur), static_cast<const T*>(v_cur), static_cast<const T*>(out),
            static_cast<const A*>(lse), static_cast<A*>(dq), static_cast<A*>(d_rows), d_err);
        check_launch("attn_bwd_simt_kernel");
        attn_bwd_kv_simt_kernel<T><<<kv_grid, 128, 0, st>>>(
            g, static_cast<const T*>(dout), static_cast<const T*>(q), sel_off, sel_ids, d_kvslot_layer, d_gslot_layer,
            static_cast<const T*>(kpool), static_cast<const T*>(vpool), static_cast<A*>(gkpool), static_cast<A*>(gvpool),
            static_cast<const T*>(k_cur), static_cast<const T*>(v_cur), static_cast<const A*>(lse),
            static_cast<const A*>(d_rows), static_cast<A*>(dk_cur), static_cast<A*>(dv_cur), n_past_pages);
        check_launch("attn_bwd_kv_simt_kernel");
    };
    if (dtype == OOMB_BF16) run(__nv_bfloat16{});
    else if (dtype == OOMB_F64) run(double{});
    else run(float{});
    OOMB_CUDA(cudaFreeAsync(d_rows, st));
}

// ===========================================================================
// Page-range split merge: rank r attended a disjoint subset of every query page's
// selected pages and produced (O_r, LSE_r), O_r normalised by its own row sum, LSE natural log
// (-inf: the rank attended no key for that row). Exact combination, parts in rank order:
//   LSE = m + ln sum_r exp(LSE_r - m),  O = sum_r exp(LSE_r - LSE) O_r.
// One warp per (token, head) row.
// ===========================================================================
template <typename T>
__global__ void lse_merge_kernel(const T* __restrict__ o_parts, const float* __restrict__ lse_parts, int parts,
                                 int64_t rows, int hd, T* __restrict__ out, float* __restrict__ lse) {
    const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float m = -INFINITY;
    for (int r = 0; r < parts; ++r) m = fmaxf(m, lse_parts[static_cast<int64_t>(r) * rows + row]);
    float l = 0.f;
    for (int r = 0; r < parts; ++r) {
        const float x = lse_parts[static_cast<int64_t>(r) * rows + row];
        if (x != -INFINITY) l += expf(x - m);
    }
    const float L = (m == -INFINITY) ? -INFINITY : m + logf(l);
    for (int d = lane; d < hd; d += 32) {
        float acc = 0.f;
        for (int r = 0; r < parts; ++r) {
            const float x = lse_parts[static_cast<int64_t>(r) * rows + row];
            if (x == -INFINITY) continue;
            acc += expf(x - L) * to_f(o_parts[(static_cast<int64_t>(r) * rows + row) * hd + d]);
        }
        out[row * hd + d] = from_f<T>(acc);
    }
    if (lane == 0) lse[row] = L;
}

void launch_lse_merge(const void* o_parts, const float* lse_parts, int parts, int64_t rows, int hd, int dtype,
                      void* out, float* lse, cudaStream_t st) {
    if (rows <= 0) return;
    ProfScope prof_(PK_OTHER, st);
    const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
    if (dtype == OOMB_BF16)
        lse_merge_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o_parts), lse_parts,
                                                              parts, rows, hd, static_cast<__nv_bfloat16*>(out), lse);
    else
        lse_merge_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(o_parts), lse_parts, parts, rows, hd,
                                                      static_cast<float*>(out), lse);
    check_launch("lse_merge_kernel");
}

// ===========================================================================
// RoPE / inverse RoPE (ops.hpp:192-230) over [rows][heads][hd]: q before attention,
// dq / dk_cur after it (rope_backward = sign -1). out may alias x.
// ===========================================================================
template <typename Tin, typename Tout>
__global__ void rope_kernel(const Tin* x, int64_t rows, int heads, int hd, int64_t pos0, int sign,
                            const double* __restrict__ inv_freq, Tout* out) {
    const int64_t pairs = rows * heads * hd / 2;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < pairs;
         q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        // one rotation pair per thread, so an in-place rotation reads both elements before writing
        const int64_t e0 = q * 2;
        const int64_t r = e0 / (static_cast<int64_t>(heads) * hd);
        const int d = static_cast<int>(e0 % hd);
        const Tin* row = x + (e0 - d);
        const double pos = static_cast<double>(sign) * static_cast<double>(pos0 + r);
        const float y0 = rope_elem(row, d, pos, inv_freq);
        const float y1 = rope_elem(row, d + 1, pos, inv_freq);
        out[e0] = from_f<Tout>(y0);
        out[e0 + 1] = from_f<Tout>(y1);
    }
}

void launch_rope(int in_dtype, int out_dtype, const void* x, int64_t rows, int heads, int hd, int64_t pos0, int sign,
                 const double* inv_freq, void* out, cudaStream_t st) {
    const int64_t pairs = rows * heads * hd / 2;
    if (pairs <= 0) return;
    ProfScope prof_(PK_OTHER, st);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>((pairs + 255) / 256, 4096));
    if (in_dtype == OOMB_BF16 && out_dtype == OOMB_BF16)
        rope_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, st>>>(
            static_cast<const __nv_bfloat16*>(x), rows, heads, hd, pos0, sign, inv_freq, static_cast<__nv_bfloat16*>(out));
    else if (in_dtype == OOMB_BF16)
        rope_kernel<__nv_bfloat16, float><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), rows, heads, hd,
                                                                 pos0, sign, inv_freq, static_cast<float*>(out));
    else if (out_dtype == OOMB_BF16)
        rope_kernel<float, __nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const float*>(x), rows, heads, hd, pos0,
                                                                 sign, inv_freq, static_cast<__nv_bfloat16*>(out));
    else
        rope_kernel<float, float><<<grid, 256, 0, st>>>(static_cast<const float*>(x), rows, heads, hd, pos0, sign,
                                                        inv_freq, static_cast<float*>(out));
    check_launch("rope_kernel");
}

}  // namespace oomb
