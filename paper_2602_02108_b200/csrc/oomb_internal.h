// SPDX-License-Identifier: Apache-2.0
//
// Internal declarations shared by the host runtime (oomb_api.cu) and the
// kernel translation units.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <tuple>
#include <mutex>
#include <set>
#include <utility>
#include <stdexcept>
#include <string>
#include <vector>

#include "oomb.h"

namespace oomb {

// Per-device one-time setup (kernel attributes apply to the current device's context): true the
// first time `key` is seen on the current device.
inline bool first_use_on_device(int key) {
    static std::mutex mu;
    static std::set<std::pair<int, int>> seen;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return true;
    std::lock_guard<std::mutex> lock(mu);
    return seen.insert({dev, key}).second;
}

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define OOMB_REQUIRE(cond, code, msg)                     \
    do {                                                  \
        if (!(cond)) throw ::oomb::Error((code), (msg));  \
    } while (0)

#define OOMB_CUDA(call)                                                                          \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            throw ::oomb::Error(OOMB_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Scratch buffer per (device, stream, slot), reused by later work on the same stream (stream order
// makes the reuse safe): the split-K partials of the forward / dQ launches, which would otherwise
// cost a cudaMallocAsync + cudaFreeAsync pair per chunk on the host. It only grows (the old buffer
// is freed in stream order) and lives until process exit.
inline void* stream_scratch(cudaStream_t st, int slot, size_t bytes) {
    static std::mutex mu;
    static std::map<std::tuple<int, cudaStream_t, int>, std::pair<void*, size_t>> bufs;
    int dev = 0;
    OOMB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    auto& b = bufs[std::make_tuple(dev, st, slot)];
    if (b.second < bytes) {
        if (b.first) OOMB_CUDA(cudaFreeAsync(b.first, st));
        OOMB_CUDA(cudaMallocAsync(&b.first, bytes, st));
        b.second = bytes;
    }
    return b.first;
}

// SM count of the current device, queried once per device.
inline int device_sms() {
    static std::atomic<int> cache[64];
    int dev = 0;
    OOMB_CUDA(cudaGetDevice(&dev));
    int n = dev < 64 ? cache[dev].load(std::memory_order_relaxed) : 0;
    if (n == 0) {
        OOMB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
        if (dev < 64) cache[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

extern std::atomic<int64_t> g_kernel_launches;
inline void count_launch(int n = 1) { g_kernel_launches.fetch_add(n, std::memory_order_relaxed); }
void check_launch(const char* what);

// ---------------------------------------------------------------------------
// Per-kernel CUDA-event timing (oomb_profile_*). A launcher brackets its kernel
// with a ProfScope; events are recorded only while a pool with profiling on is
// the active pool of the calling thread.
// ---------------------------------------------------------------------------
enum ProfKind {
    PK_APPEND = 0, PK_SCORE, PK_TOPK, PK_FWD, PK_BWD_PREP, PK_BWD_DQ, PK_BWD_DKDV, PK_BWD_SIMT, PK_GRAD_INIT,
    PK_GATHER, PK_OTHER, PK_BWD_PAIR, PK_N
};
struct Profiler {
    struct Rec {
        int kind;
        cudaEvent_t e0, e1;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> spare;
    cudaEvent_t get() {
        if (!spare.empty()) {
            cudaEvent_t e = spare.back();
            spare.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};
extern thread_local Profiler* g_prof;
struct ProfScope {
    int kind;
    cudaStream_t st;
    cudaEvent_t e0 = nullptr;
    ProfScope(int k, cudaStream_t s) : kind(k), st(s) {
        if (g_prof) {
            e0 = g_prof->get();
            cudaEventRecord(e0, st);
        }
    }
    ~ProfScope() {
        if (g_prof && e0) {
            cudaEvent_t e1 = g_prof->get();
            cudaEventRecord(e1, st);
            g_prof->recs.push_back({kind, e0, e1});
        }
    }
};

// ---------------------------------------------------------------------------
// Debug CTA timeline. OOMB_CTA_TRACE="<tag>:<launch index>:<file>" makes the chosen
// launch of kernel <tag> write, per CTA, its SM id (slot 0) and %globaltimer stamps
// (slots 1..) into a device buffer that is dumped to <file> after the launch
// (int64 header {n_ctas, slots}, then n_ctas x slots uint64). Off by default; a null
// buffer makes every mark a predicated-off branch.
// ---------------------------------------------------------------------------
struct CtaTrace {
    unsigned long long* buf = nullptr;
    int slots = 0;
};
#ifdef __CUDACC__
__device__ __forceinline__ void trace_mark(const CtaTrace& t, int slot) {
    if (t.buf) {
        unsigned long long ts;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
        const size_t cta = blockIdx.x + static_cast<size_t>(gridDim.x) * (blockIdx.y + gridDim.y * blockIdx.z);
        t.buf[cta * t.slots + slot] = ts;
    }
}
__device__ __forceinline__ void trace_value(const CtaTrace& t, int slot, unsigned long long v) {
    if (t.buf) {
        const size_t cta = blockIdx.x + static_cast<size_t>(gridDim.x) * (blockIdx.y + gridDim.y * blockIdx.z);
        t.buf[cta * t.slots + slot] = v;
    }
}
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
#endif
CtaTrace trace_begin(const char* tag, size_t n_ctas, int slots);
void trace_end(CtaTrace& t, size_t n_ctas, cudaStream_t st);

// Device error flags (bitmask) written by kernels.
enum : int { DERR_NOT_RESIDENT = 1, DERR_BAD_ID = 2 };

// ---------------------------------------------------------------------------
// Geometry passed to every attention kernel.
// ---------------------------------------------------------------------------
struct AttnGeom {
    int C;         // query rows (tokens) in the chunk
    int Hq, Hkv, hd, P;
    int group;     // Hq / Hkv
    int m;         // query pages = ceil(C / P)
    int64_t filled;  // layer fill level (valid-slot mask of past pages)
    float scale;   // 1/sqrt(hd)
    int max_pages;
    int chunk_keys;  // 1: attend the chunk's causal prefix after the selected pages (attention.hpp:187-199);
                     // 0: selected pages only (a page-range shard other than the one owning the chunk's keys)
    double scale64;  // 1/sqrt(hd) in double (fp64 pools: the reference's Real = double)
};

// ---------------------------------------------------------------------------
// Kernel launchers (kernels_simt.cu)
// ---------------------------------------------------------------------------
struct NewSlots {
    int32_t first_page;  // logical page id of slot[0]
    int32_t n;
    int32_t slot[120];
};

// Device slot of a page this pool does not store (a page-range shard's REMOTE page): append
// updates its K_avg sums only. Slot -1 is a page that is not resident (a kernel error to read).
constexpr int32_t SLOT_REMOTE = -2;

void launch_append(int dtype, const void* k, const void* v, int64_t rows, int64_t filled_before, int P, int Hkv,
                   int hd, int first_page, int n_pages_touched, const NewSlots& ns, int32_t* d_kvslot_layer,
                   void* kpool, void* vpool, void* kavg_sum_layer, int32_t* kavg_cnt_layer, int* d_err,
                   cudaStream_t st, const double* rope_inv_freq = nullptr, void* kavg_planes_layer = nullptr,
                   int64_t plane_stride = 0);
// dst CSR = the ids of src with id % stride == rank, list order kept (one CTA).
void launch_filter_owned(const int32_t* src_off, const int32_t* src_ids, int m, int stride, int rank,
                         int32_t* dst_off, int32_t* dst_ids, cudaStream_t st);
void launch_rope(int in_dtype, int out_dtype, const void* x, int64_t rows, int heads, int hd, int64_t pos0, int sign,
                 const double* inv_freq, void* out, cudaStream_t st);
// Device table inv_freq[i] = base^(-2i/hd) computed on the host with the reference's std::pow
// (ops.hpp:198-201); cached per (device, base, hd) for the life of the library.
const double* rope_inv_freq_table(float base, int hd);
// Buffers typed "void*" below hold the pool's accumulation type: float for OOMB_F32 / OOMB_BF16
// pools, double for OOMB_F64 pools (f64 = true).
void launch_mean_keys(const void* kavg_sum_layer, const int32_t* kavg_cnt_layer, int n, int row_elems,
                      void* out, cudaStream_t st, bool f64 = false);
void launch_gather(int dtype, int grads, const int32_t* d_ids, int n, const int32_t* d_slot_layer,
                   const void* pk, const void* pv, int64_t filled, int P, int Hkv, int hd, void* k_out,
                   void* v_out, uint8_t* valid_out, int* d_err, cudaStream_t st);
void launch_scatter(const int32_t* d_ids, int n, const int32_t* d_gslot_layer, void* gk, void* gv,
                    const void* dk, const void* dv, int64_t filled, int P, int Hkv, int hd, int* d_err,
                    cudaStream_t st, bool f64 = false);
void launch_accumulate_grads(const int32_t* d_ids, int n, const int32_t* d_gslot_layer, const void* gk,
                             const void* gv, int64_t filled, int P, int Hkv, int hd, void* dk, void* dv,
                             cudaStream_t st, int64_t rope_pos0 = 0,
                             const double* rope_inv_freq = nullptr, bool f64 = false, int first = 0);
void launch_grad_init(const int32_t* d_pages, const int32_t* d_slots, int n, int32_t* d_gslot_layer, void* gk,
                      void* gv, int64_t page_elems, cudaStream_t st, int elem_bytes = 4);
void launch_zero_slots(const int32_t* d_slots, int n, void* gk, void* gv, int64_t page_elems, cudaStream_t st,
                       int elem_bytes = 4);

// scale: the float score scale (fp32 / bf16), scale64 the same in double (fp64 pools). stats_scratch:
// tokens * Hq * 2 elements of the accumulation type.
void launch_score_simt(int dtype, const void* q, int64_t tokens, int Hq, int hd, const void* k_avg, int64_t n,
                       int Hkv, int P, float scale, double scale64, void* vote, void* stats_scratch, cudaStream_t st,
                       bool partial_only = false);
void launch_lse_merge(const void* o_parts, const float* lse_parts, int parts, int64_t rows, int hd, int dtype,
                      void* out, float* lse, cudaStream_t st);
void launch_topk(const void* vote, int m, int n, int k, int32_t* sel_off, int32_t* sel_ids, cudaStream_t st,
                 bool f64 = false);
void launch_fill_csr_all(int32_t* off, int32_t* ids, int m, int first, int count, cudaStream_t st);

void launch_attn_fwd_simt(int dtype, const AttnGeom& g, const void* q, const int32_t* sel_off,
                          const int32_t* sel_ids, const int32_t* d_kvslot_layer, const void* kpool,
                          const void* vpool, const void* k_cur, const void* v_cur, void* out, void* lse, int* d_err,
                          cudaStream_t st);
void launch_attn_bwd_simt(int dtype, const AttnGeom& g, const void* dout, const void* q, const int32_t* sel_off,
                          const int32_t* sel_ids, const int32_t* d_kvslot_layer, const int32_t* d_gslot_layer,
                          const void* kpool, const void* vpool, void* gkpool, void* gvpool, const void* k_cur,
                          const void* v_cur, const void* out, const void* lse, void* dq, void* dk_cur,
                          void* dv_cur, int* d_err, cudaStream_t st, int n_past_pages);

// ---------------------------------------------------------------------------
// tcgen05 / TMA kernels (attn_tc.cu)
// ---------------------------------------------------------------------------
struct TcPoolMaps {
    CUtensorMap kpool;  // [n_slots*Hkv*P rows][hd] bf16, box 128 x 64, SW128
    CUtensorMap vpool;
    CUtensorMap gkpool;  // [n_g_slots*Hkv*P rows][hd] fp32, box 128 x 32, SW128 (TMA reduce-add target)
    CUtensorMap gvpool;
    bool valid = false;
};
bool tc_supported(const AttnGeom& g, int dtype);
bool tc_bwd_available();
void make_pool_maps(TcPoolMaps& maps, const void* kpool, const void* vpool, int64_t n_slots, const float* gkpool,
                    const float* gvpool, int64_t n_g_slots, int Hkv, int P, int hd);
void launch_attn_fwd_tc(const AttnGeom& g, const TcPoolMaps& maps, const void* q, const int32_t* sel_off,
                        const int32_t* sel_ids, const int32_t* d_kvslot_layer, const void* k_cur, const void* v_cur,
                        void* out, float* lse, int* d_err, cudaStream_t st);
void launch_attn_fwd_tc4(const AttnGeom& g, const TcPoolMaps& maps, const void* q, const int32_t* sel_off,
                         const int32_t* sel_ids, const int32_t* d_kvslot_layer, const void* k_cur, const void* v_cur,
                         void* out, float* lse, int* d_err, cudaStream_t st);
void launch_attn_bwd_tc(const AttnGeom& g, const TcPoolMaps& maps, const void* dout, const void* q,
                        const int32_t* sel_off, const int32_t* sel_ids, const int32_t* d_kvslot_layer,
                        const int32_t* d_gslot_layer, float* gkpool, float* gvpool, const void* k_cur,
                        const void* v_cur, const void* out, const float* lse, float* dq, float* dk_cur,
                        float* dv_cur, int* d_err, void* workspace, size_t workspace_bytes, int nnz, int n_pages,
                        cudaStream_t st, cudaStream_t side, cudaEvent_t ev_prep, cudaEvent_t ev_dq, bool join_dq, int readback_first = -1);
size_t attn_bwd_tc_workspace(const AttnGeom& g, int max_sel_ids);
// Split-K count of the tcgen05 forward / dQ kernels for small grids (attn_fwd4.cu).
int attn_tc_splits(const AttnGeom& g, int num_sms);
bool score_tc_supported(int dtype, int hd, int P, int64_t tokens);
size_t score_tc_workspace(int64_t tokens, int Hq, int Hkv, int64_t n, int P);
void launch_score_tc(const void* q, int64_t tokens, int Hq, int Hkv, int P, const float* kavg_sum,
                     const int32_t* kavg_cnt, const float* kavg_f32, int64_t n, float scale, float* vote, void* ws,
                     cudaStream_t st, bool partial_only = false, const void* planes = nullptr,
                     int64_t plane_stride = 0);
void launch_vote_reduce(const float* part, int groups, int64_t mn, float* vote, cudaStream_t st);
void launch_debug_tc_gemm(int mode, const void* a, const void* b, float* c, int m, int n, int k, cudaStream_t st);

// Driver entry point for cuTensorMapEncodeTiled (no libcuda link dependency).
CUresult encode_tensor_map(CUtensorMap* map, CUtensorMapDataType dt, uint32_t rank, void* base,
                           const uint64_t* dims, const uint64_t* strides_bytes, const uint32_t* box,
                           CUtensorMapSwizzle swz);

}  // namespace oomb
