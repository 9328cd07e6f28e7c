// SPDX-License-Identifier: Apache-2.0
//
// oomb.hpp — C++ facade over the C ABI (oomb.h), header-only.
//
// It keeps the reference's operator API for the hot path: names, argument meaning and
// exception classes. Paths are relative to /root/reference/proj/core/include/chunktrain/.
//   PagedCache            paged_kv.hpp:41-356
//   score_pages           attention.hpp:32-67
//   select_topk(_row)     attention.hpp:71-96; select_recent / select_all :99-111
//   attn_forward          attention.hpp:156-208 (AttnSaved :117-124)
//   attn_backward         attention.hpp:222-293 (AttnGrads :210-220)
//   TieredEngine          tiered_memory.hpp:99-432; validate_schedule tiered_memory.cpp:47-138
//   ConfigError ... IoError   common.hpp:15-29
//
// Two tensor flavours:
//   * DeviceTensor — a row-major device buffer. This is the B200 path: no host copies.
//   * Tensor<Real> — the reference's host value type (shape + data). The overloads that take it
//     copy in, run on the device and copy out, so a reference call site compiles unchanged
//     (Real = double computes in fp32 on the device: the pool holds fp32 or bf16 pages).
// Selections are the reference's vector<vector<int32_t>> or a device-resident Selection.
// Every facade call throws the reference's exception class for the C status it gets back.
//
// Link: -loomb (paper_2602_02108_b200/liboomb.so) -lcudart.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "oomb.h"

namespace oomb {

// ---------------------------------------------------------------------------- errors
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& msg, int code = OOMB_ERROR) : std::runtime_error(msg), code_(code) {}
    int code() const { return code_; }

private:
    int code_;
};
struct ConfigError : Error {
    explicit ConfigError(const std::string& m) : Error(m, OOMB_CONFIG_ERROR) {}
};
struct ShapeError : Error {
    explicit ShapeError(const std::string& m) : Error(m, OOMB_SHAPE_ERROR) {}
};
struct StateError : Error {
    explicit StateError(const std::string& m) : Error(m, OOMB_STATE_ERROR) {}
};
struct ResidencyError : Error {
    explicit ResidencyError(const std::string& m) : Error(m, OOMB_RESIDENCY_ERROR) {}
};
struct IoError : Error {
    explicit IoError(const std::string& m) : Error(m, OOMB_IO_ERROR) {}
};
struct CudaError : Error {
    explicit CudaError(const std::string& m) : Error(m, OOMB_CUDA_ERROR) {}
};

[[noreturn]] inline void throw_status(int st, const std::string& msg) {
    switch (st) {
        case OOMB_CONFIG_ERROR: throw ConfigError(msg);
        case OOMB_SHAPE_ERROR: throw ShapeError(msg);
        case OOMB_STATE_ERROR: throw StateError(msg);
        case OOMB_RESIDENCY_ERROR: throw ResidencyError(msg);
        case OOMB_IO_ERROR: throw IoError(msg);
        case OOMB_CUDA_ERROR: throw CudaError(msg);
        default: throw Error(msg, st);
    }
}
inline void check(int st) {
    if (st != OOMB_OK) throw_status(st, oomb_last_error());
}
inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------- ModelConfig
enum class AttentionMode { dense, topk, local };

// config.hpp:19-49; validate() restates config.cpp:30-51 (the C ABI re-checks the fields it uses).
struct ModelConfig {
    int n_layers = 2;
    int d_model = 64;
    int n_q_heads = 4;
    int n_kv_heads = 2;
    int head_dim = 16;
    int d_ff = 256;
    int vocab_size = 256;
    int chunk_size = 64;
    int page_size = 16;
    std::vector<AttentionMode> attention_mode{AttentionMode::dense};
    int retrieval_budget = 128;
    int local_window = 4;
    double rope_base = 10000.0;
    uint64_t seed = 0;
    bool score_scale = false;

    int gqa_group() const { return n_q_heads / n_kv_heads; }
    int pages_per_chunk() const { return chunk_size / page_size; }
    int budget_pages() const { return retrieval_budget / page_size; }
    AttentionMode mode_for_layer(int layer) const {
        return attention_mode.size() == 1 ? attention_mode[0] : attention_mode.at(static_cast<size_t>(layer));
    }
    void validate() const {
        auto req = [](bool ok, const char* msg) {
            if (!ok) throw ConfigError(std::string("config: ") + msg);
        };
        req(n_layers >= 1, "n_layers must be >= 1");
        req(d_model >= 1, "d_model must be >= 1");
        req(n_q_heads >= 1 && n_kv_heads >= 1, "head counts must be >= 1");
        req(n_q_heads % n_kv_heads == 0, "n_q_heads must be divisible by n_kv_heads");
        req(head_dim >= 2 && head_dim % 2 == 0, "head_dim must be even (rotary pairs)");
        req(d_ff >= 1, "d_ff must be >= 1");
        req(vocab_size >= 2, "vocab_size must be >= 2");
        req(page_size >= 1, "page_size must be >= 1");
        req(chunk_size >= 1, "chunk_size must be >= 1");
        req(chunk_size % page_size == 0, "chunk_size must be divisible by page_size");
        req(retrieval_budget >= 0, "retrieval_budget must be >= 0");
        req(retrieval_budget % page_size == 0, "retrieval_budget must be divisible by page_size");
        req(local_window >= 0, "local_window must be >= 0");
        req(rope_base > 1.0, "rope_base must be > 1");
        req(attention_mode.size() == 1 || attention_mode.size() == static_cast<size_t>(n_layers),
            "attention_mode needs one entry or one per layer");
    }
};

// ---------------------------------------------------------------------------- tensors
enum class DType { f32 = OOMB_F32, bf16 = OOMB_BF16, f64 = OOMB_F64, i32 = 10, u8 = 11 };
inline size_t dtype_size(DType d) { return d == DType::bf16 ? 2 : d == DType::u8 ? 1 : d == DType::f64 ? 8 : 4; }
// Accumulation type of a pool dtype: K_avg, gradient pages, lse / dq / dk_cur / dv_cur and votes.
inline DType acc_dtype(DType pool) { return pool == DType::f64 ? DType::f64 : DType::f32; }

inline uint16_t f32_to_bf16(float f) {  // round to nearest even (NaN kept quiet)
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}
inline float bf16_to_f32(uint16_t b) {
    const uint32_t u = static_cast<uint32_t>(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

inline int64_t checked_numel(const std::vector<int64_t>& s) {
    int64_t n = 1;
    for (int64_t e : s) {
        if (e < 0) throw ShapeError("negative tensor extent");
        n *= e;
    }
    return n;
}

// The reference's host value type (tensor.hpp:19-125): only what the facade's overloads need.
template <class Real>
struct Tensor {
    std::vector<int64_t> shape;
    std::vector<Real> data;
    Tensor() = default;
    explicit Tensor(std::vector<int64_t> s) : shape(std::move(s)) { data.assign(static_cast<size_t>(checked_numel(shape)), Real(0)); }
    Tensor(std::vector<int64_t> s, std::vector<Real> d) : shape(std::move(s)), data(std::move(d)) {
        if (static_cast<int64_t>(data.size()) != checked_numel(shape)) throw ShapeError("tensor data size does not match shape");
    }
    int64_t numel() const { return static_cast<int64_t>(data.size()); }
    int rank() const { return static_cast<int>(shape.size()); }
    int64_t dim(int i) const { return shape.at(static_cast<size_t>(i)); }
};

// Row-major device buffer (owning, shared on copy like a handle).
class DeviceTensor {
public:
    DeviceTensor() = default;
    DeviceTensor(std::vector<int64_t> shape, DType dt, bool zero = true) : shape_(std::move(shape)), dtype_(dt) {
        const size_t n = bytes();
        void* p = nullptr;
        if (n) {
            cuda_check(cudaMalloc(&p, n), "cudaMalloc");
            if (zero) cuda_check(cudaMemset(p, 0, n), "cudaMemset");
        }
        buf_ = std::shared_ptr<void>(p, [](void* q) {
            if (q) cudaFree(q);
        });
    }
    // Upload host values, converted to dt (bf16: round to nearest even).
    template <class Real>
    static DeviceTensor from_host(const std::vector<int64_t>& shape, const Real* src, DType dt) {
        DeviceTensor t(shape, dt, false);
        const int64_t n = t.numel();
        if (dt == DType::bf16) {
            std::vector<uint16_t> h(static_cast<size_t>(n));
            for (int64_t i = 0; i < n; ++i) h[i] = f32_to_bf16(static_cast<float>(src[i]));
            t.upload(h.data());
        } else if (dt == DType::f32) {
            std::vector<float> h(static_cast<size_t>(n));
            for (int64_t i = 0; i < n; ++i) h[i] = static_cast<float>(src[i]);
            t.upload(h.data());
        } else if (dt == DType::f64) {
            std::vector<double> h(static_cast<size_t>(n));
            for (int64_t i = 0; i < n; ++i) h[i] = static_cast<double>(src[i]);
            t.upload(h.data());
        } else {
            throw ShapeError("from_host: floating-point dtypes only");
        }
        return t;
    }
    template <class Real>
    static DeviceTensor from_host(const Tensor<Real>& h, DType dt) {
        return from_host(h.shape, h.data.data(), dt);
    }
    static DeviceTensor from_ids(const std::vector<int32_t>& ids) {
        DeviceTensor t({static_cast<int64_t>(ids.size())}, DType::i32, false);
        t.upload(ids.data());
        return t;
    }
    // Download as Real (bf16 / f32 up-cast exactly).
    template <class Real = float>
    std::vector<Real> to_host() const {
        cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
        const int64_t n = numel();
        std::vector<Real> out(static_cast<size_t>(n));
        if (dtype_ == DType::bf16) {
            std::vector<uint16_t> h(static_cast<size_t>(n));
            download(h.data());
            for (int64_t i = 0; i < n; ++i) out[i] = static_cast<Real>(bf16_to_f32(h[i]));
        } else if (dtype_ == DType::f32) {
            std::vector<float> h(static_cast<size_t>(n));
            download(h.data());
            for (int64_t i = 0; i < n; ++i) out[i] = static_cast<Real>(h[i]);
        } else if (dtype_ == DType::f64) {
            std::vector<double> h(static_cast<size_t>(n));
            download(h.data());
            for (int64_t i = 0; i < n; ++i) out[i] = static_cast<Real>(h[i]);
        } else if (dtype_ == DType::i32) {
            std::vector<int32_t> h(static_cast<size_t>(n));
            download(h.data());
            for (int64_t i = 0; i < n; ++i) out[i] = static_cast<Real>(h[i]);
        } else {
            std::vector<uint8_t> h(static_cast<size_t>(n));
            download(h.data());
            for (int64_t i = 0; i < n; ++i) out[i] = static_cast<Real>(h[i]);
        }
        return out;
    }
    template <class Real>
    Tensor<Real> to_tensor() const {
        return Tensor<Real>(shape_, to_host<Real>());
    }

    void* data() { return buf_.get(); }
    const void* data() const { return buf_.get(); }
    template <class T>
    T* as() {
        return static_cast<T*>(buf_.get());
    }
    template <class T>
    const T* as() const {
        return static_cast<const T*>(buf_.get());
    }
    const std::vector<int64_t>& shape() const { return shape_; }
    int64_t dim(int i) const { return shape_.at(static_cast<size_t>(i)); }
    int rank() const { return static_cast<int>(shape_.size()); }
    int64_t numel() const { return checked_numel(shape_); }
    size_t bytes() const { return static_cast<size_t>(numel()) * dtype_size(dtype_); }
    DType dtype() const { return dtype_; }
    bool same_shape(const DeviceTensor& o) const { return shape_ == o.shape_; }

private:
    void upload(const void* h) {
        if (bytes()) cuda_check(cudaMemcpy(buf_.get(), h, bytes(), cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    }
    void download(void* h) const {
        if (bytes()) cuda_check(cudaMemcpy(h, buf_.get(), bytes(), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
    }
    std::shared_ptr<void> buf_;
    std::vector<int64_t> shape_;
    DType dtype_ = DType::f32;
};

// ---------------------------------------------------------------------------- PagedCache
enum class Tier : uint8_t { device, host };

struct MemoryReport {  // paged_kv.hpp:25-32
    uint64_t device_bytes = 0;
    uint64_t host_bytes = 0;
    uint64_t grad_bytes = 0;
    int64_t pages = 0;
    int64_t reallocs = 0;
    uint64_t copied_bytes = 0;
};
inline MemoryReport to_report(const oomb_memory_report& r) {
    return MemoryReport{r.device_bytes, r.host_bytes, r.grad_bytes, r.pages, r.reallocs, r.copied_bytes};
}

struct SlotRange {
    int64_t begin = 0;
    int64_t end = 0;  // exclusive
};

struct Gathered {  // paged_kv.hpp:110-116: [n*P][Hkv][hd] K, V and the per-slot valid mask
    DeviceTensor k, v, valid;
};

inline void* sv(cudaStream_t s) { return static_cast<void*>(s); }

class PagedCache {
public:
    // dtype: bf16 (the tcgen05 path) or f32 (1e-5 parity path). max_tokens: per-layer capacity of
    // the device page table (default 64 chunks). device_capacity_pages: KV page slots on the device
    // for all layers (default: every page resident; a TieredEngine offloads beyond it).
    // page_owner_stride / page_owner_rank: a page-range shard (oomb_config); 0 = every page.
    explicit PagedCache(const ModelConfig& cfg, DType dtype = DType::bf16, int64_t max_tokens = -1, int device = 0,
                        int64_t device_capacity_pages = -1, int page_owner_stride = 0, int page_owner_rank = 0)
        : cfg_(cfg), dtype_(dtype) {
        cfg.validate();
        if (dtype != DType::bf16 && dtype != DType::f32 && dtype != DType::f64)
            throw ConfigError("PagedCache: dtype must be bf16, f32 or f64");
        oomb_config c{cfg.n_layers,       cfg.n_q_heads,    cfg.n_kv_heads,
                      cfg.head_dim,       cfg.chunk_size,   cfg.page_size,
                      cfg.retrieval_budget, cfg.local_window, cfg.score_scale ? 1 : 0,
                      static_cast<int>(dtype), max_tokens > 0 ? max_tokens : 64LL * cfg.chunk_size,
                      device_capacity_pages, page_owner_stride, page_owner_rank};
        check(oomb_pool_create(&c, device, &pool_));
    }
    ~PagedCache() {
        if (pool_) oomb_pool_destroy(pool_);
    }
    PagedCache(const PagedCache&) = delete;
    PagedCache& operator=(const PagedCache&) = delete;

    oomb_pool_t handle() const { return pool_; }
    const ModelConfig& config() const { return cfg_; }
    DType dtype() const { return dtype_; }
    int n_layers() const { return cfg_.n_layers; }
    int page_size() const { return cfg_.page_size; }
    int64_t page_elems() const { return static_cast<int64_t>(cfg_.page_size) * cfg_.n_kv_heads * cfg_.head_dim; }
    uint64_t page_kv_bytes() const { return 2 * static_cast<uint64_t>(page_elems()) * dtype_size(dtype_); }
    static int full_pages_before(int64_t tokens, int page_size) { return static_cast<int>(tokens / page_size); }

    int64_t filled(int layer) const {
        int64_t f = 0;
        check(oomb_filled(pool_, layer, &f));
        return f;
    }
    int n_pages(int layer) const {
        int n = 0;
        check(oomb_n_pages(pool_, layer, &n));
        return n;
    }

    // paged_kv.hpp:73-108. k, v [rows][Hkv][hd] in the pool dtype.
    SlotRange append_chunk(int layer, const DeviceTensor& k, const DeviceTensor& v, cudaStream_t st = nullptr) {
        check_kv(k, v, "append_chunk");
        SlotRange r;
        check(oomb_append_chunk(pool_, layer, k.data(), v.data(), k.dim(0), sv(st), &r.begin, &r.end));
        return r;
    }
    template <class Real>
    SlotRange append_chunk(int layer, const Tensor<Real>& k, const Tensor<Real>& v) {
        return append_chunk(layer, DeviceTensor::from_host(k, dtype_), DeviceTensor::from_host(v, dtype_));
    }
    // Fused projection epilogue: k_raw is the PRE-RoPE key projection, rotated at its absolute
    // positions (ops.hpp:192-225) on its way into the page.
    SlotRange append_chunk_rope(int layer, const DeviceTensor& k_raw, const DeviceTensor& v, float rope_base,
                                cudaStream_t st = nullptr) {
        check_kv(k_raw, v, "append_chunk_rope");
        SlotRange r;
        check(oomb_append_chunk_rope(pool_, layer, k_raw.data(), v.data(), k_raw.dim(0), rope_base, sv(st), &r.begin,
                                     &r.end));
        return r;
    }

    Gathered gather_pages(int layer, std::span<const int32_t> ids, cudaStream_t st = nullptr) const {
        return gather(layer, ids, false, st);
    }
    Gathered gather_grad_pages(int layer, std::span<const int32_t> ids, cudaStream_t st = nullptr) const {
        return gather(layer, ids, true, st);
    }
    // paged_kv.hpp:135-164: dk / dv fp32 in the gather layout [n*P][Hkv][hd].
    void scatter_add_grads(int layer, std::span<const int32_t> ids, const DeviceTensor& dk, const DeviceTensor& dv,
                           cudaStream_t st = nullptr) {
        const int64_t want = static_cast<int64_t>(ids.size()) * cfg_.page_size;
        if (dk.rank() != 3 || dk.dim(0) != want || dk.dim(1) != cfg_.n_kv_heads || dk.dim(2) != cfg_.head_dim ||
            !dk.same_shape(dv) || dk.dtype() != acc_dtype(dtype_) || dv.dtype() != acc_dtype(dtype_))
            throw ShapeError("scatter_add_grads: gradient shape does not match gather layout");
        check(oomb_scatter_add_grads(pool_, layer, ids.data(), static_cast<int>(ids.size()), dk.data(), dv.data(),
                                     sv(st)));
    }
    // dM_i read-back (chunk_trainer.hpp:575-587): dk/dv += the pages' gradient rows.
    void accumulate_grad_pages(int layer, std::span<const int32_t> ids, DeviceTensor& dk, DeviceTensor& dv,
                               cudaStream_t st = nullptr) {
        check(oomb_accumulate_grad_pages(pool_, layer, ids.data(), static_cast<int>(ids.size()), dk.data(), dv.data(),
                                         sv(st)));
    }
    // The same read-back fused with rope_backward of dK (chunk_trainer.hpp:575-592): row r of dk is
    // rotated back from absolute position pos_offset + r.
    void accumulate_grad_pages_rope(int layer, std::span<const int32_t> ids, DeviceTensor& dk, DeviceTensor& dv,
                                    int64_t pos_offset, float rope_base, cudaStream_t st = nullptr) {
        check(oomb_accumulate_grad_pages_rope(pool_, layer, ids.data(), static_cast<int>(ids.size()), dk.as<float>(),
                                              dv.as<float>(), pos_offset, rope_base, sv(st)));
    }
    // paged_kv.hpp:170-183: [n][Hkv][hd] fp32.
    DeviceTensor page_mean_keys(int layer, int n_candidates = -1, cudaStream_t st = nullptr) const {
        const int n = n_candidates < 0 ? n_pages(layer) : std::min(n_candidates, n_pages(layer));
        DeviceTensor out({n, cfg_.n_kv_heads, cfg_.head_dim}, acc_dtype(dtype_), false);
        int n_out = 0;
        check(oomb_page_mean_keys(pool_, layer, n_candidates, out.data(), sv(st), &n_out));
        return out;
    }
    MemoryReport memory_report() const {
        oomb_memory_report r{};
        check(oomb_memory_report_get(pool_, &r));
        return to_report(r);
    }
    Tier tier(int layer, int page) const {
        int t = 0;
        check(oomb_get_tier(pool_, layer, page, &t));
        return static_cast<Tier>(t);
    }
    void set_tier(int layer, int page, Tier t) { check(oomb_set_tier(pool_, layer, page, static_cast<int>(t))); }
    bool grads_allocated(int layer, int page) const {
        int a = 0;
        check(oomb_grads_allocated(pool_, layer, page, &a));
        return a != 0;
    }
    void set_residency_enforced(bool on) {
        check(oomb_set_residency_enforced(pool_, on ? 1 : 0));
        enforced_ = on;
    }
    bool residency_enforced() const { return enforced_; }
    void zero_grad_pages(cudaStream_t st = nullptr) { check(oomb_zero_grad_pages(pool_, sv(st))); }
    void reset(cudaStream_t st = nullptr) { check(oomb_pool_reset(pool_, sv(st))); }
    // Logical page -> arena ids {k, v, gk, gv} as the reference numbers them (bit-exact parity).
    std::vector<int32_t> page_table(int layer) const {
        std::vector<int32_t> out(static_cast<size_t>(4) * n_pages(layer));
        check(oomb_page_table_get(pool_, layer, out.data()));
        return out;
    }
    // Surfaces a ResidencyError raised on the device (a kernel read a page tagged host).
    void check_device_errors() const { check(oomb_check_device_errors(pool_)); }

private:
    friend class TieredEngine;  // the engine turns residency enforcement on for its lifetime
    void check_kv(const DeviceTensor& k, const DeviceTensor& v, const char* op) const {
        if (k.rank() != 3 || k.dim(1) != cfg_.n_kv_heads || k.dim(2) != cfg_.head_dim || !k.same_shape(v) ||
            k.dtype() != dtype_ || v.dtype() != dtype_)
            throw ShapeError(std::string(op) + ": expected [rows x kvh x hd] K/V of equal shape in the pool dtype");
    }
    Gathered gather(int layer, std::span<const int32_t> ids, bool grads, cudaStream_t st) const {
        const int64_t rows = static_cast<int64_t>(ids.size()) * cfg_.page_size;
        Gathered g{DeviceTensor({rows, cfg_.n_kv_heads, cfg_.head_dim}, grads ? acc_dtype(dtype_) : dtype_),
                   DeviceTensor({rows, cfg_.n_kv_heads, cfg_.head_dim}, grads ? acc_dtype(dtype_) : dtype_),
                   DeviceTensor({rows}, DType::u8)};
        check(oomb_gather_pages(pool_, layer, ids.data(), static_cast<int>(ids.size()), grads ? 1 : 0, g.k.data(),
                                g.v.data(), g.valid.as<uint8_t>(), sv(st)));
        return g;
    }

    ModelConfig cfg_;
    DType dtype_;
    oomb_pool_t pool_ = nullptr;
    bool enforced_ = false;
};

// ---------------------------------------------------------------------------- selection
using PageLists = std::vector<std::vector<int32_t>>;

// AttnSaved::selected (attention.hpp:117-124) as a device CSR with a pinned host mirror.
class Selection {
public:
    Selection(const PagedCache& cache, int max_query_pages, int max_ids) {
        oomb_selection_t s = nullptr;
        check(oomb_selection_create(cache.handle(), std::max(max_query_pages, 1), std::max(max_ids, 1), &s));
        h_ = std::shared_ptr<oomb_selection_s>(s, [](oomb_selection_t p) {
            if (p) oomb_selection_destroy(p);
        });
    }
    static Selection from_lists(const PagedCache& cache, const PageLists& lists, cudaStream_t st = nullptr) {
        std::vector<int32_t> off(lists.size() + 1, 0), ids;
        for (size_t i = 0; i < lists.size(); ++i) {
            off[i + 1] = off[i] + static_cast<int32_t>(lists[i].size());
            ids.insert(ids.end(), lists[i].begin(), lists[i].end());
        }
        Selection s(cache, static_cast<int>(lists.size()), static_cast<int>(ids.size()));
        check(oomb_selection_set_host(s.handle(), off.data(), ids.empty() ? nullptr : ids.data(),
                                      static_cast<int>(lists.size()), sv(st)));
        return s;
    }
    oomb_selection_t handle() const { return h_.get(); }
    // The per-query-page lists (waits for the selection's device-to-host mirror).
    PageLists lists() const {
        int m = 0, nnz = 0;
        check(oomb_selection_get_host(handle(), nullptr, nullptr, &m, &nnz));
        std::vector<int32_t> off(static_cast<size_t>(m) + 1), ids(static_cast<size_t>(std::max(nnz, 1)));
        check(oomb_selection_get_host(handle(), off.data(), ids.data(), &m, &nnz));
        PageLists out(static_cast<size_t>(m));
        for (int i = 0; i < m; ++i) out[i].assign(ids.begin() + off[i], ids.begin() + off[i + 1]);
        return out;
    }

private:
    std::shared_ptr<oomb_selection_s> h_;
};

// ---------------------------------------------------------------------------- scoring / selection
// attention.hpp:32-67: q [tokens][Hq][hd] (bf16 or f32), k_avg [n][Hkv][hd] f32 -> vote [m][n] f32.
inline DeviceTensor score_pages(const DeviceTensor& q, const DeviceTensor& k_avg, int page_size, int gqa_group,
                                bool score_scale = false, cudaStream_t st = nullptr) {
    if (q.rank() != 3 || k_avg.rank() != 3) throw ShapeError("score_pages: expected rank-3 inputs");
    if (k_avg.dim(0) < 1) throw ShapeError("score_pages: needs at least one candidate page");
    if (q.dim(1) != static_cast<int64_t>(gqa_group) * k_avg.dim(1) || q.dim(2) != k_avg.dim(2) ||
        k_avg.dtype() != acc_dtype(q.dtype()) ||
        (q.dtype() != DType::f32 && q.dtype() != DType::bf16 && q.dtype() != DType::f64))
        throw ShapeError("score_pages: head counts / dtypes do not match");
    const int64_t m = (q.dim(0) + page_size - 1) / page_size;
    DeviceTensor vote({m, k_avg.dim(0)}, acc_dtype(q.dtype()), false);
    check(oomb_score_pages(q.data(), q.dim(0), static_cast<int>(q.dim(1)), static_cast<int>(q.dim(2)),
                           k_avg.data(), k_avg.dim(0), static_cast<int>(k_avg.dim(1)), page_size,
                           score_scale ? 1 : 0, static_cast<int>(q.dtype()), vote.data(), sv(st)));
    return vote;
}
template <class Real>
Tensor<Real> score_pages(const Tensor<Real>& q, const Tensor<Real>& k_avg, int page_size, int gqa_group,
                         bool score_scale = false) {
    if (q.rank() != 3 || k_avg.rank() != 3) throw ShapeError("score_pages: expected rank-3 inputs");
    // Real = double computes in double on the device (an OOMB_F64 path), float in fp32
    const DType dt = std::is_same_v<Real, double> ? DType::f64 : DType::f32;
    return score_pages(DeviceTensor::from_host(q, dt), DeviceTensor::from_host(k_avg, dt), page_size,
                       gqa_group, score_scale)
        .template to_tensor<Real>();
}

// attention.hpp:99-111 (host index lists, as in the reference).
inline std::vector<int32_t> select_recent(int n_pages, int window) {
    if (window < 0) throw ShapeError("select_recent: negative window");
    const int take = std::min(n_pages, window);
    std::vector<int32_t> ids(static_cast<size_t>(std::max(take, 0)));
    std::iota(ids.begin(), ids.end(), n_pages - take);
    return ids;
}
inline std::vector<int32_t> select_all(int n_pages) {
    std::vector<int32_t> ids(static_cast<size_t>(std::max(n_pages, 0)));
    std::iota(ids.begin(), ids.end(), 0);
    return ids;
}
// select_topk_row for every row of a device vote matrix [m][n], on the device (attention.hpp:71-96:
// k largest, ties to the lower id, ascending; k >= n -> all; k < 0 -> ShapeError).
inline Selection select_topk_rows(const PagedCache& cache, const DeviceTensor& vote, int budget_pages,
                                  cudaStream_t st = nullptr) {
    if (vote.rank() != 2 || vote.dtype() != acc_dtype(cache.dtype()))
        throw ShapeError("select_topk: vote must be [m x n] in the pool's accumulation type");
    const int m = static_cast<int>(vote.dim(0)), n = static_cast<int>(vote.dim(1));
    const int kk = std::min(std::max(budget_pages, 0), n);
    Selection sel(cache, m, m * kk);
    check(oomb_select_topk(sel.handle(), vote.data(), m, n, budget_pages, sv(st)));
    return sel;
}
// attention.hpp:71-96 with the reference's host signatures, computed by the device selector on a
// scratch pool, on the row as double (an fp64 scratch pool), exactly as the reference compares it.
namespace detail {
inline const PagedCache& scratch_cache() {
    static PagedCache c([] {
        ModelConfig m;
        m.n_layers = 1, m.n_q_heads = 1, m.n_kv_heads = 1, m.head_dim = 2, m.chunk_size = 1, m.page_size = 1;
        m.retrieval_budget = 0;
        return m;
    }(), DType::f64, 1);  // the reference compares scores as double (attention.hpp:71-88)
    return c;
}
}  // namespace detail
inline std::vector<int32_t> select_topk(std::span<const double> score_row, int budget_pages) {
    if (budget_pages < 0) throw ShapeError("select_topk: negative budget");
    const int64_t n = static_cast<int64_t>(score_row.size());
    if (n == 0) return {};
    auto vote = DeviceTensor::from_host(std::vector<int64_t>{1, n}, score_row.data(), DType::f64);
    return select_topk_rows(detail::scratch_cache(), vote, budget_pages).lists()[0];
}
template <class Real>
std::vector<int32_t> select_topk_row(const Tensor<Real>& score, int64_t row, int budget_pages) {
    const int64_t n = score.dim(1);
    std::vector<double> s(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) s[static_cast<size_t>(j)] = static_cast<double>(score.data[row * n + j]);
    return select_topk(s, budget_pages);
}

// The trainer's top-k selector in one device call (chunk_trainer.hpp:305-311).
inline Selection select_pages_topk(PagedCache& cache, int layer, const DeviceTensor& q, int n_candidates,
                                   cudaStream_t st = nullptr) {
    const ModelConfig& cfg = cache.config();
    const int m = static_cast<int>((q.dim(0) + cfg.page_size - 1) / cfg.page_size);
    const int n = std::min(n_candidates, cache.n_pages(layer));
    const int k = std::min(cfg.budget_pages(), std::max(n, 0));
    Selection sel(cache, m, m * k);
    DeviceTensor vote({m, std::max(n, 1)}, acc_dtype(cache.dtype()), false);
    check(oomb_select_pages_topk(cache.handle(), layer, q.data(), q.dim(0), n_candidates, sel.handle(),
                                 vote.data(), sv(st)));
    return sel;
}

// ---------------------------------------------------------------------------- attention
struct DeviceAttnSaved {  // AttnSaved on the device: out (pool dtype), lse f32 natural log
    DeviceTensor out, lse;
    Selection selected;
};
struct DeviceAttnGrads {  // AttnGrads: fp32
    DeviceTensor dq, dk_cur, dv_cur;
};
template <class Real>
struct AttnSaved {  // attention.hpp:117-124
    Tensor<Real> out;
    Tensor<Real> lse;
    PageLists selected;
};
template <class Real>
struct AttnGrads {  // attention.hpp:210-220
    Tensor<Real> dq, dk_cur, dv_cur;
};

namespace detail {
inline void check_qkv(const ModelConfig& cfg, const DeviceTensor& q, const DeviceTensor& k_cur,
                      const DeviceTensor& v_cur, const char* op) {
    if (q.rank() != 3 || q.dim(1) != cfg.n_q_heads || q.dim(2) != cfg.head_dim || k_cur.rank() != 3 ||
        k_cur.dim(0) != q.dim(0) || k_cur.dim(1) != cfg.n_kv_heads || k_cur.dim(2) != cfg.head_dim ||
        !k_cur.same_shape(v_cur))
        throw ShapeError(std::string(op) + ": q / k_cur / v_cur shape mismatch");
}
}  // namespace detail

// attention.hpp:156-208 on the device. Under residency enforcement the library checks the selected
// pages on the host before the launch (ResidencyError); the kernels' device-side flag is read by
// PagedCache::check_device_errors() (it synchronises, so it is not done per call).
inline DeviceAttnSaved attn_forward(const ModelConfig& cfg, const DeviceTensor& q, PagedCache& cache, int layer,
                                    Selection selected, const DeviceTensor& k_cur, const DeviceTensor& v_cur,
                                    cudaStream_t st = nullptr) {
    detail::check_qkv(cfg, q, k_cur, v_cur, "attn_forward");
    DeviceAttnSaved s{DeviceTensor(q.shape(), q.dtype(), false),
                      DeviceTensor({q.dim(0), q.dim(1)}, acc_dtype(cache.dtype()), false),
                      std::move(selected)};
    check(oomb_attn_forward(cache.handle(), layer, q.data(), q.dim(0), s.selected.handle(), k_cur.data(),
                            v_cur.data(), s.out.data(), s.lse.data(), sv(st)));
    return s;
}
// attention.hpp:222-293 on the device: past-page dK/dV go into the cache's fp32 gradient pages.
inline DeviceAttnGrads attn_backward(const ModelConfig& cfg, const DeviceTensor& dout, const DeviceTensor& q,
                                     PagedCache& cache, int layer, const DeviceTensor& k_cur,
                                     const DeviceTensor& v_cur, const DeviceAttnSaved& saved,
                                     cudaStream_t st = nullptr) {
    detail::check_qkv(cfg, q, k_cur, v_cur, "attn_backward");
    if (!dout.same_shape(saved.out)) throw ShapeError("attn_backward: dO shape mismatch");
    const DType acc = acc_dtype(cache.dtype());
    DeviceAttnGrads g{DeviceTensor(q.shape(), acc, false), DeviceTensor(k_cur.shape(), acc, false),
                      DeviceTensor(k_cur.shape(), acc, false)};
    check(oomb_attn_backward(cache.handle(), layer, dout.data(), q.data(), q.dim(0), saved.selected.handle(),
                             k_cur.data(), v_cur.data(), saved.out.data(), saved.lse.data(), g.dq.data(),
                             g.dk_cur.data(), g.dv_cur.data(), sv(st)));
    return g;
}

// Reference-signature overloads on host tensors (attention.hpp:156-160, 222-226).
template <class Real>
AttnSaved<Real> attn_forward(const ModelConfig& cfg, const Tensor<Real>& q, PagedCache& cache, int layer,
                             PageLists selected, const Tensor<Real>& k_cur, const Tensor<Real>& v_cur) {
    if (q.rank() != 3) throw ShapeError("attn_forward: expected [C x qh x hd] q");
    const int64_t m = (q.dim(0) + cfg.page_size - 1) / cfg.page_size;
    if (static_cast<int64_t>(selected.size()) != m)
        throw ShapeError("attn_forward: selected must have one id list per query page");
    const DType dt = cache.dtype();
    auto s = attn_forward(cfg, DeviceTensor::from_host(q, dt), cache, layer, Selection::from_lists(cache, selected),
                          DeviceTensor::from_host(k_cur, dt), DeviceTensor::from_host(v_cur, dt));
    return AttnSaved<Real>{s.out.template to_tensor<Real>(), s.lse.template to_tensor<Real>(), std::move(selected)};
}
template <class Real>
AttnGrads<Real> attn_backward(const ModelConfig& cfg, const Tensor<Real>& dout, const Tensor<Real>& q,
                              PagedCache& cache, int layer, const Tensor<Real>& k_cur, const Tensor<Real>& v_cur,
                              const AttnSaved<Real>& saved) {
    if (dout.shape != saved.out.shape) throw ShapeError("attn_backward: dO shape mismatch");
    const DType dt = cache.dtype();
    DeviceAttnSaved ds{DeviceTensor::from_host(saved.out, dt), DeviceTensor::from_host(saved.lse, acc_dtype(dt)),
                       Selection::from_lists(cache, saved.selected)};
    auto g = attn_backward(cfg, DeviceTensor::from_host(dout, dt), DeviceTensor::from_host(q, dt), cache, layer,
                           DeviceTensor::from_host(k_cur, dt), DeviceTensor::from_host(v_cur, dt), ds);
    return AttnGrads<Real>{g.dq.template to_tensor<Real>(), g.dk_cur.template to_tensor<Real>(),
                           g.dv_cur.template to_tensor<Real>()};
}

// ---------------------------------------------------------------------------- offload
enum class Phase : uint8_t { forward, backward };
enum class EventKind : uint8_t { fetch_issued, fetch_done, evict, compute_begin, compute_end, access };

struct ComputeCostModel {  // tiered_memory.hpp:58-72 (simulation mode)
    double fixed_s_per_layer = 1e-3;
    double s_per_attended_token = 1e-6;
};
struct TierConfig {  // tiered_memory.hpp:74-78
    int64_t device_capacity_pages = -1;
    double bandwidth_bytes_per_s = 16e9;
    ComputeCostModel compute;
};
struct TransferHandle {
    int64_t id = -1;
};
struct ScheduleEvent {  // tiered_memory.hpp:36-44
    EventKind kind;
    double t;
    int layer;
    int page;
    int chunk;
    uint64_t bytes;
    Phase phase;
};
struct ScheduleLog {
    double bandwidth_bytes_per_s = 0;
    std::vector<ScheduleEvent> events;
};
struct ValidationReport {  // tiered_memory.hpp:84-95
    std::vector<std::string> violations;
    double stall_seconds = 0;
    uint64_t transfer_bytes = 0;
    uint64_t h2d_bytes_forward = 0;
    uint64_t h2d_bytes_backward = 0;
    uint64_t d2h_bytes = 0;
    double overlap_fraction = 1.0;
};

// PagedCache's page-table bookkeeping without a device (drives the simulated engine).
class HostPageTable {
public:
    HostPageTable(int n_layers, int page_size, int n_kv_heads, int head_dim, int kv_elem_bytes = 4,
                  int grad_elem_bytes = 4) {
        check(oomb_pagetable_create(n_layers, page_size, n_kv_heads, head_dim, kv_elem_bytes, grad_elem_bytes, &pt_));
    }
    ~HostPageTable() {
        if (pt_) oomb_pagetable_destroy(pt_);
    }
    HostPageTable(const HostPageTable&) = delete;
    HostPageTable& operator=(const HostPageTable&) = delete;
    oomb_pagetable_t handle() const { return pt_; }
    SlotRange append_chunk(int layer, int64_t rows) {
        SlotRange r;
        check(oomb_pagetable_append(pt_, layer, rows, &r.begin, &r.end));
        return r;
    }
    void scatter_add_grads(int layer, std::span<const int32_t> ids) {
        check(oomb_pagetable_scatter(pt_, layer, ids.data(), static_cast<int>(ids.size())));
    }
    void set_tier(int layer, int page, Tier t) { check(oomb_pagetable_set_tier(pt_, layer, page, static_cast<int>(t))); }
    int n_pages(int layer) const {
        int n = 0;
        check(oomb_pagetable_n_pages(pt_, layer, &n));
        return n;
    }
    std::vector<int32_t> page_table(int layer) const {
        std::vector<int32_t> out(static_cast<size_t>(4) * n_pages(layer));
        check(oomb_pagetable_get(pt_, layer, out.data()));
        return out;
    }
    void reset() { check(oomb_pagetable_reset(pt_)); }
    MemoryReport memory_report() const {
        oomb_memory_report r{};
        check(oomb_pagetable_memory_report(pt_, &r));
        return to_report(r);
    }

private:
    oomb_pagetable_t pt_ = nullptr;
};

namespace detail {
inline std::string violation_message(int32_t code, const oomb_event* e) {  // tiered_memory.cpp:50-126
    auto where = [&] {
        char b[160];
        std::snprintf(b, sizeof b, "layer=%d page=%d t=%g", e->layer, e->page, e->t);
        return std::string(b);
    };
    switch (code) {
        case 1: return "evict of non-resident page " + where();
        case 2: return "access before fetch_done (or after evict): " + where();
        case 3: return "compute stream timestamps decrease";
        case 4: return "nested compute_begin";
        case 5: return "compute_end without begin";
        case 6: return "compute segment ends before it begins";
        default: return "unterminated compute segment";
    }
}
inline ValidationReport validate_raw(const std::vector<oomb_event>& ev, double bandwidth) {
    double out[6] = {};
    int nv = 0;
    const int64_t cap = static_cast<int64_t>(ev.size()) + 1;
    std::vector<int64_t> vev(static_cast<size_t>(cap));
    std::vector<int32_t> vcode(static_cast<size_t>(cap));
    check(oomb_validate_schedule(ev.data(), static_cast<int64_t>(ev.size()), bandwidth, out, &nv, vev.data(),
                                 vcode.data(), cap));
    ValidationReport r;
    for (int i = 0; i < nv && i < cap; ++i)
        r.violations.push_back(violation_message(vcode[i], vev[i] >= 0 ? &ev[static_cast<size_t>(vev[i])] : nullptr));
    r.stall_seconds = out[0];
    r.transfer_bytes = static_cast<uint64_t>(out[1]);
    r.h2d_bytes_forward = static_cast<uint64_t>(out[2]);
    r.h2d_bytes_backward = static_cast<uint64_t>(out[3]);
    r.d2h_bytes = static_cast<uint64_t>(out[4]);
    r.overlap_fraction = out[5];
    return r;
}
}  // namespace detail

// tiered_memory.cpp:47-138.
inline ValidationReport validate_schedule(const ScheduleLog& log) {
    std::vector<oomb_event> ev;
    ev.reserve(log.events.size());
    for (const auto& e : log.events)
        ev.push_back(oomb_event{static_cast<int32_t>(e.kind), e.layer, e.page, e.chunk, static_cast<int32_t>(e.phase), 0,
                                e.bytes, e.t});
    return detail::validate_raw(ev, log.bandwidth_bytes_per_s);
}

// TieredEngine (tiered_memory.hpp:99-432). On a PagedCache pages really move between HBM and
// pinned host memory on side streams; on a HostPageTable the reference's simulated clock runs.
class TieredEngine {
public:
    TieredEngine(PagedCache& cache, const TierConfig& cfg, cudaStream_t compute_stream = nullptr)
        : cfg_(cfg), cache_(&cache) {
        const oomb_tier_config c = to_c(cfg);
        check(oomb_tier_create(cache.handle(), &c, sv(compute_stream), &t_));
        cache.enforced_ = true;  // tiered_memory.hpp:102-113: enforcement follows the engine's lifetime
    }
    TieredEngine(HostPageTable& pt, const TierConfig& cfg) : cfg_(cfg) {
        const oomb_tier_config c = to_c(cfg);
        check(oomb_tier_create_sim(pt.handle(), &c, &t_));
    }
    ~TieredEngine() {
        if (t_) oomb_tier_destroy(t_);
        if (cache_) cache_->enforced_ = false;
    }
    TieredEngine(const TieredEngine&) = delete;
    TieredEngine& operator=(const TieredEngine&) = delete;

    void begin_phase(Phase p) { check(oomb_tier_begin_phase(t_, static_cast<int>(p))); }
    void set_prefetch_headroom_pages(int64_t pages) { check(oomb_tier_set_prefetch_headroom(t_, pages)); }
    void on_pages_appended(int layer, const SlotRange& r) {
        check(oomb_tier_on_pages_appended(t_, layer, r.begin, r.end));
    }
    void on_grads_scattered(int layer, std::span<const int32_t> ids) {
        check(oomb_tier_on_grads_scattered(t_, layer, ids.data(), static_cast<int>(ids.size())));
    }
    TransferHandle fetch_async(int layer, std::span<const int32_t> ids, int chunk = -1, bool best_effort = false) {
        TransferHandle h;
        check(oomb_tier_fetch_async(t_, layer, ids.data(), static_cast<int>(ids.size()), chunk, best_effort ? 1 : 0,
                                    &h.id));
        return h;
    }
    void wait(const TransferHandle& h) { check(oomb_tier_wait(t_, h.id)); }
    void record_access(int layer, std::span<const int32_t> ids, int chunk = -1) {
        check(oomb_tier_record_access(t_, layer, ids.data(), static_cast<int>(ids.size()), chunk));
    }
    void advance_compute(double seconds, int chunk, int layer) {
        check(oomb_tier_advance_compute(t_, seconds, chunk, layer));
    }
    void end_layer_use(int layer, std::span<const int32_t> ids) {
        check(oomb_tier_end_layer_use(t_, layer, ids.data(), static_cast<int>(ids.size())));
    }
    void release_all_reservations() { check(oomb_tier_release_all(t_)); }
    void restore_all() { check(oomb_tier_restore_all(t_)); }

    double now() const { return stats()[0]; }
    double stall_seconds() const { return stats()[1]; }
    uint64_t h2d_bytes(Phase p) const { return static_cast<uint64_t>(stats()[p == Phase::forward ? 2 : 3]); }
    uint64_t d2h_bytes() const { return static_cast<uint64_t>(stats()[4]); }
    const TierConfig& config() const { return cfg_; }

    ScheduleLog log() const {
        ScheduleLog out{cfg_.bandwidth_bytes_per_s, {}};
        for (const auto& e : raw_log())
            out.events.push_back(ScheduleEvent{static_cast<EventKind>(e.kind), e.t, e.layer, e.page, e.chunk, e.bytes,
                                               static_cast<Phase>(e.phase)});
        return out;
    }
    std::vector<oomb_event> raw_log() const {
        int64_t n = 0;
        check(oomb_tier_log(t_, nullptr, 0, &n));
        std::vector<oomb_event> ev(static_cast<size_t>(n));
        if (n) check(oomb_tier_log(t_, ev.data(), n, &n));
        ev.resize(static_cast<size_t>(n));
        return ev;
    }

private:
    static oomb_tier_config to_c(const TierConfig& c) {
        return oomb_tier_config{c.device_capacity_pages, c.bandwidth_bytes_per_s, c.compute.fixed_s_per_layer,
                                c.compute.s_per_attended_token};
    }
    std::vector<double> stats() const {
        std::vector<double> s(5);
        check(oomb_tier_stats(t_, s.data()));
        return s;
    }
    TierConfig cfg_;
    PagedCache* cache_ = nullptr;
    oomb_tier_t t_ = nullptr;
};

}  // namespace oomb
