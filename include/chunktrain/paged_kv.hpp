// SPDX-License-Identifier: Apache-2.0
//
// chunktrain/paged_kv.hpp — PagedCache<Real> (paged_kv.hpp:41-356) over the device page pool of
// liboomb.so, with the reference's host-tensor signatures. Source-compatibility header: see
// chunktrain/common.hpp.
//
// Real selects the device pool: PagedCache<float> is an OOMB_F32 pool, PagedCache<double> an
// OOMB_F64 pool whose pages, K_avg, gradients and attention arithmetic are double, as the
// reference's Real = double is.
// key_page_data returns a host mirror of the page in the reference's block layout [P][Hkv][hd],
// refreshed on every call at a stable address per (layer, page) (the device page itself never
// moves: slots are stable, paged_kv.hpp:353).
#pragma once

#include <map>
#include <span>
#include <type_traits>
#include <utility>
#include <vector>

#include "chunktrain/config.hpp"
#include "chunktrain/tensor.hpp"

namespace chunktrain {

using oomb::MemoryReport;
using oomb::SlotRange;
using oomb::Tier;

template <class Real>
class PagedCache {
public:
    struct Gathered {  // paged_kv.hpp:110-114
        Tensor<Real> k;
        Tensor<Real> v;
        std::vector<uint8_t> valid;
    };

    static constexpr oomb::DType kDType = std::is_same_v<Real, double> ? oomb::DType::f64 : oomb::DType::f32;
    explicit PagedCache(const ModelConfig& cfg) : cfg_(cfg), dev_(cfg, kDType) {}

    const ModelConfig& config() const { return cfg_; }
    int page_size() const { return cfg_.page_size; }
    int64_t page_elems() const { return dev_.page_elems(); }
    uint64_t page_buffer_bytes() const { return static_cast<uint64_t>(page_elems()) * sizeof(Real); }
    uint64_t page_kv_bytes() const { return 2 * page_buffer_bytes(); }
    int64_t filled(int layer) const { return dev_.filled(layer); }
    int n_pages(int layer) const { return dev_.n_pages(layer); }
    static int full_pages_before(int64_t tokens, int page_size) { return static_cast<int>(tokens / page_size); }

    SlotRange append_chunk(int layer, const oomb::Tensor<Real>& k, const oomb::Tensor<Real>& v) {
        return dev_.append_chunk(layer, k, v);
    }
    Gathered gather_pages(int layer, std::span<const int32_t> ids) const { return gathered(dev_.gather_pages(layer, ids)); }
    Gathered gather_grad_pages(int layer, std::span<const int32_t> ids) const {
        return gathered(dev_.gather_grad_pages(layer, ids));
    }
    void scatter_add_grads(int layer, std::span<const int32_t> ids, const oomb::Tensor<Real>& dk,
                           const oomb::Tensor<Real>& dv) {
        const int64_t want = static_cast<int64_t>(ids.size()) * cfg_.page_size;
        if (dk.rank() != 3 || dk.dim(0) != want || dk.shape != dv.shape)
            throw ShapeError("scatter_add_grads: gradient shape does not match gather layout");
        dev_.scatter_add_grads(layer, ids, oomb::DeviceTensor::from_host(dk, kDType),
                               oomb::DeviceTensor::from_host(dv, kDType));
    }
    Tensor<Real> page_mean_keys(int layer, int n_candidates = -1) const {
        return dev_.page_mean_keys(layer, n_candidates).template to_tensor<Real>();
    }
    MemoryReport memory_report() const { return dev_.memory_report(); }
    Tier tier(int layer, int page) const { return dev_.tier(layer, page); }
    void set_tier(int layer, int page, Tier t) { dev_.set_tier(layer, page, t); }
    bool grads_allocated(int layer, int page) const { return dev_.grads_allocated(layer, page); }
    void set_residency_enforced(bool on) { dev_.set_residency_enforced(on); }
    bool residency_enforced() const { return dev_.residency_enforced(); }
    void zero_grad_pages() { dev_.zero_grad_pages(); }
    void reset() { dev_.reset(); }

    const Real* key_page_data(int layer, int page) const { return mirror(layer, page, false); }
    const Real* grad_key_page_data(int layer, int page) const {
        return dev_.grads_allocated(layer, page) ? mirror(layer, page, true) : nullptr;
    }
    int64_t arena_blocks_allocated() const { return report().arena_blocks; }
    int64_t free_list_size() const { return report().free_list; }

    oomb::PagedCache& device() { return dev_; }
    const oomb::PagedCache& device() const { return dev_; }

private:
    static Gathered gathered(const oomb::Gathered& g) {
        Gathered out{g.k.template to_tensor<Real>(), g.v.template to_tensor<Real>(), g.valid.template to_host<uint8_t>()};
        return out;
    }
    oomb_memory_report report() const {
        oomb_memory_report r{};
        oomb::check(oomb_memory_report_get(dev_.handle(), &r));
        return r;
    }
    const Real* mirror(int layer, int page, bool grads) const {
        if (page < 0 || page >= n_pages(layer)) throw ShapeError("key_page_data: page out of range");
        const int32_t id = page;
        Gathered g = grads ? gather_grad_pages(layer, std::span<const int32_t>(&id, 1))
                           : gather_pages(layer, std::span<const int32_t>(&id, 1));
        std::vector<Real>& buf = mirrors_[{layer * 2 + (grads ? 1 : 0), page}];
        if (buf.empty()) buf.resize(static_cast<size_t>(page_elems()));
        std::copy(g.k.data.begin(), g.k.data.end(), buf.begin());  // in place: the address stays
        return buf.data();
    }

    ModelConfig cfg_;
    oomb::PagedCache dev_;
    mutable std::map<std::pair<int, int>, std::vector<Real>> mirrors_;
};

// ---- the contiguous-growth baseline (paged_kv.hpp:362-382, paged_kv.cpp:24-54): host arithmetic
enum class GrowthPolicy { exact_fit, doubling };

struct ReallocEvent {
    uint64_t stored_bytes_before = 0;
    uint64_t old_capacity = 0;
    uint64_t new_capacity = 0;
    uint64_t transient_bytes = 0;  // old + new buffer during the copy
};

struct ContiguousReport {
    uint64_t peak_bytes = 0;
    uint64_t copied_bytes = 0;
    int64_t reallocs = 0;
    uint64_t final_bytes = 0;
    std::vector<ReallocEvent> events;
};

// A contiguous KV buffer grown by reallocate-and-copy: each append that overflows the capacity
// allocates exact-fit or doubled capacity while the old buffer (holding `stored` bytes) is still
// live, then copies it across.
inline ContiguousReport simulate_contiguous_appends(int64_t n_appends, int64_t tokens_per_append,
                                                    uint64_t bytes_per_token, GrowthPolicy policy) {
    ContiguousReport rep;
    uint64_t cap = 0, stored = 0;
    const uint64_t step = static_cast<uint64_t>(tokens_per_append) * bytes_per_token;
    for (int64_t a = 0; a < n_appends; ++a) {
        const uint64_t need = stored + step;
        if (need > cap) {
            const uint64_t grown = policy == GrowthPolicy::doubling ? std::max<uint64_t>(2 * cap, need) : need;
            if (cap > 0) {
                ++rep.reallocs;
                rep.copied_bytes += stored;
                rep.events.push_back(ReallocEvent{stored, cap, grown, cap + grown});
            }
            rep.peak_bytes = std::max(rep.peak_bytes, cap + grown);
            cap = grown;
        }
        stored = need;
        rep.peak_bytes = std::max(rep.peak_bytes, cap);
    }
    rep.final_bytes = stored;
    return rep;
}

}  // namespace chunktrain
