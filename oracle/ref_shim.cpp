// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin extern "C" shim over the UNMODIFIED reference headers under
// /root/reference/proj/core/include (compiled in place by oracle/Makefile.ref,
// output only into oracle/_ref/). It exists so that
//   * tests/golden/make_golden.py can generate golden vectors straight from the
//     reference implementation of the hot path, and
//   * bench.py --impl reference / the cpu_baseline leg can time the reference's
//     own CPU path on the GPU box's host cores.
// Nothing here re-implements an algorithm: every entry point forwards to the
// reference function named in its comment.
//
// Private members of PagedCache (the arena ids of the page table) are exposed
// by redefining `private` for the reference headers only, after every standard
// header they use has already been included.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <numeric>
#include <optional>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#define private public
#include "chunktrain/attention.hpp"
#include "chunktrain/chunk_trainer.hpp"
#include "chunktrain/model.hpp"
#include "chunktrain/oracle.hpp"
#include "chunktrain/paged_kv.hpp"
#include "chunktrain/tiered_memory.hpp"
#undef private

using namespace chunktrain;

namespace {

thread_local std::string g_err;

enum : int { OK = 0, E_CONFIG = 1, E_SHAPE = 2, E_STATE = 3, E_RESIDENCY = 4, E_IO = 5, E_OTHER = 9 };

template <class F>
int guarded(F&& f) {
    try {
        f();
        return OK;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return E_CONFIG;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return E_SHAPE;
    } catch (const StateError& e) {
        g_err = e.what();
        return E_STATE;
    } catch (const ResidencyError& e) {
        g_err = e.what();
        return E_RESIDENCY;
    } catch (const IoError& e) {
        g_err = e.what();
        return E_IO;
    } catch (const std::exception& e) {
        g_err = e.what();
        return E_OTHER;
    }
}

}  // namespace

extern "C" {

// Mirrors the ModelConfig fields the hot path reads (config.hpp:19-49).
struct RefCfg {
    int n_layers;
    int n_q_heads;
    int n_kv_heads;
    int head_dim;
    int chunk_size;
    int page_size;
    int retrieval_budget;
    int local_window;
    int score_scale;
};

}  // extern "C"

namespace {

ModelConfig to_cfg(const RefCfg& c) {
    ModelConfig m;
    m.n_layers = c.n_layers;
    m.n_q_heads = c.n_q_heads;
    m.n_kv_heads = c.n_kv_heads;
    m.head_dim = c.head_dim;
    m.chunk_size = c.chunk_size;
    m.page_size = c.page_size;
    m.retrieval_budget = c.retrieval_budget;
    m.local_window = c.local_window;
    m.score_scale = c.score_scale != 0;
    return m;
}

template <class Real>
Tensor<Real> view3(const void* p, int64_t a, int64_t b, int64_t c) {
    Tensor<Real> t({a, b, c});
    if (t.numel()) std::memcpy(t.ptr(), p, t.bytes());
    return t;
}

template <class Real>
void put(void* dst, const Tensor<Real>& t) {
    if (t.numel()) std::memcpy(dst, t.ptr(), t.bytes());
}

std::vector<std::vector<int32_t>> csr_to_lists(const int32_t* off, const int32_t* ids, int64_t m) {
    std::vector<std::vector<int32_t>> sel(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; ++i) sel[static_cast<size_t>(i)].assign(ids + off[i], ids + off[i + 1]);
    return sel;
}

struct CacheBox {
    int real_bytes;
    ModelConfig cfg;
    std::unique_ptr<PagedCache<float>> f;
    std::unique_ptr<PagedCache<double>> d;
    std::unique_ptr<TieredEngine<float>> tf;
    std::unique_ptr<TieredEngine<double>> td;
};

template <class Real>
PagedCache<Real>& cache_of(CacheBox* b);
template <>
PagedCache<float>& cache_of<float>(CacheBox* b) { return *b->f; }
template <>
PagedCache<double>& cache_of<double>(CacheBox* b) { return *b->d; }

template <class F>
int dispatch(CacheBox* b, F&& f) {
    if (b->real_bytes == 4) return guarded([&] { f(float{}, *b->f); });
    return guarded([&] { f(double{}, *b->d); });
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// PagedCache(const ModelConfig&)  paged_kv.hpp:44-50
int ref_cache_new(int real_bytes, const RefCfg* c, void** out) {
    return guarded([&] {
        auto* b = new CacheBox{real_bytes, to_cfg(*c), nullptr, nullptr, nullptr, nullptr};
        if (real_bytes == 4) b->f = std::make_unique<PagedCache<float>>(b->cfg);
        else b->d = std::make_unique<PagedCache<double>>(b->cfg);
        *out = b;
    });
}

void ref_cache_free(void* h) { delete static_cast<CacheBox*>(h); }

// append_chunk  paged_kv.hpp:73-108
int ref_cache_append(void* h, int layer, const void* k, const void* v, int64_t rows,
                     int64_t* begin, int64_t* end) {
    auto* b = static_cast<CacheBox*>(h);
    return dispatch(b, [&](auto tag, auto& cache) {
        using Real = decltype(tag);
        const auto r = cache.append_chunk(layer, view3<Real>(k, rows, b->cfg.n_kv_heads, b->cfg.head_dim),
                                          view3<Real>(v, rows, b->cfg.n_kv_heads, b->cfg.head_dim));
        *begin = r.begin;
        *end = r.end;
    });
}

int ref_cache_n_pages(void* h, int layer) {
    auto* b = static_cast<CacheBox*>(h);
    int n = -1;
    dispatch(b, [&](auto, auto& cache) { n = cache.n_pages(layer); });
    return n;
}

int64_t ref_cache_filled(void* h, int layer) {
    auto* b = static_cast<CacheBox*>(h);
    int64_t n = -1;
    dispatch(b, [&](auto, auto& cache) { n = cache.filled(layer); });
    return n;
}

// PageEntry{k_phys, v_phys, gk_phys, gv_phys, tier}  paged_kv.hpp:256-262
int ref_cache_page_table(void* h, int layer, int32_t* out) {
    auto* b = static_cast<CacheBox*>(h);
    return dispatch(b, [&](auto, auto& cache) {
        const auto& st = cache.at_(layer);
        for (size_t i = 0; i < st.pages.size(); ++i) {
            out[4 * i + 0] = st.pages[i].k_phys;
            out[4 * i + 1] = st.pages[i].v_phys;
            out[4 * i + 2] = st.pages[i].gk_phys;
            out[4 * i + 3] = st.pages[i].gv_phys;
        }
    });
}

int ref_cache_tiers(void* h, int layer, uint8_t* out) {
    auto* b = static_cast<CacheBox*>(h);
    return dispatch(b, [&](auto, auto& cache) {
        for (int p = 0; p < cache.n_pages(layer); ++p) out[p] = static_cast<uint8_t>(cache.tier(layer, p));
    });
}

int ref_cache_set_tier(void* h, int layer, int page, int tier) {
    auto* b = static_cast<CacheBox*>(h);
    return dispatch(b, [&](auto, auto& cache) { cache.set_tier(layer, page, tier ? Tier::host : Tier::device); });
}

int ref_cache_set_residency_enforced(void* h, int on) {
    auto* b = static_cast<CacheBox*>(h);
    return dispatch(b, [&](auto, auto& cache) { cache.set_residency_enforced(on != 0); });
}

// kavg_sum / kavg_count  paged_kv.hpp:264-269
int ref_cache_kavg_raw(void* h, int layer, void* sum_out, int32_t* count_out) {
    auto* b = static_cast<CacheBox*>(h);
    return dispatch(b, [&](auto tag, auto& cache) {
        using Real = decltype(tag);
        const auto& st = cache.at_(layer);
        std::memcpy(sum_out, st.kavg_sum.data(), st.kavg_sum.size() * sizeof(Real));
        std::memcpy(count_out, st.kavg_count.data(), st.kavg_count.size() * sizeof(int32_t));
    });
}

// page_mean_keys  paged_kv.hpp:170-183
int ref_cache_mean_keys(void* h, int layer, int n, void* out, int* n_out) {
    auto* b = static_cast<CacheBox*>(h);
    return dispatch(b, [&](auto, auto& cache) {
        const auto t = cache.page_mean_keys(layer, n);
        *n_out = static_cast<int>(t.dim(0));
        put(out, t);
    });
}

// gather_pages / gather_grad_pages  paged_kv.hpp:118-130
int ref_cache_gather(void* h, int layer, const int32_t* ids, int n, int grads, void* k, void* v,
                     uint8_t* valid) {
    auto* b = static_cast<CacheBox*>(h);
    return dispatch(b, [&](auto, auto& cache) {
        std::span<const int32_t> s(ids, static_cast<size_t>(n));
        const auto g = grads ? cache.gather_grad_pages(layer, s) : cache.gather_pages(layer, s);
        put(k, g.k);
        put(v, g.v);
        if (!g.valid.empty()) std::memcpy(valid, g.valid.data(), g.valid.size());
    });
}

// scatter_add_grads  paged_kv.hpp:135-164
int ref_cache_scatter(void* h, int layer, const int32_t* ids, int n, const void* dk, const void* dv) {
    auto* b = static_cast<CacheBox*>(h);
    return dispatch(b, [&](auto tag, auto& cache) {
        using Real = decltype(tag);
        const int64_t rows = static_cast<int64_t>(n) * b->cfg.page_size;
        cache.scatter_add_grads(layer, std::span<const int32_t>(ids, static_cast<size_t>(n)),
                                view3<Real>(dk, rows, b->cfg.n_kv_heads, b->cfg.head_dim),
                                view3<Real>(dv, rows, b->cfg.n_kv_heads, b->cfg.head_dim));
    });
}

int ref_cache_reset(void* h) {
    auto* b = static_cast<CacheBox*>(h);
    return dispatch(b, [&](auto, auto& cache) { cache.reset(); });
}

int ref_cache_zero_grad(void* h) {
    auto* b = static_cast<CacheBox*>(h);
    return dispatch(b, [&](auto, auto& cache) { cache.zero_grad_pages(); });
}

// memory_report  paged_kv.hpp:185-197 ; arena/free-list introspection :244-251
int ref_cache_memory_report(void* h, uint64_t* out) {
    auto* b = static_cast<CacheBox*>(h);
    return dispatch(b, [&](auto, auto& cache) {
        const auto r = cache.memory_report();
        out[0] = r.device_bytes;
        out[1] = r.host_bytes;
        out[2] = r.grad_bytes;
        out[3] = static_cast<uint64_t>(r.pages);
        out[4] = static_cast<uint64_t>(r.reallocs);
        out[5] = r.copied_bytes;
        out[6] = static_cast<uint64_t>(cache.arena_blocks_allocated());
        out[7] = static_cast<uint64_t>(cache.free_list_size());
    });
}

// score_pages  attention.hpp:32-67
int ref_score_pages(int real_bytes, const void* q, int64_t tokens, int qh, int hd, const void* k_avg,
                    int64_t n, int kvh, int page_size, int gqa_group, int score_scale, void* out) {
    return guarded([&] {
        if (real_bytes == 4) {
            put(out, score_pages(view3<float>(q, tokens, qh, hd), view3<float>(k_avg, n, kvh, hd),
                                 page_size, gqa_group, score_scale != 0));
        } else {
            put(out, score_pages(view3<double>(q, tokens, qh, hd), view3<double>(k_avg, n, kvh, hd),
                                 page_size, gqa_group, score_scale != 0));
        }
    });
}

// select_topk  attention.hpp:71-88 ; returns the id count
int ref_select_topk(const double* row, int n, int budget, int32_t* out, int* count) {
    return guarded([&] {
        const auto ids = select_topk(std::span<const double>(row, static_cast<size_t>(n)), budget);
        std::copy(ids.begin(), ids.end(), out);
        *count = static_cast<int>(ids.size());
    });
}

// select_topk_row  attention.hpp:90-96 (score rows stored as Real)
int ref_select_topk_row(int real_bytes, const void* score, int64_t m, int64_t n, int64_t row,
                        int budget, int32_t* out, int* count) {
    return guarded([&] {
        std::vector<int32_t> ids;
        if (real_bytes == 4) {
            Tensor<float> s({m, n});
            std::memcpy(s.ptr(), score, s.bytes());
            ids = select_topk_row(s, row, budget);
        } else {
            Tensor<double> s({m, n});
            std::memcpy(s.ptr(), score, s.bytes());
            ids = select_topk_row(s, row, budget);
        }
        std::copy(ids.begin(), ids.end(), out);
        *count = static_cast<int>(ids.size());
    });
}

// select_recent / select_all  attention.hpp:99-111
int ref_select_recent(int n_pages, int window, int32_t* out, int* count) {
    return guarded([&] {
        const auto ids = select_recent(n_pages, window);
        std::copy(ids.begin(), ids.end(), out);
        *count = static_cast<int>(ids.size());
    });
}

// attn_forward  attention.hpp:156-208. Selection is CSR over the m query pages.
int ref_attn_forward(void* h, int layer, const void* q, int64_t c, const int32_t* sel_off,
                     const int32_t* sel_ids, int64_t m, const void* k_cur, const void* v_cur, void* out,
                     void* lse) {
    auto* b = static_cast<CacheBox*>(h);
    const auto& cfg = b->cfg;
    return dispatch(b, [&](auto tag, auto& cache) {
        using Real = decltype(tag);
        auto saved = attn_forward(cfg, view3<Real>(q, c, cfg.n_q_heads, cfg.head_dim), cache, layer,
                                  csr_to_lists(sel_off, sel_ids, m),
                                  view3<Real>(k_cur, c, cfg.n_kv_heads, cfg.head_dim),
                                  view3<Real>(v_cur, c, cfg.n_kv_heads, cfg.head_dim));
        put(out, saved.out);
        put(lse, saved.lse);
    });
}

// attn_backward  attention.hpp:222-293 (saved O / LSE passed back in)
int ref_attn_backward(void* h, int layer, const void* dout, const void* q, int64_t c,
                      const int32_t* sel_off, const int32_t* sel_ids, int64_t m, const void* k_cur,
                      const void* v_cur, const void* out, const void* lse, void* dq, void* dk_cur,
                      void* dv_cur) {
    auto* b = static_cast<CacheBox*>(h);
    const auto& cfg = b->cfg;
    return dispatch(b, [&](auto tag, auto& cache) {
        using Real = decltype(tag);
        AttnSaved<Real> saved;
        saved.out = view3<Real>(out, c, cfg.n_q_heads, cfg.head_dim);
        saved.lse = Tensor<Real>({c, static_cast<int64_t>(cfg.n_q_heads)});
        std::memcpy(saved.lse.ptr(), lse, saved.lse.bytes());
        saved.selected = csr_to_lists(sel_off, sel_ids, m);
        auto g = attn_backward(cfg, view3<Real>(dout, c, cfg.n_q_heads, cfg.head_dim),
                               view3<Real>(q, c, cfg.n_q_heads, cfg.head_dim), cache, layer,
                               view3<Real>(k_cur, c, cfg.n_kv_heads, cfg.head_dim),
                               view3<Real>(v_cur, c, cfg.n_kv_heads, cfg.head_dim), saved);
        put(dq, g.dq);
        put(dk_cur, g.dk_cur);
        put(dv_cur, g.dv_cur);
    });
}

// naive_attention_fwd_bwd  oracle.hpp:293-357
int ref_naive_attention(int real_bytes, const void* q, int64_t tq, int qh, int hd, const void* k,
                        const void* v, int64_t tk, int kvh, int64_t past_len, const void* dout,
                        int gqa_group, void* out, void* dq, void* dk, void* dv) {
    return guarded([&] {
        auto run = [&](auto tag) {
            using Real = decltype(tag);
            auto r = naive_attention_fwd_bwd(view3<Real>(q, tq, qh, hd), view3<Real>(k, tk, kvh, hd),
                                             view3<Real>(v, tk, kvh, hd), past_len,
                                             view3<Real>(dout, tq, qh, hd), gqa_group);
            put(out, r.out);
            put(dq, r.dq);
            put(dk, r.dk);
            put(dv, r.dv);
        };
        if (real_bytes == 4) run(float{});
        else run(double{});
    });
}

// ---------------------------------------------------------------------------
// TieredEngine (tiered_memory.hpp:99-432) driven op by op, for policy parity.
// ---------------------------------------------------------------------------

struct RefTierCfg {
    int64_t device_capacity_pages;
    double bandwidth_bytes_per_s;
    double fixed_s_per_layer;
    double s_per_attended_token;
};

struct RefEvent {
    int32_t kind;
    int32_t layer;
    int32_t page;
    int32_t chunk;
    int32_t phase;
    int32_t pad;
    uint64_t bytes;
    double t;
};

int ref_tier_new(void* h, const RefTierCfg* c) {
    auto* b = static_cast<CacheBox*>(h);
    return guarded([&] {
        TierConfig tc;
        tc.device_capacity_pages = c->device_capacity_pages;
        tc.bandwidth_bytes_per_s = c->bandwidth_bytes_per_s;
        tc.compute.fixed_s_per_layer = c->fixed_s_per_layer;
        tc.compute.s_per_attended_token = c->s_per_attended_token;
        if (b->real_bytes == 4) b->tf = std::make_unique<TieredEngine<float>>(*b->f, tc);
        else b->td = std::make_unique<TieredEngine<double>>(*b->d, tc);
    });
}

#define TIER_DISPATCH(b, expr)                          \
    guarded([&] {                                       \
        if ((b)->real_bytes == 4) { auto& eng = *(b)->tf; expr; } \
        else { auto& eng = *(b)->td; expr; }            \
    })

int ref_tier_free(void* h) {
    auto* b = static_cast<CacheBox*>(h);
    b->tf.reset();
    b->td.reset();
    return OK;
}

int ref_tier_begin_phase(void* h, int phase) {
    auto* b = static_cast<CacheBox*>(h);
    return TIER_DISPATCH(b, eng.begin_phase(phase ? Phase::backward : Phase::forward));
}

int ref_tier_set_headroom(void* h, int64_t pages) {
    auto* b = static_cast<CacheBox*>(h);
    return TIER_DISPATCH(b, eng.set_prefetch_headroom_pages(pages));
}

int ref_tier_on_pages_appended(void* h, int layer, int64_t begin, int64_t end) {
    auto* b = static_cast<CacheBox*>(h);
    return TIER_DISPATCH(b, eng.on_pages_appended(layer, SlotRange{begin, end}));
}

int ref_tier_on_grads_scattered(void* h, int layer, const int32_t* ids, int n) {
    auto* b = static_cast<CacheBox*>(h);
    return TIER_DISPATCH(b, eng.on_grads_scattered(layer, std::span<const int32_t>(ids, static_cast<size_t>(n))));
}

int ref_tier_fetch_async(void* h, int layer, const int32_t* ids, int n, int chunk, int best_effort,
                         int64_t* handle) {
    auto* b = static_cast<CacheBox*>(h);
    return TIER_DISPATCH(b, *handle = eng.fetch_async(layer, std::span<const int32_t>(ids, static_cast<size_t>(n)),
                                                      chunk, best_effort != 0).id);
}

int ref_tier_wait(void* h, int64_t handle) {
    auto* b = static_cast<CacheBox*>(h);
    TransferHandle th;
    th.id = handle;
    return TIER_DISPATCH(b, eng.wait(th));
}

int ref_tier_record_access(void* h, int layer, const int32_t* ids, int n, int chunk) {
    auto* b = static_cast<CacheBox*>(h);
    return TIER_DISPATCH(b, eng.record_access(layer, std::span<const int32_t>(ids, static_cast<size_t>(n)), chunk));
}

int ref_tier_advance_compute(void* h, double seconds, int chunk, int layer) {
    auto* b = static_cast<CacheBox*>(h);
    return TIER_DISPATCH(b, eng.advance_compute(seconds, chunk, layer));
}

int ref_tier_end_layer_use(void* h, int layer, const int32_t* ids, int n) {
    auto* b = static_cast<CacheBox*>(h);
    return TIER_DISPATCH(b, eng.end_layer_use(layer, std::span<const int32_t>(ids, static_cast<size_t>(n))));
}

int ref_tier_release_all(void* h) {
    auto* b = static_cast<CacheBox*>(h);
    return TIER_DISPATCH(b, eng.release_all_reservations());
}

int ref_tier_stats(void* h, double* out) {
    auto* b = static_cast<CacheBox*>(h);
    return TIER_DISPATCH(b, {
        out[0] = eng.now();
        out[1] = eng.stall_seconds();
        out[2] = static_cast<double>(eng.h2d_bytes(Phase::forward));
        out[3] = static_cast<double>(eng.h2d_bytes(Phase::backward));
        out[4] = static_cast<double>(eng.d2h_bytes());
    });
}

int64_t ref_tier_log_size(void* h) {
    auto* b = static_cast<CacheBox*>(h);
    int64_t n = 0;
    TIER_DISPATCH(b, n = static_cast<int64_t>(eng.log().events.size()));
    return n;
}

int ref_tier_log(void* h, RefEvent* out) {
    auto* b = static_cast<CacheBox*>(h);
    return TIER_DISPATCH(b, {
        const auto& ev = eng.log().events;
        for (size_t i = 0; i < ev.size(); ++i) {
            out[i].kind = static_cast<int32_t>(ev[i].kind);
            out[i].layer = ev[i].layer;
            out[i].page = ev[i].page;
            out[i].chunk = ev[i].chunk;
            out[i].phase = static_cast<int32_t>(ev[i].phase);
            out[i].pad = 0;
            out[i].bytes = ev[i].bytes;
            out[i].t = ev[i].t;
        }
    });
}

// validate_schedule  tiered_memory.cpp:47-138 over an externally built log
// dump_schedule_jsonl (tiered_memory.cpp:28-45) of an event list into a caller buffer.
int ref_dump_schedule_jsonl(const RefEvent* ev, int64_t n, double bandwidth, char* out, int64_t cap, int64_t* len) {
    return guarded([&] {
        ScheduleLog log;
        log.bandwidth_bytes_per_s = bandwidth;
        for (int64_t i = 0; i < n; ++i) {
            ScheduleEvent e;
            e.kind = static_cast<EventKind>(ev[i].kind);
            e.t = ev[i].t;
            e.layer = ev[i].layer;
            e.page = ev[i].page;
            e.chunk = ev[i].chunk;
            e.bytes = ev[i].bytes;
            e.phase = static_cast<Phase>(ev[i].phase);
            log.events.push_back(e);
        }
        std::ostringstream os;
        dump_schedule_jsonl(log, os);
        const std::string str = os.str();
        *len = static_cast<int64_t>(str.size());
        if (out && cap > 0) std::memcpy(out, str.data(), static_cast<size_t>(std::min<int64_t>(cap, *len)));
    });
}

int ref_validate_schedule(const RefEvent* ev, int64_t n, double bandwidth, double* out, int* n_violations) {
    return guarded([&] {
        ScheduleLog log;
        log.bandwidth_bytes_per_s = bandwidth;
        for (int64_t i = 0; i < n; ++i) {
            ScheduleEvent e;
            e.kind = static_cast<EventKind>(ev[i].kind);
            e.t = ev[i].t;
            e.layer = ev[i].layer;
            e.page = ev[i].page;
            e.chunk = ev[i].chunk;
            e.bytes = ev[i].bytes;
            e.phase = static_cast<Phase>(ev[i].phase);
            log.events.push_back(e);
        }
        const auto rep = validate_schedule(log);
        out[0] = rep.stall_seconds;
        out[1] = static_cast<double>(rep.transfer_bytes);
        out[2] = static_cast<double>(rep.h2d_bytes_forward);
        out[3] = static_cast<double>(rep.h2d_bytes_backward);
        out[4] = static_cast<double>(rep.d2h_bytes);
        out[5] = rep.overlap_fraction;
        *n_violations = static_cast<int>(rep.violations.size());
    });
}

// ---- whole-model chunked training step: ChunkTrainer::train_step
// (chunk_trainer.hpp:131-186) on caller-provided parameters, flattened in ModelParams::visit
// order (model.hpp:66-81). Test infrastructure: the GPU chunk loop is compared against it.
struct RefModelCfg {
    int n_layers, d_model, n_q_heads, n_kv_heads, head_dim, d_ff, vocab_size, chunk_size, page_size;
    int retrieval_budget, local_window, score_scale;
    int mode;  // 0 dense, 1 topk, 2 local (one mode for every layer)
    double rope_base;
    uint64_t seed;
};

}  // extern "C"

namespace {
ModelConfig to_model_cfg(const RefModelCfg& c) {
    ModelConfig m;
    m.n_layers = c.n_layers;
    m.d_model = c.d_model;
    m.n_q_heads = c.n_q_heads;
    m.n_kv_heads = c.n_kv_heads;
    m.head_dim = c.head_dim;
    m.d_ff = c.d_ff;
    m.vocab_size = c.vocab_size;
    m.chunk_size = c.chunk_size;
    m.page_size = c.page_size;
    m.retrieval_budget = c.retrieval_budget;
    m.local_window = c.local_window;
    m.score_scale = c.score_scale != 0;
    m.attention_mode = {c.mode == 0 ? AttentionMode::dense
                                    : (c.mode == 1 ? AttentionMode::topk_sparse : AttentionMode::local)};
    m.rope_base = c.rope_base;
    m.seed = c.seed;
    return m;
}
template <class Real>
void flat_in(ModelParams<Real>& p, const void* src) {
    const Real* s = static_cast<const Real*>(src);
    p.visit([&](const char*, int, Tensor<Real>& t) {
        std::memcpy(t.ptr(), s, t.bytes());
        s += t.numel();
    });
}
template <class Real>
void flat_out(const ModelParams<Real>& p, void* dst) {
    Real* d = static_cast<Real*>(dst);
    p.visit([&](const char*, int, const Tensor<Real>& t) {
        std::memcpy(d, t.ptr(), t.bytes());
        d += t.numel();
    });
}
template <class Real>
void train_step_impl(const RefModelCfg* c, const void* params, const int32_t* tokens, int64_t n, void* grads,
                     double* loss, int32_t* sel_counts) {
    const ModelConfig cfg = to_model_cfg(*c);
    ModelParams<Real> p = ModelParams<Real>::zeros_like_config(cfg);
    flat_in(p, params);
    ParamGrads<Real> g = ParamGrads<Real>::zeros_like_config(cfg);
    ChunkTrainer<Real> tr(cfg);
    const StepMetrics m = tr.train_step(p, std::span<const int32_t>(tokens, static_cast<size_t>(n)), g);
    flat_out(g, grads);
    *loss = m.loss;
    if (sel_counts) {  // number of selected ids per (chunk, layer, query page), for the caller's checks
        int64_t k = 0;
        for (const auto& ch : tr.last_chunks())
            for (const auto& per_layer : ch.selected)
                for (const auto& ids : per_layer) sel_counts[k++] = static_cast<int32_t>(ids.size());
    }
}
}  // namespace

extern "C" {

int64_t ref_model_numel(const RefModelCfg* c) {
    int64_t n = 0;
    guarded([&] { n = ModelParams<double>::zeros_like_config(to_model_cfg(*c)).param_count(); });
    return n;
}

// init_params (model.hpp:127-145) flattened in visit order.
int ref_init_params(int real_bytes, const RefModelCfg* c, uint64_t seed, void* out) {
    return guarded([&] {
        if (real_bytes == 4) flat_out(init_params<float>(to_model_cfg(*c), seed), out);
        else flat_out(init_params<double>(to_model_cfg(*c), seed), out);
    });
}

// full_forward_backward (oracle.hpp:89-276): the exact non-chunked model pass (monolithic causal
// softmax), the reference's ground truth for the chunked trainer.
int ref_full_forward_backward(int real_bytes, const RefModelCfg* c, const void* params, const int32_t* tokens,
                              int64_t n, void* grads, double* loss) {
    return guarded([&] {
        const ModelConfig cfg = to_model_cfg(*c);
        auto run = [&](auto zero) {
            using Real = decltype(zero);
            ModelParams<Real> p = ModelParams<Real>::zeros_like_config(cfg);
            flat_in(p, params);
            const auto r = full_forward_backward(cfg, p, std::span<const int32_t>(tokens, static_cast<size_t>(n)));
            flat_out(r.grads, grads);
            *loss = r.loss;
        };
        if (real_bytes == 4) run(float{});
        else run(double{});
    });
}

// ChunkTrainer::train_step with enable_offload(tier) (chunk_trainer.hpp:118-186): gradients, loss and
// the step's ScheduleLog (last_schedule()) as RefEvent records; *n_events = log size.
int ref_train_step_offload(int real_bytes, const RefModelCfg* c, const void* params, const int32_t* tokens, int64_t n,
                           const RefTierCfg* tc, void* grads, double* loss, RefEvent* events, int64_t cap,
                           int64_t* n_events) {
    return guarded([&] {
        const ModelConfig cfg = to_model_cfg(*c);
        TierConfig tier;
        tier.device_capacity_pages = tc->device_capacity_pages;
        tier.bandwidth_bytes_per_s = tc->bandwidth_bytes_per_s;
        tier.compute.fixed_s_per_layer = tc->fixed_s_per_layer;
        tier.compute.s_per_attended_token = tc->s_per_attended_token;
        auto run = [&](auto zero) {
            using Real = decltype(zero);
            ModelParams<Real> p = ModelParams<Real>::zeros_like_config(cfg);
            flat_in(p, params);
            ParamGrads<Real> g = ParamGrads<Real>::zeros_like_config(cfg);
            ChunkTrainer<Real> tr(cfg);
            tr.enable_offload(tier);
            const StepMetrics m = tr.train_step(p, std::span<const int32_t>(tokens, static_cast<size_t>(n)), g);
            flat_out(g, grads);
            *loss = m.loss;
            const ScheduleLog* log = tr.last_schedule();
            *n_events = log ? static_cast<int64_t>(log->events.size()) : 0;
            for (int64_t i = 0; log && i < std::min(cap, *n_events); ++i) {
                const auto& e = log->events[static_cast<size_t>(i)];
                events[i] = RefEvent{static_cast<int32_t>(e.kind), e.layer, e.page, e.chunk,
                                     static_cast<int32_t>(e.phase), 0, e.bytes, e.t};
            }
        };
        if (real_bytes == 4) run(float{});
        else run(double{});
    });
}

int ref_train_step(int real_bytes, const RefModelCfg* c, const void* params, const int32_t* tokens, int64_t n,
                   void* grads, double* loss, int32_t* sel_counts) {
    return guarded([&] {
        if (real_bytes == 4) train_step_impl<float>(c, params, tokens, n, grads, loss, sel_counts);
        else train_step_impl<double>(c, params, tokens, n, grads, loss, sel_counts);
    });
}

}  // extern "C"
