// SPDX-License-Identifier: Apache-2.0
//
// Host-side state shared by the C-ABI runtime (oomb_api.cu) and the offload
// engine (tier.cu): the reference page-table mirror, the device pool and
// selection handles, and the exception guard.
#pragma once

#include <algorithm>
#include <deque>
#include <string>
#include <memory>
#include <vector>

#include "oomb_internal.h"

namespace oomb {

extern thread_local std::string g_last_error;

template <class F>
int guard(F&& f) {
    struct Reset {
        ~Reset() { g_prof = nullptr; }
    } reset_prof;
    try {
        f();
        return OOMB_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return OOMB_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return OOMB_ERROR;
    }
}

// ---------------------------------------------------------------------------
// Host mirror of PagedCache's page table (paged_kv.hpp:41-356): arena ids are
// allocated exactly like the reference (LIFO free list; k then v per new page
// at append; gk then gv lazily at first scatter; reset frees k, v, gk, gv per
// page per layer) so page tables compare bit-exactly.
// ---------------------------------------------------------------------------
// Page tiers. DEVICE / HOST are the reference's Tier (paged_kv.hpp:34). REMOTE marks a page whose
// K/V and gradients live on another page-range shard (pool page ownership, oomb_config
// page_owner_stride); LOST marks a host-tier page whose host copy was dropped when a real offload
// engine detached without room to bring it back. Reads of REMOTE / LOST pages always raise
// ResidencyError, enforcement or not.
enum : uint8_t { TIER_DEVICE = 0, TIER_HOST = 1, TIER_REMOTE = 2, TIER_LOST = 3 };

struct PageTable {
    struct Entry {
        int32_t k = -1, v = -1, gk = -1, gv = -1;
        uint8_t tier = TIER_DEVICE;
    };
    int n_layers, P, kvh, hd, kv_elem, grad_elem;
    std::vector<std::vector<Entry>> pages;
    std::vector<int64_t> filled;
    int64_t arena_n = 0;
    std::vector<int32_t> free_list;

    PageTable(int L, int P_, int kvh_, int hd_, int kve, int ge)
        : n_layers(L), P(P_), kvh(kvh_), hd(hd_), kv_elem(kve), grad_elem(ge), pages(L), filled(L, 0) {}

    void check_layer(int layer) const {
        OOMB_REQUIRE(layer >= 0 && layer < n_layers, OOMB_SHAPE_ERROR, "cache: layer out of range");
    }
    int32_t alloc() {  // alloc_page_ paged_kv.hpp:280-288
        if (!free_list.empty()) {
            const int32_t id = free_list.back();
            free_list.pop_back();
            return id;
        }
        return static_cast<int32_t>(arena_n++);
    }
    // append_chunk's page bookkeeping (paged_kv.hpp:73-108). Returns [first_new, n_new).
    void append(int layer, int64_t rows, int64_t* b, int64_t* e, int* first_new, int* n_new) {
        check_layer(layer);
        OOMB_REQUIRE(rows >= 0, OOMB_SHAPE_ERROR, "append_chunk: expected [rows x kvh x hd] K/V of equal shape");
        auto& st = pages[layer];
        *b = filled[layer];
        *e = filled[layer] + rows;
        *first_new = static_cast<int>(st.size());
        *n_new = 0;
        if (rows > 0) {
            const int64_t last_page = (filled[layer] + rows - 1) / P;
            while (static_cast<int64_t>(st.size()) <= last_page) {
                Entry en;
                en.k = alloc();
                en.v = alloc();
                st.push_back(en);
                ++*n_new;
            }
        }
        filled[layer] += rows;
    }
    void check_ids(int layer, const int32_t* ids, int n, bool enforce, const char* op,
                   bool allow_remote = false) const {
        check_layer(layer);
        const auto& st = pages[layer];
        for (int i = 0; i < n; ++i) {
            OOMB_REQUIRE(ids[i] >= 0 && ids[i] < static_cast<int32_t>(st.size()), OOMB_SHAPE_ERROR,
                         std::string(op) + ": page id out of range");
            const uint8_t t = st[ids[i]].tier;
            if (allow_remote && t == TIER_REMOTE) continue;
            OOMB_REQUIRE(t != TIER_REMOTE, OOMB_RESIDENCY_ERROR,
                         std::string(op) + ": page " + std::to_string(ids[i]) + " of layer " + std::to_string(layer) +
                             " is owned by another page-range shard");
            OOMB_REQUIRE(t != TIER_LOST, OOMB_RESIDENCY_ERROR,
                         std::string(op) + ": page " + std::to_string(ids[i]) + " of layer " + std::to_string(layer) +
                             " lost its data when an offload engine detached without room to restore it");
            OOMB_REQUIRE(!enforce || t == TIER_DEVICE, OOMB_RESIDENCY_ERROR,
                         std::string(op) + ": page " + std::to_string(ids[i]) + " of layer " + std::to_string(layer) +
                             " is not device-resident");
        }
    }
    // scatter_add_grads' lazy allocation (paged_kv.hpp:148-153), in call order.
    std::vector<int32_t> scatter(int layer, const int32_t* ids, int n) {
        std::vector<int32_t> fresh;
        auto& st = pages[layer];
        for (int i = 0; i < n; ++i) {
            Entry& en = st[ids[i]];
            if (en.gk < 0) {
                en.gk = alloc();
                en.gv = alloc();
                fresh.push_back(ids[i]);
            }
        }
        return fresh;
    }
    void reset() {  // paged_kv.hpp:227-242
        for (int l = 0; l < n_layers; ++l) {
            for (const auto& en : pages[l]) {
                free_list.push_back(en.k);
                free_list.push_back(en.v);
                if (en.gk >= 0) {
                    free_list.push_back(en.gk);
                    free_list.push_back(en.gv);
                }
            }
            pages[l].clear();
            filled[l] = 0;
        }
    }
    oomb_memory_report report() const {  // paged_kv.hpp:185-197
        oomb_memory_report r{};
        const uint64_t pe = static_cast<uint64_t>(P) * kvh * hd;
        for (const auto& st : pages)
            for (const auto& en : st) {
                r.pages += 1;
                if (en.tier == TIER_DEVICE) r.device_bytes += 2 * pe * kv_elem;
                else if (en.tier == TIER_HOST) r.host_bytes += 2 * pe * kv_elem;
                if (en.gk >= 0) r.grad_bytes += 2 * pe * grad_elem;
            }
        r.arena_blocks = arena_n;
        r.free_list = static_cast<int64_t>(free_list.size());
        return r;
    }
};

}  // namespace oomb

using namespace oomb;

struct oomb_pagetable_s {
    PageTable pt;
};

struct oomb_tier_s;

struct oomb_pool_s {
    oomb_config cfg{};
    oomb_tier_s* engine = nullptr;  // the attached real offload engine (orphaned if the pool dies first)
    int device = 0;
    int64_t max_pages = 0;
    std::shared_ptr<void> loop_state;  // oomb_layer_step's streams / selections (layer_loop.cu)
    int elem = 4;   // K/V element bytes (bf16 2, fp32 4, fp64 8)
    int aelem = 4;  // accumulation element bytes: K_avg sums, gradient pages, lse / dq / votes (fp64 pools: 8)
    bool f64() const { return aelem == 8; }
    int64_t page_elems = 0;
    PageTable* pt = nullptr;
    int64_t n_kv_slots = 0, n_g_slots = 0;
    // Free device slots, FIFO: a slot freed by an eviction goes to the back, so the slot handed out
    // next is the one freed longest ago, whose write-back has most likely drained already.
    std::deque<int32_t> kv_free, g_free;
    std::vector<std::vector<int32_t>> kvslot, gslot;
    void* kpool = nullptr;
    void* vpool = nullptr;
    float* gkpool = nullptr;
    float* gvpool = nullptr;
    int32_t* d_kvslot = nullptr;
    int32_t* d_gslot = nullptr;
    void* d_kavg_sum = nullptr;  // accumulation type (see aelem)
    int32_t* d_kavg_cnt = nullptr;
    uint8_t* d_kavg_planes = nullptr;  // bf16 (see kavg_planes_layer)
    int64_t plane_stride = 0;
    int* d_err = nullptr;
    bool enforce = false;
    int policy = 0;
    // page-range shard ownership (oomb_config page_owner_*): this pool stores K/V / gradients only
    // for pages with id % owner_stride == owner_rank; others are TIER_REMOTE with kvslot SLOT_REMOTE
    int owner_stride = 1, owner_rank = 0;
    bool owns(int64_t page) const { return owner_stride <= 1 || page % owner_stride == owner_rank; }
    TcPoolMaps maps;
    // tcgen05 backward: dQ runs on bwd_side concurrently with dK/dV on the caller's stream. Two
    // workspaces alternate between calls so that, with OOMB_ATTN_DEFER_DQ, chunk i-1's prep and
    // dK/dV can start while chunk i's dQ still reads its workspace (bwd_ev_dq[b] marks its end).
    void* bwd_ws[2] = {nullptr, nullptr};
    size_t bwd_ws_bytes[2] = {0, 0};
    bool bwd_ws_used[2] = {false, false};
    int bwd_parity = 0;
    cudaStream_t bwd_side = nullptr;
    cudaEvent_t bwd_ev_prep = nullptr;
    cudaEvent_t bwd_ev_dq[2] = {nullptr, nullptr};
    cudaEvent_t bwd_last_dq = nullptr;
    bool prof_on = false;
    Profiler prof;
    // Write-back tickets (offload engine): a slot freed by an eviction carries the number of
    // the D2H batch that reads it out, and so does the page's host block it was written to. Each
    // batch records an event on the (in-order) D2H stream; a stream about to write into a recycled
    // slot, or to read a host block back, waits for that batch only if it has not completed yet
    // (and at most once per newer batch).
    std::vector<uint64_t> kv_ticket, g_ticket;
    uint64_t wb_ticket = 0;                                    // newest write-back batch
    int64_t compute_ticket_waits = 0;                          // diagnostics: waits put on a compute stream
    uint64_t wb_completed = 0;                                 // every batch <= this has drained
    std::deque<std::pair<uint64_t, cudaEvent_t>> wb_events;    // batches not yet seen complete
    std::vector<cudaEvent_t> wb_spare;
    std::vector<std::pair<cudaStream_t, uint64_t>> waited;     // newest batch each stream has waited for

    // Victim slots (offload engine): a slot freed by an eviction keeps the evicted page's data until
    // it is handed out again; `holder` names that page (layer * max_pages + page, -1: none). A fetch
    // of the page before then takes the slot back off the free list instead of copying the page in.
    std::vector<int64_t> kv_holder, g_holder;
    void set_holder(bool grad, int32_t s, int64_t idx) {
        auto& h = grad ? g_holder : kv_holder;
        if (h.empty()) h.assign(grad ? n_g_slots : n_kv_slots, -1);
        h[s] = idx;
    }
    // Deferred write-back (offload engine): a victim slot may hold the only current copy of its page;
    // the engine's hook copies it out before the slot is handed to anything else.
    void* victim_ctx = nullptr;
    void (*victim_flush)(void* ctx, bool grad, int32_t slot) = nullptr;
    int32_t pop_free(bool grad) {  // the oldest free slot (FIFO), no longer holding any page's data
        auto& fl = grad ? g_free : kv_free;
        const int32_t s = fl.front();
        auto& h = grad ? g_holder : kv_holder;
        if (victim_flush && !h.empty() && h[s] >= 0) victim_flush(victim_ctx, grad, s);
        fl.pop_front();
        if (!h.empty()) h[s] = -1;
        return s;
    }
    bool holds(bool grad, int32_t s, int64_t idx) const {  // free slot s still holds page idx's data
        const auto& h = grad ? g_holder : kv_holder;
        return s >= 0 && !h.empty() && h[s] == idx;
    }
    bool reclaim(bool grad, int32_t s, int64_t idx) {  // take victim slot s back for page idx
        auto& h = grad ? g_holder : kv_holder;
        if (s < 0 || h.empty() || h[s] != idx) return false;
        auto& fl = grad ? g_free : kv_free;
        const auto it = std::find(fl.begin(), fl.end(), s);
        if (it == fl.end()) return false;
        fl.erase(it);
        h[s] = -1;
        return true;
    }
    void clear_holders() {
        kv_holder.clear();
        g_holder.clear();
    }

    void free_slot_after_writeback(bool grad, int32_t s) {
        auto& v = grad ? g_ticket : kv_ticket;
        if (v.empty()) v.assign(grad ? n_g_slots : n_kv_slots, 0);
        v[s] = wb_ticket;
    }
    void record_writeback(cudaStream_t d2h) {  // after the copies of batch wb_ticket
        cudaEvent_t e;
        if (wb_spare.empty()) {
            OOMB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        } else {
            e = wb_spare.back();
            wb_spare.pop_back();
        }
        OOMB_CUDA(cudaEventRecord(e, d2h));
        wb_events.emplace_back(wb_ticket, e);
    }
    void retire_writebacks() {
        while (!wb_events.empty()) {
            const cudaError_t q = cudaEventQuery(wb_events.front().second);
            if (q == cudaErrorNotReady) return;
            OOMB_CUDA(q);
            wb_completed = wb_events.front().first;
            wb_spare.push_back(wb_events.front().second);
            wb_events.pop_front();
        }
    }
    bool wait_slot(bool grad, int32_t s, cudaStream_t st) {
        const auto& v = grad ? g_ticket : kv_ticket;
        return !v.empty() && wait_ticket(v[s], st);
    }
    // Make stream st wait until write-back batch t has drained (no-op when it has, or when st
    // already waited for a batch >= t).
    bool wait_ticket(uint64_t t, cudaStream_t st) {  // true: st now waits on a pending batch
        if (t <= wb_completed) return false;
        retire_writebacks();
        if (t <= wb_completed) return false;
        auto it = std::find_if(waited.begin(), waited.end(), [&](const auto& w) { return w.first == st; });
        if (it != waited.end() && it->second >= t) return false;
        for (const auto& b : wb_events)
            if (b.first >= t) {  // the first pending batch at or after the slot's: covers it (in-order stream)
                OOMB_CUDA(cudaStreamWaitEvent(st, b.second, 0));
                if (it != waited.end()) it->second = b.first;
                else waited.emplace_back(st, b.first);
                return true;
            }
        return false;
    }
    void destroy_writeback_events() {
        for (auto& b : wb_events) cudaEventDestroy(b.second);
        for (auto e : wb_spare) cudaEventDestroy(e);
        wb_events.clear();
        wb_spare.clear();
    }

    int32_t* kvslot_layer(int l) { return d_kvslot + static_cast<int64_t>(l) * max_pages; }
    int32_t* gslot_layer(int l) { return d_gslot + static_cast<int64_t>(l) * max_pages; }
    void* kavg_sum_layer(int l) {
        return static_cast<uint8_t*>(d_kavg_sum) + static_cast<int64_t>(l) * max_pages * cfg.n_kv_heads * cfg.head_dim * aelem;
    }
    int32_t* kavg_cnt_layer(int l) { return d_kavg_cnt + static_cast<int64_t>(l) * max_pages; }
    // bf16 hi / lo planes of K_avg for the tcgen05 scorer ([layer][2][Hkv][plane_stride][hd]); null when
    // the pool's dtype / head dim never use it
    void* kavg_planes_layer(int l) {
        return d_kavg_planes ? static_cast<void*>(d_kavg_planes + static_cast<int64_t>(l) * 2 * cfg.n_kv_heads *
                                                                       plane_stride * cfg.head_dim * 2)
                             : nullptr;
    }
};

struct oomb_selection_s {
    oomb_pool_s* pool = nullptr;
    bool nnz_from_host = false;  // nnz is known only once the host mirror lands (filter_owned)
    int max_m = 0, max_ids = 0;
    int32_t* d_off = nullptr;
    int32_t* d_ids = nullptr;
    int32_t* h_off = nullptr;  // pinned
    int32_t* h_ids = nullptr;  // pinned
    int m = 0, nnz = 0;
    cudaEvent_t ev = nullptr;
    bool host_pending = false;  // device -> host mirror copy in flight
};


inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
inline void set_dev(oomb_pool_s* p) {
    OOMB_CUDA(cudaSetDevice(p->device));
    g_prof = p->prof_on ? &p->prof : nullptr;
}
