// SPDX-License-Identifier: Apache-2.0
//
// Tiered residency engine — TieredEngine (tiered_memory.hpp:99-432) for B200.
//
// The decision logic is the reference's, statement for statement: the same LRU
// counter, reserved / pinned flags, best-effort all-or-nothing prefetch with append
// headroom, write-back of dirty K/V and gradient pages only, the same capacity
// error. On a bare page table it also runs the reference's simulated clock, so its
// ScheduleLog equals the reference's event for event (tests/test_tier_cpu.py).
//
// On a pool the pages really move:
//   evict  -> D2H stream waits for the compute stream's tail, copies the dirty K/V
//             (and dK/dV) blocks of the page's device slots into its pinned host
//             blocks, records an event; the device slots return to the free list
//             tagged with that event; the device page-table entries are cleared on
//             the compute stream.
//   fetch  -> a device slot is taken (the H2D stream first waits for the slot's
//             last write-back), K/V (+dK/dV) are copied H2D, an event is recorded.
//   wait   -> the compute stream waits for the transfer's event, then the new
//             slots are published in the device page table (one small kernel).
// Log timestamps then come from CUDA events recorded at each point, so
// validate_schedule checks residency-before-use on the real GPU timeline.

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <set>
#include <tuple>

#include "pool.h"

namespace oomb {

enum EventKind { EV_FETCH_ISSUED = 0, EV_FETCH_DONE, EV_EVICT, EV_COMPUTE_BEGIN, EV_COMPUTE_END, EV_ACCESS };

// Device page-table update list, applied by one kernel on the compute stream.
struct TableUpdates {
    int32_t n;
    int32_t idx[480];  // (layer*max_pages + page) entries
    int32_t kv[480];
    int32_t g[480];
};

__global__ void table_update_kernel(TableUpdates u, int32_t* kvslot, int32_t* gslot) {
    for (int i = threadIdx.x; i < u.n; i += blockDim.x) {
        kvslot[u.idx[i]] = u.kv[i];
        gslot[u.idx[i]] = u.g[i];
    }
}

// Staged page moves: a flush's pieces are packed back to back in a device staging buffer, so the
// host link sees one cudaMemcpyAsync per run of host-contiguous pieces (a page's K | V, or dK | dV,
// and pages with adjacent ids) instead of one per piece, and the scatter into (gather out of) the
// pool's slots is one kernel over HBM. One CTA per piece, 16-byte vectors.
struct StagePiece {
    uint8_t* dev;  // the piece's place in a pool (K, V, dK or dV slot)
    int64_t off;   // its offset in the staging buffer
    int64_t n;     // bytes (a multiple of 16)
};

__global__ void stage_move_kernel(const StagePiece* __restrict__ pc, uint8_t* __restrict__ stg, int to_pool) {
    const StagePiece q = pc[blockIdx.x];
    uint4* a = reinterpret_cast<uint4*>(to_pool ? q.dev : stg + q.off);
    const uint4* b = reinterpret_cast<const uint4*>(to_pool ? stg + q.off : q.dev);
    for (int64_t i = threadIdx.x; i < q.n / 16; i += blockDim.x) a[i] = b[i];
}

}  // namespace oomb

using namespace oomb;

struct oomb_tier_s {
    struct PageState {
        bool kv_host_valid = true;
        bool grad_host_valid = true;
        bool reserved = false;
        bool pinned = false;
        double in_flight_done = 0;
        double writeback_done = 0;
        uint64_t lru = 0;
        bool host_has_kv = false;    // real mode: host block holds data
        bool host_has_grad = false;
        uint64_t wb_batch = 0;       // real mode: the write-back batch that last filled the host block
        int32_t vkv = -1, vg = -1;   // real mode: the slots the page was evicted from (victim slots)
        bool pend_kv = false, pend_g = false;  // real mode: the host block is stale, the victim slot (or,
                                               // once fetched back, the page's slot) holds the data
    };
    struct Transfer {
        int layer = 0;
        std::vector<int32_t> pages;
        double ready = 0;
        cudaEvent_t ev = nullptr;  // real mode: copies done
    };
    struct LogEv {
        oomb_event e;
        cudaEvent_t ev;  // real mode timestamp (nullptr: use e.t)
    };

    oomb_tier_config cfg{};
    PageTable* pt = nullptr;
    oomb_pool_s* pool = nullptr;  // nullptr = simulation mode
    bool orphaned = false;        // real mode: the pool was destroyed before the engine
    int phase = 0;
    double clock = 0, h2d_free = 0, d2h_free = 0, stall_s = 0;
    uint64_t h2d_fwd = 0, h2d_bwd = 0, d2h = 0, lru_counter = 0;
    int64_t headroom = 0;
    std::vector<std::vector<PageState>> pages;
    std::vector<Transfer> transfers;
    std::vector<LogEv> log;

    // ---- real mode
    cudaStream_t compute = nullptr, h2d_stream = nullptr, d2h_stream = nullptr;
    // OOMB_TIER_DEBUG counters: best-effort issued / refused, pages prefetched / fetched on demand,
    // H2D waits on a page's own pending write-back, H2D waits on a recycled slot's write-back
    int64_t dbg[6] = {};
    uint64_t h2d_moved = 0;  // real mode: bytes actually copied in (victim-slot reclaims move none)
    uint64_t d2h_moved = 0;  // real mode: bytes actually copied out (deferred write-backs of reclaimed pages: none)
    // Deferred write-back (OOMB_TIER_LAZY_WB=1; default off): an eviction frees the page's slots
    // without copying them out; a victim slot is copied out only when it comes within clean_ahead
    // (OOMB_TIER_CLEAN_AHEAD) slots of the front of its free list, or is handed out, so a page fetched
    // back before then moves nothing either way. The engine's decisions and its transfer accounting
    // are the reference's. Measured at c3 low locality (profiles/r02_perf_notes.md): 22-56 % less D2H,
    // but a copy-out issued close to the slot's reuse makes the taker wait for it, so the step is
    // faster only with spare slots (7,168: 549 vs 561 ms backward) and slower with the bench's 6,656.
    bool lazy_wb = false;
    int64_t forced_flushes = 0;  // deferred victims copied out only when their slot was handed out
    int64_t clean_ahead = 256;
    cudaEvent_t t0 = nullptr;
    std::vector<cudaEvent_t> spare_events;
    // pinned [layer][page] x (K, V, dK, dV) blocks, one allocation: a page's four pieces are adjacent,
    // so a move of its K/V and gradients is one host-contiguous run (one copy, staged flushes)
    uint8_t* host_kv = nullptr;    // K, V of block 0 (stride page_block)
    uint8_t* host_grad = nullptr;  // dK, dV of block 0 (host_kv + kv_block, stride page_block)
    size_t kv_block = 0, grad_block = 0, page_block = 0;
    TableUpdates pending{};

    bool real() const { return pool != nullptr; }

    cudaEvent_t new_event() {
        if (!spare_events.empty()) {
            cudaEvent_t e = spare_events.back();
            spare_events.pop_back();
            return e;
        }
        cudaEvent_t e;
        OOMB_CUDA(cudaEventCreate(&e));
        return e;
    }

    void sync_pages() {
        pages.resize(pt->n_layers);
        for (int l = 0; l < pt->n_layers; ++l) pages[l].resize(pt->pages[l].size());
    }
    PageState& state(int layer, int page) {
        sync_pages();
        return pages.at(layer).at(page);
    }
    uint8_t tier(int layer, int page) const { return pt->pages[layer][page].tier; }
    void set_tier(int layer, int page, uint8_t t) { pt->pages[layer][page].tier = t; }
    int64_t device_page_count() const {  // tiered_memory.hpp:328-336
        int64_t n = 0;
        for (int l = 0; l < pt->n_layers; ++l)
            for (const auto& e : pt->pages[l]) n += e.tier == 0;
        return n;
    }
    bool grads_allocated(int layer, int page) const { return pt->pages[layer][page].gk >= 0; }
    uint64_t kv_bytes() const {  // page_kv_bytes: K+V of one page, all kv heads
        return 2ull * pt->P * pt->kvh * pt->hd * pt->kv_elem;
    }
    uint64_t grad_bytes() const { return 2ull * pt->P * pt->kvh * pt->hd * pt->grad_elem; }
    uint64_t page_transfer_bytes(int layer, int page) const {  // tiered_memory.hpp:322-326
        uint64_t b = kv_bytes();
        if (grads_allocated(layer, page)) b += grad_bytes();
        return b;
    }

    // `on`: the stream whose timeline stamps the event in real mode (the compute stream may be the
    // legacy default stream, i.e. a null handle, so the choice is explicit rather than a pointer).
    enum On { ON_NONE = 0, ON_COMPUTE, ON_H2D, ON_D2H };
    // Real-mode log timestamps: one CUDA event per engine operation and stream, shared by every
    // log entry it stamps (one event per page would be one API call per page). `stamp` records
    // now; `later` creates an event that the caller records once the batch it stamps is enqueued.
    std::vector<cudaEvent_t> log_events;  // owned, destroyed with the engine
    cudaStream_t stream_of(On on) const { return on == ON_COMPUTE ? compute : (on == ON_H2D ? h2d_stream : d2h_stream); }
    cudaEvent_t later() {
        if (!real()) return nullptr;
        cudaEvent_t e;
        OOMB_CUDA(cudaEventCreate(&e));
        log_events.push_back(e);
        return e;
    }
    cudaEvent_t stamp(On on) {
        cudaEvent_t e = later();
        if (e) OOMB_CUDA(cudaEventRecord(e, stream_of(on)));
        return e;
    }
    void push(int kind, double t, int layer, int32_t page, uint64_t bytes, int chunk, cudaEvent_t ev = nullptr) {
        LogEv le{};
        le.e.kind = kind;
        le.e.t = t;
        le.e.layer = layer;
        le.e.page = page;
        le.e.chunk = chunk;
        le.e.bytes = bytes;
        le.e.phase = phase;
        le.ev = ev;
        log.push_back(le);
    }

    // ---- queued page copies (real mode): flushed per direction and operation as one
    // cudaMemcpyAsync per run of copies that are contiguous on both sides (adjacent slots of
    // adjacent host blocks merge into one transfer)
    std::vector<void*> cp_dst[2], cp_src[2];
    std::vector<size_t> cp_size[2];
    int64_t copy_calls = 0;              // diagnostics: cudaMemcpyAsync calls issued by flushes
    cudaEvent_t d2h_batch_ev = nullptr;  // the current write-back batch's completion stamp
    void queue_copy(int dir, void* dst, const void* src, size_t n) {  // dir 0: H2D, 1: D2H
        auto& d = cp_dst[dir];
        auto& s = cp_src[dir];
        auto& z = cp_size[dir];
        if (!d.empty() && static_cast<uint8_t*>(d.back()) + z.back() == dst &&
            static_cast<const uint8_t*>(s.back()) + z.back() == src) {
            z.back() += n;  // extends the previous run on both sides
            return;
        }
        d.push_back(dst);
        s.push_back(const_cast<void*>(src));
        z.push_back(n);
    }
    // OOMB_TIER_STAGED: bit 0 stages H2D flushes, bit 1 D2H flushes (default 3); an unstaged flush
    // is one cudaMemcpyAsync per queued run, straight between host block and slot
    const int staged_dirs = [] {
        const char* e = std::getenv("OOMB_TIER_STAGED");
        return e ? std::atoi(e) : 3;
    }();
    std::vector<StagePiece> stage_pcs;
    void flush_copies(int dir) {
        auto& dv = cp_dst[dir];
        auto& sv = cp_src[dir];
        auto& zv = cp_size[dir];
        if (dv.empty()) return;
        const cudaStream_t st = dir ? d2h_stream : h2d_stream;
        const cudaMemcpyKind kind = dir ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice;
        const size_t n = dv.size();
        bool aligned = true;
        for (size_t i = 0; i < n; ++i)
            aligned = aligned && ((reinterpret_cast<uintptr_t>(dv[i]) | reinterpret_cast<uintptr_t>(sv[i]) | zv[i]) & 15) == 0;
        if (!(staged_dirs & (1 << dir)) || n < 3 || !aligned) {
            for (size_t i = 0; i < n; ++i) OOMB_CUDA(cudaMemcpyAsync(dv[i], sv[i], zv[i], kind, st));
            copy_calls += static_cast<int64_t>(n);
        } else {
            // pieces back to back in staging; the device side of each piece is the pool side
            stage_pcs.resize(n);
            int64_t total = 0;
            for (size_t i = 0; i < n; ++i) {
                stage_pcs[i].dev = static_cast<uint8_t*>(dir ? sv[i] : dv[i]);
                stage_pcs[i].off = total;
                stage_pcs[i].n = static_cast<int64_t>(zv[i]);
                total += stage_pcs[i].n;
            }
            const int64_t desc_off = (total + 255) & ~int64_t(255);
            uint8_t* stg = nullptr;
            OOMB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&stg), desc_off + n * sizeof(StagePiece), st));
            auto* desc = reinterpret_cast<StagePiece*>(stg + desc_off);
            // pageable source: the call returns once the descriptors are staged by the driver
            OOMB_CUDA(cudaMemcpyAsync(desc, stage_pcs.data(), n * sizeof(StagePiece), cudaMemcpyHostToDevice, st));
            // host runs: consecutive pieces whose host blocks are adjacent move in one copy
            auto host_runs = [&](auto&& copy) {
                size_t i = 0;
                while (i < n) {
                    uint8_t* h = static_cast<uint8_t*>(dir ? dv[i] : sv[i]);
                    int64_t len = stage_pcs[i].n;
                    size_t j = i + 1;
                    while (j < n && static_cast<uint8_t*>(dir ? dv[j] : sv[j]) == h + len) len += stage_pcs[j++].n;
                    copy(h, stage_pcs[i].off, len);
                    i = j;
                }
            };
            if (dir) {  // D2H: gather the slots, then the runs to their host blocks
                stage_move_kernel<<<static_cast<unsigned>(n), 256, 0, st>>>(desc, stg, 0);
                OOMB_CUDA(cudaGetLastError());
                host_runs([&](uint8_t* h, int64_t off, int64_t len) {
                    OOMB_CUDA(cudaMemcpyAsync(h, stg + off, len, cudaMemcpyDeviceToHost, st));
                    ++copy_calls;
                });
            } else {  // H2D: the runs into staging, then scatter into the slots
                host_runs([&](uint8_t* h, int64_t off, int64_t len) {
                    OOMB_CUDA(cudaMemcpyAsync(stg + off, h, len, cudaMemcpyHostToDevice, st));
                    ++copy_calls;
                });
                stage_move_kernel<<<static_cast<unsigned>(n), 256, 0, st>>>(desc, stg, 1);
                OOMB_CUDA(cudaGetLastError());
            }
            OOMB_CUDA(cudaFreeAsync(stg, st));
        }
        dv.clear();
        sv.clear();
        zv.clear();
    }
    // A write-back batch: the D2H stream follows everything enqueued on the compute stream so
    // far, then copies every evicted page, then stamps the batch; slots freed by it carry its
    // ticket (pool.h) so a later write into a recycled slot waits for the read-out.
    void begin_writeback() {
        if (!real()) return;
        cudaEvent_t tail = new_event();
        OOMB_CUDA(cudaEventRecord(tail, compute));
        OOMB_CUDA(cudaStreamWaitEvent(d2h_stream, tail, 0));
        spare_events.push_back(tail);
        ++pool->wb_ticket;
        d2h_batch_ev = later();
    }
    void end_writeback() {
        if (!real()) return;
        flush_copies(1);
        pool->record_writeback(d2h_stream);
        OOMB_CUDA(cudaEventRecord(d2h_batch_ev, d2h_stream));
        d2h_batch_ev = nullptr;
    }

    // ---- device table publication (real mode)
    void queue_table(int layer, int page) {
        const int idx = static_cast<int>(layer * pool->max_pages + page);
        // one entry per (layer, page) per batch, holding the newest slots: the kernel applies
        // entries in parallel, so two entries for one page would race (eviction then refetch)
        int at = -1;
        for (int i = 0; i < pending.n; ++i)
            if (pending.idx[i] == idx) {
                at = i;
                break;
            }
        if (at < 0) {
            if (pending.n == 480) flush_table();
            at = pending.n++;
            pending.idx[at] = idx;
        }
        pending.kv[at] = pool->kvslot[layer][page];
        pending.g[at] = pool->gslot[layer][page];
    }
    void flush_table() {
        if (!real() || pending.n == 0) return;
        table_update_kernel<<<1, 256, 0, compute>>>(pending, pool->d_kvslot, pool->d_gslot);
        check_launch("table_update_kernel");
        pending.n = 0;
    }

    // ---- capacity (tiered_memory.hpp:341-384)
    bool fits_after_eviction(int64_t incoming) {
        if (cfg.device_capacity_pages < 0) return true;
        sync_pages();
        int64_t evictable = 0;
        for (int l = 0; l < pt->n_layers; ++l)
            for (size_t p = 0; p < pages[l].size(); ++p)
                if (tier(l, static_cast<int>(p)) == 0 && !pages[l][p].reserved) ++evictable;
        return device_page_count() - evictable + incoming <= cfg.device_capacity_pages;
    }

    void enforce_capacity(int64_t incoming) {
        // The reference evicts one page at a time, each time the non-reserved resident page with
        // the smallest (pinned, lru) key (tiered_memory.hpp:341-384). Evicting a page changes no
        // other page's key, so the victims are exactly the `need` smallest keys in ascending order:
        // one scan + partial sort gives the same evictions and log, O(n + k log k) instead of O(n k).
        if (cfg.device_capacity_pages < 0) return;
        sync_pages();
        const int64_t need = device_page_count() + incoming - cfg.device_capacity_pages;
        if (need <= 0) return;
        struct Cand {
            bool pinned;
            uint64_t lru;
            int l, p;
        };
        std::vector<Cand> cand;
        for (int l = 0; l < pt->n_layers; ++l)
            for (size_t p = 0; p < pages[l].size(); ++p) {
                const PageState& ps = pages[l][p];
                if (tier(l, static_cast<int>(p)) != 0 || ps.reserved) continue;
                cand.push_back({ps.pinned, ps.lru, l, static_cast<int>(p)});
            }
        const size_t k = std::min<size_t>(cand.size(), static_cast<size_t>(need));
        auto key_less = [](const Cand& a, const Cand& b) {
            return std::make_pair(a.pinned, a.lru) < std::make_pair(b.pinned, b.lru);
        };
        std::partial_sort(cand.begin(), cand.begin() + k, cand.end(), key_less);
        begin_writeback();
        for (size_t i = 0; i < k; ++i) {
            pages[cand[i].l][cand[i].p].pinned = false;
            evict(cand[i].l, cand[i].p);
        }
        end_writeback();
        clean_front();
        if (static_cast<int64_t>(k) < need)
            throw Error(OOMB_CONFIG_ERROR, "tiered_memory: device capacity smaller than the working set (capacity " +
                                               std::to_string(cfg.device_capacity_pages) + " pages)");
    }

    // ---- eviction (tiered_memory.hpp:386-403)
    void evict(int layer, int page) {
        PageState& ps = state(layer, page);
        uint64_t bytes = 0;
        const bool wb_kv = !ps.kv_host_valid;
        const bool wb_grad = grads_allocated(layer, page) && !ps.grad_host_valid;
        if (wb_kv) bytes += kv_bytes();
        if (wb_grad) bytes += grad_bytes();
        if (bytes > 0) {
            const double start = std::max(d2h_free, clock);
            ps.writeback_done = start + static_cast<double>(bytes) / cfg.bandwidth_bytes_per_s;
            d2h_free = ps.writeback_done;
            d2h += bytes;
            ps.kv_host_valid = true;
            ps.grad_host_valid = true;
        }
        if (real()) real_evict(layer, page, wb_kv, wb_grad);
        set_tier(layer, page, 1);
        push(EV_EVICT, clock, layer, page, bytes, -1, d2h_batch_ev);
    }

    void real_evict(int layer, int page, bool wb_kv, bool wb_grad) {
        auto& p = *pool;
        const int32_t ks = p.kvslot[layer][page], gs = p.gslot[layer][page];
        const size_t hidx = static_cast<size_t>(layer) * p.max_pages + page;
        const size_t kvb = static_cast<size_t>(p.page_elems) * p.elem;
        const size_t gb = static_cast<size_t>(p.page_elems) * sizeof(float);
        PageState& ps = pages[layer][page];
        // a page fetched back into its victim slots with a write-back still deferred has a stale host
        // block even when the reference's flags say clean
        const bool need_kv = (wb_kv || ps.pend_kv) && ks >= 0;
        const bool need_g = (wb_grad || ps.pend_g) && gs >= 0;
        ps.pend_kv = lazy_wb && need_kv;
        ps.pend_g = lazy_wb && need_g;
        if (need_kv && !lazy_wb) {
            uint8_t* h = host_kv + hidx * page_block;
            queue_copy(1, h, static_cast<uint8_t*>(p.kpool) + ks * kvb, kvb);
            queue_copy(1, h + kvb, static_cast<uint8_t*>(p.vpool) + ks * kvb, kvb);
            ps.host_has_kv = true;
            ps.wb_batch = p.wb_ticket;
            d2h_moved += 2 * kvb;
        }
        if (need_g && !lazy_wb) {
            uint8_t* h = host_grad + hidx * page_block;
            queue_copy(1, h, reinterpret_cast<uint8_t*>(p.gkpool) + gs * gb, gb);
            queue_copy(1, h + gb, reinterpret_cast<uint8_t*>(p.gvpool) + gs * gb, gb);
            ps.host_has_grad = true;
            ps.wb_batch = p.wb_ticket;
            d2h_moved += 2 * gb;
        }
        if (ks >= 0) {
            p.free_slot_after_writeback(false, ks);
            p.kv_free.push_back(ks);
            p.set_holder(false, ks, static_cast<int64_t>(hidx));
        }
        if (gs >= 0) {
            p.free_slot_after_writeback(true, gs);
            p.g_free.push_back(gs);
            p.set_holder(true, gs, static_cast<int64_t>(hidx));
        }
        ps.vkv = ks;
        ps.vg = gs;
        p.kvslot[layer][page] = -1;
        p.gslot[layer][page] = -1;
        queue_table(layer, page);
    }

    int32_t take_slot(bool grad, cudaStream_t st, const char* what) {
        auto& fl = grad ? pool->g_free : pool->kv_free;
        OOMB_REQUIRE(!fl.empty(), OOMB_CONFIG_ERROR,
                     std::string("offload: no free device ") + what +
                         " slot for an in-flight fetch (raise the pool's device_capacity_pages above the tier "
                         "capacity)");
        const int32_t s = pool->pop_free(grad);
        dbg[5] += pool->wait_slot(grad, s, st);
        return s;
    }

    // Copy a deferred victim out of free slot s into its page's host block (inside a write-back
    // batch: the D2H stream already follows the compute stream). The slot's ticket moves to this batch.
    void flush_victim(bool grad, int32_t s) {
        auto& p = *pool;
        const auto& hold = grad ? p.g_holder : p.kv_holder;
        if (hold.empty() || hold[s] < 0) return;
        const int64_t idx = hold[s];
        const int layer = static_cast<int>(idx / p.max_pages), page = static_cast<int>(idx % p.max_pages);
        PageState& ps = pages[layer][page];
        if (grad ? !(ps.pend_g && ps.vg == s) : !(ps.pend_kv && ps.vkv == s)) return;
        const size_t kvb = static_cast<size_t>(p.page_elems) * p.elem;
        const size_t gb = static_cast<size_t>(p.page_elems) * sizeof(float);
        if (grad) {
            uint8_t* h = host_grad + static_cast<size_t>(idx) * page_block;
            queue_copy(1, h, reinterpret_cast<uint8_t*>(p.gkpool) + s * gb, gb);
            queue_copy(1, h + gb, reinterpret_cast<uint8_t*>(p.gvpool) + s * gb, gb);
            ps.host_has_grad = true;
            ps.pend_g = false;
            d2h_moved += 2 * gb;
        } else {
            uint8_t* h = host_kv + static_cast<size_t>(idx) * page_block;
            queue_copy(1, h, static_cast<uint8_t*>(p.kpool) + s * kvb, kvb);
            queue_copy(1, h + kvb, static_cast<uint8_t*>(p.vpool) + s * kvb, kvb);
            ps.host_has_kv = true;
            ps.pend_kv = false;
            d2h_moved += 2 * kvb;
        }
        ps.wb_batch = p.wb_ticket;
        p.free_slot_after_writeback(grad, s);
    }
    // Copy out the deferred victims among the first clean_ahead slots of both free lists.
    void clean_front() {
        if (!real() || !lazy_wb) return;
        bool open = false;
        for (int g = 0; g < 2; ++g) {
            const auto& fl = g ? pool->g_free : pool->kv_free;
            const auto& hold = g ? pool->g_holder : pool->kv_holder;
            if (hold.empty()) continue;
            int64_t n = 0;
            for (auto it = fl.begin(); it != fl.end() && n < clean_ahead; ++it, ++n) {
                const int64_t idx = hold[*it];
                if (idx < 0) continue;
                const PageState& ps = pages[idx / pool->max_pages][idx % pool->max_pages];
                if (!(g ? (ps.pend_g && ps.vg == *it) : (ps.pend_kv && ps.vkv == *it))) continue;
                if (!open) begin_writeback();
                open = true;
                flush_victim(g != 0, *it);
            }
        }
        if (open) end_writeback();
    }
    // The pool hands out a free slot that still holds a deferred victim: copy it out first (its own
    // batch; the taker waits for it through the slot's ticket).
    static void forced_flush(void* ctx, bool grad, int32_t s) {
        auto* t = static_cast<oomb_tier_s*>(ctx);
        const auto& hold = grad ? t->pool->g_holder : t->pool->kv_holder;
        const int64_t idx = hold[s];
        const PageState& ps = t->pages[idx / t->pool->max_pages][idx % t->pool->max_pages];
        if (!(grad ? (ps.pend_g && ps.vg == s) : (ps.pend_kv && ps.vkv == s))) return;
        // slots are only handed out outside a write-back batch (evictions and clean-ahead take none)
        OOMB_REQUIRE(t->d2h_batch_ev == nullptr, OOMB_STATE_ERROR, "offload: slot taken inside a write-back batch");
        t->begin_writeback();
        t->flush_victim(grad, s);
        t->end_writeback();
        ++t->forced_flushes;
    }

    // H2D of one page into fresh device slots (real mode).
    void real_fetch(int layer, int page) {
        auto& p = *pool;
        const size_t hidx = static_cast<size_t>(layer) * p.max_pages + page;
        const size_t kvb = static_cast<size_t>(p.page_elems) * p.elem;
        const size_t gb = static_cast<size_t>(p.page_elems) * sizeof(float);
        PageState& ps = pages[layer][page];
        // A page whose victim slots were not handed out since its eviction still has its data there
        // (a write-back, deferred or not, only reads them): it takes them back, no copy and no wait for
        // the read-out. A later write into a reclaimed slot (scatter, append) marks the host copy
        // stale, so a torn read-out is always written again before the host block is used. Otherwise
        // the host block is read, only after the write-back that filled it has landed; the
        // destination slots wait for their own read-outs in take_slot.
        const int64_t idx = static_cast<int64_t>(hidx);
        const bool g_need = grads_allocated(layer, page);
        const int32_t vkv = ps.vkv, vg = ps.vg;
        const bool kv_held = p.holds(false, vkv, idx), g_held = g_need && p.holds(true, vg, idx);
        OOMB_REQUIRE(kv_held || ps.host_has_kv, OOMB_STATE_ERROR,
                     "offload: page " + std::to_string(page) + " of layer " + std::to_string(layer) +
                         " is host-tier but its host block holds no data");
        OOMB_REQUIRE((kv_held || !ps.pend_kv) && (g_held || !g_need || !ps.pend_g), OOMB_STATE_ERROR,
                     "offload: page " + std::to_string(page) + " has a deferred write-back but no victim slot");
        ps.vkv = ps.vg = -1;
        const bool kv_back = kv_held && p.reclaim(false, vkv, idx);
        const bool g_back = g_held && p.reclaim(true, vg, idx);
        if (!kv_back || (g_need && !g_back && ps.host_has_grad)) dbg[4] += p.wait_ticket(ps.wb_batch, h2d_stream);
        const int32_t ks = kv_back ? vkv : take_slot(false, h2d_stream, "KV");
        p.kvslot[layer][page] = ks;
        if (!kv_back && ps.host_has_kv) {
            const uint8_t* h = host_kv + hidx * page_block;
            queue_copy(0, static_cast<uint8_t*>(p.kpool) + ks * kvb, h, kvb);
            queue_copy(0, static_cast<uint8_t*>(p.vpool) + ks * kvb, h + kvb, kvb);
            h2d_moved += 2 * kvb;
        }
        if (g_back) {
            p.gslot[layer][page] = vg;
        } else if (g_need) {
            const int32_t gs = take_slot(true, h2d_stream, "gradient");
            p.gslot[layer][page] = gs;
            if (ps.host_has_grad) {
                h2d_moved += 2 * gb;
                const uint8_t* h = host_grad + hidx * page_block;
                queue_copy(0, reinterpret_cast<uint8_t*>(p.gkpool) + gs * gb, h, gb);
                queue_copy(0, reinterpret_cast<uint8_t*>(p.gvpool) + gs * gb, h + gb, gb);
            } else {
                OOMB_CUDA(cudaMemsetAsync(reinterpret_cast<uint8_t*>(p.gkpool) + gs * gb, 0, gb, h2d_stream));
                OOMB_CUDA(cudaMemsetAsync(reinterpret_cast<uint8_t*>(p.gvpool) + gs * gb, 0, gb, h2d_stream));
            }
        }
    }

    // ---- public operations
    void on_pages_appended(int layer, int64_t b, int64_t e) {  // tiered_memory.hpp:131-145
        sync_pages();
        if (e <= b) return;
        const int first = static_cast<int>(b / pt->P);
        const int last = static_cast<int>((e - 1) / pt->P);
        cudaEvent_t ev = stamp(ON_COMPUTE);
        for (int p = first; p <= last; ++p) {
            PageState& ps = state(layer, p);
            ps.kv_host_valid = false;
            ps.reserved = true;
            ps.lru = ++lru_counter;
            push(EV_FETCH_DONE, clock, layer, p, 0, -1, ev);
        }
        enforce_capacity(0);
    }

    int64_t fetch_async(int layer, const int32_t* ids, int n, int chunk, bool best_effort) {  // :163-229
        sync_pages();
        Transfer tr;
        tr.layer = layer;
        std::vector<int32_t> to_transfer, to_pin;
        double ready = clock;
        for (int i = 0; i < n; ++i) {
            const int32_t p = ids[i];
            if (p < 0 || p >= static_cast<int32_t>(pt->pages[layer].size()))
                throw Error(OOMB_STATE_ERROR, "fetch_pages: unknown page " + std::to_string(p));
            PageState& ps = state(layer, p);
            if (tier(layer, p) >= TIER_REMOTE)
                throw Error(OOMB_RESIDENCY_ERROR, "fetch_pages: page " + std::to_string(p) +
                                                      (tier(layer, p) == TIER_REMOTE
                                                           ? " is owned by another page-range shard"
                                                           : " lost its data when an engine detached"));
            if (tier(layer, p) == 0) {
                if (best_effort) {
                    if (!ps.reserved && !ps.pinned) to_pin.push_back(p);
                } else {
                    ps.reserved = true;
                    ps.pinned = false;
                    ps.lru = ++lru_counter;
                }
                continue;
            }
            if (ps.in_flight_done > 0) {
                tr.pages.push_back(p);
                ready = std::max(ready, ps.in_flight_done);
                continue;
            }
            to_transfer.push_back(p);
        }
        if (best_effort) {
            const int64_t hr = phase == 0 ? headroom : 0;
            const int64_t demand = static_cast<int64_t>(to_transfer.size()) + static_cast<int64_t>(to_pin.size()) + hr;
            ++dbg[0];
            if (!fits_after_eviction(demand)) {
                ++dbg[1];
                to_transfer.clear();
            } else {
                for (int32_t p : to_pin) {
                    PageState& ps = state(layer, p);
                    ps.pinned = true;
                    ps.lru = ++lru_counter;
                }
            }
        }
        dbg[best_effort ? 2 : 3] += static_cast<int64_t>(to_transfer.size());
        cudaEvent_t ev_issue = to_transfer.empty() ? nullptr : stamp(ON_H2D);
        cudaEvent_t ev_done = to_transfer.empty() ? nullptr : later();
        for (int32_t p : to_transfer) {
            PageState& ps = state(layer, p);
            const uint64_t bytes = page_transfer_bytes(layer, p);
            push(EV_FETCH_ISSUED, clock, layer, p, 0, chunk, ev_issue);
            const double start = std::max({h2d_free, clock, ps.writeback_done});
            const double done = start + static_cast<double>(bytes) / cfg.bandwidth_bytes_per_s;
            h2d_free = done;
            ps.in_flight_done = done;
            if (phase == 0) h2d_fwd += bytes;
            else h2d_bwd += bytes;
            // a page listed twice is logged twice, as in the reference, but moved once (its second
            // occurrence finds the slots the first one took)
            if (real() && pool->kvslot[layer][p] < 0) real_fetch(layer, p);
            push(EV_FETCH_DONE, done, layer, p, bytes, chunk, ev_done);
            ready = std::max(ready, done);
            tr.pages.push_back(p);
        }
        if (real()) {
            flush_copies(0);
            if (ev_done) OOMB_CUDA(cudaEventRecord(ev_done, h2d_stream));
            tr.ev = new_event();
            OOMB_CUDA(cudaEventRecord(tr.ev, h2d_stream));
        }
        tr.ready = ready;
        transfers.push_back(std::move(tr));
        return static_cast<int64_t>(transfers.size()) - 1;
    }

    void wait(int64_t h) {  // :234-254
        if (h < 0 || h >= static_cast<int64_t>(transfers.size()))
            throw Error(OOMB_STATE_ERROR, "wait: handle was never issued");
        Transfer& tr = transfers[h];
        if (tr.ready > clock) {
            stall_s += tr.ready - clock;
            clock = tr.ready;
        }
        if (real() && tr.ev) OOMB_CUDA(cudaStreamWaitEvent(compute, tr.ev, 0));
        // The reference enforces capacity for one incoming page before each page turns resident;
        // the pages of this transfer are not eviction candidates either way (still host-tier, or
        // already resident and reserved), so one enforcement for all of them evicts the same pages
        // in the same order.
        // Only the pages still host-tier at entry land here: a page of this transfer that is already
        // resident (it landed via another handle) is skipped, as in the reference, even if the
        // enforcement below evicts it (the reference checks it before any of its evictions).
        std::set<int32_t> coming;
        for (int32_t p : tr.pages)
            if (tier(tr.layer, p) != 0) coming.insert(p);
        const int64_t incoming = static_cast<int64_t>(coming.size());
        if (incoming > 0) enforce_capacity(incoming);
        for (int32_t p : tr.pages) {
            PageState& ps = state(tr.layer, p);
            if (!coming.erase(p)) continue;
            set_tier(tr.layer, p, 0);
            ps.in_flight_done = 0;
            ps.reserved = true;
            ps.pinned = false;
            ps.lru = ++lru_counter;
            if (real()) queue_table(tr.layer, p);
        }
        tr.pages.clear();
        flush_table();
    }

    // Real mode: bring every host-tier page back into free device slots so the pool holds all
    // K/V and gradient data again once the engine detaches (the reference's engine only tags
    // pages, so its pool never loses them). All-or-nothing: ConfigError, and nothing moves, when
    // the pool has fewer free slots than host-tier pages.
    void restore_all() {
        if (!real()) return;
        sync_pages();
        size_t need_kv = 0, need_g = 0;
        for (int l = 0; l < pt->n_layers; ++l)
            for (size_t p = 0; p < pages[l].size(); ++p)
                if (tier(l, static_cast<int>(p)) == TIER_HOST && pages[l][p].in_flight_done <= 0) {
                    ++need_kv;
                    if (grads_allocated(l, static_cast<int>(p))) ++need_g;
                }
        OOMB_REQUIRE(need_kv <= pool->kv_free.size() && need_g <= pool->g_free.size(), OOMB_CONFIG_ERROR,
                     "restore_all: the pool has fewer free device slots than host-tier pages");
        for (int l = 0; l < pt->n_layers; ++l)
            for (size_t i = 0; i < pages[l].size(); ++i) {
                const int p = static_cast<int>(i);
                if (tier(l, p) != TIER_HOST) continue;
                PageState& ps = pages[l][i];
                if (ps.in_flight_done <= 0) real_fetch(l, p);  // an in-flight page already has its slots
                set_tier(l, p, 0);
                ps.in_flight_done = 0;
                queue_table(l, p);
            }
        flush_copies(0);
        cudaEvent_t done = new_event();
        OOMB_CUDA(cudaEventRecord(done, h2d_stream));
        OOMB_CUDA(cudaStreamWaitEvent(compute, done, 0));
        spare_events.push_back(done);
        flush_table();
    }

    void record_access(int layer, const int32_t* ids, int n, int chunk) {  // :256-264
        flush_table();
        cudaEvent_t ev = n > 0 ? stamp(ON_COMPUTE) : nullptr;
        for (int i = 0; i < n; ++i) {
            const int32_t p = ids[i];
            if (tier(layer, p) != 0) throw Error(OOMB_RESIDENCY_ERROR, "access to non-resident page " + std::to_string(p));
            state(layer, p).lru = ++lru_counter;
            push(EV_ACCESS, clock, layer, p, 0, chunk, ev);
        }
    }

    void advance_compute(double seconds, int chunk, int layer) {
        push(EV_COMPUTE_BEGIN, clock, layer, -1, 0, chunk, stamp(ON_COMPUTE));
        clock += seconds;
        push(EV_COMPUTE_END, clock, layer, -1, 0, chunk, stamp(ON_COMPUTE));
    }

    void end_layer_use(int layer, const int32_t* ids, int n) {  // :274-280
        for (int i = 0; i < n; ++i) {
            state(layer, ids[i]).reserved = false;
            state(layer, ids[i]).pinned = false;
        }
        enforce_capacity(0);
        flush_table();
    }

    // Real mode, at attach: the engine takes over pages the pool already holds. A device page
    // appended before the engine existed has no host copy yet (its first eviction must write it
    // back); a page tagged host without an engine (set_tier, as the reference's tests do before
    // constructing one) still has its data in device slots: it is written back now and its slots
    // are freed, so the page really lives in the host tier.
    void adopt_pool_pages() {
        sync_pages();
        bool wb = false;
        for (int l = 0; l < pt->n_layers; ++l)
            for (size_t i = 0; i < pages[l].size(); ++i) {
                const int p = static_cast<int>(i);
                PageState& ps = pages[l][i];
                const bool has_g = grads_allocated(l, p);
                if (tier(l, p) == TIER_DEVICE) {
                    ps.kv_host_valid = false;
                    ps.grad_host_valid = !has_g;
                } else if (tier(l, p) == TIER_HOST) {
                    if (pool->kvslot[l][p] >= 0) {
                        if (!wb) begin_writeback();
                        wb = true;
                        real_evict(l, p, true, has_g);
                        ps.kv_host_valid = true;
                        ps.grad_host_valid = true;
                    } else {
                        set_tier(l, p, TIER_LOST);  // no copy anywhere (cannot happen through this API)
                    }
                }
            }
        if (wb) end_writeback();
        flush_table();
    }

    void release_all() {
        for (auto& l : pages)
            for (auto& ps : l) {
                ps.reserved = false;
                ps.pinned = false;
            }
        enforce_capacity(0);
        flush_table();
    }

};

extern "C" {

// (internal, hidden) oomb_pool_destroy of a pool whose engine is still attached
// (internal, hidden) oomb_pool_reset with an engine attached: the pages are new, so are their states
void tier_on_pool_reset(oomb_tier_s* t) {
    for (auto& l : t->pages) l.clear();
}

void tier_orphan(oomb_tier_s* t) {
    t->orphaned = true;
    t->pt = nullptr;
    t->pool->victim_flush = nullptr;
    t->pool->victim_ctx = nullptr;
}

// (internal, hidden) the stream the engine orders its write-backs after and its fetch waits into
void* tier_compute_stream(oomb_tier_s* t) { return t->compute; }
// (internal) the event real-mode log timestamps are measured from
void* tier_t0(oomb_tier_s* t) { return t->t0; }

int oomb_tier_create_sim(oomb_pagetable_t pt, const oomb_tier_config* cfg, oomb_tier_t* out) {
    return guard([&] {
        OOMB_REQUIRE(cfg->bandwidth_bytes_per_s > 0, OOMB_CONFIG_ERROR, "tiered_memory: bandwidth must be positive");
        auto* t = new oomb_tier_s();
        t->cfg = *cfg;
        t->pt = &pt->pt;
        t->sync_pages();
        *out = t;
    });
}

int oomb_tier_create(oomb_pool_t pool, const oomb_tier_config* cfg, void* compute_stream, oomb_tier_t* out) {
    return guard([&] {
        set_dev(pool);
        OOMB_REQUIRE(cfg->bandwidth_bytes_per_s > 0, OOMB_CONFIG_ERROR, "tiered_memory: bandwidth must be positive");
        OOMB_REQUIRE(!pool->f64(), OOMB_CONFIG_ERROR, "tiered_memory: real page moves support fp32 / bf16 pools");
        auto* t = new oomb_tier_s();
        try {
            t->cfg = *cfg;
            t->pt = pool->pt;
            t->pool = pool;
            t->compute = S(compute_stream);
            // OOMB_TIER_PRIO=1: the copy streams at the highest priority, so the staged flushes'
            // scatter / gather CTAs take SMs ahead of the attention's queued CTAs; measured neutral at
            // c3 (profiles/r03_perf_notes.md), so default priority
            int prio_lo = 0, prio_hi = 0;
            OOMB_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
            const char* pe = std::getenv("OOMB_TIER_PRIO");
            const int prio = (pe && pe[0] == '1') ? prio_hi : 0;
            OOMB_CUDA(cudaStreamCreateWithPriority(&t->h2d_stream, cudaStreamNonBlocking, prio));
            OOMB_CUDA(cudaStreamCreateWithPriority(&t->d2h_stream, cudaStreamNonBlocking, prio));
            t->kv_block = 2 * static_cast<size_t>(pool->page_elems) * pool->elem;
            t->grad_block = 2 * static_cast<size_t>(pool->page_elems) * sizeof(float);
            const size_t n_host = static_cast<size_t>(pool->cfg.n_layers) * pool->max_pages;
            t->page_block = t->kv_block + t->grad_block;
            OOMB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&t->host_kv), n_host * t->page_block, cudaHostAllocDefault));
            t->host_grad = t->host_kv + t->kv_block;
            OOMB_CUDA(cudaEventCreate(&t->t0));
            OOMB_CUDA(cudaEventRecord(t->t0, t->compute));
            OOMB_REQUIRE(pool->engine == nullptr, OOMB_STATE_ERROR, "tiered_memory: the pool already has an engine");
            pool->enforce = true;  // the engine turns residency enforcement on (tiered_memory.hpp:102-108)
            pool->engine = t;
            if (const char* e = std::getenv("OOMB_TIER_LAZY_WB")) t->lazy_wb = e[0] != '0';
            if (const char* e = std::getenv("OOMB_TIER_CLEAN_AHEAD")) t->clean_ahead = std::atoll(e);
            pool->victim_ctx = t;
            pool->victim_flush = &oomb_tier_s::forced_flush;
            t->adopt_pool_pages();
        } catch (...) {
            oomb_tier_destroy(t);
            throw;
        }
        *out = t;
    });
}

int oomb_tier_destroy(oomb_tier_t t) {
    if (!t) return OOMB_OK;
    if (std::getenv("OOMB_TIER_DEBUG"))
        std::fprintf(stderr, "tier: best-effort %lld refused %lld | pages prefetched %lld on-demand %lld | "
                     "H2D waits: page write-back %lld, slot write-back %lld | compute-stream slot waits %lld | "
                     "forced victim flushes %lld, d2h moved %.2f GB\n",
                     (long long)t->dbg[0], (long long)t->dbg[1], (long long)t->dbg[2], (long long)t->dbg[3],
                     (long long)t->dbg[4], (long long)t->dbg[5],
                     (long long)(t->real() && !t->orphaned ? t->pool->compute_ticket_waits : -1),
                     (long long)t->forced_flushes, static_cast<double>(t->d2h_moved) / 1e9);
    if (t->real()) {
#ifndef OOMB_TIER_RESTORE_ON_DESTROY
#define OOMB_TIER_RESTORE_ON_DESTROY 1
#endif
        int64_t lost = 0;
        if (!t->orphaned) {
            cudaSetDevice(t->pool->device);
            if (OOMB_TIER_RESTORE_ON_DESTROY) {
                try {
                    t->restore_all();
                } catch (...) {
                }
            }
            // Pages still host-tier now (no room in the pool, or restore disabled) lose their data with
            // the pinned blocks freed below. They are tagged lost: every later read of their K/V or
            // gradients raises ResidencyError (pool.h check_ids), whether or not enforcement is on.
            try {
                t->sync_pages();
                for (int l = 0; l < t->pt->n_layers; ++l)
                    for (size_t i = 0; i < t->pages[l].size(); ++i)
                        if (t->tier(l, static_cast<int>(i)) == TIER_HOST) {
                            t->set_tier(l, static_cast<int>(i), TIER_LOST);
                            ++lost;
                        }
            } catch (...) {
            }
            cudaDeviceSynchronize();
            t->pool->enforce = false;
            t->pool->engine = nullptr;
            t->pool->victim_flush = nullptr;
            t->pool->victim_ctx = nullptr;
            t->pool->clear_holders();  // victim data dies with the engine's host blocks
        } else {
            cudaDeviceSynchronize();
        }
        if (lost > 0)
            g_last_error = "tier_destroy: " + std::to_string(lost) +
                           " host-tier page(s) could not be restored to the device (no free slots) and are marked "
                           "lost; reads of them raise ResidencyError";
        for (auto e : t->log_events) cudaEventDestroy(e);
        for (auto& tr : t->transfers)
            if (tr.ev) cudaEventDestroy(tr.ev);
        for (auto e : t->spare_events) cudaEventDestroy(e);
        if (t->t0) cudaEventDestroy(t->t0);
        if (t->h2d_stream) cudaStreamDestroy(t->h2d_stream);
        if (t->d2h_stream) cudaStreamDestroy(t->d2h_stream);
        cudaFreeHost(t->host_kv);  // host_grad points into the same allocation
        delete t;
        return lost > 0 ? OOMB_RESIDENCY_ERROR : OOMB_OK;
    }
    delete t;
    return OOMB_OK;
}

#define TIER_CALL(t, body)                                                                          \
    guard([&] {                                                                                     \
        OOMB_REQUIRE(!(t)->orphaned, OOMB_STATE_ERROR, "tiered_memory: the engine's pool was destroyed"); \
        if ((t)->real()) set_dev((t)->pool);                                                        \
        body;                                                                                       \
    })

int oomb_tier_begin_phase(oomb_tier_t t, int phase) { return TIER_CALL(t, t->phase = phase ? 1 : 0); }
int oomb_tier_set_prefetch_headroom(oomb_tier_t t, int64_t pages) { return TIER_CALL(t, t->headroom = pages); }
int oomb_tier_on_pages_appended(oomb_tier_t t, int layer, int64_t b, int64_t e) {
    return TIER_CALL(t, t->on_pages_appended(layer, b, e));
}
int oomb_tier_on_grads_scattered(oomb_tier_t t, int layer, const int32_t* ids, int n) {
    return TIER_CALL(t, for (int i = 0; i < n; ++i) t->state(layer, ids[i]).grad_host_valid = false);
}
int oomb_tier_fetch_async(oomb_tier_t t, int layer, const int32_t* ids, int n, int chunk, int best_effort,
                          int64_t* handle) {
    return TIER_CALL(t, *handle = t->fetch_async(layer, ids, n, chunk, best_effort != 0));
}
int oomb_tier_wait(oomb_tier_t t, int64_t handle) { return TIER_CALL(t, t->wait(handle)); }
int oomb_tier_record_access(oomb_tier_t t, int layer, const int32_t* ids, int n, int chunk) {
    return TIER_CALL(t, t->record_access(layer, ids, n, chunk));
}
int oomb_tier_advance_compute(oomb_tier_t t, double seconds, int chunk, int layer) {
    return TIER_CALL(t, t->advance_compute(seconds, chunk, layer));
}
int oomb_tier_end_layer_use(oomb_tier_t t, int layer, const int32_t* ids, int n) {
    return TIER_CALL(t, t->end_layer_use(layer, ids, n));
}
int oomb_tier_release_all(oomb_tier_t t) { return TIER_CALL(t, t->release_all()); }
int oomb_tier_restore_all(oomb_tier_t t) { return TIER_CALL(t, t->restore_all()); }

int oomb_tier_stats(oomb_tier_t t, double* out) {
    return guard([&] {
        out[0] = t->clock;
        out[1] = t->stall_s;
        out[2] = static_cast<double>(t->h2d_fwd);
        out[3] = static_cast<double>(t->h2d_bwd);
        out[4] = static_cast<double>(t->d2h);
    });
}

int oomb_tier_moved_bytes(oomb_tier_t t, int64_t* h2d_moved, int64_t* d2h_moved) {
    return guard([&] {
        *h2d_moved = static_cast<int64_t>(t->h2d_moved);
        if (d2h_moved) *d2h_moved = static_cast<int64_t>(t->d2h_moved);
    });
}

int oomb_tier_log(oomb_tier_t t, oomb_event* out, int64_t cap, int64_t* n) {
    return guard([&] {
        *n = static_cast<int64_t>(t->log.size());
        if (!out) return;
        if (t->real()) {
            set_dev(t->pool);
            OOMB_CUDA(cudaDeviceSynchronize());
        }
        for (int64_t i = 0; i < std::min(cap, *n); ++i) {
            out[i] = t->log[i].e;
            if (t->real() && t->log[i].ev) {
                float ms = 0.f;
                OOMB_CUDA(cudaEventElapsedTime(&ms, t->t0, t->log[i].ev));
                out[i].t = ms * 1e-3;
            }
        }
    });
}

// validate_schedule (tiered_memory.cpp:47-138)
int oomb_validate_schedule(const oomb_event* ev, int64_t n, double bw, double* out, int* n_viol, int64_t* viol_event,
                           int32_t* viol_code, int64_t viol_cap) {
    return guard([&] {
        struct Track {
            bool resident = false;
            double since = 0;
        };
        std::map<std::pair<int, int32_t>, Track> track;
        int viol = 0;
        int64_t cur = -1;
        auto violate = [&](int32_t code) {
            if (viol_event && viol_code && viol < viol_cap) {
                viol_event[viol] = cur;
                viol_code[viol] = code;
            }
            ++viol;
        };
        double last_compute_t = -1, prev_end = 0, begin_t = 0, busy = 0, stall = 0;
        bool in_compute = false;
        uint64_t transfer = 0, h2d_f = 0, h2d_b = 0, d2h_b = 0;
        for (int64_t i = 0; i < n; ++i) {
            const oomb_event& e = ev[i];
            cur = i;
            const auto key = std::make_pair(e.layer, e.page);
            switch (e.kind) {
                case EV_FETCH_ISSUED: break;
                case EV_FETCH_DONE:
                    track[key].resident = true;
                    track[key].since = e.t;
                    transfer += e.bytes;
                    if (e.phase == 0) h2d_f += e.bytes;
                    else h2d_b += e.bytes;
                    if (bw > 0) busy += static_cast<double>(e.bytes) / bw;
                    break;
                case EV_EVICT: {
                    auto it = track.find(key);
                    if (it == track.end() || !it->second.resident) violate(1);
                    else it->second.resident = false;
                    transfer += e.bytes;
                    d2h_b += e.bytes;
                    if (e.bytes > 0 && bw > 0) busy += static_cast<double>(e.bytes) / bw;
                    break;
                }
                case EV_ACCESS: {
                    auto it = track.find(key);
                    if (it == track.end() || !it->second.resident || it->second.since > e.t) violate(2);
                    break;
                }
                case EV_COMPUTE_BEGIN:
                    if (e.t < last_compute_t) violate(3);
                    last_compute_t = e.t;
                    if (in_compute) violate(4);
                    in_compute = true;
                    begin_t = e.t;
                    stall += std::max(0.0, e.t - prev_end);
                    break;
                case EV_COMPUTE_END:
                    if (!in_compute) violate(5);
                    if (e.t < begin_t) violate(6);
                    in_compute = false;
                    prev_end = e.t;
                    last_compute_t = e.t;
                    break;
            }
        }
        cur = -1;
        if (in_compute) violate(7);
        out[0] = stall;
        out[1] = static_cast<double>(transfer);
        out[2] = static_cast<double>(h2d_f);
        out[3] = static_cast<double>(h2d_b);
        out[4] = static_cast<double>(d2h_b);
        out[5] = busy > 0 ? std::clamp(1.0 - stall / busy, 0.0, 1.0) : 1.0;
        *n_viol = viol;
    });
}

}  // extern "C"
