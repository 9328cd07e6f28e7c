// SPDX-License-Identifier: Apache-2.0
//
// The attention layer's chunk-recurrent step as native code: the hot path's own call sequence of
// ChunkTrainer::train_step (chunk_trainer.hpp:131-186) restricted to one attention layer, so a
// whole 1M-token layer pass is one C call instead of ~10 host calls per chunk.
//
//   forward, chunks ascending (chunk_trainer.hpp:409-437):
//       select over the pages of earlier chunks (dense: all; local: recent window; top-k:
//       K_avg -> score_pages -> select_topk_row, :292-316) -> append_chunk -> attn_forward
//   backward, chunks descending (:531-592):
//       attn_backward (past-page dK/dV into the gradient pool) -> dM_i read-back of the chunk's
//       own pages into its dk_cur / dv_cur (:575-587)
//
// The dependencies the loop does NOT have are exploited exactly as bench.py's Python loop does
// (same results, bitwise): chunk i+1's selection reads only K_avg of chunks <= i, so it runs on a
// high-priority stream under chunk i's attention; consecutive chunks' forwards run on two streams
// (chunk i reads pages of chunks < i and its own k / v); each chunk's dQ is deferred
// (OOMB_ATTN_DEFER_DQ) so it overlaps the previous chunk's dK/dV, whose launches stay ordered.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <numeric>
#include <vector>

#include "oomb_internal.h"
#include "pool.h"

namespace oomb {
namespace {

// Streams, events, per-chunk selections and vote buffers of a pool's layer loop, kept across calls
// (pool->loop_state) so a step issues no allocation and no host synchronisation of its own.
struct LayerLoop {
    cudaStream_t sel = nullptr, att[2] = {nullptr, nullptr};
    cudaEvent_t ev_app[2] = {}, ev_sel[2] = {}, ev_att[2] = {};
    std::vector<oomb_selection_t> sels;
    int sel_ids = 0;  // id capacity of every selection
    void* votes[2] = {nullptr, nullptr};
    int64_t vote_bytes = 0;
    int fwd_chunks = 0;  // chunks of the last forward (their selections are kept for the backward)
    // engine path: host copies of selections and per-chunk residency records of the last step
    std::vector<int32_t> h_off, h_ids;
    std::vector<int64_t> stats;  // {phase, chunk, pages resident for the chunk, H2D bytes, D2H bytes}
    explicit LayerLoop(int device) {
        cudaSetDevice(device);
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        cudaStreamCreateWithPriority(&sel, cudaStreamNonBlocking, hi);  // selection ahead of the attention
        for (int i = 0; i < 2; ++i) {
            cudaStreamCreateWithFlags(&att[i], cudaStreamNonBlocking);
            cudaEventCreateWithFlags(&ev_app[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&ev_sel[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&ev_att[i], cudaEventDisableTiming);
        }
    }
    ~LayerLoop() {
        for (auto s : sels) oomb_selection_destroy(s);
        for (int i = 0; i < 2; ++i) {
            if (votes[i]) cudaFree(votes[i]);
            if (ev_app[i]) cudaEventDestroy(ev_app[i]);
            if (ev_sel[i]) cudaEventDestroy(ev_sel[i]);
            if (ev_att[i]) cudaEventDestroy(ev_att[i]);
            if (att[i]) cudaStreamDestroy(att[i]);
        }
        if (sel) cudaStreamDestroy(sel);
    }
};

void ok(int rc) {
    if (rc != OOMB_OK) throw Error(rc, oomb_last_error());
}

// Ascending distinct ids of a selection (waits for its host mirror): the chunk's residency working
// set (AttentionChunkLoop.union). `extra_from` >= 0 adds the m own pages extra_from.. (union1d).
std::vector<int32_t> sel_union(LayerLoop& L, oomb_selection_t s, int64_t extra_from = -1, int m = 0) {
    int mq = 0, nnz = 0;
    ok(oomb_selection_get_host(s, nullptr, nullptr, &mq, &nnz));
    L.h_off.resize(static_cast<size_t>(mq) + 1);
    L.h_ids.resize(static_cast<size_t>(std::max(nnz, 1)));
    ok(oomb_selection_get_host(s, L.h_off.data(), L.h_ids.data(), &mq, &nnz));
    std::vector<int32_t> u(L.h_ids.begin(), L.h_ids.begin() + nnz);
    for (int j = 0; extra_from >= 0 && j < m; ++j) u.push_back(static_cast<int32_t>(extra_from + j));
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    return u;
}

void tier_io(oomb_tier_t t, int64_t* h2d, int64_t* d2h) {
    double st[5];
    ok(oomb_tier_stats(t, st));
    *h2d = static_cast<int64_t>(st[2] + st[3]);
    *d2h = static_cast<int64_t>(st[4]);
}

}  // namespace
}  // namespace oomb

using namespace oomb;

extern "C" void* tier_compute_stream(oomb_tier_s* t);  // tier.cu (internal)
extern "C" void* tier_t0(oomb_tier_s* t);              // tier.cu (internal)

extern "C" int oomb_layer_step(oomb_pool_t p, int layer, int n_chunks, int mode, const void* q, int q_cycle,
                               const void* k, const void* v, const void* dout, int dout_cycle, void* out, void* lse,
                               void* dq, void* dk_cur, void* dv_cur, int64_t grad_stride_chunks, int flags,
                               void* stream) {
    return guard([&] {
        OOMB_REQUIRE(p != nullptr, OOMB_STATE_ERROR, "layer_step: null pool");
        OOMB_CUDA(cudaSetDevice(p->device));
        const oomb_config& c = p->cfg;
        OOMB_REQUIRE(n_chunks >= 1 && q_cycle >= 1 && dout_cycle >= 1, OOMB_SHAPE_ERROR, "layer_step: bad counts");
        OOMB_REQUIRE(mode >= OOMB_MODE_DENSE && mode <= OOMB_MODE_LOCAL, OOMB_CONFIG_ERROR, "layer_step: bad mode");
        oomb_tier_t eng = p->engine;
        OOMB_REQUIRE(eng == nullptr || tier_compute_stream(eng) == stream, OOMB_STATE_ERROR,
                     "layer_step: with a TieredEngine attached, `stream` must be the engine's compute stream");
        OOMB_REQUIRE(p->owner_stride == 1, OOMB_CONFIG_ERROR, "layer_step: page-range shards use the host loop");
        const int C = c.chunk_size, P = c.page_size, m = C / P;
        const int64_t qe = static_cast<int64_t>(C) * c.n_q_heads * c.head_dim;   // q / out / dout / dq per chunk
        const int64_t ke = static_cast<int64_t>(C) * c.n_kv_heads * c.head_dim;  // k / v / dk / dv per chunk
        const size_t el = static_cast<size_t>(p->elem), ae = static_cast<size_t>(p->aelem);
        auto at = [](const void* b, int64_t elems, size_t es) {
            return static_cast<const void*>(static_cast<const uint8_t*>(b) + elems * es);
        };
        auto atw = [](void* b, int64_t elems, size_t es) { return static_cast<void*>(static_cast<uint8_t*>(b) + elems * es); };
        cudaStream_t comp = S(stream);
        if (!p->loop_state) p->loop_state = std::shared_ptr<void>(new LayerLoop(p->device), [](void* x) {
            delete static_cast<LayerLoop*>(x);
        });
        LayerLoop& L = *static_cast<LayerLoop*>(p->loop_state.get());
        const int64_t max_pages = p->max_pages;
        const int k_sel = c.retrieval_budget / P;
        const int64_t per_qp = mode == OOMB_MODE_TOPK ? k_sel : mode == OOMB_MODE_LOCAL ? c.local_window : max_pages;
        const int need_ids = static_cast<int>(std::max<int64_t>(1, m * per_qp));
        if (need_ids > L.sel_ids) {  // (re)size the per-chunk selections
            for (auto s_ : L.sels) oomb_selection_destroy(s_);
            L.sels.clear();
            L.sel_ids = need_ids;
        }
        while (static_cast<int>(L.sels.size()) < n_chunks) {
            oomb_selection_t s_ = nullptr;
            ok(oomb_selection_create(p, m, L.sel_ids, &s_));
            L.sels.push_back(s_);
        }
        const int64_t vb = std::max<int64_t>(1, m * max_pages) * static_cast<int64_t>(ae);
        if (mode == OOMB_MODE_TOPK && vb > L.vote_bytes) {
            for (int i = 0; i < 2; ++i) {
                if (L.votes[i]) OOMB_CUDA(cudaFree(L.votes[i]));
                OOMB_CUDA(cudaMalloc(&L.votes[i], vb));
            }
            L.vote_bytes = vb;
        }

        if (flags & OOMB_LAYER_BACKWARD_ONLY) {
            OOMB_REQUIRE(L.fwd_chunks >= n_chunks, OOMB_STATE_ERROR,
                         "layer_step: backward-only needs this pool's forward of the same chunks first");
            if (!eng) goto backward;
        }
        if (!(flags & OOMB_LAYER_BACKWARD_ONLY)) L.stats.clear();
        if (eng) {
            // ---- forward under the residency protocol (AttentionChunkLoop.forward_chunk with an engine;
            // chunk_trainer.hpp:328-363, 409-462): the selection of chunk i+1 is issued on the side
            // stream right after chunk i's append; every fetch decision waits for the selection's ids.
            // The attention runs on the engine's compute stream, which its write-backs follow.
            auto fwd_engine = [&] {
                ok(oomb_tier_begin_phase(eng, 0));
                OOMB_CUDA(cudaEventRecord(L.ev_app[1], comp));
                OOMB_CUDA(cudaStreamWaitEvent(L.sel, L.ev_app[1], 0));
                auto select = [&](int i) {
                    const void* qi = at(q, (i % q_cycle) * qe, el);
                    const int n_cand = i * m;
                    if (mode == OOMB_MODE_TOPK && n_cand > 0)
                        ok(oomb_select_pages_topk(p, layer, qi, C, n_cand, L.sels[i], L.votes[i & 1], L.sel));
                    else if (mode == OOMB_MODE_LOCAL && n_cand > 0)
                        ok(oomb_select_recent(L.sels[i], n_cand, c.local_window, m, L.sel));
                    else
                        ok(oomb_select_all(L.sels[i], n_cand, m, L.sel));
                    OOMB_CUDA(cudaEventRecord(L.ev_sel[i & 1], L.sel));
                };
                select(0);
                for (int i = 0; i < n_chunks; ++i) {
                    const void* qi = at(q, (i % q_cycle) * qe, el);
                    const void* ki = at(k, i * ke, el);
                    const void* vi = at(v, i * ke, el);
                    OOMB_CUDA(cudaStreamWaitEvent(comp, L.ev_sel[i & 1], 0));
                    int64_t h0 = 0, d0 = 0, h1 = 0, d1 = 0, hnd = 0, hnd2 = 0;
                    tier_io(eng, &h0, &d0);
                    std::vector<int32_t> ids = sel_union(L, L.sels[i]);
                    const int n_ids = static_cast<int>(ids.size());
                    ok(oomb_tier_fetch_async(eng, layer, ids.data(), n_ids, i, 0, &hnd));
                    int64_t b = 0, e = 0;
                    ok(oomb_append_chunk(p, layer, ki, vi, C, comp, &b, &e));
                    if (i + 1 < n_chunks) {
                        OOMB_CUDA(cudaEventRecord(L.ev_app[i & 1], comp));
                        OOMB_CUDA(cudaStreamWaitEvent(L.sel, L.ev_app[i & 1], 0));
                        select(i + 1);
                    }
                    ok(oomb_tier_on_pages_appended(eng, layer, b, e));
                    ok(oomb_tier_wait(eng, hnd));
                    ok(oomb_tier_fetch_async(eng, layer, ids.data(), n_ids, i, 0, &hnd2));
                    ok(oomb_tier_wait(eng, hnd2));
                    ok(oomb_tier_record_access(eng, layer, ids.data(), n_ids, i));
                    ok(oomb_attn_forward_ex(p, layer, qi, C, L.sels[i], ki, vi, atw(out, i * qe, el),
                                            atw(lse, static_cast<int64_t>(i) * C * c.n_q_heads, ae), 0, comp));
                    for (int j = 0; j < m; ++j) ids.push_back(static_cast<int32_t>(i * m + j));
                    ok(oomb_tier_end_layer_use(eng, layer, ids.data(), static_cast<int>(ids.size())));
                    tier_io(eng, &h1, &d1);
                    L.stats.insert(L.stats.end(), {0, i, n_ids, h1 - h0, d1 - d0});
                }
                OOMB_CUDA(cudaEventRecord(L.ev_sel[0], L.sel));
                OOMB_CUDA(cudaStreamWaitEvent(comp, L.ev_sel[0], 0));
                L.fwd_chunks = n_chunks;
            };
            auto bwd_engine = [&] {  // AttentionChunkLoop.begin_backward + backward_chunk with an engine
                ok(oomb_tier_release_all(eng));
                ok(oomb_tier_begin_phase(eng, 1));
                // OOMB_LOOP_TIMELINE=<file>: every chunk's backward start / end on the compute stream in ms
                // from the engine log's origin (diagnostics of the copy / compute overlap)
                const char* tl_path = std::getenv("OOMB_LOOP_TIMELINE");
                std::vector<cudaEvent_t> tl;
                std::vector<double> th;  // host ms: fetch + wait + record_access, prefetch, attn_backward, rest
                auto now_ms = [] {
                    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
                        .count();
                };
                auto mark = [&] {
                    if (!tl_path) return;
                    tl.emplace_back();
                    OOMB_CUDA(cudaEventCreate(&tl.back()));
                    OOMB_CUDA(cudaEventRecord(tl.back(), comp));
                };
                for (int i = n_chunks - 1; i >= 0; --i) {
                    const int64_t gi = grad_stride_chunks ? i : 0;
                    void* dki = atw(dk_cur, gi * ke, ae);
                    void* dvi = atw(dv_cur, gi * ke, ae);
                    int64_t h0 = 0, d0 = 0, h1 = 0, d1 = 0, hnd = 0, pend = 0;
                    const double hs0 = tl_path ? now_ms() : 0;
                    tier_io(eng, &h0, &d0);
                    std::vector<int32_t> ids = sel_union(L, L.sels[i], static_cast<int64_t>(i) * m, m);
                    ok(oomb_tier_fetch_async(eng, layer, ids.data(), static_cast<int>(ids.size()), i, 0, &hnd));
                    ok(oomb_tier_wait(eng, hnd));
                    ok(oomb_tier_record_access(eng, layer, ids.data(), static_cast<int>(ids.size()), i));
                    const double hs1 = tl_path ? now_ms() : 0;
                    if (i > 0) {  // step-ahead prefetch: cached ids of the next (earlier) chunk + its own pages
                        std::vector<int32_t> nxt = sel_union(L, L.sels[i - 1], static_cast<int64_t>(i - 1) * m, m);
                        ok(oomb_tier_fetch_async(eng, layer, nxt.data(), static_cast<int>(nxt.size()), i - 1, 1, &pend));
                    }
                    const double hs2 = tl_path ? now_ms() : 0;
                    mark();
                    ok(oomb_attn_backward_readback(p, layer, at(dout, (i % dout_cycle) * qe, el),
                                               at(q, (i % q_cycle) * qe, el), C, L.sels[i], at(k, i * ke, el),
                                               at(v, i * ke, el), at(out, i * qe, el),
                                               at(lse, static_cast<int64_t>(i) * C * c.n_q_heads, ae),
                                               atw(dq, gi * qe, ae), dki, dvi, 0, static_cast<int64_t>(i) * m,
                                               comp));  // + the dM_i read-back
                    mark();
                    const double hs3 = tl_path ? now_ms() : 0;
                    std::vector<int32_t> su = sel_union(L, L.sels[i]);
                    ok(oomb_tier_on_grads_scattered(eng, layer, su.data(), static_cast<int>(su.size())));
                    ok(oomb_tier_end_layer_use(eng, layer, ids.data(), static_cast<int>(ids.size())));
                    tier_io(eng, &h1, &d1);
                    L.stats.insert(L.stats.end(), {1, i, static_cast<int64_t>(ids.size()), h1 - h0, d1 - d0});
                    if (tl_path) th.insert(th.end(), {hs1 - hs0, hs2 - hs1, hs3 - hs2, now_ms() - hs3});
                }
                if (tl_path) {
                    OOMB_CUDA(cudaStreamSynchronize(comp));
                    auto t0 = static_cast<cudaEvent_t>(tier_t0(eng));
                    if (FILE* f = std::fopen(tl_path, "w")) {
                        for (size_t j = 0; j + 1 < tl.size(); j += 2) {
                            float ta = 0, tb = 0;
                            cudaEventElapsedTime(&ta, t0, tl[j]);
                            cudaEventElapsedTime(&tb, t0, tl[j + 1]);
                            const double* h = th.data() + 4 * (j / 2);
                            std::fprintf(f, "%d %.4f %.4f %.4f %.4f %.4f %.4f\n", n_chunks - 1 - static_cast<int>(j / 2),
                                         ta, tb, h[0], h[1], h[2], h[3]);
                        }
                        std::fclose(f);
                    }
                    for (auto e_ : tl) cudaEventDestroy(e_);
                }
            };
            if (!(flags & OOMB_LAYER_BACKWARD_ONLY)) fwd_engine();
            if (!(flags & OOMB_LAYER_FORWARD_ONLY)) bwd_engine();
            return;
        }
        {  // ---- forward (a block: the backward-only goto skips it whole)
        // OOMB_LOOP_HOSTPROF=1: host microseconds spent issuing each part of the forward (stderr)
        static const bool host_prof = std::getenv("OOMB_LOOP_HOSTPROF") != nullptr;
        double hp[4] = {0, 0, 0, 0};  // select, append, attn_forward, events
        auto hnow = [] {
            return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
        };
        double ht = host_prof ? hnow() : 0;
        auto hmark = [&](int k) {
            if (!host_prof) return;
            const double t = hnow();
            hp[k] += t - ht;
            ht = t;
        };
        OOMB_CUDA(cudaEventRecord(L.ev_app[1], comp));  // earlier work precedes this step's selections
        OOMB_CUDA(cudaStreamWaitEvent(L.sel, L.ev_app[1], 0));
        for (int i = 0; i < 2; ++i) OOMB_CUDA(cudaStreamWaitEvent(L.att[i], L.ev_app[1], 0));
        for (int i = 0; i < n_chunks; ++i) {
            const void* qi = at(q, (i % q_cycle) * qe, el);
            const void* ki = at(k, i * ke, el);
            const void* vi = at(v, i * ke, el);
            const int n_cand = i * m;
            if (i > 0) OOMB_CUDA(cudaStreamWaitEvent(L.sel, L.ev_app[(i - 1) & 1], 0));  // K_avg of chunks < i
            hmark(3);
            if (mode == OOMB_MODE_TOPK && n_cand > 0)
                ok(oomb_select_pages_topk(p, layer, qi, C, n_cand, L.sels[i], L.votes[i & 1], L.sel));
            else if (mode == OOMB_MODE_LOCAL && n_cand > 0)
                ok(oomb_select_recent(L.sels[i], n_cand, c.local_window, m, L.sel));
            else
                ok(oomb_select_all(L.sels[i], n_cand, m, L.sel));
            hmark(0);
            OOMB_CUDA(cudaEventRecord(L.ev_sel[i & 1], L.sel));
            hmark(3);
            int64_t b = 0, e = 0;
            ok(oomb_append_chunk(p, layer, ki, vi, C, comp, &b, &e));
            hmark(1);
            OOMB_CUDA(cudaEventRecord(L.ev_app[i & 1], comp));
            cudaStream_t a = L.att[i & 1];
            OOMB_CUDA(cudaStreamWaitEvent(a, L.ev_app[i & 1], 0));
            OOMB_CUDA(cudaStreamWaitEvent(a, L.ev_sel[i & 1], 0));
            hmark(3);
            ok(oomb_attn_forward_ex(p, layer, qi, C, L.sels[i], ki, vi, atw(out, i * qe, el),
                                    atw(lse, static_cast<int64_t>(i) * C * c.n_q_heads, ae), 0, a));
            hmark(2);
        }
        if (host_prof)
            std::fprintf(stderr, "layer_step forward host us: select %.1f append %.1f attn_forward %.1f events %.1f (%d chunks)\n",
                         hp[0], hp[1], hp[2], hp[3], n_chunks);
        for (int i = 0; i < 2; ++i) {
            OOMB_CUDA(cudaEventRecord(L.ev_att[i], L.att[i]));
            OOMB_CUDA(cudaStreamWaitEvent(comp, L.ev_att[i], 0));
        }
        OOMB_CUDA(cudaEventRecord(L.ev_sel[0], L.sel));
        OOMB_CUDA(cudaStreamWaitEvent(comp, L.ev_sel[0], 0));
        L.fwd_chunks = n_chunks;
        if (flags & OOMB_LAYER_FORWARD_ONLY) return;
        }

    backward:  // ---- backward (dQ deferred: chunk i's dQ overlaps chunk i-1's dK/dV)
        for (int i = n_chunks - 1; i >= 0; --i) {
            const int64_t gi = grad_stride_chunks ? i : 0;
            const void* qi = at(q, (i % q_cycle) * qe, el);
            const void* di = at(dout, (i % dout_cycle) * qe, el);
            void* dqi = atw(dq, gi * qe, ae);
            void* dki = atw(dk_cur, gi * ke, ae);
            void* dvi = atw(dv_cur, gi * ke, ae);
            // dQ deferred; the dM_i read-back of the chunk's own pages runs in the dK/dV kernel's store
            ok(oomb_attn_backward_readback(p, layer, di, qi, C, L.sels[i], at(k, i * ke, el), at(v, i * ke, el),
                                           at(out, i * qe, el), at(lse, static_cast<int64_t>(i) * C * c.n_q_heads, ae),
                                           dqi, dki, dvi, OOMB_ATTN_DEFER_DQ, static_cast<int64_t>(i) * m, comp));
        }
        ok(oomb_attn_join_dq(p, comp));
    });
}

extern "C" int oomb_layer_stats(oomb_pool_t p, int64_t* out, int64_t cap, int64_t* n) {
    return guard([&] {
        OOMB_REQUIRE(p != nullptr && n != nullptr, OOMB_STATE_ERROR, "layer_stats: null argument");
        const auto* L = static_cast<const LayerLoop*>(p->loop_state.get());
        const int64_t recs = L ? static_cast<int64_t>(L->stats.size() / 5) : 0;
        *n = recs;
        if (out)
            for (int64_t r = 0; r < std::min(recs, cap); ++r)
                for (int j = 0; j < 5; ++j) out[r * 5 + j] = L->stats[static_cast<size_t>(r * 5 + j)];
    });
}
