// SPDX-License-Identifier: Apache-2.0
//
// C++ facade tests (include/oomb.hpp). They read like the reference's own Catch2 suites
// (/root/reference/proj/tests/test_attention.cpp, test_paged_kv.cpp, test_tiered_memory.cpp):
// the same calls with the same arguments, through the facade instead of the CPU templates.
// The checker is the C oracle (oracle/oomb_oracle.c, test infrastructure only).
//
//   test_facade cpu   host-only cases (config, errors, page table, simulated TieredEngine,
//                     validate_schedule); no CUDA device needed.
//   test_facade gpu   device cases: score/select known answers, fwd/bwd against the oracle in
//                     fp32 (1e-5) and bf16 on the tcgen05 shape (2e-2), replay, residency.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "oomb.hpp"

// ---- oracle (oracle/oomb_oracle.c)
extern "C" {
struct OcCache;
int oc_cache_new(int real_bytes, int n_layers, int kv_heads, int head_dim, int page_size, OcCache** out);
void oc_cache_free(OcCache* c);
int oc_cache_page_table(const OcCache* c, int layer, int32_t* out);
int oc_cache_n_pages(const OcCache* c, int layer);
int oc_append_f32(OcCache* c, int layer, const float* k, const float* v, int64_t rows, int64_t* b, int64_t* e);
int oc_scatter_f32(OcCache* c, int layer, const int32_t* ids, int n, const float* dk, const float* dv);
int oc_gather_f32(const OcCache* c, int layer, const int32_t* ids, int n, int grads, float* k, float* v,
                  uint8_t* valid);
int oc_attn_forward_f32(OcCache* c, int layer, int n_q_heads, const float* q, int64_t C, const int32_t* sel_off,
                        const int32_t* sel_ids, int64_t m, const float* k_cur, const float* v_cur, float* out,
                        float* lse);
int oc_attn_backward_f32(OcCache* c, int layer, int n_q_heads, const float* dout, const float* q, int64_t C,
                         const int32_t* sel_off, const int32_t* sel_ids, int64_t m, const float* k_cur,
                         const float* v_cur, const float* saved_out, const float* saved_lse, float* dq, float* dk_cur,
                         float* dv_cur);
}

namespace {

using namespace oomb;

int g_failed = 0, g_checks = 0;
std::string g_case;

#define CHECK(cond)                                                                                    \
    do {                                                                                               \
        ++g_checks;                                                                                    \
        if (!(cond)) {                                                                                 \
            ++g_failed;                                                                                \
            std::fprintf(stderr, "FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond);  \
        }                                                                                              \
    } while (0)

template <class E>
bool throws(const std::function<void()>& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

void run_case(const char* name, const std::function<void()>& f) {
    g_case = name;
    const int before = g_failed;
    try {
        f();
    } catch (const std::exception& e) {
        ++g_failed;
        std::fprintf(stderr, "FAIL [%s] unexpected exception: %s\n", name, e.what());
    }
    std::printf("%s %s\n", g_failed == before ? "ok  " : "FAIL", name);
}

std::vector<float> randn(int64_t n, std::mt19937_64& rng, float sd = 1.0f) {
    std::normal_distribution<float> d(0.f, sd);
    std::vector<float> v(static_cast<size_t>(n));
    for (auto& x : v) x = d(rng);
    return v;
}
std::vector<float> bf16_round(std::vector<float> v) {
    for (auto& x : v) x = bf16_to_f32(f32_to_bf16(x));
    return v;
}
double rel_l2(const std::vector<float>& a, const std::vector<float>& b) {  // tensor.hpp:157-163
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += (static_cast<double>(a[i]) - b[i]) * (static_cast<double>(a[i]) - b[i]);
        den += static_cast<double>(b[i]) * b[i];
    }
    return std::sqrt(num) / std::max(std::sqrt(den), 1e-30);
}

ModelConfig attn_config() {  // the reference test geometry (test_attention.cpp attn_config)
    ModelConfig cfg;
    cfg.n_layers = 1;
    cfg.n_q_heads = 4;
    cfg.n_kv_heads = 2;
    cfg.head_dim = 8;
    cfg.page_size = 4;
    cfg.chunk_size = 8;
    cfg.retrieval_budget = 8;
    return cfg;
}

// ============================================================================ CPU cases
void cpu_cases() {
    run_case("ModelConfig::validate rejects what config.cpp rejects", [] {
        ModelConfig ok;
        ok.validate();
        auto bad = [](auto mut) {
            ModelConfig c;
            mut(c);
            return throws<ConfigError>([&] { c.validate(); });
        };
        CHECK(bad([](ModelConfig& c) { c.n_kv_heads = 3; }));
        CHECK(bad([](ModelConfig& c) { c.head_dim = 7; }));
        CHECK(bad([](ModelConfig& c) { c.chunk_size = 60; }));
        CHECK(bad([](ModelConfig& c) { c.retrieval_budget = 10; }));
        CHECK(bad([](ModelConfig& c) { c.rope_base = 1.0; }));
        CHECK(bad([](ModelConfig& c) { c.attention_mode = {AttentionMode::dense, AttentionMode::topk, AttentionMode::local}; }));
        CHECK(ok.gqa_group() == 2 && ok.pages_per_chunk() == 4 && ok.budget_pages() == 8);
    });
    run_case("C ABI statuses map onto the reference exception classes", [] {
        oomb_config c{};  // all zero: invalid before any device call
        oomb_pool_t p = nullptr;
        CHECK(throws<ConfigError>([&] { check(oomb_pool_create(&c, 0, &p)); }));
        CHECK(std::string(oomb_last_error()).size() > 0);
        CHECK(throws<ShapeError>([] { select_recent(4, -1); }));
        CHECK(throws<StateError>([] { throw_status(OOMB_STATE_ERROR, "x"); }));
        CHECK(throws<ResidencyError>([] { throw_status(OOMB_RESIDENCY_ERROR, "x"); }));
        CHECK(throws<IoError>([] { throw_status(OOMB_IO_ERROR, "x"); }));
        CHECK(throws<Error>([] { throw_status(OOMB_CUDA_ERROR, "x"); }));
    });
    run_case("select_recent / select_all windows (test_attention.cpp:106-110)", [] {
        CHECK(select_recent(10, 3) == (std::vector<int32_t>{7, 8, 9}));
        CHECK(select_recent(2, 5) == (std::vector<int32_t>{0, 1}));
        CHECK(select_recent(4, 0).empty());
        CHECK(select_all(3) == (std::vector<int32_t>{0, 1, 2}));
    });
    run_case("bf16 conversion rounds to nearest even", [] {
        CHECK(f32_to_bf16(1.0f) == 0x3f80);
        CHECK(bf16_to_f32(f32_to_bf16(1.0f + 1.0f / 256)) == 1.0f);          // tie -> even (down)
        CHECK(bf16_to_f32(f32_to_bf16(1.0f + 3.0f / 256)) == 1.0f + 4.0f / 256);  // tie -> even (up)
        CHECK(std::isnan(bf16_to_f32(f32_to_bf16(std::nanf("")))));
    });
    run_case("page table: arena ids and lazy grad pages equal the oracle's", [] {
        const int L = 2, P = 4, H = 2, D = 8;
        HostPageTable pt(L, P, H, D);
        OcCache* oc = nullptr;
        CHECK(oc_cache_new(4, L, H, D, P, &oc) == 0);
        std::mt19937_64 rng(5);
        const int64_t rows_seq[] = {6, 3, 9, 1};
        for (int i = 0; i < 4; ++i) {
            const int layer = i % L;
            const int64_t rows = rows_seq[i];
            auto k = randn(rows * H * D, rng), v = randn(rows * H * D, rng);
            SlotRange r = pt.append_chunk(layer, rows);
            int64_t b = 0, e = 0;
            oc_append_f32(oc, layer, k.data(), v.data(), rows, &b, &e);
            CHECK(r.begin == b && r.end == e);
        }
        const std::vector<int32_t> ids{2, 0};
        pt.scatter_add_grads(0, ids);
        std::vector<float> g(ids.size() * P * H * D, 1.0f);
        oc_scatter_f32(oc, 0, ids.data(), 2, g.data(), g.data());
        for (int layer = 0; layer < L; ++layer) {
            CHECK(pt.n_pages(layer) == oc_cache_n_pages(oc, layer));
            std::vector<int32_t> ref(static_cast<size_t>(4) * oc_cache_n_pages(oc, layer));
            oc_cache_page_table(oc, layer, ref.data());
            CHECK(pt.page_table(layer) == ref);
        }
        const MemoryReport rep = pt.memory_report();
        CHECK(rep.pages == pt.n_pages(0) + pt.n_pages(1));
        CHECK(rep.grad_bytes == 2ull * 2 * P * H * D * 4);
        CHECK(rep.reallocs == 0 && rep.copied_bytes == 0);
        oc_cache_free(oc);
    });
    run_case("TieredEngine (simulated) keeps capacity, logs a valid schedule", [] {
        const int P = 4, H = 1, D = 8;
        HostPageTable pt(1, P, H, D);
        TierConfig tc;
        tc.device_capacity_pages = 4;
        tc.bandwidth_bytes_per_s = 1e9;
        TieredEngine eng(pt, tc);
        eng.begin_phase(Phase::forward);
        for (int chunk = 0; chunk < 4; ++chunk) {
            SlotRange r = pt.append_chunk(0, 2 * P);
            eng.on_pages_appended(0, r);
            const int n = pt.n_pages(0);
            std::vector<int32_t> ids;
            for (int p = std::max(0, n - 4); p < n - 2; ++p) ids.push_back(p);
            if (!ids.empty()) {
                TransferHandle h = eng.fetch_async(0, ids, chunk);
                eng.wait(h);
                eng.record_access(0, ids, chunk);
            }
            eng.advance_compute(1e-6, chunk, 0);
            std::vector<int32_t> own{n - 2, n - 1};
            eng.end_layer_use(0, own);
            if (!ids.empty()) eng.end_layer_use(0, ids);
        }
        const ScheduleLog log = eng.log();
        CHECK(!log.events.empty());
        CHECK(eng.h2d_bytes(Phase::forward) > 0);
        CHECK(eng.d2h_bytes() > 0);  // appended pages are dirty: evicting them writes back
        const ValidationReport rep = validate_schedule(log);
        CHECK(rep.violations.empty());
        CHECK(rep.transfer_bytes == eng.h2d_bytes(Phase::forward) + eng.h2d_bytes(Phase::backward) + eng.d2h_bytes());
        CHECK(rep.overlap_fraction >= 0.0 && rep.overlap_fraction <= 1.0);
    });
    run_case("validate_schedule reports the reference's violation messages", [] {
        ScheduleLog log{1e9, {}};
        log.events.push_back({EventKind::access, 0.0, 0, 3, 0, 0, Phase::forward});
        log.events.push_back({EventKind::evict, 1.0, 0, 5, 0, 0, Phase::forward});
        log.events.push_back({EventKind::compute_begin, 2.0, 0, -1, 0, 0, Phase::forward});
        const ValidationReport rep = validate_schedule(log);
        CHECK(rep.violations.size() == 3);
        CHECK(rep.violations.size() > 0 &&
              rep.violations[0].rfind("access before fetch_done (or after evict): layer=0 page=3", 0) == 0);
        CHECK(rep.violations.size() > 1 && rep.violations[1].rfind("evict of non-resident page layer=0 page=5", 0) == 0);
        CHECK(rep.violations.size() > 2 && rep.violations[2] == "unterminated compute segment");
    });
}

// ============================================================================ GPU cases
struct Csr {
    std::vector<int32_t> off, ids;
};
Csr to_csr(const PageLists& l) {
    Csr c;
    c.off.push_back(0);
    for (const auto& x : l) {
        c.ids.insert(c.ids.end(), x.begin(), x.end());
        c.off.push_back(static_cast<int32_t>(c.ids.size()));
    }
    return c;
}

// One chunk after `past_pages` pages of history through the facade (host-Tensor overloads, the
// reference's own signatures) and through the oracle; returns max rel-L2 over every output.
double chunk_vs_oracle(const ModelConfig& cfg, DType dt, int past_pages, int k_pages, uint64_t seed,
                       bool device_path) {
    std::mt19937_64 rng(seed);
    const int P = cfg.page_size, H = cfg.n_kv_heads, Hq = cfg.n_q_heads, D = cfg.head_dim, C = cfg.chunk_size;
    auto rnd = [&](int64_t n) { return dt == DType::bf16 ? bf16_round(randn(n, rng)) : randn(n, rng); };
    const int64_t past_rows = static_cast<int64_t>(past_pages) * P;
    auto kp = rnd(past_rows * H * D), vp = rnd(past_rows * H * D);
    auto q = rnd(static_cast<int64_t>(C) * Hq * D), kc = rnd(static_cast<int64_t>(C) * H * D),
         vc = rnd(static_cast<int64_t>(C) * H * D), dout = rnd(static_cast<int64_t>(C) * Hq * D);

    PagedCache cache(cfg, dt, past_rows + C);
    OcCache* oc = nullptr;
    oc_cache_new(4, cfg.n_layers, H, D, P, &oc);
    if (past_rows) {
        cache.append_chunk(0, Tensor<float>({past_rows, H, D}, kp), Tensor<float>({past_rows, H, D}, vp));
        int64_t b, e;
        oc_append_f32(oc, 0, kp.data(), vp.data(), past_rows, &b, &e);
    }
    // a fixed pseudo-random selection of k_pages pages per query page (ascending)
    const int m = C / P;
    PageLists sel(static_cast<size_t>(m));
    for (int qp = 0; qp < m; ++qp) {
        std::vector<int32_t> all = select_all(past_pages);
        std::shuffle(all.begin(), all.end(), rng);
        all.resize(static_cast<size_t>(std::min(k_pages, past_pages)));
        std::sort(all.begin(), all.end());
        sel[qp] = all;
    }
    const Csr csr = to_csr(sel);
    std::vector<float> ro(q.size()), rl(static_cast<size_t>(C) * Hq), rdq(q.size()), rdk(kc.size()), rdv(vc.size());
    oc_attn_forward_f32(oc, 0, Hq, q.data(), C, csr.off.data(), csr.ids.data(), m, kc.data(), vc.data(), ro.data(),
                        rl.data());
    // each side's backward consumes its own forward's saved O / LSE, as the reference's does
    double err = 0;
    std::vector<float> out, lse, dq, dk, dv;
    if (device_path) {  // DeviceTensor API: the B200 path without host round trips per call
        auto dq_t = DeviceTensor::from_host(std::vector<int64_t>{C, Hq, D}, q.data(), dt);
        auto saved = attn_forward(cfg, dq_t, cache, 0, Selection::from_lists(cache, sel),
                                  DeviceTensor::from_host(std::vector<int64_t>{C, H, D}, kc.data(), dt),
                                  DeviceTensor::from_host(std::vector<int64_t>{C, H, D}, vc.data(), dt));
        auto g = attn_backward(cfg, DeviceTensor::from_host(std::vector<int64_t>{C, Hq, D}, dout.data(), dt), dq_t,
                               cache, 0, DeviceTensor::from_host(std::vector<int64_t>{C, H, D}, kc.data(), dt),
                               DeviceTensor::from_host(std::vector<int64_t>{C, H, D}, vc.data(), dt), saved);
        out = saved.out.to_host(), lse = saved.lse.to_host();
        dq = g.dq.to_host(), dk = g.dk_cur.to_host(), dv = g.dv_cur.to_host();
    } else {  // the reference's own signatures on host tensors
        auto saved = attn_forward(cfg, Tensor<float>({C, Hq, D}, q), cache, 0, sel, Tensor<float>({C, H, D}, kc),
                                  Tensor<float>({C, H, D}, vc));
        CHECK(saved.selected == sel);
        auto g = attn_backward(cfg, Tensor<float>({C, Hq, D}, dout), Tensor<float>({C, Hq, D}, q), cache, 0,
                               Tensor<float>({C, H, D}, kc), Tensor<float>({C, H, D}, vc), saved);
        out = saved.out.data, lse = saved.lse.data, dq = g.dq.data, dk = g.dk_cur.data, dv = g.dv_cur.data;
    }
    oc_attn_backward_f32(oc, 0, Hq, dout.data(), q.data(), C, csr.off.data(), csr.ids.data(), m, kc.data(), vc.data(),
                         ro.data(), rl.data(), rdq.data(), rdk.data(), rdv.data());
    err = std::max({rel_l2(out, ro), rel_l2(lse, rl), rel_l2(dq, rdq), rel_l2(dk, rdk), rel_l2(dv, rdv)});
    if (past_pages) {  // the gradient pool of the selected pages
        const std::vector<int32_t> ids = select_all(past_pages);
        Gathered gg = cache.gather_grad_pages(0, ids);
        std::vector<float> gk_ref(static_cast<size_t>(past_rows) * H * D), gv_ref(gk_ref.size());
        std::vector<uint8_t> valid(static_cast<size_t>(past_rows));
        oc_gather_f32(oc, 0, ids.data(), past_pages, 1, gk_ref.data(), gv_ref.data(), valid.data());
        err = std::max({err, rel_l2(gg.k.to_host(), gk_ref), rel_l2(gg.v.to_host(), gv_ref)});
        std::vector<int32_t> ref_pt(static_cast<size_t>(4) * past_pages);  // page table bit-exact
        oc_cache_page_table(oc, 0, ref_pt.data());
        CHECK(cache.page_table(0) == ref_pt);
    }
    oc_cache_free(oc);
    return err;
}

void gpu_cases() {
    run_case("score_pages matches the reference softmax on a one-token case (test_attention.cpp:54-64)", [] {
        Tensor<double> q({1, 1, 2}, {1.0, 0.0});
        Tensor<double> k_avg({2, 1, 2}, {1.0, 0.0, 0.0, 1.0});
        auto score = score_pages(q, k_avg, /*page_size=*/8, /*gqa_group=*/1);
        CHECK(score.dim(0) == 1 && score.dim(1) == 2);
        CHECK(std::abs(score.data[0] - 0.731058578) < 1e-6);
        CHECK(std::abs(score.data[1] - 0.268941421) < 1e-6);
    });
    run_case("score_pages: identical representatives give uniform votes (test_attention.cpp:66-83)", [] {
        std::mt19937_64 rng(1);
        const int page = 4;
        auto qv = randn(2 * page * 2 * 8, rng);
        Tensor<double> q({2 * page, 2, 8}, std::vector<double>(qv.begin(), qv.end()));
        Tensor<double> k_avg({3, 1, 8});
        for (int p = 0; p < 3; ++p)
            for (int j = 0; j < 8; ++j) k_avg.data[p * 8 + j] = 0.37 * j;
        auto score = score_pages(q, k_avg, page, /*gqa_group=*/2);
        CHECK(score.dim(0) == 2 && score.dim(1) == 3);
        for (double s : score.data) CHECK(std::abs(s - page * 2 / 3.0) < 1e-5);
    });
    run_case("select_topk budget arithmetic, ties, and degeneracy (test_attention.cpp:94-112)", [] {
        std::vector<double> scores{5.0, 5.0, 1.0};
        CHECK(select_topk(scores, 1) == std::vector<int32_t>{0});
        CHECK(select_topk(scores, 7) == (std::vector<int32_t>{0, 1, 2}));
        CHECK(select_topk(scores, 0).empty());
        std::vector<double> s2{0.1, 9.0, 3.0, 7.0, 0.2};
        CHECK(select_topk(s2, 3) == (std::vector<int32_t>{1, 2, 3}));
        CHECK(throws<ShapeError>([&] { select_topk(s2, -1); }));
    });
    run_case("single token with no past attends only itself (test_attention.cpp:120-135)", [] {
        ModelConfig cfg = attn_config();
        cfg.chunk_size = cfg.page_size;
        PagedCache cache(cfg, DType::f32, cfg.chunk_size);
        std::mt19937_64 rng(3);
        Tensor<float> q({1, cfg.n_q_heads, cfg.head_dim}, randn(cfg.n_q_heads * cfg.head_dim, rng));
        Tensor<float> k({1, cfg.n_kv_heads, cfg.head_dim}, randn(cfg.n_kv_heads * cfg.head_dim, rng));
        Tensor<float> v({1, cfg.n_kv_heads, cfg.head_dim}, randn(cfg.n_kv_heads * cfg.head_dim, rng));
        auto saved = attn_forward(cfg, q, cache, 0, {{}}, k, v);
        for (int h = 0; h < cfg.n_q_heads; ++h)
            for (int j = 0; j < cfg.head_dim; ++j)
                CHECK(std::abs(saved.out.data[h * cfg.head_dim + j] - v.data[(h / cfg.gqa_group()) * cfg.head_dim + j]) <
                      1e-6);
    });
    run_case("attn_forward rejects a selection of the wrong length", [] {
        ModelConfig cfg = attn_config();
        PagedCache cache(cfg, DType::f32, 64);
        Tensor<float> q({cfg.chunk_size, cfg.n_q_heads, cfg.head_dim});
        Tensor<float> k({cfg.chunk_size, cfg.n_kv_heads, cfg.head_dim});
        CHECK(throws<ShapeError>([&] { attn_forward(cfg, q, cache, 0, {{}}, k, k); }));
    });
    run_case("fp32 forward + backward + grad pages match the oracle within 1e-5 (host Tensor API)", [] {
        const double e = chunk_vs_oracle(attn_config(), DType::f32, 6, 2, 11, false);
        std::printf("     rel_l2 %.3g\n", e);
        CHECK(e < 1e-5);
    });
    run_case("bf16 tcgen05 shape (hd 128, P 128, 28/4 heads) matches the oracle within 2e-2 (DeviceTensor API)", [] {
        ModelConfig cfg;
        cfg.n_layers = 1, cfg.n_q_heads = 28, cfg.n_kv_heads = 4, cfg.head_dim = 128;
        cfg.page_size = 128, cfg.chunk_size = 256, cfg.retrieval_budget = 256;
        const double e = chunk_vs_oracle(cfg, DType::bf16, 5, 2, 12, true);
        std::printf("     rel_l2 %.3g\n", e);
        CHECK(e < 2e-2);
    });
    run_case("forward replay is bitwise identical (test_attention.cpp:207-226)", [] {
        ModelConfig cfg;
        cfg.n_layers = 1, cfg.n_q_heads = 28, cfg.n_kv_heads = 4, cfg.head_dim = 128;
        cfg.page_size = 128, cfg.chunk_size = 256, cfg.retrieval_budget = 256;
        PagedCache cache(cfg, DType::bf16, 1024);
        std::mt19937_64 rng(13);
        auto kv = DeviceTensor::from_host(std::vector<int64_t>{512, 4, 128}, randn(512 * 4 * 128, rng).data(), DType::bf16);
        cache.append_chunk(0, kv, kv);
        auto q = DeviceTensor::from_host(std::vector<int64_t>{256, 28, 128}, randn(256 * 28 * 128, rng).data(), DType::bf16);
        auto kc = DeviceTensor::from_host(std::vector<int64_t>{256, 4, 128}, randn(256 * 4 * 128, rng).data(), DType::bf16);
        Selection sel = select_pages_topk(cache, 0, q, cache.n_pages(0));
        auto a = attn_forward(cfg, q, cache, 0, sel, kc, kc);
        auto b = attn_forward(cfg, q, cache, 0, sel, kc, kc);
        CHECK(a.out.to_host() == b.out.to_host());
        CHECK(a.lse.to_host() == b.lse.to_host());
        CHECK(sel.lists().size() == 2 && sel.lists()[0].size() == 2);
    });
    run_case("a page tagged host under enforcement raises ResidencyError (paged_kv.hpp:301-312)", [] {
        ModelConfig cfg = attn_config();
        PagedCache cache(cfg, DType::f32, 64);
        std::mt19937_64 rng(14);
        const int64_t rows = 2 * cfg.page_size;
        Tensor<float> k({rows, cfg.n_kv_heads, cfg.head_dim}, randn(rows * cfg.n_kv_heads * cfg.head_dim, rng));
        cache.append_chunk(0, k, k);
        cache.set_tier(0, 1, Tier::host);
        CHECK(cache.tier(0, 1) == Tier::host);
        cache.set_residency_enforced(true);
        const std::vector<int32_t> ids{0, 1};
        CHECK(throws<ResidencyError>([&] { cache.gather_pages(0, ids); }));
        cache.set_residency_enforced(false);
        Gathered g = cache.gather_pages(0, ids);
        CHECK(g.k.to_host() == k.data);
    });
}

}  // namespace

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "cpu";
    if (mode == "cpu" || mode == "all") cpu_cases();
    if (mode == "gpu" || mode == "all") gpu_cases();
    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed == 0 ? 0 : 1;
}
