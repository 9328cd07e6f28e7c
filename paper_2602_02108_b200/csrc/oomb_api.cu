// SPDX-License-Identifier: Apache-2.0
//
// Host runtime behind include/oomb.h: the device page pool, the host mirror of
// the reference page table (arena ids, LIFO free list, lazy gradient pages),
// selections (device CSR + pinned host mirror), and dispatch to the sm_100a
// kernels. Every entry point catches and converts exceptions to oomb_status.

#include <map>
#include <tuple>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "pool.h"

namespace oomb {

thread_local std::string g_last_error;
thread_local Profiler* g_prof = nullptr;

const double* rope_inv_freq_table(float base, int hd) {
    static std::mutex mu;
    static std::map<std::tuple<int, float, int>, double*> tables;
    int dev = 0;
    OOMB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_tuple(dev, base, hd);
    auto it = tables.find(key);
    if (it != tables.end()) return it->second;
    std::vector<double> h(static_cast<size_t>(hd / 2));
    for (int i = 0; i < hd / 2; ++i)
        h[static_cast<size_t>(i)] = std::pow(static_cast<double>(base), -2.0 * static_cast<double>(i) / static_cast<double>(hd));
    double* d = nullptr;
    OOMB_CUDA(cudaMalloc(reinterpret_cast<void**>(&d), h.size() * sizeof(double)));
    OOMB_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
    tables[key] = d;
    return d;
}

namespace {
struct TraceReq {
    std::string tag, path;
    long index = -1;
    std::map<std::string, long> counts;
    std::string pending_path;
};
TraceReq& trace_req() {
    static TraceReq r = [] {
        TraceReq t;
        if (const char* e = getenv("OOMB_CTA_TRACE")) {
            std::string v(e);
            const size_t a = v.find(':'), b = v.find(':', a + 1);
            if (a != std::string::npos && b != std::string::npos) {
                t.tag = v.substr(0, a);
                t.index = std::stol(v.substr(a + 1, b - a - 1));
                t.path = v.substr(b + 1);
            }
        }
        return t;
    }();
    return r;
}
}  // namespace

CtaTrace trace_begin(const char* tag, size_t n_ctas, int slots) {
    TraceReq& r = trace_req();
    CtaTrace t;
    if (r.index < 0 || r.tag != tag) return t;
    if (r.counts[tag]++ != r.index) return t;
    OOMB_CUDA(cudaMalloc(reinterpret_cast<void**>(&t.buf), n_ctas * slots * sizeof(unsigned long long)));
    OOMB_CUDA(cudaMemset(t.buf, 0, n_ctas * slots * sizeof(unsigned long long)));
    t.slots = slots;
    return t;
}

void trace_end(CtaTrace& t, size_t n_ctas, cudaStream_t st) {
    if (!t.buf) return;
    OOMB_CUDA(cudaStreamSynchronize(st));
    std::vector<unsigned long long> h(n_ctas * t.slots);
    OOMB_CUDA(cudaMemcpy(h.data(), t.buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(trace_req().path.c_str(), "wb")) {
        const int64_t hdr[2] = {static_cast<int64_t>(n_ctas), t.slots};
        fwrite(hdr, sizeof(hdr), 1, f);
        fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
        fclose(f);
    }
    cudaFree(t.buf);
    t.buf = nullptr;
}

// ---------------------------------------------------------------------------
// cuTensorMapEncodeTiled through the runtime's driver entry point.
// ---------------------------------------------------------------------------
CUresult encode_tensor_map(CUtensorMap* map, CUtensorMapDataType dt, uint32_t rank, void* base, const uint64_t* dims,
                           const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw Error(OOMB_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    uint32_t estr[5] = {1, 1, 1, 1, 1};
    return fn(map, dt, rank, base, dims, strides_bytes, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

namespace {

void validate_cfg(const oomb_config& c) {  // ModelConfig::validate (config.cpp:30-51), path subset
    auto req = [](bool ok, const char* m) {
        if (!ok) throw Error(OOMB_CONFIG_ERROR, std::string("config: ") + m);
    };
    req(c.n_layers >= 1, "n_layers must be >= 1");
    req(c.n_q_heads >= 1 && c.n_kv_heads >= 1, "head counts must be >= 1");
    req(c.n_q_heads % c.n_kv_heads == 0, "n_q_heads must be divisible by n_kv_heads");
    req(c.head_dim >= 2 && c.head_dim % 2 == 0, "head_dim must be even (rotary pairs)");
    req(c.page_size >= 1, "page_size must be >= 1");
    req(c.chunk_size >= 1, "chunk_size must be >= 1");
    req(c.chunk_size % c.page_size == 0, "chunk_size must be divisible by page_size");
    req(c.retrieval_budget >= 0, "retrieval_budget must be >= 0");
    req(c.retrieval_budget % c.page_size == 0, "retrieval_budget must be divisible by page_size");
    req(c.local_window >= 0, "local_window must be >= 0");
    req(c.dtype == OOMB_F32 || c.dtype == OOMB_BF16 || c.dtype == OOMB_F64, "dtype must be OOMB_F32, OOMB_BF16 or OOMB_F64");
    req(c.head_dim <= 256, "head_dim must be <= 256");
    req(c.max_tokens >= 1, "max_tokens must be >= 1");
}


int32_t pop_slot(oomb_pool_s* p, bool grad, const char* what) {
    OOMB_REQUIRE(!(grad ? p->g_free : p->kv_free).empty(), OOMB_CONFIG_ERROR,
                 std::string("device ") + what + " capacity exhausted (raise device_capacity_pages or offload)");
    return p->pop_free(grad);
}

// Copy a small host int32 array into a stream-ordered temporary device buffer.
int32_t* upload_ids(const int32_t* host, int n, cudaStream_t st) {
    int32_t* d = nullptr;
    OOMB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), std::max(n, 1) * sizeof(int32_t), st));
    if (n > 0) OOMB_CUDA(cudaMemcpyAsync(d, host, n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    return d;
}

AttnGeom geom(oomb_pool_s* p, int64_t tokens, int layer) {
    AttnGeom g{};
    g.C = static_cast<int>(tokens);
    g.Hq = p->cfg.n_q_heads;
    g.Hkv = p->cfg.n_kv_heads;
    g.hd = p->cfg.head_dim;
    g.P = p->cfg.page_size;
    g.group = g.Hq / g.Hkv;
    g.m = static_cast<int>((tokens + g.P - 1) / g.P);
    g.filled = p->pt->filled[layer];
    g.scale = 1.0f / std::sqrt(static_cast<float>(g.hd));
    g.scale64 = 1.0 / std::sqrt(static_cast<double>(g.hd));
    g.max_pages = static_cast<int>(p->max_pages);
    g.chunk_keys = 1;
    return g;
}

void sel_host_sync(oomb_selection_s* s) {
    if (s->host_pending) {
        OOMB_CUDA(cudaEventSynchronize(s->ev));
        s->host_pending = false;
    }
    if (s->nnz_from_host) {
        s->nnz = s->h_off[s->m];
        s->nnz_from_host = false;
    }
}

// Lazy grad pages for every list of the selection, reference order (qp asc, list order).
void ensure_grad_pages(oomb_pool_s* p, int layer, const int32_t* h_off, const int32_t* h_ids, int m, cudaStream_t st) {
    std::vector<int32_t> pages, slots;
    for (int qp = 0; qp < m; ++qp) {
        const int n = h_off[qp + 1] - h_off[qp];
        if (n == 0) continue;
        p->pt->check_ids(layer, h_ids + h_off[qp], n, p->enforce, "scatter_add_grads");
        for (int32_t pid : p->pt->scatter(layer, h_ids + h_off[qp], n)) {
            const int32_t gs = pop_slot(p, true, "gradient page");
            p->compute_ticket_waits += p->wait_slot(true, gs, st);
            p->gslot[layer][pid] = gs;
            pages.push_back(pid);
            slots.push_back(gs);
        }
    }
    if (pages.empty()) return;
    const int n = static_cast<int>(pages.size());
    int32_t* d = nullptr;
    OOMB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), 2 * n * sizeof(int32_t), st));
    std::vector<int32_t> both(pages);
    both.insert(both.end(), slots.begin(), slots.end());
    OOMB_CUDA(cudaMemcpyAsync(d, both.data(), 2 * n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    launch_grad_init(d, d + n, n, p->gslot_layer(layer), p->gkpool, p->gvpool, p->page_elems, st, p->aelem);
    OOMB_CUDA(cudaFreeAsync(d, st));
}

bool use_tc(oomb_pool_s* p, const AttnGeom& g) {
    if (p->policy == 1) return false;
    const bool ok = tc_supported(g, p->cfg.dtype) && p->maps.valid;
    OOMB_REQUIRE(p->policy != 2 || ok, OOMB_CONFIG_ERROR, "tcgen05 kernels do not support this shape/dtype");
    return ok;
}

}  // namespace
}  // namespace oomb

using namespace oomb;

extern "C" {

const char* oomb_last_error(void) { return g_last_error.c_str(); }
int oomb_version(void) { return 1; }
int64_t oomb_kernel_launches(void) { return g_kernel_launches.load(); }

// ---------------------------------------------------------------------------
// page table host logic
// ---------------------------------------------------------------------------
int oomb_pagetable_create(int n_layers, int page_size, int n_kv_heads, int head_dim, int kv_elem_bytes,
                          int grad_elem_bytes, oomb_pagetable_t* out) {
    return guard([&] {
        OOMB_REQUIRE(n_layers >= 1 && page_size >= 1 && n_kv_heads >= 1 && head_dim >= 1, OOMB_CONFIG_ERROR,
                     "pagetable: bad geometry");
        *out = new oomb_pagetable_s{PageTable(n_layers, page_size, n_kv_heads, head_dim, kv_elem_bytes,
                                              grad_elem_bytes)};
    });
}
int oomb_pagetable_destroy(oomb_pagetable_t pt) {
    delete pt;
    return OOMB_OK;
}
int oomb_pagetable_append(oomb_pagetable_t pt, int layer, int64_t rows, int64_t* b, int64_t* e) {
    return guard([&] {
        int fn, nn;
        pt->pt.append(layer, rows, b, e, &fn, &nn);
    });
}
int oomb_pagetable_scatter(oomb_pagetable_t pt, int layer, const int32_t* ids, int n) {
    return guard([&] {
        pt->pt.check_ids(layer, ids, n, false, "scatter_add_grads");
        pt->pt.scatter(layer, ids, n);
    });
}
int oomb_pagetable_reset(oomb_pagetable_t pt) {
    return guard([&] { pt->pt.reset(); });
}
int oomb_pagetable_n_pages(oomb_pagetable_t pt, int layer, int* n) {
    return guard([&] {
        pt->pt.check_layer(layer);
        *n = static_cast<int>(pt->pt.pages[layer].size());
    });
}
int oomb_pagetable_get(oomb_pagetable_t pt, int layer, int32_t* out) {
    return guard([&] {
        pt->pt.check_layer(layer);
        const auto& st = pt->pt.pages[layer];
        for (size_t i = 0; i < st.size(); ++i) {
            out[4 * i + 0] = st[i].k;
            out[4 * i + 1] = st[i].v;
            out[4 * i + 2] = st[i].gk;
            out[4 * i + 3] = st[i].gv;
        }
    });
}
int oomb_pagetable_set_tier(oomb_pagetable_t pt, int layer, int page, int tier) {
    return guard([&] {
        pt->pt.check_layer(layer);
        OOMB_REQUIRE(page >= 0 && page < static_cast<int>(pt->pt.pages[layer].size()), OOMB_SHAPE_ERROR,
                     "set_tier: page out of range");
        pt->pt.pages[layer][page].tier = tier ? 1 : 0;
    });
}
int oomb_pagetable_memory_report(oomb_pagetable_t pt, oomb_memory_report* out) {
    return guard([&] { *out = pt->pt.report(); });
}

// ---------------------------------------------------------------------------
// pool lifecycle
// ---------------------------------------------------------------------------
int oomb_pool_create(const oomb_config* cfg, int device, oomb_pool_t* out) {
    return guard([&] {
        validate_cfg(*cfg);
        auto* p = new oomb_pool_s();
        try {
            p->cfg = *cfg;
            p->device = device;
            OOMB_CUDA(cudaSetDevice(device));
            {  // stream-ordered scratch (scoring workspace, id lists) is reused chunk after chunk: keep
               // freed blocks in the device's default pool instead of unmapping them at every sync
                cudaMemPool_t mp;
                OOMB_CUDA(cudaDeviceGetDefaultMemPool(&mp, device));
                uint64_t keep = UINT64_MAX;
                OOMB_CUDA(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep));
            }
            const auto& c = p->cfg;
            p->max_pages = (c.max_tokens + c.page_size - 1) / c.page_size;
            OOMB_REQUIRE(c.dtype == OOMB_F32 || c.dtype == OOMB_BF16 || c.dtype == OOMB_F64, OOMB_CONFIG_ERROR,
                         "dtype must be OOMB_F32, OOMB_BF16 or OOMB_F64");
            p->elem = c.dtype == OOMB_BF16 ? 2 : c.dtype == OOMB_F64 ? 8 : 4;
            p->aelem = c.dtype == OOMB_F64 ? 8 : 4;
            p->page_elems = static_cast<int64_t>(c.page_size) * c.n_kv_heads * c.head_dim;
            p->pt = new PageTable(c.n_layers, c.page_size, c.n_kv_heads, c.head_dim, p->elem, p->aelem);
            OOMB_REQUIRE(c.page_owner_stride >= 0 && (c.page_owner_stride <= 1 ||
                                                     (c.page_owner_rank >= 0 && c.page_owner_rank < c.page_owner_stride)),
                         OOMB_CONFIG_ERROR, "page_owner_rank must be in [0, page_owner_stride)");
            p->owner_stride = std::max(1, c.page_owner_stride);
            p->owner_rank = p->owner_stride > 1 ? c.page_owner_rank : 0;
            const int64_t owned_pages = (p->max_pages + p->owner_stride - 1) / p->owner_stride;
            p->n_kv_slots = c.device_capacity_pages > 0 ? c.device_capacity_pages : c.n_layers * owned_pages;
            p->n_g_slots = p->n_kv_slots;
            // FIFO (pool.h): slot 0 is handed out first.
            for (int64_t i = 0; i < p->n_kv_slots; ++i) p->kv_free.push_back(static_cast<int32_t>(i));
            for (int64_t i = 0; i < p->n_g_slots; ++i) p->g_free.push_back(static_cast<int32_t>(i));
            p->kvslot.assign(c.n_layers, std::vector<int32_t>(p->max_pages, -1));
            p->gslot.assign(c.n_layers, std::vector<int32_t>(p->max_pages, -1));
            const size_t kv_bytes = static_cast<size_t>(p->n_kv_slots) * p->page_elems * p->elem;
            const size_t g_bytes = static_cast<size_t>(p->n_g_slots) * p->page_elems * p->aelem;
            OOMB_CUDA(cudaMalloc(&p->kpool, kv_bytes));
            OOMB_CUDA(cudaMalloc(&p->vpool, kv_bytes));
            OOMB_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->gkpool), g_bytes));
            OOMB_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->gvpool), g_bytes));
            const size_t tab = static_cast<size_t>(c.n_layers) * p->max_pages * sizeof(int32_t);
            OOMB_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->d_kvslot), tab));
            OOMB_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->d_gslot), tab));
            OOMB_CUDA(cudaMemset(p->d_kvslot, 0xFF, tab));
            OOMB_CUDA(cudaMemset(p->d_gslot, 0xFF, tab));
            const size_t ks = static_cast<size_t>(c.n_layers) * p->max_pages * c.n_kv_heads * c.head_dim;
            OOMB_CUDA(cudaMalloc(&p->d_kavg_sum, ks * p->aelem));
            OOMB_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->d_kavg_cnt), tab));
            OOMB_CUDA(cudaMemset(p->d_kavg_sum, 0, ks * p->aelem));
            OOMB_CUDA(cudaMemset(p->d_kavg_cnt, 0, tab));
            if (c.dtype == OOMB_BF16 && c.head_dim == 128 && c.page_size % 128 == 0) {  // the tcgen05 scorer's shape
                p->plane_stride = (p->max_pages + 127) / 128 * 128;
                const size_t pb = static_cast<size_t>(c.n_layers) * 2 * c.n_kv_heads * p->plane_stride * c.head_dim * 2;
                OOMB_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->d_kavg_planes), pb));
                OOMB_CUDA(cudaMemset(p->d_kavg_planes, 0, pb));
            }
            OOMB_CUDA(cudaMalloc(reinterpret_cast<void**>(&p->d_err), sizeof(int)));
            OOMB_CUDA(cudaMemset(p->d_err, 0, sizeof(int)));
            if (c.dtype == OOMB_BF16 && (c.head_dim == 128 || c.head_dim == 64) &&
                (c.page_size % 128 == 0 || c.page_size == 64))
                make_pool_maps(p->maps, p->kpool, p->vpool, p->n_kv_slots, p->gkpool, p->gvpool, p->n_g_slots,
                               c.n_kv_heads, c.page_size, c.head_dim);
        } catch (...) {
            oomb_pool_destroy(p);
            throw;
        }
        *out = p;
    });
}

void tier_orphan(oomb_tier_s* t);  // tier.cu
void tier_on_pool_reset(oomb_tier_s* t);  // tier.cu

int oomb_pool_destroy(oomb_pool_t p) {
    if (!p) return OOMB_OK;
    cudaSetDevice(p->device);
    cudaDeviceSynchronize();
    p->loop_state.reset();  // the layer loop's selections refer to the pool
    if (p->engine) tier_orphan(p->engine);  // an engine outliving its pool frees only its own memory
    cudaFree(p->kpool);
    cudaFree(p->vpool);
    cudaFree(p->gkpool);
    cudaFree(p->gvpool);
    cudaFree(p->d_kvslot);
    cudaFree(p->d_gslot);
    cudaFree(p->d_kavg_sum);
    cudaFree(p->d_kavg_cnt);
    cudaFree(p->d_kavg_planes);
    cudaFree(p->d_err);
    for (int b = 0; b < 2; ++b) {
        cudaFree(p->bwd_ws[b]);
        if (p->bwd_ev_dq[b]) cudaEventDestroy(p->bwd_ev_dq[b]);
    }
    if (p->bwd_ev_prep) cudaEventDestroy(p->bwd_ev_prep);
    if (p->bwd_side) cudaStreamDestroy(p->bwd_side);
    p->destroy_writeback_events();
    for (auto& r : p->prof.recs) {
        cudaEventDestroy(r.e0);
        cudaEventDestroy(r.e1);
    }
    for (auto e : p->prof.spare) cudaEventDestroy(e);
    delete p->pt;
    delete p;
    return OOMB_OK;
}

int oomb_pool_reset(oomb_pool_t p, void* stream) {
    return guard([&] {
        set_dev(p);
        for (int l = 0; l < p->cfg.n_layers; ++l) {
            for (int64_t pg = 0; pg < static_cast<int64_t>(p->pt->pages[l].size()); ++pg) {
                if (p->kvslot[l][pg] >= 0) p->kv_free.push_back(p->kvslot[l][pg]);
                if (p->gslot[l][pg] >= 0) p->g_free.push_back(p->gslot[l][pg]);
                p->kvslot[l][pg] = -1;
                p->gslot[l][pg] = -1;
            }
        }
        p->pt->reset();
        p->clear_holders();  // freed slots hold no page of the new sequence
        if (p->engine) tier_on_pool_reset(p->engine);
        const size_t tab = static_cast<size_t>(p->cfg.n_layers) * p->max_pages * sizeof(int32_t);
        OOMB_CUDA(cudaMemsetAsync(p->d_kvslot, 0xFF, tab, S(stream)));
        OOMB_CUDA(cudaMemsetAsync(p->d_gslot, 0xFF, tab, S(stream)));
        OOMB_CUDA(cudaMemsetAsync(p->d_kavg_cnt, 0, tab, S(stream)));
    });
}

int oomb_zero_grad_pages(oomb_pool_t p, void* stream) {
    return guard([&] {
        set_dev(p);
        std::vector<int32_t> slots;
        for (int l = 0; l < p->cfg.n_layers; ++l)
            for (size_t pg = 0; pg < p->pt->pages[l].size(); ++pg)
                if (p->gslot[l][pg] >= 0) slots.push_back(p->gslot[l][pg]);
        if (slots.empty()) return;
        int32_t* d = upload_ids(slots.data(), static_cast<int>(slots.size()), S(stream));
        launch_zero_slots(d, static_cast<int>(slots.size()), p->gkpool, p->gvpool, p->page_elems, S(stream), p->aelem);
        OOMB_CUDA(cudaFreeAsync(d, S(stream)));
    });
}

int oomb_memory_report_get(oomb_pool_t p, oomb_memory_report* out) {
    return guard([&] { *out = p->pt->report(); });
}

int oomb_check_device_errors(oomb_pool_t p) {
    return guard([&] {
        set_dev(p);
        int h = 0;
        OOMB_CUDA(cudaDeviceSynchronize());
        OOMB_CUDA(cudaMemcpy(&h, p->d_err, sizeof(int), cudaMemcpyDeviceToHost));
        OOMB_CUDA(cudaMemset(p->d_err, 0, sizeof(int)));
        OOMB_REQUIRE(!(h & DERR_BAD_ID), OOMB_SHAPE_ERROR, "kernel read a page id out of range");
        OOMB_REQUIRE(!(h & DERR_NOT_RESIDENT), OOMB_RESIDENCY_ERROR, "kernel read a page that is not device-resident");
    });
}

int oomb_set_kernel_policy(oomb_pool_t p, int policy) {
    return guard([&] {
        OOMB_REQUIRE(policy >= 0 && policy <= 2, OOMB_CONFIG_ERROR, "policy must be 0, 1 or 2");
        p->policy = policy;
    });
}

// ---------------------------------------------------------------------------
// page table ops
// ---------------------------------------------------------------------------
static int append_impl(oomb_pool_t p, int layer, const void* k, const void* v, int64_t rows, void* stream,
                       int64_t* slot_begin, int64_t* slot_end, float rope_base) {
    return guard([&] {
        set_dev(p);
        p->pt->check_layer(layer);
        const int P = p->cfg.page_size;
        OOMB_REQUIRE(p->pt->filled[layer] + rows <= p->max_pages * P, OOMB_CONFIG_ERROR,
                     "append_chunk: layer capacity (max_tokens) exceeded");
        const double* inv_freq = rope_base > 0.f ? rope_inv_freq_table(rope_base, p->cfg.head_dim) : nullptr;
        int64_t b, e;
        int first_new, n_new;
        const int64_t filled0 = p->pt->filled[layer];
        if (rows > 0 && filled0 % P != 0) {  // rows land in the partly filled tail page: it must be here
            const int tail = static_cast<int>(filled0 / P);
            const uint8_t t = p->pt->pages[layer][tail].tier;
            OOMB_REQUIRE(t == TIER_REMOTE || (t == TIER_DEVICE && p->kvslot[layer][tail] >= 0), OOMB_RESIDENCY_ERROR,
                         "append_chunk: the partly filled tail page " + std::to_string(tail) + " of layer " +
                             std::to_string(layer) + " is not device-resident (fetch it before appending)");
        }
        {  // every new page this shard stores needs a free slot: check before touching the page table
            const int64_t n_before = static_cast<int64_t>(p->pt->pages[layer].size());
            const int64_t last = rows > 0 ? (filled0 + rows - 1) / P : n_before - 1;
            int64_t need = 0;
            for (int64_t pg = n_before; pg <= last; ++pg) need += p->owns(pg);
            OOMB_REQUIRE(need <= static_cast<int64_t>(p->kv_free.size()), OOMB_CONFIG_ERROR,
                         "device KV page capacity exhausted (raise device_capacity_pages or offload)");
        }
        p->pt->append(layer, rows, &b, &e, &first_new, &n_new);
        for (int i = 0; i < n_new; ++i) {
            const int pg = first_new + i;
            if (!p->owns(pg)) {  // another page-range shard stores it; K_avg sums are kept here too
                p->kvslot[layer][pg] = SLOT_REMOTE;
                p->pt->pages[layer][pg].tier = TIER_REMOTE;
                continue;
            }
            const int32_t s = pop_slot(p, false, "KV page");
            p->compute_ticket_waits += p->wait_slot(false, s, S(stream));  // a recycled slot may still be draining
            p->kvslot[layer][pg] = s;
        }
        *slot_begin = b;
        *slot_end = e;
        // Launch in segments that create at most 100 new pages each.
        const int64_t re = static_cast<int64_t>(p->cfg.n_kv_heads) * p->cfg.head_dim;
        int64_t done = 0;
        int published = first_new;  // first new page whose slot is not yet in d_kvslot
        while (done < rows) {
            const int64_t seg = std::min<int64_t>(rows - done, static_cast<int64_t>(100) * P);
            const int64_t f = filled0 + done;
            const int first_page = static_cast<int>(f / P);
            const int last_page = static_cast<int>((f + seg - 1) / P);
            NewSlots ns{};
            ns.first_page = std::max(first_page, published);
            ns.n = 0;
            for (int pg = ns.first_page; pg <= last_page; ++pg) ns.slot[ns.n++] = p->kvslot[layer][pg];
            const char* kb = static_cast<const char*>(k) + done * re * p->elem;
            const char* vb = static_cast<const char*>(v) + done * re * p->elem;
            launch_append(p->cfg.dtype, kb, vb, seg, f, P, p->cfg.n_kv_heads, p->cfg.head_dim, first_page,
                          last_page - first_page + 1, ns, p->kvslot_layer(layer), p->kpool, p->vpool,
                          p->kavg_sum_layer(layer), p->kavg_cnt_layer(layer), p->d_err, S(stream), inv_freq,
                          p->kavg_planes_layer(layer), p->plane_stride);
            published = std::max(published, last_page + 1);
            done += seg;
        }
    });
}

int oomb_append_chunk(oomb_pool_t p, int layer, const void* k, const void* v, int64_t rows, void* stream,
                      int64_t* slot_begin, int64_t* slot_end) {
    return append_impl(p, layer, k, v, rows, stream, slot_begin, slot_end, 0.f);
}
int oomb_append_chunk_rope(oomb_pool_t p, int layer, const void* k_raw, const void* v, int64_t rows, float rope_base,
                           void* stream, int64_t* slot_begin, int64_t* slot_end) {
    const int rc = guard([&] {
        OOMB_REQUIRE(rope_base > 0.f, OOMB_CONFIG_ERROR, "append_chunk_rope: rope base must be positive");
        OOMB_REQUIRE(p->cfg.dtype != OOMB_F64, OOMB_CONFIG_ERROR, "append_chunk_rope: fp32 / bf16 pools");
    });
    if (rc != OOMB_OK) return rc;
    return append_impl(p, layer, k_raw, v, rows, stream, slot_begin, slot_end, rope_base);
}
int oomb_rope(const void* x, int64_t rows, int heads, int hd, int64_t pos_offset, float base, int sign, int in_dtype,
              int out_dtype, void* out, void* stream) {
    return guard([&] {
        OOMB_REQUIRE(rows >= 0 && heads >= 1 && hd >= 2 && hd % 2 == 0, OOMB_SHAPE_ERROR,
                     "rope: head dimension must be even");  // ops.hpp:194-196
        OOMB_REQUIRE(base > 0.f && (sign == 1 || sign == -1), OOMB_CONFIG_ERROR, "rope: base > 0, sign +-1");
        OOMB_REQUIRE(in_dtype != OOMB_F64 && out_dtype != OOMB_F64, OOMB_CONFIG_ERROR, "rope: fp32 / bf16");
        launch_rope(in_dtype, out_dtype, x, rows, heads, hd, pos_offset, sign, rope_inv_freq_table(base, hd), out,
                    S(stream));
    });
}

int oomb_n_pages(oomb_pool_t p, int layer, int* n) {
    return guard([&] {
        p->pt->check_layer(layer);
        *n = static_cast<int>(p->pt->pages[layer].size());
    });
}
int oomb_filled(oomb_pool_t p, int layer, int64_t* f) {
    return guard([&] {
        p->pt->check_layer(layer);
        *f = p->pt->filled[layer];
    });
}
int oomb_page_table_get(oomb_pool_t p, int layer, int32_t* out) {
    return guard([&] {
        p->pt->check_layer(layer);
        const auto& st = p->pt->pages[layer];
        for (size_t i = 0; i < st.size(); ++i) {
            out[4 * i + 0] = st[i].k;
            out[4 * i + 1] = st[i].v;
            out[4 * i + 2] = st[i].gk;
            out[4 * i + 3] = st[i].gv;
        }
    });
}
int oomb_device_slots_get(oomb_pool_t p, int layer, int32_t* out) {
    return guard([&] {
        p->pt->check_layer(layer);
        for (size_t i = 0; i < p->pt->pages[layer].size(); ++i) {
            out[2 * i + 0] = p->kvslot[layer][i];
            out[2 * i + 1] = p->gslot[layer][i];
        }
    });
}
int oomb_page_mean_keys(oomb_pool_t p, int layer, int n_candidates, void* out, void* stream, int* n_out) {
    return guard([&] {
        set_dev(p);
        p->pt->check_layer(layer);
        const int np = static_cast<int>(p->pt->pages[layer].size());
        const int n = n_candidates < 0 ? np : std::min(n_candidates, np);
        launch_mean_keys(p->kavg_sum_layer(layer), p->kavg_cnt_layer(layer), n, p->cfg.n_kv_heads * p->cfg.head_dim,
                         out, S(stream), p->f64());
        *n_out = n;
    });
}
int oomb_kavg_raw(oomb_pool_t p, int layer, void* sum_out, int32_t* count_out, void* stream) {
    return guard([&] {
        set_dev(p);
        p->pt->check_layer(layer);
        const int64_t np = static_cast<int64_t>(p->pt->pages[layer].size());
        const int64_t re = static_cast<int64_t>(p->cfg.n_kv_heads) * p->cfg.head_dim;
        if (np == 0) return;
        OOMB_CUDA(cudaMemcpyAsync(sum_out, p->kavg_sum_layer(layer), np * re * p->aelem,
                                  cudaMemcpyDeviceToDevice, S(stream)));
        OOMB_CUDA(cudaMemcpyAsync(count_out, p->kavg_cnt_layer(layer), np * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                  S(stream)));
    });
}
int oomb_gather_pages(oomb_pool_t p, int layer, const int32_t* ids, int n, int grads, void* k_out, void* v_out,
                      uint8_t* valid_out, void* stream) {
    return guard([&] {
        set_dev(p);
        p->pt->check_ids(layer, ids, n, p->enforce, grads ? "gather_grad_pages" : "gather_pages");
        if (n == 0) return;
        int32_t* d = upload_ids(ids, n, S(stream));
        launch_gather(p->cfg.dtype, grads, d, n, grads ? p->gslot_layer(layer) : p->kvslot_layer(layer),
                      grads ? static_cast<const void*>(p->gkpool) : p->kpool,
                      grads ? static_cast<const void*>(p->gvpool) : p->vpool, p->pt->filled[layer],
                      p->cfg.page_size, p->cfg.n_kv_heads, p->cfg.head_dim, k_out, v_out, valid_out, p->d_err,
                      S(stream));
        OOMB_CUDA(cudaFreeAsync(d, S(stream)));
    });
}
int oomb_scatter_add_grads(oomb_pool_t p, int layer, const int32_t* ids, int n, const void* dk, const void* dv,
                           void* stream) {
    return guard([&] {
        set_dev(p);
        p->pt->check_ids(layer, ids, n, p->enforce, "scatter_add_grads");
        if (n == 0) return;
        const int32_t off[2] = {0, n};
        ensure_grad_pages(p, layer, off, ids, 1, S(stream));
        int32_t* d = upload_ids(ids, n, S(stream));
        launch_scatter(d, n, p->gslot_layer(layer), p->gkpool, p->gvpool, dk, dv, p->pt->filled[layer],
                       p->cfg.page_size, p->cfg.n_kv_heads, p->cfg.head_dim, p->d_err, S(stream), p->f64());
        OOMB_CUDA(cudaFreeAsync(d, S(stream)));
    });
}
int oomb_set_tier(oomb_pool_t p, int layer, int page, int tier) {
    return guard([&] {
        p->pt->check_layer(layer);
        OOMB_REQUIRE(page >= 0 && page < static_cast<int>(p->pt->pages[layer].size()), OOMB_SHAPE_ERROR,
                     "set_tier: page out of range");
        OOMB_REQUIRE(p->pt->pages[layer][page].tier <= TIER_HOST, OOMB_STATE_ERROR,
                     "set_tier: page is owned by another shard or lost");
        p->pt->pages[layer][page].tier = tier ? TIER_HOST : TIER_DEVICE;
    });
}
int oomb_get_tier(oomb_pool_t p, int layer, int page, int* tier) {
    return guard([&] {
        p->pt->check_layer(layer);
        OOMB_REQUIRE(page >= 0 && page < static_cast<int>(p->pt->pages[layer].size()), OOMB_SHAPE_ERROR,
                     "tier: page out of range");
        *tier = p->pt->pages[layer][page].tier;
    });
}
int oomb_set_residency_enforced(oomb_pool_t p, int on) {
    return guard([&] { p->enforce = on != 0; });
}
int oomb_grads_allocated(oomb_pool_t p, int layer, int page, int* a) {
    return guard([&] {
        p->pt->check_layer(layer);
        OOMB_REQUIRE(page >= 0 && page < static_cast<int>(p->pt->pages[layer].size()), OOMB_SHAPE_ERROR,
                     "grads_allocated: page out of range");
        *a = p->pt->pages[layer][page].gk >= 0;
    });
}

// ---------------------------------------------------------------------------
// selections
// ---------------------------------------------------------------------------
int oomb_selection_create(oomb_pool_t p, int max_m, int max_ids, oomb_selection_t* out) {
    return guard([&] {
        set_dev(p);
        OOMB_REQUIRE(max_m >= 1 && max_ids >= 0, OOMB_CONFIG_ERROR, "selection: bad capacity");
        auto* s = new oomb_selection_s();
        s->pool = p;
        s->max_m = max_m;
        s->max_ids = max_ids;
        OOMB_CUDA(cudaMalloc(reinterpret_cast<void**>(&s->d_off), (max_m + 1) * sizeof(int32_t)));
        OOMB_CUDA(cudaMalloc(reinterpret_cast<void**>(&s->d_ids), std::max(max_ids, 1) * sizeof(int32_t)));
        OOMB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&s->h_off), (max_m + 1) * sizeof(int32_t)));
        OOMB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&s->h_ids), std::max(max_ids, 1) * sizeof(int32_t)));
        OOMB_CUDA(cudaEventCreateWithFlags(&s->ev, cudaEventDisableTiming));
        s->h_off[0] = 0;
        *out = s;
    });
}
int oomb_selection_destroy(oomb_selection_t s) {
    if (!s) return OOMB_OK;
    cudaSetDevice(s->pool->device);
    if (s->ev) cudaEventSynchronize(s->ev);
    cudaFree(s->d_off);
    cudaFree(s->d_ids);
    cudaFreeHost(s->h_off);
    cudaFreeHost(s->h_ids);
    if (s->ev) cudaEventDestroy(s->ev);
    delete s;
    return OOMB_OK;
}
int oomb_selection_set_host(oomb_selection_t s, const int32_t* off, const int32_t* ids, int m, void* stream) {
    return guard([&] {
        set_dev(s->pool);
        OOMB_REQUIRE(m >= 0 && m <= s->max_m, OOMB_SHAPE_ERROR, "selection: too many query pages");
        const int nnz = m > 0 ? off[m] : 0;
        OOMB_REQUIRE(nnz >= 0 && nnz <= s->max_ids, OOMB_SHAPE_ERROR, "selection: too many ids");
        OOMB_CUDA(cudaEventSynchronize(s->ev));  // previous async copy out of the pinned mirror is done
        s->host_pending = false;
        s->nnz_from_host = false;
        std::memcpy(s->h_off, off, (m + 1) * sizeof(int32_t));
        if (nnz) std::memcpy(s->h_ids, ids, nnz * sizeof(int32_t));
        OOMB_CUDA(cudaMemcpyAsync(s->d_off, s->h_off, (m + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, S(stream)));
        if (nnz)
            OOMB_CUDA(cudaMemcpyAsync(s->d_ids, s->h_ids, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, S(stream)));
        OOMB_CUDA(cudaEventRecord(s->ev, S(stream)));
        s->m = m;
        s->nnz = nnz;
    });
}
int oomb_selection_get_host(oomb_selection_t s, int32_t* off, int32_t* ids, int* m, int* nnz) {
    return guard([&] {
        set_dev(s->pool);
        sel_host_sync(s);
        *m = s->m;
        *nnz = s->nnz;
        if (off) std::memcpy(off, s->h_off, (s->m + 1) * sizeof(int32_t));
        if (ids && s->nnz) std::memcpy(ids, s->h_ids, s->nnz * sizeof(int32_t));
    });
}
int oomb_selection_device(oomb_selection_t s, const int32_t** off, const int32_t** ids, int* m) {
    return guard([&] {
        *off = s->d_off;
        *ids = s->d_ids;
        *m = s->m;
    });
}
static void select_range(oomb_selection_t s, int first, int count, int m, cudaStream_t st) {
    OOMB_REQUIRE(m >= 0 && m <= s->max_m, OOMB_SHAPE_ERROR, "selection: too many query pages");
    OOMB_REQUIRE(static_cast<int64_t>(m) * count <= s->max_ids, OOMB_SHAPE_ERROR, "selection: too many ids");
    OOMB_CUDA(cudaEventSynchronize(s->ev));
    s->host_pending = false;
    s->nnz_from_host = false;
    for (int qp = 0; qp <= m; ++qp) s->h_off[qp] = qp * count;
    for (int qp = 0; qp < m; ++qp)
        for (int i = 0; i < count; ++i) s->h_ids[static_cast<int64_t>(qp) * count + i] = first + i;
    s->m = m;
    s->nnz = m * count;
    launch_fill_csr_all(s->d_off, s->d_ids, m, first, count, st);
}
int oomb_select_all(oomb_selection_t s, int n_pages, int m, void* stream) {
    return guard([&] {
        set_dev(s->pool);
        OOMB_REQUIRE(n_pages >= 0, OOMB_SHAPE_ERROR, "select_all: negative page count");
        select_range(s, 0, n_pages, m, S(stream));
    });
}
int oomb_select_recent(oomb_selection_t s, int n_pages, int window, int m, void* stream) {
    return guard([&] {
        set_dev(s->pool);
        OOMB_REQUIRE(window >= 0, OOMB_SHAPE_ERROR, "select_recent: negative window");  // attention.hpp:100
        const int take = std::min(n_pages, window);
        select_range(s, n_pages - take, take, m, S(stream));
    });
}
static void select_topk_impl(oomb_selection_t s, const void* vote, int m, int n, int k, cudaStream_t st) {
    OOMB_REQUIRE(k >= 0, OOMB_SHAPE_ERROR, "select_topk: negative budget");  // attention.hpp:73
    OOMB_REQUIRE(m >= 0 && m <= s->max_m, OOMB_SHAPE_ERROR, "selection: too many query pages");
    const int kk = std::min(k, n);
    OOMB_REQUIRE(static_cast<int64_t>(m) * kk <= s->max_ids, OOMB_SHAPE_ERROR, "selection: too many ids");
    OOMB_CUDA(cudaEventSynchronize(s->ev));
    launch_topk(vote, m, n, k, s->d_off, s->d_ids, st, s->pool->f64());
    OOMB_CUDA(cudaMemcpyAsync(s->h_off, s->d_off, (m + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    if (m * kk)
        OOMB_CUDA(cudaMemcpyAsync(s->h_ids, s->d_ids, static_cast<size_t>(m) * kk * sizeof(int32_t),
                                  cudaMemcpyDeviceToHost, st));
    OOMB_CUDA(cudaEventRecord(s->ev, st));
    s->host_pending = true;
    s->nnz_from_host = false;
    s->m = m;
    s->nnz = m * kk;
}

int oomb_selection_filter_owned(oomb_pool_t p, oomb_selection_t src, oomb_selection_t dst, void* stream) {
    return guard([&] {
        set_dev(p);
        OOMB_REQUIRE(src != nullptr && dst != nullptr && src != dst, OOMB_STATE_ERROR,
                     "filter_owned: needs two distinct selections");
        OOMB_REQUIRE(src->m <= dst->max_m && src->nnz <= dst->max_ids, OOMB_SHAPE_ERROR,
                     "filter_owned: destination selection too small");
        OOMB_CUDA(cudaEventSynchronize(dst->ev));  // the previous mirror copy out of dst is done
        const int m = src->m;
        launch_filter_owned(src->d_off, src->d_ids, m, p->owner_stride, p->owner_rank, dst->d_off, dst->d_ids,
                            S(stream));
        OOMB_CUDA(cudaMemcpyAsync(dst->h_off, dst->d_off, (m + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                  S(stream)));
        if (src->nnz)  // an upper bound: the exact count is h_off[m] once the mirror lands
            OOMB_CUDA(cudaMemcpyAsync(dst->h_ids, dst->d_ids, static_cast<size_t>(src->nnz) * sizeof(int32_t),
                                      cudaMemcpyDeviceToHost, S(stream)));
        OOMB_CUDA(cudaEventRecord(dst->ev, S(stream)));
        dst->host_pending = true;
        dst->nnz_from_host = true;
        dst->m = m;
        dst->nnz = src->nnz;
    });
}
int oomb_page_owner(oomb_pool_t p, int* stride, int* rank) {
    return guard([&] {
        if (stride) *stride = p->owner_stride;
        if (rank) *rank = p->owner_rank;
    });
}

int oomb_select_topk(oomb_selection_t s, const void* vote, int m, int n, int k, void* stream) {
    return guard([&] {
        set_dev(s->pool);
        select_topk_impl(s, vote, m, n, k, S(stream));
    });
}

// ---------------------------------------------------------------------------
// scoring
// ---------------------------------------------------------------------------
// score_pages on fp32 representatives (k_avg [n][Hkv][hd]) or, when kavg_sum/kavg_cnt are given,
// on the pool's K_avg sums (mean formed on the fly, paged_kv.hpp:170-183). bf16 + hd 128 +
// 128-aligned chunks use the tcgen05 scorer; everything else the exact SIMT scorer.
static void score_impl(const void* q, int64_t tokens, int Hq, int hd, const void* k_avg, const void* kavg_sum,
                       const int32_t* kavg_cnt, int64_t n, int Hkv, int P, int score_scale, int dtype, bool allow_tc,
                       void* vote, cudaStream_t st, bool partial_only = false, const void* planes = nullptr,
                       int64_t plane_stride = 0) {
    OOMB_REQUIRE(n >= 1, OOMB_SHAPE_ERROR, "score_pages: needs at least one candidate page");
    OOMB_REQUIRE(Hq >= 1 && Hkv >= 1 && Hq % Hkv == 0 && hd >= 1 && hd <= 256 && P >= 1, OOMB_SHAPE_ERROR,
                 "score_pages: bad shape");
    const float scale = score_scale ? 1.0f / std::sqrt(static_cast<float>(hd)) : 1.0f;
    const double scale64 = score_scale ? 1.0 / std::sqrt(static_cast<double>(hd)) : 1.0;
    const bool f64 = dtype == OOMB_F64;
    const size_t ae = f64 ? 8 : 4;
    if (allow_tc && score_tc_supported(dtype, hd, P, tokens)) {
        void* ws = nullptr;
        OOMB_CUDA(cudaMallocAsync(&ws, score_tc_workspace(tokens, Hq, Hkv, n, P), st));
        launch_score_tc(q, tokens, Hq, Hkv, P, static_cast<const float*>(kavg_sum), kavg_cnt,
                        static_cast<const float*>(k_avg), n, scale, static_cast<float*>(vote), ws, st, partial_only,
                        planes, plane_stride);
        OOMB_CUDA(cudaFreeAsync(ws, st));
        return;
    }
    void* kavg = const_cast<void*>(k_avg);
    if (!kavg) {
        OOMB_CUDA(cudaMallocAsync(&kavg, n * Hkv * hd * ae, st));
        launch_mean_keys(kavg_sum, kavg_cnt, static_cast<int>(n), Hkv * hd, kavg, st, f64);
    }
    void* stats = nullptr;
    OOMB_CUDA(cudaMallocAsync(&stats, std::max<int64_t>(tokens * Hq, 1) * 2 * ae, st));
    launch_score_simt(dtype, q, tokens, Hq, hd, kavg, n, Hkv, P, scale, scale64, vote, stats, st, partial_only);
    OOMB_CUDA(cudaFreeAsync(stats, st));
    if (!k_avg) OOMB_CUDA(cudaFreeAsync(kavg, st));
}

int oomb_score_pages(const void* q, int64_t tokens, int Hq, int hd, const void* k_avg, int64_t n, int Hkv,
                     int page_size, int score_scale, int dtype, void* vote, void* stream) {
    return guard([&] {
        score_impl(q, tokens, Hq, hd, k_avg, nullptr, nullptr, n, Hkv, page_size, score_scale, dtype, true, vote,
                   S(stream));
    });
}

static void select_topk_impl(oomb_selection_t s, const void* vote, int m, int n, int k, cudaStream_t st);

int oomb_score_pages_partial(oomb_pool_t p, int layer, const void* q, int64_t tokens, int n_candidates,
                             void* partials, void* stream) {
    return guard([&] {
        set_dev(p);
        p->pt->check_layer(layer);
        const int n = std::min(n_candidates, static_cast<int>(p->pt->pages[layer].size()));
        OOMB_REQUIRE(n >= 1, OOMB_SHAPE_ERROR, "score_pages: needs at least one candidate page");
        score_impl(q, tokens, p->cfg.n_q_heads, p->cfg.head_dim, nullptr, p->kavg_sum_layer(layer),
                   p->kavg_cnt_layer(layer), n, p->cfg.n_kv_heads, p->cfg.page_size, p->cfg.score_scale,
                   p->cfg.dtype, p->policy != 1, partials, S(stream), /*partial_only=*/true, p->kavg_planes_layer(layer),
                   p->plane_stride);
    });
}

int oomb_lse_merge(const void* o_parts, const float* lse_parts, int parts, int64_t rows, int hd, int dtype,
                   void* out, float* lse, void* stream) {
    return guard([&] {
        OOMB_REQUIRE(parts >= 1 && rows >= 0 && hd >= 1 && hd <= 256, OOMB_SHAPE_ERROR, "lse_merge: bad shape");
        OOMB_REQUIRE(dtype == OOMB_BF16 || dtype == OOMB_F32, OOMB_CONFIG_ERROR, "lse_merge: dtype");
        launch_lse_merge(o_parts, lse_parts, parts, rows, hd, dtype, out, lse, S(stream));
    });
}

int oomb_vote_reduce(const float* partials, int groups, int64_t m, int64_t n, float* vote, void* stream) {
    return guard([&] {
        OOMB_REQUIRE(groups >= 1 && m >= 0 && n >= 0, OOMB_SHAPE_ERROR, "vote_reduce: bad shape");
        if (m * n > 0) launch_vote_reduce(partials, groups, m * n, vote, S(stream));
    });
}

int oomb_select_pages_topk(oomb_pool_t p, int layer, const void* q, int64_t tokens, int n_candidates,
                           oomb_selection_t sel, void* vote_scratch, void* stream) {
    return guard([&] {
        set_dev(p);
        p->pt->check_layer(layer);
        const int np = static_cast<int>(p->pt->pages[layer].size());
        const int n = std::min(n_candidates, np);
        const int m = static_cast<int>((tokens + p->cfg.page_size - 1) / p->cfg.page_size);
        if (n <= 0) {  // chunk_trainer.hpp:297: no candidates -> empty lists
            select_range(sel, 0, 0, m, S(stream));
            return;
        }
        score_impl(q, tokens, p->cfg.n_q_heads, p->cfg.head_dim, nullptr, p->kavg_sum_layer(layer),
                   p->kavg_cnt_layer(layer), n, p->cfg.n_kv_heads, p->cfg.page_size, p->cfg.score_scale,
                   p->cfg.dtype, p->policy != 1, vote_scratch, S(stream), false, p->kavg_planes_layer(layer),
                   p->plane_stride);
        select_topk_impl(sel, vote_scratch, m, n, p->cfg.retrieval_budget / p->cfg.page_size, S(stream));
    });
}

// ---------------------------------------------------------------------------
// attention
// ---------------------------------------------------------------------------
int oomb_attn_forward_ex(oomb_pool_t p, int layer, const void* q, int64_t tokens, oomb_selection_t sel,
                         const void* k_cur, const void* v_cur, void* out, void* lse, int flags, void* stream) {
    return guard([&] {
        set_dev(p);
        p->pt->check_layer(layer);
        OOMB_REQUIRE(tokens >= 1, OOMB_SHAPE_ERROR, "attn_forward: empty chunk");
        AttnGeom g = geom(p, tokens, layer);
        if (flags & OOMB_ATTN_PAST_ONLY) g.chunk_keys = 0;
        OOMB_REQUIRE(sel->m == g.m, OOMB_SHAPE_ERROR,
                     "attn_forward: one selected-page list per query page required");  // attention.hpp:172-174
        if (p->enforce) {  // gather_pages' residency check (paged_kv.hpp:118-122)
            sel_host_sync(sel);
            for (int qp = 0; qp < g.m; ++qp)
                p->pt->check_ids(layer, sel->h_ids + sel->h_off[qp], sel->h_off[qp + 1] - sel->h_off[qp], true,
                                 "gather_pages");
        }
        if (use_tc(p, g))
            launch_attn_fwd_tc(g, p->maps, q, sel->d_off, sel->d_ids, p->kvslot_layer(layer), k_cur, v_cur, out,
                               static_cast<float*>(lse), p->d_err, S(stream));
        else
            launch_attn_fwd_simt(p->cfg.dtype, g, q, sel->d_off, sel->d_ids, p->kvslot_layer(layer), p->kpool, p->vpool,
                                 k_cur, v_cur, out, lse, p->d_err, S(stream));
    });
}

int oomb_attn_forward(oomb_pool_t p, int layer, const void* q, int64_t tokens, oomb_selection_t sel,
                      const void* k_cur, const void* v_cur, void* out, void* lse, void* stream) {
    return oomb_attn_forward_ex(p, layer, q, tokens, sel, k_cur, v_cur, out, lse, 0, stream);
}

namespace {
int attn_backward_impl(oomb_pool_t p, int layer, const void* dout, const void* q, int64_t tokens,
                       oomb_selection_t sel, const void* k_cur, const void* v_cur, const void* out, const void* lse,
                       void* dq, void* dk_cur, void* dv_cur, int flags, int64_t own_first, void* stream) {
    return guard([&] {
        set_dev(p);
        p->pt->check_layer(layer);
        OOMB_REQUIRE(tokens >= 1, OOMB_SHAPE_ERROR, "attn_backward: empty chunk");
        AttnGeom g = geom(p, tokens, layer);
        if (flags & OOMB_ATTN_PAST_ONLY) g.chunk_keys = 0;
        OOMB_REQUIRE(sel->m == g.m, OOMB_SHAPE_ERROR, "attn_backward: one selected-page list per query page required");
        sel_host_sync(sel);
        for (int qp = 0; qp < g.m; ++qp)
            p->pt->check_ids(layer, sel->h_ids + sel->h_off[qp], sel->h_off[qp + 1] - sel->h_off[qp], p->enforce,
                             "attn_backward");
        ensure_grad_pages(p, layer, sel->h_off, sel->h_ids, g.m, S(stream));
        // own_first >= 0: the dM_i read-back of the chunk's own pages (oomb_accumulate_grad_pages of
        // pages own_first .. own_first + tokens / P - 1) folded into this call
        int rb_first = -1, rb_n = 0;
        if (own_first >= 0) {
            OOMB_REQUIRE(!(flags & OOMB_ATTN_PAST_ONLY) && tokens % g.P == 0 &&
                             (own_first + tokens / g.P) * g.P <= p->pt->filled[layer],
                         OOMB_SHAPE_ERROR,
                         "attn_backward_readback: the chunk's own keys must fill whole appended pages");
            rb_first = static_cast<int>(own_first);
            rb_n = static_cast<int>(tokens / g.P);
            std::vector<int32_t> own(static_cast<size_t>(rb_n));
            for (int i = 0; i < rb_n; ++i) own[static_cast<size_t>(i)] = rb_first + i;
            p->pt->check_ids(layer, own.data(), rb_n, p->enforce, "gather_grad_pages", /*allow_remote=*/true);
        }
        const size_t kvb = static_cast<size_t>(tokens) * g.Hkv * g.hd * p->aelem;
        const bool tc = p->policy != 1 && p->maps.valid && tc_supported(g, p->cfg.dtype) && tc_bwd_available();
        if (tc) {
            if (!p->bwd_side) {
                OOMB_CUDA(cudaStreamCreateWithFlags(&p->bwd_side, cudaStreamNonBlocking));
                OOMB_CUDA(cudaEventCreateWithFlags(&p->bwd_ev_prep, cudaEventDisableTiming));
                for (int b = 0; b < 2; ++b) OOMB_CUDA(cudaEventCreateWithFlags(&p->bwd_ev_dq[b], cudaEventDisableTiming));
            }
            const bool defer = (flags & OOMB_ATTN_DEFER_DQ) != 0;
            const int b = p->bwd_parity;
            p->bwd_parity ^= 1;
            const size_t need = attn_bwd_tc_workspace(g, sel->nnz);
            // the dQ that last used this workspace has finished reading it
            if (p->bwd_ws_used[b]) OOMB_CUDA(cudaStreamWaitEvent(S(stream), p->bwd_ev_dq[b], 0));
            if (need > p->bwd_ws_bytes[b]) {  // regrow in stream order: no device-wide synchronisation
                if (p->bwd_ws[b]) OOMB_CUDA(cudaFreeAsync(p->bwd_ws[b], S(stream)));
                p->bwd_ws[b] = nullptr;
                OOMB_CUDA(cudaMallocAsync(&p->bwd_ws[b], need, S(stream)));
                p->bwd_ws_bytes[b] = need;
            }
            launch_attn_bwd_tc(g, p->maps, dout, q, sel->d_off, sel->d_ids, p->kvslot_layer(layer),
                               p->gslot_layer(layer), p->gkpool, p->gvpool, k_cur, v_cur, out,
                               static_cast<const float*>(lse), static_cast<float*>(dq), static_cast<float*>(dk_cur),
                               static_cast<float*>(dv_cur), p->d_err, p->bwd_ws[b], p->bwd_ws_bytes[b], sel->nnz,
                               static_cast<int>(p->pt->pages[layer].size()), S(stream), p->bwd_side,
                               p->bwd_ev_prep, p->bwd_ev_dq[b], !defer, rb_first);
            p->bwd_ws_used[b] = true;
            p->bwd_last_dq = p->bwd_ev_dq[b];
        } else {
            OOMB_CUDA(cudaMemsetAsync(dk_cur, 0, kvb, S(stream)));
            OOMB_CUDA(cudaMemsetAsync(dv_cur, 0, kvb, S(stream)));
            launch_attn_bwd_simt(p->cfg.dtype, g, dout, q, sel->d_off, sel->d_ids, p->kvslot_layer(layer),
                                 p->gslot_layer(layer), p->kpool, p->vpool, p->gkpool, p->gvpool, k_cur, v_cur, out,
                                 lse, dq, dk_cur, dv_cur, p->d_err, S(stream),
                                 static_cast<int>(p->pt->pages[layer].size()));
            if (rb_first >= 0)
                launch_accumulate_grads(nullptr, rb_n, p->gslot_layer(layer), p->gkpool, p->gvpool,
                                        p->pt->filled[layer], p->cfg.page_size, p->cfg.n_kv_heads, p->cfg.head_dim,
                                        dk_cur, dv_cur, S(stream), 0, nullptr, p->f64(), rb_first);
        }
    });
}

}  // namespace

int oomb_attn_backward_ex(oomb_pool_t p, int layer, const void* dout, const void* q, int64_t tokens,
                          oomb_selection_t sel, const void* k_cur, const void* v_cur, const void* out, const void* lse,
                          void* dq, void* dk_cur, void* dv_cur, int flags, void* stream) {
    return attn_backward_impl(p, layer, dout, q, tokens, sel, k_cur, v_cur, out, lse, dq, dk_cur, dv_cur, flags, -1,
                              stream);
}

int oomb_attn_backward_readback(oomb_pool_t p, int layer, const void* dout, const void* q, int64_t tokens,
                                oomb_selection_t sel, const void* k_cur, const void* v_cur, const void* out,
                                const void* lse, void* dq, void* dk_cur, void* dv_cur, int flags, int64_t own_first_page,
                                void* stream) {
    if (own_first_page < 0)
        return guard([&] { OOMB_REQUIRE(false, OOMB_SHAPE_ERROR, "attn_backward_readback: negative own_first_page"); });
    return attn_backward_impl(p, layer, dout, q, tokens, sel, k_cur, v_cur, out, lse, dq, dk_cur, dv_cur, flags,
                              own_first_page, stream);
}

int oomb_attn_backward(oomb_pool_t p, int layer, const void* dout, const void* q, int64_t tokens,
                       oomb_selection_t sel, const void* k_cur, const void* v_cur, const void* out, const void* lse,
                       void* dq, void* dk_cur, void* dv_cur, void* stream) {
    return oomb_attn_backward_ex(p, layer, dout, q, tokens, sel, k_cur, v_cur, out, lse, dq, dk_cur, dv_cur, 0, stream);
}

int oomb_attn_join_dq(oomb_pool_t p, void* stream) {
    return guard([&] {
        set_dev(p);
        if (p->bwd_last_dq) OOMB_CUDA(cudaStreamWaitEvent(S(stream), p->bwd_last_dq, 0));
    });
}

int oomb_accumulate_grad_pages(oomb_pool_t p, int layer, const int32_t* ids, int n, void* dk, void* dv,
                               void* stream) {
    return guard([&] {
        set_dev(p);
        // on a page-range shard the REMOTE pages among ids add nothing here: their owners add them to
        // their partial dk / dv, which the range group sums (sharding.ShardedLayer.backward)
        p->pt->check_ids(layer, ids, n, p->enforce, "gather_grad_pages", /*allow_remote=*/true);
        if (n == 0) return;
        // a consecutive run of pages (the dM_i read-back of a chunk's own pages) needs no id upload
        bool run = true;
        for (int i = 1; i < n && run; ++i) run = ids[i] == ids[0] + i;
        int32_t* d = run ? nullptr : upload_ids(ids, n, S(stream));
        launch_accumulate_grads(d, n, p->gslot_layer(layer), p->gkpool, p->gvpool, p->pt->filled[layer],
                                p->cfg.page_size, p->cfg.n_kv_heads, p->cfg.head_dim, dk, dv, S(stream), 0, nullptr,
                                p->f64(), ids[0]);
        if (d) OOMB_CUDA(cudaFreeAsync(d, S(stream)));
    });
}

int oomb_accumulate_grad_pages_rope(oomb_pool_t p, int layer, const int32_t* ids, int n, float* dk, float* dv,
                                    int64_t pos_offset, float rope_base, void* stream) {
    return guard([&] {
        set_dev(p);
        p->pt->check_ids(layer, ids, n, p->enforce, "gather_grad_pages", /*allow_remote=*/true);
        OOMB_REQUIRE(rope_base > 1.f, OOMB_CONFIG_ERROR, "rope_base must be > 1");
        OOMB_REQUIRE(!p->f64(), OOMB_CONFIG_ERROR, "the fused RoPE epilogues support fp32 / bf16 pools");
        if (n == 0) return;
        int32_t* d = upload_ids(ids, n, S(stream));
        launch_accumulate_grads(d, n, p->gslot_layer(layer), p->gkpool, p->gvpool, p->pt->filled[layer],
                                p->cfg.page_size, p->cfg.n_kv_heads, p->cfg.head_dim, dk, dv, S(stream), pos_offset,
                                rope_inv_freq_table(rope_base, p->cfg.head_dim));
        OOMB_CUDA(cudaFreeAsync(d, S(stream)));
    });
}

int oomb_profile_enable(oomb_pool_t p, int on) {
    return guard([&] { p->prof_on = on != 0; });
}

int oomb_profile_collect(oomb_pool_t p, int64_t* counts, double* ms, int n_kinds) {
    return guard([&] {
        OOMB_CUDA(cudaSetDevice(p->device));
        OOMB_CUDA(cudaDeviceSynchronize());
        for (int k = 0; k < n_kinds; ++k) {
            counts[k] = 0;
            ms[k] = 0.0;
        }
        for (auto& r : p->prof.recs) {
            float t = 0.f;
            OOMB_CUDA(cudaEventElapsedTime(&t, r.e0, r.e1));
            if (r.kind < n_kinds) {
                counts[r.kind] += 1;
                ms[r.kind] += t;
            }
            p->prof.spare.push_back(r.e0);
            p->prof.spare.push_back(r.e1);
        }
        p->prof.recs.clear();
    });
}

int oomb_debug_tc_gemm(int mode, const void* a, const void* b, float* c, int m, int n, int k, void* stream) {
    return guard([&] {
        OOMB_REQUIRE(m == 128 && (n == 64 || n == 128 || n == 256) && k % 64 == 0 && k > 0, OOMB_SHAPE_ERROR,
                     "debug_tc_gemm: M=128, N in {64,128,256}, K%64==0");
        launch_debug_tc_gemm(mode, a, b, c, m, n, k, S(stream));
    });
}

}  // extern "C"
