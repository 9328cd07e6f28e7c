/* SPDX-License-Identifier: Apache-2.0
 *
 * oomb_oracle.c — CPU restatement of the OOMB hot path. TEST INFRASTRUCTURE.
 *
 * This file is the CHECKER, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. The product
 * path (paper_2602_02108_b200) never links or calls it and fails loudly if its
 * CUDA library is missing.
 *
 * It restates, in plain C with the same floating-point operation order, the
 * reference's CPU algorithm for the path (all citations relative to
 * /root/reference/proj/core/include/chunktrain/):
 *   page manager     paged_kv.hpp:41-356   (LIFO free-list arena, lazy grad pages, K_avg)
 *   score_pages      attention.hpp:32-67
 *   select_topk      attention.hpp:71-88, select_recent :99-105, select_all :107-111
 *   attn_forward     attention.hpp:117-208 (OnlineRow :128-147)
 *   attn_backward    attention.hpp:210-293
 *   naive attention  oracle.hpp:293-357
 * Built with -O2 -ffp-contract=off (no -march=native) it is BIT-IDENTICAL to the
 * reference compiled the same way (oracle/Makefile.ref); tests/test_oracle_golden.py
 * pins that against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py). Parity is therefore pinned, not assumed.
 *
 * Every entry point returns 0 or an error code that maps 1:1 onto the
 * reference's exception classes (common.hpp:15-29).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OC_OK = 0, OC_CONFIG = 1, OC_SHAPE = 2, OC_STATE = 3, OC_RESIDENCY = 4, OC_IO = 5, OC_OTHER = 9 };

static const char* g_err = "";
const char* oc_last_error(void) { return g_err; }
#define FAIL(code, msg) do { g_err = (msg); return (code); } while (0)

/* ------------------------------------------------------------------------ */
/* Page manager (paged_kv.hpp:41-356)                                        */
/* ------------------------------------------------------------------------ */

typedef struct {
    int32_t k_phys, v_phys, gk_phys, gv_phys; /* PageEntry paged_kv.hpp:256-262 */
    uint8_t tier;                              /* 0 = device, 1 = host */
} OcPage;

typedef struct {
    OcPage* pages;
    int n_pages, cap_pages;
    void* kavg_sum;       /* [n_pages x kvh x hd] Real */
    int32_t* kavg_count;  /* [n_pages] */
    int64_t filled;
} OcLayer;

typedef struct {
    int real_bytes, page_size, kv_heads, head_dim, n_layers;
    OcLayer* layers;
    void** arena; int64_t arena_n, arena_cap;
    int32_t* free_list; int64_t free_n, free_cap;
    int enforce_residency;
} OcCache;

static int64_t row_elems(const OcCache* c) { return (int64_t)c->kv_heads * c->head_dim; }
static int64_t page_elems(const OcCache* c) { return (int64_t)c->page_size * row_elems(c); }

/* ModelConfig::validate subset (config.cpp:30-51) for the fields the path uses. */
int oc_validate(int n_layers, int n_q_heads, int n_kv_heads, int head_dim, int chunk_size,
                int page_size, int retrieval_budget, int local_window) {
    if (n_layers < 1) FAIL(OC_CONFIG, "config: n_layers must be >= 1");
    if (n_q_heads < 1 || n_kv_heads < 1) FAIL(OC_CONFIG, "config: head counts must be >= 1");
    if (n_q_heads % n_kv_heads != 0) FAIL(OC_CONFIG, "config: n_q_heads must be divisible by n_kv_heads");
    if (head_dim < 2 || head_dim % 2 != 0) FAIL(OC_CONFIG, "config: head_dim must be even (rotary pairs)");
    if (page_size < 1) FAIL(OC_CONFIG, "config: page_size must be >= 1");
    if (chunk_size < 1) FAIL(OC_CONFIG, "config: chunk_size must be >= 1");
    if (chunk_size % page_size != 0) FAIL(OC_CONFIG, "config: chunk_size must be divisible by page_size");
    if (retrieval_budget < 0) FAIL(OC_CONFIG, "config: retrieval_budget must be >= 0");
    if (retrieval_budget % page_size != 0) FAIL(OC_CONFIG, "config: retrieval_budget must be divisible by page_size");
    if (local_window < 0) FAIL(OC_CONFIG, "config: local_window must be >= 0");
    return OC_OK;
}

int oc_cache_new(int real_bytes, int n_layers, int kv_heads, int head_dim, int page_size, OcCache** out) {
    if (real_bytes != 4 && real_bytes != 8) FAIL(OC_CONFIG, "oracle: real_bytes must be 4 or 8");
    if (n_layers < 1 || kv_heads < 1 || head_dim < 1 || page_size < 1) FAIL(OC_CONFIG, "oracle: bad cache shape");
    OcCache* c = (OcCache*)calloc(1, sizeof(OcCache));
    c->real_bytes = real_bytes;
    c->page_size = page_size;
    c->kv_heads = kv_heads;
    c->head_dim = head_dim;
    c->n_layers = n_layers;
    c->layers = (OcLayer*)calloc((size_t)n_layers, sizeof(OcLayer));
    *out = c;
    return OC_OK;
}

void oc_cache_free(OcCache* c) {
    if (!c) return;
    for (int l = 0; l < c->n_layers; ++l) {
        free(c->layers[l].pages);
        free(c->layers[l].kavg_sum);
        free(c->layers[l].kavg_count);
    }
    for (int64_t i = 0; i < c->arena_n; ++i) free(c->arena[i]);
    free(c->arena);
    free(c->free_list);
    free(c->layers);
    free(c);
}

static int layer_ok(const OcCache* c, int layer) { return layer >= 0 && layer < c->n_layers; }

/* alloc_page_  paged_kv.hpp:280-288: LIFO free list first, else a new arena block. */
static int32_t alloc_page(OcCache* c) {
    if (c->free_n > 0) return c->free_list[--c->free_n];
    if (c->arena_n == c->arena_cap) {
        c->arena_cap = c->arena_cap ? 2 * c->arena_cap : 64;
        c->arena = (void**)realloc(c->arena, (size_t)c->arena_cap * sizeof(void*));
    }
    c->arena[c->arena_n] = calloc((size_t)page_elems(c), (size_t)c->real_bytes);
    return (int32_t)(c->arena_n++);
}

static void push_free(OcCache* c, int32_t id) {
    if (c->free_n == c->free_cap) {
        c->free_cap = c->free_cap ? 2 * c->free_cap : 64;
        c->free_list = (int32_t*)realloc(c->free_list, (size_t)c->free_cap * sizeof(int32_t));
    }
    c->free_list[c->free_n++] = id;
}

/* valid_in_page_  paged_kv.hpp:295-299 */
static int valid_in_page(const OcCache* c, const OcLayer* st, int pid) {
    const int64_t start = (int64_t)pid * c->page_size;
    int64_t v = st->filled - start;
    if (v > c->page_size) v = c->page_size;
    return (int)(v < 0 ? 0 : v);
}

/* check_resident_  paged_kv.hpp:301-312 */
static int check_resident(const OcCache* c, int layer, const int32_t* ids, int n) {
    const OcLayer* st = &c->layers[layer];
    for (int i = 0; i < n; ++i) {
        if (ids[i] < 0 || ids[i] >= st->n_pages) FAIL(OC_SHAPE, "page id out of range");
        if (c->enforce_residency && st->pages[ids[i]].tier != 0) FAIL(OC_RESIDENCY, "page is not device-resident");
    }
    return OC_OK;
}

int oc_cache_n_pages(const OcCache* c, int layer) { return layer_ok(c, layer) ? c->layers[layer].n_pages : -1; }
int64_t oc_cache_filled(const OcCache* c, int layer) { return layer_ok(c, layer) ? c->layers[layer].filled : -1; }

int oc_cache_page_table(const OcCache* c, int layer, int32_t* out) {
    if (!layer_ok(c, layer)) FAIL(OC_SHAPE, "cache: layer out of range");
    const OcLayer* st = &c->layers[layer];
    for (int p = 0; p < st->n_pages; ++p) {
        out[4 * p + 0] = st->pages[p].k_phys;
        out[4 * p + 1] = st->pages[p].v_phys;
        out[4 * p + 2] = st->pages[p].gk_phys;
        out[4 * p + 3] = st->pages[p].gv_phys;
    }
    return OC_OK;
}

int oc_cache_set_tier(OcCache* c, int layer, int page, int tier) {
    if (!layer_ok(c, layer) || page < 0 || page >= c->layers[layer].n_pages) FAIL(OC_SHAPE, "set_tier: out of range");
    c->layers[layer].pages[page].tier = (uint8_t)(tier ? 1 : 0);
    return OC_OK;
}

void oc_cache_set_residency_enforced(OcCache* c, int on) { c->enforce_residency = on != 0; }

/* reset  paged_kv.hpp:227-242 */
void oc_cache_reset(OcCache* c) {
    for (int l = 0; l < c->n_layers; ++l) {
        OcLayer* st = &c->layers[l];
        for (int p = 0; p < st->n_pages; ++p) {
            push_free(c, st->pages[p].k_phys);
            push_free(c, st->pages[p].v_phys);
            if (st->pages[p].gk_phys >= 0) {
                push_free(c, st->pages[p].gk_phys);
                push_free(c, st->pages[p].gv_phys);
            }
        }
        st->n_pages = 0;
        st->filled = 0;
    }
}

/* zero_grad_pages  paged_kv.hpp:214-223 */
void oc_cache_zero_grad(OcCache* c) {
    for (int l = 0; l < c->n_layers; ++l) {
        const OcLayer* st = &c->layers[l];
        for (int p = 0; p < st->n_pages; ++p) {
            if (st->pages[p].gk_phys >= 0) {
                memset(c->arena[st->pages[p].gk_phys], 0, (size_t)page_elems(c) * (size_t)c->real_bytes);
                memset(c->arena[st->pages[p].gv_phys], 0, (size_t)page_elems(c) * (size_t)c->real_bytes);
            }
        }
    }
}

/* memory_report  paged_kv.hpp:185-197 (+ arena_blocks_allocated / free_list_size) */
void oc_cache_memory_report(const OcCache* c, uint64_t* out) {
    memset(out, 0, 8 * sizeof(uint64_t));
    const uint64_t buf = (uint64_t)page_elems(c) * (uint64_t)c->real_bytes;
    for (int l = 0; l < c->n_layers; ++l) {
        const OcLayer* st = &c->layers[l];
        for (int p = 0; p < st->n_pages; ++p) {
            out[3] += 1;
            if (st->pages[p].tier == 0) out[0] += 2 * buf;
            else out[1] += 2 * buf;
            if (st->pages[p].gk_phys >= 0) out[2] += 2 * buf;
        }
    }
    out[6] = (uint64_t)c->arena_n;
    out[7] = (uint64_t)c->free_n;
}

static void ensure_page_capacity(OcCache* c, OcLayer* st, int need) {
    if (need <= st->cap_pages) return;
    int cap = st->cap_pages ? st->cap_pages : 16;
    while (cap < need) cap *= 2;
    st->pages = (OcPage*)realloc(st->pages, (size_t)cap * sizeof(OcPage));
    st->kavg_sum = realloc(st->kavg_sum, (size_t)cap * (size_t)row_elems(c) * (size_t)c->real_bytes);
    st->kavg_count = (int32_t*)realloc(st->kavg_count, (size_t)cap * sizeof(int32_t));
    st->cap_pages = cap;
}

/* ------------------------------------------------------------------------ */
/* select_topk / select_recent / select_all (attention.hpp:71-111)          */
/* ------------------------------------------------------------------------ */

static const double* g_sort_scores;
/* The reference's partial_sort comparator: score descending, then id ascending. */
static int cmp_score_desc_id_asc(const void* pa, const void* pb) {
    const int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
    const double sa = g_sort_scores[a], sb = g_sort_scores[b];
    if (sa != sb) return sa > sb ? -1 : 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}
static int cmp_i32(const void* pa, const void* pb) {
    const int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* The comparator is a strict total order, so the kept set equals the
 * reference's partial_sort prefix; the output is then sorted ascending. */
int oc_select_topk(const double* row, int n, int budget, int32_t* out, int* count) {
    if (budget < 0) FAIL(OC_SHAPE, "select_topk: negative budget");
    int32_t* ids = (int32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
    for (int i = 0; i < n; ++i) ids[i] = i;
    int keep = n;
    if (budget < n) {
        g_sort_scores = row;
        qsort(ids, (size_t)n, sizeof(int32_t), cmp_score_desc_id_asc);
        keep = budget;
    }
    qsort(ids, (size_t)keep, sizeof(int32_t), cmp_i32);
    memcpy(out, ids, (size_t)keep * sizeof(int32_t));
    *count = keep;
    free(ids);
    return OC_OK;
}

int oc_select_recent(int n_pages, int window, int32_t* out, int* count) {
    if (window < 0) FAIL(OC_SHAPE, "select_recent: negative window");
    const int take = n_pages < window ? n_pages : window;
    for (int i = 0; i < take; ++i) out[i] = n_pages - take + i;
    *count = take;
    return OC_OK;
}

int oc_select_all(int n_pages, int32_t* out, int* count) {
    for (int i = 0; i < n_pages; ++i) out[i] = i;
    *count = n_pages;
    return OC_OK;
}

/* ------------------------------------------------------------------------ */
/* Typed part: instantiated for float (f32) and double (f64).               */
/* ------------------------------------------------------------------------ */

#define DEFINE_ORACLE(REAL, SUF, EXP, LOG, SQRT)                                                   \
                                                                                                   \
/* append_chunk  paged_kv.hpp:73-108 */                                                            \
int oc_append_##SUF(OcCache* c, int layer, const REAL* k, const REAL* v, int64_t rows,            \
                    int64_t* begin, int64_t* end) {                                                \
    if (c->real_bytes != (int)sizeof(REAL)) FAIL(OC_CONFIG, "oracle: dtype mismatch");             \
    if (!layer_ok(c, layer)) FAIL(OC_SHAPE, "cache: layer out of range");                          \
    OcLayer* st = &c->layers[layer];                                                               \
    const int64_t re = row_elems(c);                                                               \
    *begin = st->filled;                                                                           \
    *end = st->filled + rows;                                                                      \
    for (int64_t r = 0; r < rows; ++r) {                                                           \
        const int64_t slot = st->filled + r;                                                       \
        const int page = (int)(slot / c->page_size);                                               \
        const int off = (int)(slot % c->page_size);                                                \
        if (page == st->n_pages) {                                                                 \
            ensure_page_capacity(c, st, page + 1);                                                 \
            OcPage e = {-1, -1, -1, -1, 0};                                                        \
            e.k_phys = alloc_page(c);                                                              \
            e.v_phys = alloc_page(c);                                                              \
            st->pages[page] = e;                                                                   \
            memset((REAL*)st->kavg_sum + (int64_t)page * re, 0, (size_t)re * sizeof(REAL));        \
            st->kavg_count[page] = 0;                                                              \
            st->n_pages += 1;                                                                      \
        }                                                                                          \
        const OcPage* e = &st->pages[page];                                                        \
        REAL* kd = (REAL*)c->arena[e->k_phys] + off * re;                                          \
        REAL* vd = (REAL*)c->arena[e->v_phys] + off * re;                                          \
        const REAL* ks = k + r * re;                                                               \
        const REAL* vs = v + r * re;                                                               \
        REAL* sum = (REAL*)st->kavg_sum + (int64_t)page * re;                                      \
        for (int64_t j = 0; j < re; ++j) {                                                         \
            kd[j] = ks[j];                                                                         \
            vd[j] = vs[j];                                                                         \
            sum[j] += ks[j];                                                                       \
        }                                                                                          \
        st->kavg_count[page] += 1;                                                                 \
    }                                                                                              \
    st->filled += rows;                                                                            \
    return OC_OK;                                                                                  \
}                                                                                                  \
                                                                                                   \
/* page_mean_keys  paged_kv.hpp:170-183: sum * (1/count), a reciprocal multiply. */                \
int oc_mean_keys_##SUF(const OcCache* c, int layer, int n_candidates, REAL* out, int* n_out) {    \
    if (!layer_ok(c, layer)) FAIL(OC_SHAPE, "cache: layer out of range");                          \
    const OcLayer* st = &c->layers[layer];                                                         \
    const int n = n_candidates < 0 ? st->n_pages                                                   \
                                   : (n_candidates < st->n_pages ? n_candidates : st->n_pages);    \
    const int64_t re = row_elems(c);                                                               \
    for (int p = 0; p < n; ++p) {                                                                  \
        const REAL inv = (REAL)1 / (REAL)st->kavg_count[p];                                        \
        const REAL* sum = (const REAL*)st->kavg_sum + (int64_t)p * re;                             \
        for (int64_t j = 0; j < re; ++j) out[(int64_t)p * re + j] = sum[j] * inv;                  \
    }                                                                                              \
    *n_out = n;                                                                                    \
    return OC_OK;                                                                                  \
}                                                                                                  \
                                                                                                   \
/* gather_pages / gather_grad_pages  paged_kv.hpp:118-130, gather_impl_ :314-347 */                \
int oc_gather_##SUF(const OcCache* c, int layer, const int32_t* ids, int n, int grads,            \
                    REAL* k, REAL* v, uint8_t* valid) {                                            \
    if (!layer_ok(c, layer)) FAIL(OC_SHAPE, "cache: layer out of range");                          \
    int rc = check_resident(c, layer, ids, n);                                                     \
    if (rc) return rc;                                                                             \
    const OcLayer* st = &c->layers[layer];                                                         \
    const int64_t re = row_elems(c), P = c->page_size;                                             \
    memset(k, 0, (size_t)(n * P * re) * sizeof(REAL));                                             \
    memset(v, 0, (size_t)(n * P * re) * sizeof(REAL));                                             \
    memset(valid, 0, (size_t)(n * P));                                                             \
    for (int i = 0; i < n; ++i) {                                                                  \
        const OcPage* e = &st->pages[ids[i]];                                                      \
        const int vs = valid_in_page(c, st, ids[i]);                                               \
        const REAL* sk = NULL;                                                                     \
        const REAL* sv = NULL;                                                                     \
        if (grads) {                                                                               \
            if (e->gk_phys >= 0) { sk = c->arena[e->gk_phys]; sv = c->arena[e->gv_phys]; }         \
        } else {                                                                                   \
            sk = c->arena[e->k_phys];                                                              \
            sv = c->arena[e->v_phys];                                                              \
        }                                                                                          \
        if (sk) {                                                                                  \
            memcpy(k + (int64_t)i * P * re, sk, (size_t)(vs * re) * sizeof(REAL));                 \
            memcpy(v + (int64_t)i * P * re, sv, (size_t)(vs * re) * sizeof(REAL));                 \
        }                                                                                          \
        for (int s = 0; s < vs; ++s) valid[(int64_t)i * P + s] = 1;                                \
    }                                                                                              \
    return OC_OK;                                                                                  \
}                                                                                                  \
                                                                                                   \
/* scatter_add_grads  paged_kv.hpp:135-164 */                                                      \
int oc_scatter_##SUF(OcCache* c, int layer, const int32_t* ids, int n, const REAL* dk,            \
                     const REAL* dv) {                                                             \
    if (!layer_ok(c, layer)) FAIL(OC_SHAPE, "cache: layer out of range");                          \
    int rc = check_resident(c, layer, ids, n);                                                     \
    if (rc) return rc;                                                                             \
    OcLayer* st = &c->layers[layer];                                                               \
    const int64_t re = row_elems(c), P = c->page_size;                                             \
    for (int i = 0; i < n; ++i) {                                                                  \
        OcPage* e = &st->pages[ids[i]];                                                            \
        if (e->gk_phys < 0) {                                                                      \
            e->gk_phys = alloc_page(c);                                                            \
            e->gv_phys = alloc_page(c);                                                            \
            memset(c->arena[e->gk_phys], 0, (size_t)page_elems(c) * sizeof(REAL));                 \
            memset(c->arena[e->gv_phys], 0, (size_t)page_elems(c) * sizeof(REAL));                 \
        }                                                                                          \
        const int vs = valid_in_page(c, st, ids[i]);                                               \
        REAL* gk = (REAL*)c->arena[e->gk_phys];                                                    \
        REAL* gv = (REAL*)c->arena[e->gv_phys];                                                    \
        const REAL* sk = dk + (int64_t)i * P * re;                                                 \
        const REAL* sv = dv + (int64_t)i * P * re;                                                 \
        for (int64_t j = 0; j < vs * re; ++j) {                                                    \
            gk[j] += sk[j];                                                                        \
            gv[j] += sv[j];                                                                        \
        }                                                                                          \
    }                                                                                              \
    return OC_OK;                                                                                  \
}                                                                                                  \
                                                                                                   \
/* score_pages  attention.hpp:32-67. Loop order t asc, h asc, p asc; Real accumulation. */         \
int oc_score_pages_##SUF(const REAL* q, int64_t tokens, int qh, int hd, const REAL* k_avg,        \
                         int64_t n, int kvh, int page_size, int gqa_group, int score_scale,        \
                         REAL* score) {                                                            \
    if (n < 1) FAIL(OC_SHAPE, "score_pages: needs at least one candidate page");                   \
    const int64_t m = (tokens + page_size - 1) / page_size;                                        \
    memset(score, 0, (size_t)(m * n) * sizeof(REAL));                                              \
    const REAL scale = score_scale ? (REAL)1 / SQRT((REAL)hd) : (REAL)1;                           \
    REAL* raw = (REAL*)malloc((size_t)n * sizeof(REAL));                                           \
    for (int64_t t = 0; t < tokens; ++t) {                                                         \
        const int64_t qpage = t / page_size;                                                       \
        for (int64_t h = 0; h < qh; ++h) {                                                         \
            const int64_t kh = h / gqa_group;                                                      \
            const REAL* qv = q + (t * qh + h) * hd;                                                \
            REAL mx = -(REAL)INFINITY;                                                             \
            for (int64_t p = 0; p < n; ++p) {                                                      \
                const REAL* kv = k_avg + (p * kvh + kh) * hd;                                      \
                REAL dot = 0;                                                                      \
                for (int64_t j = 0; j < hd; ++j) dot += qv[j] * kv[j];                             \
                raw[p] = dot * scale;                                                              \
                mx = (mx < raw[p]) ? raw[p] : mx;                                                  \
            }                                                                                      \
            REAL sum = 0;                                                                          \
            for (int64_t p = 0; p < n; ++p) {                                                      \
                raw[p] = EXP(raw[p] - mx);                                                         \
                sum += raw[p];                                                                     \
            }                                                                                      \
            const REAL inv = (REAL)1 / sum;                                                        \
            REAL* srow = score + qpage * n;                                                        \
            for (int64_t p = 0; p < n; ++p) srow[p] += raw[p] * inv;                               \
        }                                                                                          \
    }                                                                                              \
    free(raw);                                                                                     \
    return OC_OK;                                                                                  \
}                                                                                                  \
                                                                                                   \
/* OnlineRow::update  attention.hpp:128-147 */                                                     \
static void online_update_##SUF(REAL* m, REAL* l, REAL* acc, REAL logit, const REAL* v,           \
                                int64_t hd) {                                                      \
    if (logit > *m) {                                                                              \
        const REAL corr = (*l == (REAL)0) ? (REAL)0 : EXP(*m - logit);                             \
        for (int64_t j = 0; j < hd; ++j) acc[j] *= corr;                                           \
        *l *= corr;                                                                                \
        *m = logit;                                                                                \
    }                                                                                              \
    const REAL w = EXP(logit - *m);                                                                \
    *l += w;                                                                                       \
    for (int64_t j = 0; j < hd; ++j) acc[j] += w * v[j];                                           \
}                                                                                                  \
                                                                                                   \
/* attn_forward  attention.hpp:156-208. Selection as CSR over the m query pages:                   \
 * past pages in list order (valid slots only), then the chunk's causal prefix s = 0..t. */        \
int oc_attn_forward_##SUF(OcCache* c, int layer, int n_q_heads, const REAL* q, int64_t C,        \
                          const int32_t* sel_off, const int32_t* sel_ids, int64_t m,               \
                          const REAL* k_cur, const REAL* v_cur, REAL* out, REAL* lse) {            \
    const int64_t qh = n_q_heads, hd = c->head_dim, kvh_n = c->kv_heads;                           \
    const int64_t group = qh / kvh_n;                                                              \
    const REAL scale = (REAL)1 / SQRT((REAL)hd);                                                   \
    const int64_t P = c->page_size;                                                                \
    const int64_t n_qpages = (C + P - 1) / P;                                                      \
    if (m != n_qpages) FAIL(OC_SHAPE, "attn_forward: one selected-page list per query page required"); \
    REAL* acc = (REAL*)malloc((size_t)hd * sizeof(REAL));                                          \
    for (int64_t qp = 0; qp < n_qpages; ++qp) {                                                    \
        const int32_t* ids = sel_ids + sel_off[qp];                                                \
        const int n_ids = sel_off[qp + 1] - sel_off[qp];                                           \
        const int64_t past_rows = (int64_t)n_ids * P;                                              \
        REAL* gk = (REAL*)malloc((size_t)(past_rows * kvh_n * hd + 1) * sizeof(REAL));            \
        REAL* gv = (REAL*)malloc((size_t)(past_rows * kvh_n * hd + 1) * sizeof(REAL));            \
        uint8_t* valid = (uint8_t*)malloc((size_t)past_rows + 1);                                  \
        int rc = oc_gather_##SUF(c, layer, ids, n_ids, 0, gk, gv, valid);                          \
        if (rc) { free(gk); free(gv); free(valid); free(acc); return rc; }                         \
        const int64_t row_begin = qp * P;                                                          \
        const int64_t row_end = (C < row_begin + P) ? C : row_begin + P;                           \
        for (int64_t t = row_begin; t < row_end; ++t) {                                            \
            for (int64_t h = 0; h < qh; ++h) {                                                     \
                const int64_t kh = h / group;                                                      \
                const REAL* qv = q + (t * qh + h) * hd;                                            \
                REAL mm = -(REAL)INFINITY, l = 0;                                                  \
                for (int64_t j = 0; j < hd; ++j) acc[j] = 0;                                       \
                for (int64_t s = 0; s < past_rows; ++s) {                                          \
                    if (!valid[s]) continue;                                                       \
                    const REAL* kv = gk + (s * kvh_n + kh) * hd;                                   \
                    REAL dot = 0;                                                                  \
                    for (int64_t j = 0; j < hd; ++j) dot += qv[j] * kv[j];                         \
                    online_update_##SUF(&mm, &l, acc, dot * scale, gv + (s * kvh_n + kh) * hd, hd); \
                }                                                                                  \
                for (int64_t s = 0; s <= t; ++s) {                                                 \
                    const REAL* kv = k_cur + (s * kvh_n + kh) * hd;                                \
                    REAL dot = 0;                                                                  \
                    for (int64_t j = 0; j < hd; ++j) dot += qv[j] * kv[j];                         \
                    online_update_##SUF(&mm, &l, acc, dot * scale, v_cur + (s * kvh_n + kh) * hd, hd); \
                }                                                                                  \
                REAL* o = out + (t * qh + h) * hd;                                                 \
                const REAL inv = (REAL)1 / l;                                                      \
                for (int64_t j = 0; j < hd; ++j) o[j] = acc[j] * inv;                              \
                lse[t * qh + h] = mm + LOG(l);                                                     \
            }                                                                                      \
        }                                                                                          \
        free(gk); free(gv); free(valid);                                                           \
    }                                                                                              \
    free(acc);                                                                                     \
    return OC_OK;                                                                                  \
}                                                                                                  \
                                                                                                   \
/* attn_backward  attention.hpp:222-293. D = rowsum(dO*O) from the SAVED O; p rebuilt from the    \
 * saved LSE; past dK/dV accumulate per query page then scatter_add in qp order. */                \
int oc_attn_backward_##SUF(OcCache* c, int layer, int n_q_heads, const REAL* dout,               \
                           const REAL* q, int64_t C, const int32_t* sel_off,                       \
                           const int32_t* sel_ids, int64_t m, const REAL* k_cur,                   \
                           const REAL* v_cur, const REAL* saved_out, const REAL* saved_lse,        \
                           REAL* dq, REAL* dk_cur, REAL* dv_cur) {                                 \
    const int64_t qh = n_q_heads, hd = c->head_dim, kvh_n = c->kv_heads;                           \
    const int64_t group = qh / kvh_n;                                                              \
    const REAL scale = (REAL)1 / SQRT((REAL)hd);                                                   \
    const int64_t P = c->page_size;                                                                \
    const int64_t n_qpages = (C + P - 1) / P;                                                      \
    if (m != n_qpages) FAIL(OC_SHAPE, "attn_backward: one selected-page list per query page required"); \
    memset(dq, 0, (size_t)(C * qh * hd) * sizeof(REAL));                                           \
    memset(dk_cur, 0, (size_t)(C * kvh_n * hd) * sizeof(REAL));                                    \
    memset(dv_cur, 0, (size_t)(C * kvh_n * hd) * sizeof(REAL));                                    \
    for (int64_t qp = 0; qp < n_qpages; ++qp) {                                                    \
        const int32_t* ids = sel_ids + sel_off[qp];                                                \
        const int n_ids = sel_off[qp + 1] - sel_off[qp];                                           \
        const int64_t past_rows = (int64_t)n_ids * P;                                              \
        const size_t pe = (size_t)(past_rows * kvh_n * hd + 1);                                    \
        REAL* gk = (REAL*)malloc(pe * sizeof(REAL));                                               \
        REAL* gv = (REAL*)malloc(pe * sizeof(REAL));                                               \
        REAL* dk_past = (REAL*)calloc(pe, sizeof(REAL));                                           \
        REAL* dv_past = (REAL*)calloc(pe, sizeof(REAL));                                           \
        uint8_t* valid = (uint8_t*)malloc((size_t)past_rows + 1);                                  \
        int rc = oc_gather_##SUF(c, layer, ids, n_ids, 0, gk, gv, valid);                          \
        if (rc) { free(gk); free(gv); free(dk_past); free(dv_past); free(valid); return rc; }      \
        const int64_t row_begin = qp * P;                                                          \
        const int64_t row_end = (C < row_begin + P) ? C : row_begin + P;                           \
        for (int64_t t = row_begin; t < row_end; ++t) {                                            \
            for (int64_t h = 0; h < qh; ++h) {                                                     \
                const int64_t kh = h / group;                                                      \
                const REAL* qv = q + (t * qh + h) * hd;                                            \
                const REAL* dov = dout + (t * qh + h) * hd;                                        \
                const REAL* ov = saved_out + (t * qh + h) * hd;                                    \
                const REAL l_se = saved_lse[t * qh + h];                                           \
                REAL dcorr = 0;                                                                    \
                for (int64_t j = 0; j < hd; ++j) dcorr += dov[j] * ov[j];                          \
                REAL* dqv = dq + (t * qh + h) * hd;                                                \
                for (int64_t s = 0; s < past_rows + t + 1; ++s) {                                  \
                    const REAL *kv, *vv;                                                           \
                    REAL *dkv, *dvv;                                                               \
                    if (s < past_rows) {                                                           \
                        if (!valid[s]) continue;                                                   \
                        kv = gk + (s * kvh_n + kh) * hd;                                           \
                        vv = gv + (s * kvh_n + kh) * hd;                                           \
                        dkv = dk_past + (s * kvh_n + kh) * hd;                                     \
                        dvv = dv_past + (s * kvh_n + kh) * hd;                                     \
                    } else {                                                                       \
                        const int64_t sc = s - past_rows;                                          \
                        kv = k_cur + (sc * kvh_n + kh) * hd;                                       \
                        vv = v_cur + (sc * kvh_n + kh) * hd;                                       \
                        dkv = dk_cur + (sc * kvh_n + kh) * hd;                                     \
                        dvv = dv_cur + (sc * kvh_n + kh) * hd;                                     \
                    }                                                                              \
                    REAL dot = 0;                                                                  \
                    for (int64_t j = 0; j < hd; ++j) dot += qv[j] * kv[j];                         \
                    const REAL p = EXP(dot * scale - l_se);                                        \
                    REAL dov_dot_v = 0;                                                            \
                    for (int64_t j = 0; j < hd; ++j) dov_dot_v += dov[j] * vv[j];                  \
                    const REAL dlogit = p * (dov_dot_v - dcorr) * scale;                           \
                    for (int64_t j = 0; j < hd; ++j) {                                             \
                        dqv[j] += dlogit * kv[j];                                                  \
                        dkv[j] += dlogit * qv[j];                                                  \
                        dvv[j] += p * dov[j];                                                      \
                    }                                                                              \
                }                                                                                  \
            }                                                                                      \
        }                                                                                          \
        if (n_ids > 0) rc = oc_scatter_##SUF(c, layer, ids, n_ids, dk_past, dv_past);              \
        free(gk); free(gv); free(dk_past); free(dv_past); free(valid);                             \
        if (rc) return rc;                                                                         \
    }                                                                                              \
    return OC_OK;                                                                                  \
}                                                                                                  \
                                                                                                   \
/* naive_attention_fwd_bwd  oracle.hpp:293-357: query row t attends keys [0, past_len + t],        \
 * probabilities materialised; shares nothing with the streaming path. */                          \
int oc_naive_attention_##SUF(const REAL* q, int64_t tq, int qh, int hd, const REAL* k,            \
                             const REAL* v, int64_t tk, int kvh, int64_t past_len,                 \
                             const REAL* dout, int gqa_group, REAL* out, REAL* dq, REAL* dk,       \
                             REAL* dv) {                                                           \
    const REAL scale = (REAL)1 / SQRT((REAL)hd);                                                   \
    memset(out, 0, (size_t)(tq * qh * hd) * sizeof(REAL));                                         \
    memset(dq, 0, (size_t)(tq * qh * hd) * sizeof(REAL));                                          \
    memset(dk, 0, (size_t)(tk * kvh * hd) * sizeof(REAL));                                         \
    memset(dv, 0, (size_t)(tk * kvh * hd) * sizeof(REAL));                                         \
    REAL* p = (REAL*)malloc((size_t)(tk > 0 ? tk : 1) * sizeof(REAL));                             \
    for (int64_t t = 0; t < tq; ++t) {                                                             \
        const int64_t limit = (tk - 1 < past_len + t) ? tk - 1 : past_len + t;                     \
        for (int64_t hh = 0; hh < qh; ++hh) {                                                      \
            const int64_t kv = hh / gqa_group;                                                     \
            const REAL* qv = q + (t * qh + hh) * hd;                                               \
            REAL mx = -(REAL)INFINITY;                                                             \
            for (int64_t s = 0; s <= limit; ++s) {                                                 \
                REAL dot = 0;                                                                      \
                const REAL* kr = k + (s * kvh + kv) * hd;                                          \
                for (int64_t j = 0; j < hd; ++j) dot += qv[j] * kr[j];                             \
                p[s] = dot * scale;                                                                \
                mx = (mx < p[s]) ? p[s] : mx;                                                      \
            }                                                                                      \
            REAL sum = 0;                                                                          \
            for (int64_t s = 0; s <= limit; ++s) {                                                 \
                p[s] = EXP(p[s] - mx);                                                             \
                sum += p[s];                                                                       \
            }                                                                                      \
            for (int64_t s = 0; s <= limit; ++s) p[s] /= sum;                                      \
            REAL* ov = out + (t * qh + hh) * hd;                                                   \
            for (int64_t s = 0; s <= limit; ++s) {                                                 \
                const REAL* vr = v + (s * kvh + kv) * hd;                                          \
                for (int64_t j = 0; j < hd; ++j) ov[j] += p[s] * vr[j];                            \
            }                                                                                      \
            const REAL* dov = dout + (t * qh + hh) * hd;                                           \
            REAL dcorr = 0;                                                                        \
            for (int64_t s = 0; s <= limit; ++s) {                                                 \
                const REAL* vr = v + (s * kvh + kv) * hd;                                          \
                REAL dot = 0;                                                                      \
                for (int64_t j = 0; j < hd; ++j) dot += dov[j] * vr[j];                            \
                dcorr += p[s] * dot;                                                               \
            }                                                                                      \
            REAL* dqv = dq + (t * qh + hh) * hd;                                                   \
            for (int64_t s = 0; s <= limit; ++s) {                                                 \
                const REAL* kr = k + (s * kvh + kv) * hd;                                          \
                const REAL* vr = v + (s * kvh + kv) * hd;                                          \
                REAL dov_dot_v = 0;                                                                \
                for (int64_t j = 0; j < hd; ++j) dov_dot_v += dov[j] * vr[j];                      \
                const REAL dlogit = p[s] * (dov_dot_v - dcorr) * scale;                            \
                REAL* dkr = dk + (s * kvh + kv) * hd;                                              \
                REAL* dvr = dv + (s * kvh + kv) * hd;                                              \
                for (int64_t j = 0; j < hd; ++j) {                                                 \
                    dqv[j] += dlogit * kr[j];                                                      \
                    dkr[j] += dlogit * qv[j];                                                      \
                    dvr[j] += p[s] * dov[j];                                                       \
                }                                                                                  \
            }                                                                                      \
        }                                                                                          \
    }                                                                                              \
    free(p);                                                                                       \
    return OC_OK;                                                                                  \
}

DEFINE_ORACLE(float, f32, expf, logf, sqrtf)
DEFINE_ORACLE(double, f64, exp, log, sqrt)

/* kavg raw state for bit-exact checks of the device K_avg sums. */
int oc_cache_kavg_raw(const OcCache* c, int layer, void* sum_out, int32_t* count_out) {
    if (!layer_ok(c, layer)) FAIL(OC_SHAPE, "cache: layer out of range");
    const OcLayer* st = &c->layers[layer];
    memcpy(sum_out, st->kavg_sum, (size_t)st->n_pages * (size_t)row_elems(c) * (size_t)c->real_bytes);
    memcpy(count_out, st->kavg_count, (size_t)st->n_pages * sizeof(int32_t));
    return OC_OK;
}
