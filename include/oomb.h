/* SPDX-License-Identifier: Apache-2.0
 *
 * oomb.h — C ABI of the B200-native OOMB hot path (liboomb.so).
 *
 * The reference (/root/reference/proj) has no FFI: its operator API is the C++
 * template surface of paged_kv.hpp / attention.hpp / tiered_memory.hpp. Each
 * entry point below replaces one of those calls; the citation next to it is
 * the reference interface it stands in for (paths relative to
 * /root/reference/proj/core/include/chunktrain/). The host side of that API is
 * the C++ facade include/oomb.hpp (reference names and exceptions), mirrored in
 * Python (paper_2602_02108_b200/, ctypes); INTEGRATION.md shows the binding a
 * maintainer of the reference would add.
 *
 * Conventions
 *  - Every function returns an oomb_status; OOMB_OK == 0. The codes map 1:1
 *    onto the reference's exception classes (common.hpp:15-29) plus
 *    OOMB_CUDA_ERROR. oomb_last_error() holds the message (thread-local).
 *  - Tensor arguments are DEVICE pointers unless the name ends in _host.
 *    Layouts are the reference's row-major ones: q/out/dout/dq [tokens][Hq][hd],
 *    k/v/k_cur/v_cur/dk_cur/dv_cur [rows][Hkv][hd], lse [tokens][Hq].
 *  - Element types: q, k, v, k_cur, v_cur, out, dout use the pool dtype
 *    (OOMB_F32, OOMB_BF16 or OOMB_F64). lse, votes, dq, dk_cur, dv_cur, K_avg and the
 *    gradient pool use the pool's ACCUMULATION type: float for OOMB_F32 / OOMB_BF16 pools,
 *    double for OOMB_F64 pools (the reference's Real = double). Those arguments are
 *    declared void* (float* / double* convert implicitly). OOMB_F64 pools run the exact
 *    SIMT kernels; the tcgen05 kernels, RoPE epilogues, real offload and the page-range
 *    merge are bf16 / fp32 paths.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *    every call is stream-ordered and asynchronous unless documented.
 *  - Handles are not thread-safe.
 */
#ifndef OOMB_H_
#define OOMB_H_

#include <stdint.h>

#if defined(__GNUC__)
#define OOMB_API __attribute__((visibility("default")))
#else
#define OOMB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    OOMB_OK = 0,
    OOMB_CONFIG_ERROR = 1,    /* chunktrain::ConfigError    common.hpp:15-17 */
    OOMB_SHAPE_ERROR = 2,     /* chunktrain::ShapeError     common.hpp:18-20 */
    OOMB_STATE_ERROR = 3,     /* chunktrain::StateError     common.hpp:21-23 */
    OOMB_RESIDENCY_ERROR = 4, /* chunktrain::ResidencyError common.hpp:24-26 */
    OOMB_IO_ERROR = 5,        /* chunktrain::IoError        common.hpp:27-29 */
    OOMB_CUDA_ERROR = 6,
    OOMB_ERROR = 9
} oomb_status;

typedef enum { OOMB_F32 = 0, OOMB_BF16 = 1, OOMB_F64 = 2 } oomb_dtype;

/* ModelConfig fields on the path (config.hpp:19-49) + device sizing. */
typedef struct {
    int n_layers;
    int n_q_heads;
    int n_kv_heads;
    int head_dim;
    int chunk_size;       /* C */
    int page_size;        /* P */
    int retrieval_budget; /* B tokens; k = B / P pages per query page (config.hpp:41) */
    int local_window;     /* W pages */
    int score_scale;      /* 0 = unscaled vote (config.hpp:35-37) */
    int dtype;            /* oomb_dtype of the KV pool and the attention inputs */
    int64_t max_tokens;   /* per-layer capacity of the device page table */
    int64_t device_capacity_pages; /* KV page slots on the device, all layers; <= 0: n_layers*max_pages */
    /* Page-range shard ownership (appended fields, zero = off). With page_owner_stride
     * R > 1 this pool stores K/V and gradients only for the pages with id % R == page_owner_rank.
     * Every other page is REMOTE (tier 2): append still adds its rows to the page's K_avg sums
     * (pinned metadata, replicated on every shard, so every shard scores every candidate) but
     * stores no K/V, and any read of a REMOTE page raises OOMB_RESIDENCY_ERROR. The arena ids of
     * the reference page table are still assigned for every page. device_capacity_pages <= 0 then
     * defaults to the owned share, n_layers * ceil(max_pages / R): per-shard HBM is 1/R. */
    int page_owner_stride;
    int page_owner_rank;
} oomb_config;

typedef struct {
    uint64_t device_bytes; /* MemoryReport paged_kv.hpp:25-32 */
    uint64_t host_bytes;
    uint64_t grad_bytes;
    int64_t pages;
    int64_t reallocs;      /* always 0 */
    uint64_t copied_bytes; /* always 0 */
    int64_t arena_blocks;  /* PagedCache::arena_blocks_allocated paged_kv.hpp:249 */
    int64_t free_list;     /* PagedCache::free_list_size        paged_kv.hpp:250 */
} oomb_memory_report;

typedef struct oomb_pool_s* oomb_pool_t;           /* PagedCache<Real>          paged_kv.hpp:41 */
typedef struct oomb_selection_s* oomb_selection_t; /* AttnSaved::selected       attention.hpp:117-124 */
typedef struct oomb_pagetable_s* oomb_pagetable_t; /* PagedCache page table only (host logic) */

OOMB_API const char* oomb_last_error(void);
OOMB_API int oomb_version(void);
/* Number of sm_100a kernel launches issued by this process (for bench evidence). */
OOMB_API int64_t oomb_kernel_launches(void);

/* ---- lifecycle ---------------------------------------------------------- */
/* PagedCache(const ModelConfig&) + ModelConfig::validate  paged_kv.hpp:44-50, config.cpp:30-51 */
OOMB_API int oomb_pool_create(const oomb_config* cfg, int device, oomb_pool_t* out);
OOMB_API int oomb_pool_destroy(oomb_pool_t pool);
/* PagedCache::reset  paged_kv.hpp:227-242 */
OOMB_API int oomb_pool_reset(oomb_pool_t pool, void* stream);
/* PagedCache::zero_grad_pages  paged_kv.hpp:214-223 */
OOMB_API int oomb_zero_grad_pages(oomb_pool_t pool, void* stream);
/* PagedCache::memory_report  paged_kv.hpp:185-197 */
OOMB_API int oomb_memory_report_get(oomb_pool_t pool, oomb_memory_report* out);
/* Sticky device-side error flag raised by kernels; synchronises, reports, then clears it.
 * The forward does not copy a selection to the host unless residency is enforced, so a
 * selected id outside the layer's pages is skipped by the kernel and reported here as
 * OOMB_SHAPE_ERROR (the reference's gather throws ShapeError at the call); a read of a
 * non-resident slot is OOMB_RESIDENCY_ERROR. The backward and the enforced forward check the
 * ids on the host and fail at the call instead. */
OOMB_API int oomb_check_device_errors(oomb_pool_t pool);

/* ---- page table --------------------------------------------------------- */
/* PagedCache::append_chunk  paged_kv.hpp:73-108. k, v: [rows][Hkv][hd] device, pool dtype.
 * Writes tail slots in place and updates the K_avg fp32 sums in append order. */
OOMB_API int oomb_append_chunk(oomb_pool_t pool, int layer, const void* k, const void* v, int64_t rows, void* stream,
                      int64_t* slot_begin, int64_t* slot_end);
/* Fused projection epilogue (chunk_trainer.hpp:424-432): k_raw is the PRE-RoPE
 * key projection; every row is rotated at its absolute position (ops.hpp:192-225, angles and trig
 * in double) on its way into the page, and K_avg accumulates the rotated keys — the rotated K is
 * never written back to HBM separately. Same slot semantics as oomb_append_chunk. */
OOMB_API int oomb_append_chunk_rope(oomb_pool_t pool, int layer, const void* k_raw, const void* v, int64_t rows,
                                    float rope_base, void* stream, int64_t* slot_begin, int64_t* slot_end);
/* rope / rope_backward (ops.hpp:192-230) over [rows][heads][hd]: row r at position pos_offset + r,
 * sign +1 forward, -1 backward (the inverse rotation). dtypes OOMB_F32 / OOMB_BF16; out may
 * alias x. */
OOMB_API int oomb_rope(const void* x, int64_t rows, int heads, int hd, int64_t pos_offset, float base, int sign,
                       int in_dtype, int out_dtype, void* out, void* stream);
OOMB_API int oomb_n_pages(oomb_pool_t pool, int layer, int* n_pages);   /* paged_kv.hpp:62 */
OOMB_API int oomb_filled(oomb_pool_t pool, int layer, int64_t* filled); /* paged_kv.hpp:61 */
/* Reference arena ids {k_phys, v_phys, gk_phys, gv_phys} per logical page (PageEntry paged_kv.hpp:256-262). */
OOMB_API int oomb_page_table_get(oomb_pool_t pool, int layer, int32_t* out_host);
/* Device slots {kv_slot, grad_slot} per logical page (-1 = none / not resident). */
OOMB_API int oomb_device_slots_get(oomb_pool_t pool, int layer, int32_t* out_host);
/* PagedCache::page_mean_keys  paged_kv.hpp:170-183 -> out [n][Hkv][hd] fp32 device. */
OOMB_API int oomb_page_mean_keys(oomb_pool_t pool, int layer, int n_candidates, void* out, void* stream, int* n_out);
/* Raw K_avg state (sums [n][Hkv][hd] in the accumulation type, counts int32 [n]; device). */
OOMB_API int oomb_kavg_raw(oomb_pool_t pool, int layer, void* sum_out, int32_t* count_out, void* stream);
/* PagedCache::gather_pages / gather_grad_pages  paged_kv.hpp:118-130. ids on host; k/v out
 * [n*P][Hkv][hd] device (pool dtype for KV, fp32 for grads); valid [n*P] uint8 device. */
OOMB_API int oomb_gather_pages(oomb_pool_t pool, int layer, const int32_t* ids_host, int n, int grads, void* k_out,
                      void* v_out, uint8_t* valid_out, void* stream);
/* PagedCache::scatter_add_grads  paged_kv.hpp:135-164. dk/dv fp32 [n*P][Hkv][hd] device. */
OOMB_API int oomb_scatter_add_grads(oomb_pool_t pool, int layer, const int32_t* ids_host, int n, const void* dk,
                           const void* dv, void* stream);
/* Tier tags and residency enforcement  paged_kv.hpp:199-211. Tiers: 0 device, 1 host (the
 * reference's two), 2 remote (owned by another page-range shard), 3 lost (a host-tier page whose
 * pinned copy was dropped when a real offload engine detached without room to restore it).
 * Pages in tiers 2 and 3 cannot be re-tagged, and reading them always raises
 * OOMB_RESIDENCY_ERROR, enforcement or not. */
OOMB_API int oomb_set_tier(oomb_pool_t pool, int layer, int page, int tier);
OOMB_API int oomb_get_tier(oomb_pool_t pool, int layer, int page, int* tier);
OOMB_API int oomb_set_residency_enforced(oomb_pool_t pool, int on);
OOMB_API int oomb_grads_allocated(oomb_pool_t pool, int layer, int page, int* allocated);

/* ---- selection ---------------------------------------------------------- */
/* A selection is per query page: CSR (offsets[m+1], ids[]) in device memory, with an
 * asynchronously-maintained pinned host mirror. */
OOMB_API int oomb_selection_create(oomb_pool_t pool, int max_query_pages, int max_ids, oomb_selection_t* out);
OOMB_API int oomb_selection_destroy(oomb_selection_t sel);
/* Upload caller-provided lists (the reference's vector<vector<int32_t>>). */
OOMB_API int oomb_selection_set_host(oomb_selection_t sel, const int32_t* offsets_host, const int32_t* ids_host, int m,
                            void* stream);
/* Read back (waits for the mirror). offsets_host needs m+1 entries; ids_host nnz entries. */
OOMB_API int oomb_selection_get_host(oomb_selection_t sel, int32_t* offsets_host, int32_t* ids_host, int* m, int* nnz);
/* Device CSR pointers (int32). */
OOMB_API int oomb_selection_device(oomb_selection_t sel, const int32_t** offsets, const int32_t** ids, int* m);
/* select_all / select_recent  attention.hpp:99-111, broadcast to m query pages (chunk_trainer.hpp:301-304). */
OOMB_API int oomb_select_all(oomb_selection_t sel, int n_pages, int m, void* stream);
OOMB_API int oomb_select_recent(oomb_selection_t sel, int n_pages, int window, int m, void* stream);
/* Page-range shard: dst = the part of src this pool owns (ids with
 * id % page_owner_stride == page_owner_rank, each list's order kept), built on the device; the
 * host mirror follows asynchronously, as select_topk's does. A pool that owns every page copies. */
OOMB_API int oomb_selection_filter_owned(oomb_pool_t pool, oomb_selection_t src, oomb_selection_t dst, void* stream);
/* The pool's ownership (stride 1 / rank 0 when it owns every page). */
OOMB_API int oomb_page_owner(oomb_pool_t pool, int* stride, int* rank);
/* select_topk_row per row of a device vote matrix [m][n] fp32  attention.hpp:71-96:
 * k largest, ties to the lower id, ascending; k >= n -> all; k < 0 -> SHAPE_ERROR. */
OOMB_API int oomb_select_topk(oomb_selection_t sel, const void* vote, int m, int n, int k, void* stream);

/* ---- scoring ------------------------------------------------------------ */
/* score_pages  attention.hpp:32-67 on explicit representatives:
 * q [tokens][Hq][hd] (dtype), k_avg [n][Hkv][hd] fp32 -> vote [ceil(tokens/P)][n] fp32 device. */
OOMB_API int oomb_score_pages(const void* q, int64_t tokens, int n_q_heads, int head_dim, const void* k_avg, int64_t n,
                     int n_kv_heads, int page_size, int score_scale, int dtype, void* vote, void* stream);
/* The trainer's top-k selector in one call (chunk_trainer.hpp:305-311): K_avg of the first
 * n_candidates pages of `layer` (pinned metadata) -> score_pages -> select_topk_row per query page. */
OOMB_API int oomb_select_pages_topk(oomb_pool_t pool, int layer, const void* q, int64_t tokens, int n_candidates,
                           oomb_selection_t sel, void* vote_scratch, void* stream);

/* KV-group sharding support: the vote of score_pages sums over ALL q-heads
 * (attention.hpp:44-64). A rank holding a subset of KV groups computes per-group partial votes
 * [Hkv_local][m][n] fp32; after an all-gather in global group order, oomb_vote_reduce sums them in
 * that fixed order, so every rank (and the single-GPU path) selects identically. */
OOMB_API int oomb_score_pages_partial(oomb_pool_t pool, int layer, const void* q, int64_t tokens, int n_candidates,
                                      void* partials, void* stream);
OOMB_API int oomb_vote_reduce(const float* partials, int groups, int64_t m, int64_t n, float* vote, void* stream);

/* ---- attention ---------------------------------------------------------- */
/* attn_forward  attention.hpp:156-208: q [C][Hq][hd], k_cur/v_cur [C][Hkv][hd] (pool dtype) ->
 * out [C][Hq][hd] (pool dtype), lse [C][Hq] fp32 (natural log). */
OOMB_API int oomb_attn_forward(oomb_pool_t pool, int layer, const void* q, int64_t tokens, oomb_selection_t sel,
                      const void* k_cur, const void* v_cur, void* out, void* lse, void* stream);
/* attn_backward  attention.hpp:222-293: rebuilds P from the saved lse, D from the saved out;
 * past-page dK/dV are accumulated IN PLACE into the fp32 gradient pool (lazily allocated
 * and zeroed per page, reference order); dq/dk_cur/dv_cur fp32 are overwritten. */
OOMB_API int oomb_attn_backward(oomb_pool_t pool, int layer, const void* dout, const void* q, int64_t tokens,
                       oomb_selection_t sel, const void* k_cur, const void* v_cur, const void* out,
                       const void* lse, void* dq, void* dk_cur, void* dv_cur, void* stream);
/* Page-range split: a shard attends only its share of every query page's
 * selected pages. flags = OOMB_ATTN_PAST_ONLY drops the chunk's own causal keys (the shard that
 * owns them passes 0). The forward then writes that shard's partial (out, lse) — lse = -inf and
 * out = 0 for rows that attended no key; the backward, given the MERGED out / lse, writes the
 * shard's partial dq (summed over shards afterwards), its pages' dK/dV, and zeros in
 * dk_cur / dv_cur when the chunk's keys are not its own. Replaces the reference call sites
 * chunk_trainer.hpp:437 / :565 on a page-range shard. */
#define OOMB_ATTN_PAST_ONLY 1
/* Backward only: do not make `stream` wait for dq. The dQ kernel runs on the pool's side stream
 * concurrently with dK/dV and keeps running under the caller's next work (the next chunk's
 * backward); oomb_attn_join_dq makes a stream wait for every deferred dq. q, dout, k_cur, v_cur,
 * the selection and dq must stay untouched until then. */
#define OOMB_ATTN_DEFER_DQ 2
OOMB_API int oomb_attn_forward_ex(oomb_pool_t pool, int layer, const void* q, int64_t tokens, oomb_selection_t sel,
                                  const void* k_cur, const void* v_cur, void* out, void* lse, int flags,
                                  void* stream);
OOMB_API int oomb_attn_backward_ex(oomb_pool_t pool, int layer, const void* dout, const void* q, int64_t tokens,
                                   oomb_selection_t sel, const void* k_cur, const void* v_cur, const void* out,
                                   const void* lse, void* dq, void* dk_cur, void* dv_cur, int flags,
                                   void* stream);
/* Exact merge of page-range shards' partial attention outputs, shards in rank order:
 * o_parts [parts][rows][hd] (dtype), lse_parts [parts][rows] fp32 natural log ->
 * lse = ln sum_r e^{lse_r}, out = sum_r e^{lse_r - lse} o_r. rows = tokens * n_q_heads. */
/* The attention layer's whole chunk-recurrent step in one native call (chunk_trainer.hpp:131-186,
 * attention only): for chunks i = 0..n-1 select (mode: dense / top-k K_avg vote / local window over
 * the pages of chunks < i, :292-316) -> append_chunk -> attn_forward, then for i = n-1..0
 * attn_backward -> the dM_i read-back of the chunk's own pages into its dk_cur / dv_cur (:575-587).
 * Chunk i reads q[i % q_cycle], k[i], v[i], dout[i % dout_cycle] ([C][H][hd] blocks, pool dtype)
 * and writes out[i], lse[i] (accumulation type); its dq / dk_cur / dv_cur go to block
 * i * grad_stride_chunks of dq / dk_cur / dv_cur (grad_stride_chunks = 0: every chunk reuses block
 * 0). Selection of chunk i+1 overlaps chunk i's attention on a high-priority stream, consecutive
 * forwards run on two streams and dQ is deferred under the previous chunk's dK/dV: the same
 * results as the host loop, bitwise. Requires no page-range split (that runs in the host loop).
 * With a TieredEngine attached (oomb_tier_create on this pool, `stream` = its compute stream) the
 * step follows the residency protocol of chunk_trainer.hpp:328-363 / 409-462 / 531-592 exactly as
 * AttentionChunkLoop does: per chunk, fetch of the selection's union -> append -> on_pages_appended
 * -> wait + fill fetch + record_access -> attn_forward -> end_layer_use; backward after
 * release_all + begin_phase(backward): fetch + record_access of union(sel) + own pages, a
 * best-effort step-ahead prefetch of the previous chunk's, attn_backward (dQ not deferred: the
 * engine's write-backs follow the compute stream), on_grads_scattered, dM_i read-back,
 * end_layer_use. Every fetch decision waits for the selection's ids on the host; the selection of
 * chunk i+1 still runs on the side stream under chunk i's work. flags: OOMB_LAYER_FORWARD_ONLY runs
 * the forward alone; OOMB_LAYER_BACKWARD_ONLY then runs the backward of that forward (its
 * selections are kept). */
#define OOMB_MODE_DENSE 0
#define OOMB_MODE_TOPK 1
#define OOMB_MODE_LOCAL 2
#define OOMB_LAYER_FORWARD_ONLY 1
#define OOMB_LAYER_BACKWARD_ONLY 2
OOMB_API int oomb_layer_step(oomb_pool_t pool, int layer, int n_chunks, int mode, const void* q, int q_cycle,
                             const void* k, const void* v, const void* dout, int dout_cycle, void* out, void* lse,
                             void* dq, void* dk_cur, void* dv_cur, int64_t grad_stride_chunks, int flags,
                             void* stream);
/* Per-chunk residency records of the pool's last engine-attached oomb_layer_step: *n records of 5
 * int64 {phase (0 forward, 1 backward), chunk, pages the chunk needed resident, H2D bytes, D2H bytes
 * the engine moved during the chunk}; the first min(*n, cap) are written to out (may be null). */
OOMB_API int oomb_layer_stats(oomb_pool_t pool, int64_t* out, int64_t cap, int64_t* n);
/* oomb_attn_backward_ex + the dM_i read-back of the chunk's own pages own_first_page ..
 * own_first_page + tokens / P - 1 into dk_cur / dv_cur (what oomb_accumulate_grad_pages of those
 * pages does after the backward, chunk_trainer.hpp:575-587), done in the dK/dV kernel's store of the
 * chunk's own keys: the same two fp32 roundings, bit for bit, one launch fewer. tokens must be a
 * multiple of the page size and those pages appended. */
OOMB_API int oomb_attn_backward_readback(oomb_pool_t pool, int layer, const void* dout, const void* q, int64_t tokens,
                                         oomb_selection_t sel, const void* k_cur, const void* v_cur, const void* out,
                                         const void* lse, void* dq, void* dk_cur, void* dv_cur, int flags,
                                         int64_t own_first_page, void* stream);
/* Make `stream` wait for the dq of every earlier oomb_attn_backward_ex(..., OOMB_ATTN_DEFER_DQ). */
OOMB_API int oomb_attn_join_dq(oomb_pool_t pool, void* stream);
OOMB_API int oomb_lse_merge(const void* o_parts, const float* lse_parts, int parts, int64_t rows, int hd, int dtype,
                            void* out, float* lse, void* stream);
/* Kernel family selection: 0 = auto (tcgen05 when dtype bf16, hd 128, P % 128 == 0),
 * 1 = force the SIMT kernels, 2 = force tcgen05 (error if the shape is unsupported). */
OOMB_API int oomb_set_kernel_policy(oomb_pool_t pool, int policy);

/* dM_i read-back (chunk_trainer.hpp:575-587): dk[i*P+s] += grad_k(ids[i], s) and the same for
 * dv, reference layout [n*P][Hkv][hd] fp32 device; pages without gradients add 0. */
OOMB_API int oomb_accumulate_grad_pages(oomb_pool_t pool, int layer, const int32_t* ids_host, int n, void* dk,
                                        void* dv, void* stream);
/* The reverse projection epilogue (chunk_trainer.hpp:575-592): the dM_i read-back
 * followed by rope_backward of dK (ops.hpp:227-230) in one pass: dk <- rope^-1(dk + grad_k),
 * dv <- dv + grad_v, row r at absolute position pos_offset + r. Bitwise equal to
 * oomb_accumulate_grad_pages followed by oomb_rope(sign -1) on dk. */
OOMB_API int oomb_accumulate_grad_pages_rope(oomb_pool_t pool, int layer, const int32_t* ids_host, int n, float* dk,
                                             float* dv, int64_t pos_offset, float rope_base, void* stream);

/* ---- kernel timing evidence ---------------------------------------------
 * When enabled, every kernel the pool launches is bracketed by CUDA events on its
 * stream; oomb_profile_collect synchronises and returns, per kernel kind, the number of
 * launches and the summed device milliseconds, then clears the record.
 * Kinds: 0 append, 1 score, 2 topk, 3 attn_fwd, 4 bwd_prep, 5 bwd_dq, 6 bwd_dkdv,
 * 7 bwd_simt, 8 grad_init, 9 gather/scatter, 10 other, 11 bwd_pair (the span of the dq and dkdv
 * kernels, which run concurrently: dq on a library side stream). */
OOMB_API int oomb_profile_enable(oomb_pool_t pool, int on);
OOMB_API int oomb_profile_collect(oomb_pool_t pool, int64_t* counts, double* ms, int n_kinds);

/* ---- tiered residency / offload (TieredEngine, tiered_memory.hpp:99-432) ----
 * The policy is the reference's, decision for decision: LRU eviction of unreserved pages
 * (unpinned first), reserved / pinned states, all-or-nothing best-effort prefetch with
 * append headroom, write-back of dirty K/V and gradient pages only, capacity errors.
 * Created on a pool, pages really move: evictions D2H-copy dirty K/V (+dK/dV) into a
 * pinned host pool on a D2H stream and free the device slot; fetches H2D-copy into a fresh
 * slot on an H2D stream; wait() makes the compute stream wait on the copy and publishes
 * the slot in the device page table. Log timestamps then come from CUDA events.
 * Created on a bare page table (no device), the engine runs the reference's simulated
 * clock (bandwidth + cost model) and its log matches the reference event for event. */
typedef struct oomb_tier_s* oomb_tier_t;
typedef struct {
    int64_t device_capacity_pages; /* -1 = unlimited (TierConfig, tiered_memory.hpp:74-78) */
    double bandwidth_bytes_per_s;  /* simulated link (simulation mode) */
    double fixed_s_per_layer;      /* ComputeCostModel :58-72 */
    double s_per_attended_token;
} oomb_tier_config;
typedef struct { /* ScheduleEvent tiered_memory.hpp:36-44 */
    int32_t kind; /* 0 fetch_issued, 1 fetch_done, 2 evict, 3 compute_begin, 4 compute_end, 5 access */
    int32_t layer;
    int32_t page;
    int32_t chunk;
    int32_t phase; /* 0 forward, 1 backward */
    int32_t pad;
    uint64_t bytes;
    double t;
} oomb_event;
OOMB_API int oomb_tier_create_sim(oomb_pagetable_t pt, const oomb_tier_config* cfg, oomb_tier_t* out);
OOMB_API int oomb_tier_create(oomb_pool_t pool, const oomb_tier_config* cfg, void* compute_stream, oomb_tier_t* out);
OOMB_API int oomb_tier_destroy(oomb_tier_t t);
OOMB_API int oomb_tier_begin_phase(oomb_tier_t t, int phase);
OOMB_API int oomb_tier_set_prefetch_headroom(oomb_tier_t t, int64_t pages);
OOMB_API int oomb_tier_on_pages_appended(oomb_tier_t t, int layer, int64_t slot_begin, int64_t slot_end);
OOMB_API int oomb_tier_on_grads_scattered(oomb_tier_t t, int layer, const int32_t* ids_host, int n);
OOMB_API int oomb_tier_fetch_async(oomb_tier_t t, int layer, const int32_t* ids_host, int n, int chunk, int best_effort,
                                   int64_t* handle);
OOMB_API int oomb_tier_wait(oomb_tier_t t, int64_t handle);
OOMB_API int oomb_tier_record_access(oomb_tier_t t, int layer, const int32_t* ids_host, int n, int chunk);
OOMB_API int oomb_tier_advance_compute(oomb_tier_t t, double seconds, int chunk, int layer);
OOMB_API int oomb_tier_end_layer_use(oomb_tier_t t, int layer, const int32_t* ids_host, int n);
OOMB_API int oomb_tier_release_all(oomb_tier_t t);
/* Real engine: fetch every host-tier page back into free device slots (K/V and gradient blocks)
 * and mark it resident; OOMB_CONFIG_ERROR, moving nothing, if the pool lacks the slots. Not in
 * the reference (its engine only tags pages); oomb_tier_destroy calls it when the pool has room,
 * so detaching an engine does not drop the data of pages it left on the host. */
OOMB_API int oomb_tier_restore_all(oomb_tier_t t);
/* out[5] = {now, stall_seconds, h2d_bytes forward, h2d_bytes backward, d2h_bytes} */
OOMB_API int oomb_tier_stats(oomb_tier_t t, double* out);
OOMB_API int oomb_tier_log(oomb_tier_t t, oomb_event* out, int64_t cap, int64_t* n);
/* Real engine: bytes actually copied host->device and device->host (d2h_moved may be null).
 * oomb_tier_stats counts the reference's transfer bytes (every fetch and write-back decision,
 * tiered_memory.hpp:322-326, 386-403). A page fetched back before the device slots its eviction
 * freed are handed out again takes them back without a copy. With OOMB_TIER_LAZY_WB=1 in the
 * environment at engine creation, the write-back itself is deferred until the freed slot nears the
 * front of its free list (OOMB_TIER_CLEAN_AHEAD slots, default 256) or is handed out, and dropped
 * if the page is fetched back first. */
OOMB_API int oomb_tier_moved_bytes(oomb_tier_t t, int64_t* h2d_moved, int64_t* d2h_moved);
/* validate_schedule (tiered_memory.cpp:47-138): out[6] = {stall_s, transfer_bytes, h2d_fwd, h2d_bwd,
 * d2h, overlap_fraction}; n_violations = residency/order violations found. When viol_event / viol_code
 * are non-null, the first viol_cap violations are described by the index of the offending event (-1 for
 * the end-of-log check) and a code: 1 evict of non-resident page, 2 access before fetch_done (or after
 * evict), 3 compute timestamps decrease, 4 nested compute_begin, 5 compute_end without begin, 6 compute
 * segment ends before it begins, 7 unterminated compute segment — the reference's message list. */
OOMB_API int oomb_validate_schedule(const oomb_event* events, int64_t n, double bandwidth, double* out,
                                    int* n_violations, int64_t* viol_event, int32_t* viol_code, int64_t viol_cap);

/* ---- page-table host logic (no device) -----------------------------------
 * The arena / LIFO free-list / lazy-gradient-page bookkeeping of PagedCache
 * (paged_kv.hpp:73-108,135-164,227-242,280-288), exposed on its own so that it is
 * testable without a GPU. The pool owns one of these. */
OOMB_API int oomb_pagetable_create(int n_layers, int page_size, int n_kv_heads, int head_dim, int kv_elem_bytes,
                          int grad_elem_bytes, oomb_pagetable_t* out);
OOMB_API int oomb_pagetable_destroy(oomb_pagetable_t pt);
OOMB_API int oomb_pagetable_append(oomb_pagetable_t pt, int layer, int64_t rows, int64_t* slot_begin, int64_t* slot_end);
OOMB_API int oomb_pagetable_scatter(oomb_pagetable_t pt, int layer, const int32_t* ids_host, int n);
OOMB_API int oomb_pagetable_reset(oomb_pagetable_t pt);
OOMB_API int oomb_pagetable_n_pages(oomb_pagetable_t pt, int layer, int* n);
OOMB_API int oomb_pagetable_get(oomb_pagetable_t pt, int layer, int32_t* out_host);
OOMB_API int oomb_pagetable_set_tier(oomb_pagetable_t pt, int layer, int page, int tier);
OOMB_API int oomb_pagetable_memory_report(oomb_pagetable_t pt, oomb_memory_report* out);

/* ---- debug / evidence ------------------------------------------------------ */
/* One 128xNxK bf16 tcgen05 GEMM tile through the same TMA/UMMA building blocks the
 * attention kernels use (validation of descriptor layouts). mode 0: C = A B^T with
 * A [M][K], B [N][K] (both K-major); mode 1: C = A B with B [K][N] (MN-major B).
 * M = 128, N in {64,128,256}, K % 64 == 0. C fp32 [M][N]. */
OOMB_API int oomb_debug_tc_gemm(int mode, const void* a, const void* b, float* c, int m, int n, int k, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* OOMB_H_ */
