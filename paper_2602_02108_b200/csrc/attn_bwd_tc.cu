// SPDX-License-Identifier: Apache-2.0
//
// tcgen05 backward of the paged chunk attention (attention.hpp:222-293),
// deterministic (no floating-point atomics):
//
//   bwd_prep      D[h][t] = sum_d dO*O (saved O, attention.hpp:253-256) and
//                 L[h][t] = lse*log2(e), head-major for broadcast reads.
//   bwd_sched     per past page: bitmask of the query pages that selected it; the ascending union
//                 of selected pages (the backward's key blocks); the dK/dV units longest first.
//   attn_bwd_dq   query-major: S = Q K^T, dP = dO V^T, dS = P (dP - D),
//                 dQ += dS K over the query page's selected pages then the
//                 chunk's causal prefix; dQ written once (fp32).
//   attn_bwd_dkdv key-major: one CTA owns one (key block, kv head) and loops over
//                 every (128-row query tile, q-head of the group) that attends it:
//                 S^T = K Q^T, dP^T = V dO^T, dV += P^T dO, dK += dS^T Q with
//                 dK/dV accumulated in TMEM, then ONE read-modify-write into the
//                 fp32 gradient pool (past pages) or a store to dk_cur/dv_cur
//                 (the chunk's own keys). Pages never selected are not touched.

#include <algorithm>
#include <cub/block/block_scan.cuh>

#include "tc_common.cuh"

namespace oomb {

#ifndef OOMB_BWD_KV_FIRST
#define OOMB_BWD_KV_FIRST 0  // launch order of the pair (both orders measured equal at c3)
#endif

using namespace tc;

namespace {

#ifndef OOMB_BWD_POLY
#define OOMB_BWD_POLY 0  // measured: no gain (the P phase is latency-, not MUFU-bound)
#endif
#ifndef OOMB_DQ_POLY_N
#define OOMB_DQ_POLY_N 4  // measured: dQ 44.75 -> 41.67 ms (256K c3, serialized) with OOMB_DQ_X2
#endif
#ifndef OOMB_KV_POLY_N
#define OOMB_KV_POLY_N (OOMB_BWD_POLY ? 4 : 0)
#endif
constexpr int kDqPolyN = OOMB_DQ_POLY_N;  // dQ kernel: 1 in N exp2 of P on the FMA pipe (ex2_poly; 0: none)
constexpr int kKvPolyN = OOMB_KV_POLY_N;  // dK/dV kernel: the same for P^T
#ifndef OOMB_POLY_LEAN
#define OOMB_POLY_LEAN 1  // ex2_lean (1 ALU op) instead of ex2_poly (4) for the FMA-pipe share
#endif
#ifndef OOMB_DQ_X2
#define OOMB_DQ_X2 1  // dQ kernel softmax arithmetic as packed fp32 pairs (FFMA2 / FADD2 / FMUL2)
#endif
#ifndef OOMB_KV_X2
#define OOMB_KV_X2 0  // the same in the dK/dV kernel
#endif
__device__ __forceinline__ float ex2_mix(float x, int c, int n) {
    return (n > 0 && c % n == n - 1) ? (OOMB_POLY_LEAN ? ex2_lean(x) : ex2_poly(x)) : ex2(x);
}
// Elements c, c + 1 (c even): 1 pair in n on the FMA pipe as a packed pair (ex2_lean2: 10 issue
// slots for two exponentials instead of 16), the others on the MUFU. n = 0: all on the MUFU.
__device__ __forceinline__ float2 ex2_pair(float2 x, int c, int n) {
    if (n > 0 && (c >> 1) % n == n - 1) return ex2_lean2(x);
    return make_float2(ex2(x.x), ex2(x.y));
}
#ifndef OOMB_DQ_PAIR_N
#define OOMB_DQ_PAIR_N 4  // dQ: 1 pair in N of P's exponentials as an FMA-pipe packed pair (replaces
                          // OOMB_DQ_POLY_N): 42.13 -> 41.62 ms serialized (256K c3)
#endif
#ifndef OOMB_KV_PAIR_N
#define OOMB_KV_PAIR_N 4  // the same for the dK/dV kernel's P^T: 57.53 -> 56.01 ms (N = 2: 56.30)
#endif
constexpr int kDqPairN = OOMB_DQ_PAIR_N, kKvPairN = OOMB_KV_PAIR_N;

#ifndef OOMB_BWD_LPT
#define OOMB_BWD_LPT 1  // dK/dV units longest first (bwd_order_kernel); 0: own blocks, then union order
#endif

#ifndef OOMB_DQ_SPLIT
#define OOMB_DQ_SPLIT 1  // split-K of the dQ kernel over key blocks when the grid is small (attn_tc_splits)
#endif

#ifndef OOMB_KV_TRACE
#define OOMB_KV_TRACE 0  // per-CTA wait / phase cycle counters of the dK/dV kernel (OOMB_CTA_TRACE=dkdv:i:file)
#endif
#if OOMB_KV_TRACE
#define KVT_WAIT(acc, bar, ph)                      \
    do {                                            \
        const long long t0_ = clock64();            \
        mbar_wait(bar, ph);                         \
        acc += clock64() - t0_;                     \
    } while (0)
#define KVT(...) __VA_ARGS__
#else
#define KVT_WAIT(acc, bar, ph) mbar_wait(bar, ph)
#define KVT(...)
#endif


// ---------------------------------------------------------------- workspace
struct BwdWs {
    float* Dt;        // [Hq][C]
    float* Lt;        // [Hq][C]
    uint64_t* mask;   // [max_pages]
    int32_t* uni;     // [max_pages]
    int32_t* n_uni;   // [1] (+ the dK/dV work counter)
    int32_t* order;   // [chunk blocks + max_pages * blocks per page]: dK/dV units, longest first
};

inline int bwd_blocks_per_page(const AttnGeom& g) { return g.P == kHalf ? 1 : std::max(1, g.P / kTile); }

BwdWs carve(const AttnGeom& g, void* ws) {
    uint8_t* p = static_cast<uint8_t*>(ws);
    BwdWs w;
    const size_t hc = static_cast<size_t>(g.Hq) * g.C * sizeof(float);
    w.Dt = reinterpret_cast<float*>(p);
    w.Lt = reinterpret_cast<float*>(p + hc);
    size_t off = (2 * hc + 255) & ~size_t(255);
    w.mask = reinterpret_cast<uint64_t*>(p + off);
    off += static_cast<size_t>(g.max_pages) * 8;
    w.uni = reinterpret_cast<int32_t*>(p + off);
    off += static_cast<size_t>(g.max_pages) * 4;
    w.n_uni = reinterpret_cast<int32_t*>(p + off);
    off = (off + 8 + 255) & ~size_t(255);
    w.order = reinterpret_cast<int32_t*>(p + off);
    return w;
}

// ---------------------------------------------------------------- prep kernels
__device__ __forceinline__ void bwd_prep_body(const __nv_bfloat16* __restrict__ o,
                                              const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse,
                                              int C, int Hq, int hd, float* __restrict__ Dt, float* __restrict__ Lt,
                                              int block) {
    // two (token, head) rows per warp: up to 16 lanes x 16 B of O and dO each (hd 64: 8 lanes)
    const int64_t row = (static_cast<int64_t>(block) * (blockDim.x / 32) + (threadIdx.x >> 5)) * 2 +
                        ((threadIdx.x >> 4) & 1);
    const int l16 = threadIdx.x & 15;
    const bool ok = row < static_cast<int64_t>(C) * Hq;
    float s = 0.f;
    if (ok && l16 * 8 < hd) {
        const uint4 a = reinterpret_cast<const uint4*>(o + row * hd)[l16];
        const uint4 b = reinterpret_cast<const uint4*>(dout + row * hd)[l16];
        const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 fa = __bfloat1622float2(a2[i]);
            const float2 fb = __bfloat1622float2(b2[i]);
            s += fa.x * fb.x + fa.y * fb.y;
        }
    }
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (ok && l16 == 0) {
        const int t = static_cast<int>(row / Hq), h = static_cast<int>(row % Hq);
        Dt[static_cast<int64_t>(h) * C + t] = s;
        Lt[static_cast<int64_t>(h) * C + t] = lse[row] * kLog2e;
    }
}

// pages the layer holds: ids at or past this are out of range (never past the pool's table)
inline int layer_pages(const AttnGeom& g) {
    return static_cast<int>(std::min<int64_t>(g.max_pages, (g.filled + g.P - 1) / g.P));
}



// The backward's schedule in ONE single-CTA launch (a chunk's backward is a dozen small launches
// on short histories, so each one counts): clear the page -> query-page bitmask and the dK/dV
// work counter, build the mask from the selection, the ascending union of the selected pages and,
// when `order` is given, the dK/dV work units longest first (LPT) so the persistent grid does not
// end on a long unit: unit codes [0, ncb) are the chunk's own key blocks (block b is attended by the
// ncb - b query tiles from its diagonal on), codes ncb + k * bpp + sub the past blocks of the k-th
// union page (attended by popcount(mask) query pages x tpq tiles each). Units write disjoint
// gradient rows, so the order changes the schedule only, never a result bit.
__device__ __forceinline__ void bwd_sched_body(const int32_t* __restrict__ off, const int32_t* __restrict__ ids,
                                               int m, int layer_pages, int n_pages, uint64_t* __restrict__ mask,
                                               int32_t* __restrict__ uni, int32_t* __restrict__ n_uni, int ncb,
                                               int bpp, int tpq, int32_t* __restrict__ order, int* err) {
    using Scan = cub::BlockScan<int, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    constexpr int kKeys = 256;
    __shared__ int hist[kKeys], cur[kKeys];
    const int tid = threadIdx.x;
    for (int p = tid; p < n_pages; p += 1024) mask[p] = 0ull;
    for (int i = tid; i < kKeys; i += 1024) hist[i] = 0;
    if (tid == 0) n_uni[1] = 0;  // the dK/dV kernel's work counter
    __syncthreads();
    const int nnz = m > 0 ? off[m] : 0;
    for (int i = tid; i < nnz; i += 1024) {
        int lo = 0, hi = m;  // the list holding entry i: the last qp with off[qp] <= i
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (off[mid] <= i) lo = mid;
            else hi = mid;
        }
        const int pid = ids[i];
        if (pid < 0 || pid >= layer_pages) {
            atomicOr(err, DERR_BAD_ID);
            continue;
        }
        atomicOr(reinterpret_cast<unsigned long long*>(mask + pid), 1ull << lo);
    }
    __syncthreads();
    const int per = (n_pages + 1023) / 1024;
    const int p0 = min(n_pages, tid * per), p1 = min(n_pages, p0 + per);
    int cnt = 0;
    for (int p = p0; p < p1; ++p) cnt += mask[p] != 0ull;
    int pos, total;
    Scan(tmp).ExclusiveSum(cnt, pos, total);
    for (int p = p0; p < p1; ++p)
        if (mask[p] != 0ull) uni[pos++] = p;
    if (tid == 0) n_uni[0] = total;
    if (!order) return;
    __syncthreads();
    const int units = ncb + total * bpp;
    auto key = [&](int u) {
        const int k = u < ncb ? ncb - u : __popcll(mask[uni[(u - ncb) / bpp]]) * tpq;
        return min(k, kKeys - 1);
    };
    for (int u = tid; u < units; u += 1024) atomicAdd(&hist[key(u)], 1);
    __syncthreads();
    if (tid == 0) {
        int at = 0;
        for (int k = kKeys - 1; k >= 0; --k) {
            cur[k] = at;
            at += hist[k];
        }
    }
    __syncthreads();
    for (int u = tid; u < units; u += 1024) order[atomicAdd(&cur[key(u)], 1)] = u;
}

// The backward's two preparation steps in ONE launch of 1024-thread blocks: block 0 builds the
// schedule (bwd_sched_body) while blocks 1.. compute D = rowsum(dO * O) and the log2 LSE, 64
// (token, head) rows each.
__global__ void __launch_bounds__(1024) bwd_prep_sched_kernel(
    const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse, int C,
    int Hq, int hd, float* __restrict__ Dt, float* __restrict__ Lt, const int32_t* __restrict__ off,
    const int32_t* __restrict__ ids, int m, int layer_pages, int n_pages, uint64_t* __restrict__ mask,
    int32_t* __restrict__ uni, int32_t* __restrict__ n_uni, int ncb, int bpp, int tpq, int32_t* __restrict__ order,
    int* err) {
    if (blockIdx.x == 0) bwd_sched_body(off, ids, m, layer_pages, n_pages, mask, uni, n_uni, ncb, bpp, tpq, order, err);
    else bwd_prep_body(o, dout, lse, C, Hq, hd, Dt, Lt, static_cast<int>(blockIdx.x) - 1);
}

// ===========================================================================
// dQ kernel (query-major): one CTA per (128-row query tile, q-head), looping over the key
// blocks the tile attends (its query page's selected pages, then the chunk's causal prefix).
//
// Every MMA is a TS-MMA (A from TMEM), so shared memory supplies only B operands:
//   Q and dO are staged into TMEM once (bf16 packed, 64 columns each);
//   S = Q K^T and dP = dO V^T land in TMEM; the softmax warpgroups turn S into P as soon as
//   S is ready (the exp work, overlapping dQ of the previous block and dP of this one), then
//   dS = P (dP - D) is written back IN PLACE of dP as packed bf16 and dQ += dS K runs with
//   dS as the TMEM A operand. dQ is scaled and stored once, by TMA, at the end.
// TMEM (the CTA owns all 512 columns, base 0): Q [0,64) dO [64,128) S [128,256) dP [256,384)
// dQ [384,512). Warpgroup w owns key columns [64w, 64w+64) of every block; its packed dS
// goes to dP columns [256+64w, 256+64w+32) (its own region: the other group may still be
// reading its dP columns).
// ===========================================================================
#ifndef OOMB_DQ_KST
#define OOMB_DQ_KST 3
#endif
#ifndef OOMB_DQ_ALIAS
#define OOMB_DQ_ALIAS 0  // measured equal at c3 (468.4 vs 468.7 ms backward pass)
#endif
// Q and dO are read from shared memory only once (staged into TMEM at the start), so with
// OOMB_DQ_ALIAS their tiles double as the 4th K stage and the 1st V stage (layout
// K0 K1 K2 Q=K3 | dO=V0 V1 V2); the producers wait for the TMEM staging before first reuse.
constexpr bool kDqAlias = OOMB_DQ_ALIAS != 0;
constexpr int kDqKSt = kDqAlias ? 4 : OOMB_DQ_KST;
constexpr int kDqVSt = kDqAlias ? 3 : 5 - OOMB_DQ_KST;  // K / V stages (3 / 2: 2 / 3 measured 6 % slower)
constexpr int kDqK = kDqAlias ? 0 : 2 * kTileBytes;     // kDqKSt stages
constexpr int kDqQ = kDqAlias ? 3 * kTileBytes : 0;
constexpr int kDqDO = kDqQ + kTileBytes;
constexpr int kDqV = kDqAlias ? kDqDO : kDqK + kDqKSt * kTileBytes;  // kDqVSt stages
constexpr int kDqBar = kDqV + kDqVSt * kTileBytes;
constexpr int kDqNv = kDqBar + 256;                 // uint8 valid-key counts of the past blocks
constexpr int kDqNvCap = 1024;
constexpr int kDqSmem = kDqNv + kDqNvCap + 1024;
static_assert(kDqSmem <= 232448, "dynamic shared memory above the 227 KB opt-in limit");
constexpr uint32_t kDqTmQ = 0, kDqTmDO = 64, kDqTmS = 128, kDqTmDP = 256, kDqTmDQ = 384;

struct DqBars {
    uint64_t qdo_full, qdo_tmem;
    uint64_t k_full[kDqKSt], k_empty[kDqKSt], v_full[kDqVSt], v_empty[kDqVSt];
    uint64_t s_full, s_free, dp_full, ds_full, dq_done;
    uint32_t tmem_base;
};

struct BwdParams {
    AttnGeom g;
    const int32_t* sel_off;
    const int32_t* sel_ids;
    const int32_t* kvslot;
    const int32_t* gslot;
    float* gk;
    float* gv;
    const float* Dt;
    const float* Lt;
    const uint64_t* mask;
    const int32_t* uni;
    const int32_t* n_uni;
    const int32_t* order;  // dK/dV unit order (null: identity)
    float* dq;
    float* dk_cur;
    float* dv_cur;
    int* err;
    CtaTrace tr;  // debug CTA timeline (OOMB_CTA_TRACE)
    // >= 0: first page id of the chunk's own pages; the dK/dV epilogue of the chunk's own key blocks
    // adds those pages' pool gradients (the dM_i read-back, chunk_trainer.hpp:575-587) before the
    // store: fl(fl(dK * scale) + pool), the same two roundings as the store + accumulate_grads pass
    int readback_first;
};

// dQ-kernel K step ks (16 keys) of the packed dS operand: keys [64w, 64w+64) of warpgroup w
// sit in dP columns [64w, 64w+32).
__host__ __device__ constexpr uint32_t ds_col(int ks) { return (ks >> 2) * 64 + (ks & 3) * 8; }

__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_kc, const __grid_constant__ CUtensorMap tm_vc,
                       const __grid_constant__ CUtensorMap tm_kp, const __grid_constant__ CUtensorMap tm_vp,
                       const __grid_constant__ CUtensorMap tmap_dq, BwdParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    DqBars* bars = reinterpret_cast<DqBars*>(smem + kDqBar);
    const AttnGeom& g = p.g;
    const int h = blockIdx.x;
    const int qt = (g.C / kTile) - 1 - blockIdx.y;  // longest causal prefixes first
    const int kvh = h / g.group;
    const bool p64 = g.P == kHalf;  // two query pages per tile, 64-key half blocks (tc_common.cuh)
    const int qp = (qt * kTile) / g.P;
    const int sel_begin = p.sel_off[qp];
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        mbar_init(&bars->qdo_full, 1);
        mbar_init(&bars->qdo_tmem, 256);
        for (int i = 0; i < kDqKSt; ++i) {
            mbar_init(&bars->k_full[i], 1);
            mbar_init(&bars->k_empty[i], 1);
        }
        for (int i = 0; i < kDqVSt; ++i) {
            mbar_init(&bars->v_full[i], 1);
            mbar_init(&bars->v_empty[i], 1);
        }
        mbar_init(&bars->s_full, 1);
        mbar_init(&bars->s_free, 256);
        mbar_init(&bars->dp_full, 1);
        mbar_init(&bars->ds_full, 256);
        mbar_init(&bars->dq_done, 1);
        fence_barrier_init();
    }
    if (warp == 3) tmem_alloc<512>(&bars->tmem_base);
    tc_fence_before();
    HalfList hl{};
    if (p64) hl = half_list_sync(p.sel_off, p.sel_ids, qt);  // (a barrier, like the one it replaces)
    else __syncthreads();
    tc_fence_after();
    if (bars->tmem_base != 0) __trap();  // all 512 columns: base column 0 (the constants rely on it)
    const int n_past = p64 ? hl.blocks() : (p.sel_off[qp + 1] - sel_begin) * (g.P / kTile);
    const int nb_all = n_past + (g.chunk_keys ? qt + 1 : 0);
    // split-K (small grids, attn_tc_splits): CTA z attends key blocks [j0, j0 + nb) and stores its
    // partial dQ at rows z C + t of the partial buffer; dq_split_sum adds the splits in z order
    const int zs = static_cast<int>(gridDim.z), z = static_cast<int>(blockIdx.z);
    const int j0 = static_cast<int>(static_cast<int64_t>(nb_all) * z / zs);
    const int nb = static_cast<int>(static_cast<int64_t>(nb_all) * (z + 1) / zs) - j0;
    uint8_t* sQ = smem + kDqQ;
    uint8_t* sDO = smem + kDqDO;
    uint8_t* sK = smem + kDqK;
    uint8_t* sV = smem + kDqV;

    if (warp == 0) {
        if (lane == 0) {  // Q, dO, K producer
            mbar_expect_tx(&bars->qdo_full, 2 * kTileBytes);
            for (int r = 0; r < 2; ++r) {
                tma_load_3d(sQ + r * kRegion, &tm_q, &bars->qdo_full, r * 64, h, qt * kTile);
                tma_load_3d(sDO + r * kRegion, &tm_do, &bars->qdo_full, r * 64, h, qt * kTile);
            }
            for (int j = 0; j < nb; ++j) {
                const int st = j % kDqKSt;
                if (j >= kDqKSt) mbar_wait(&bars->k_empty[st], ((j / kDqKSt) - 1) & 1);
                if (kDqAlias && j == 3) mbar_wait(&bars->qdo_tmem, 0);  // K stage 3 is the Q tile
                mbar_expect_tx(&bars->k_full[st], kTileBytes);
                uint8_t* dst = sK + st * kTileBytes;
                const int jb = j0 + j;
                if (jb < n_past && p64) {
                    for (int hh = 0; hh < 2; ++hh) {
                        const int row = past_half_row(g, p.sel_ids, p.kvslot, hl, 2 * jb + hh, kvh, p.err);
                        for (int r = 0; r < 2; ++r)
                            tma_load_2d(dst + r * kRegion + hh * (kRegion / 2), &tm_kp, &bars->k_full[st], r * 64, row);
                    }
                } else if (jb < n_past) {
                    const PastBlock b = past_block(g, p.sel_ids, p.kvslot, sel_begin, jb, kvh, p.err);
                    for (int r = 0; r < 2; ++r) tma_load_2d(dst + r * kRegion, &tm_kp, &bars->k_full[st], r * 64, b.row);
                } else {
                    for (int r = 0; r < 2; ++r)
                        tma_load_3d(dst + r * kRegion, &tm_kc, &bars->k_full[st], r * 64, kvh, (jb - n_past) * kTile);
                }
            }
        }
    } else if (warp == 2) {
        if (lane == 0) {  // V producer
            for (int j = 0; j < nb; ++j) {
                const int st = j % kDqVSt;
                if (j >= kDqVSt) mbar_wait(&bars->v_empty[st], ((j / kDqVSt) - 1) & 1);
                if (kDqAlias && j == 0) mbar_wait(&bars->qdo_tmem, 0);  // V stage 0 is the dO tile
                mbar_expect_tx(&bars->v_full[st], kTileBytes);
                uint8_t* dst = sV + st * kTileBytes;
                const int jb = j0 + j;
                if (jb < n_past && p64) {
                    for (int hh = 0; hh < 2; ++hh) {
                        const int row = past_half_row(g, p.sel_ids, p.kvslot, hl, 2 * jb + hh, kvh, nullptr);
                        for (int r = 0; r < 2; ++r)
                            tma_load_2d(dst + r * kRegion + hh * (kRegion / 2), &tm_vp, &bars->v_full[st], r * 64, row);
                    }
                } else if (jb < n_past) {
                    const PastBlock b = past_block(g, p.sel_ids, p.kvslot, sel_begin, jb, kvh, nullptr);
                    for (int r = 0; r < 2; ++r) tma_load_2d(dst + r * kRegion, &tm_vp, &bars->v_full[st], r * 64, b.row);
                } else {
                    for (int r = 0; r < 2; ++r)
                        tma_load_3d(dst + r * kRegion, &tm_vc, &bars->v_full[st], r * 64, kvh, (jb - n_past) * kTile);
                }
            }
        }
    } else if (warp == 1) {
        // MMA warp (converged). Order: S(0) dP(0) | S(1) dQ(0) dP(1) | S(2) dQ(1) dP(2) | ... dQ(nb-1).
        constexpr uint32_t idesc_s = make_idesc_bf16(kTile, kTile, 0, 0);  // [128 q] x [128 keys], K = hd
        // N = hd: at head dim 64 only the 64 real columns (the epilogue never reads the others)
        const uint32_t idesc_q = make_idesc_bf16(kTile, g.hd == 64 ? 64 : kHd, 0, 1);  // [128 q] x [hd], K = keys
        // K = hd contractions: at head dim 64 the k-steps over the zero-padded columns 64-127 would
        // add exact zeros, so they are not issued
        const int nks_hd = g.hd / 16;
        const uint64_t dK = sdesc_k(smem_u32(sK)), dV = sdesc_k(smem_u32(sV));
        const uint64_t dKmn = sdesc_mn(smem_u32(sK), kRegion);
        mbar_wait(&bars->qdo_tmem, 0);
        tc_fence_after();
        auto mma_s = [&](int j) {
            const int st = j % kDqKSt;
            mbar_wait(&bars->k_full[st], (j / kDqKSt) & 1);
            if (j >= 1) mbar_wait(&bars->s_free, (j - 1) & 1);  // softmax read S(j-1) into registers
            tc_fence_after();
            const uint64_t so = boff(st * kTileBytes);
            if (nks_hd == kHd / 16) {
#pragma unroll
                for (int ks = 0; ks < kHd / 16; ++ks) umma_ts_w(kDqTmS, kDqTmQ + ks * 8, dK + so + koff(ks, kRegion), idesc_s, ks);
            } else {  // head dim 64
#pragma unroll
                for (int ks = 0; ks < kHd / 32; ++ks) umma_ts_w(kDqTmS, kDqTmQ + ks * 8, dK + so + koff(ks, kRegion), idesc_s, ks);
            }
            umma_commit_w(&bars->s_full);
        };
        auto mma_dp = [&](int j) {
            const int st = j % kDqVSt;
            mbar_wait(&bars->v_full[st], (j / kDqVSt) & 1);
            tc_fence_after();
            const uint64_t so = boff(st * kTileBytes);
            if (nks_hd == kHd / 16) {
#pragma unroll
                for (int ks = 0; ks < kHd / 16; ++ks) umma_ts_w(kDqTmDP, kDqTmDO + ks * 8, dV + so + koff(ks, kRegion), idesc_s, ks);
            } else {  // head dim 64
#pragma unroll
                for (int ks = 0; ks < kHd / 32; ++ks) umma_ts_w(kDqTmDP, kDqTmDO + ks * 8, dV + so + koff(ks, kRegion), idesc_s, ks);
            }
            umma_commit_w(&bars->dp_full);
            umma_commit_w(&bars->v_empty[st]);
        };
        auto mma_dq = [&](int j) {
            const int st = j % kDqKSt;
            mbar_wait(&bars->ds_full, j & 1);
            tc_fence_after();
            const uint64_t so = boff(st * kTileBytes);
            const uint32_t first = j == 0 ? 0u : 1u;
#pragma unroll
            for (int ks = 0; ks < kTile / 16; ++ks)
                umma_ts_w(kDqTmDQ, kDqTmDP + ds_col(ks), dKmn + so + mnoff(ks), idesc_q, first | ks);
            umma_commit_w(&bars->k_empty[st]);
        };
        if (nb > 0) {
            mma_s(0);
            mma_dp(0);
            for (int j = 1; j < nb; ++j) {
                mma_s(j);
                mma_dq(j - 1);  // dS(j-1) lives in the dP columns: dP(j) is issued after it
                mma_dp(j);
            }
            mma_dq(nb - 1);
        }
        umma_commit_w(&bars->dq_done);
    } else if (warp >= 4) {
        const int quarter = warp & 3, wg = (warp - 4) >> 2;
        const int r = quarter * 32 + lane;  // query row of the tile = TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        // ---- stage Q (group 0) / dO (group 1) rows into TMEM
        mbar_wait(&bars->qdo_full, 0);
        stage_row_tmem(wg ? sDO : sQ, kRegion, r, (wg ? kDqTmDO : kDqTmQ) + lane_off);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars->qdo_tmem);
        const int t = qt * kTile + r;
        const float sl2 = g.scale * kLog2e;
        const float L2 = p.Lt[static_cast<int64_t>(h) * g.C + t];
        const float Dr = p.Dt[static_cast<int64_t>(h) * g.C + t];
        const uint32_t tS = kDqTmS + wg * 64 + lane_off, tDP = kDqTmDP + wg * 64 + lane_off;
        uint8_t* nvt = smem + kDqNv;
        uint16_t* hvt = reinterpret_cast<uint16_t*>(nvt);
        if (p64) stage_half_valid(g, p.sel_ids, hl, hvt, kDqNvCap / 2, threadIdx.x - 128, 256);
        else stage_past_valid(g, p.sel_ids, sel_begin, n_past, nvt, kDqNvCap, threadIdx.x - 128, 256);
        named_bar_sync(3, 256);
        for (int j = 0; j < nb; ++j) {
            int lim;  // keep key columns c <= lim (of this group's 64)
            const int jb = j0 + j;
            if (jb < n_past && p64) {  // the group's 64 columns are half block 2 jb + wg
                lim = half_lim(half_valid(g, p.sel_ids, hl, hvt, kDqNvCap / 2, 2 * jb + wg), r);
            } else if (jb < n_past) {
                lim = past_valid(g, p.sel_ids, sel_begin, nvt, kDqNvCap, jb) - 1 - wg * 64;
            } else {
                lim = ((jb - n_past == qt) ? r : kTile - 1) - wg * 64;
            }
            // ---- P = exp2(S * scale * log2e - L) for this group's 64 key columns
            mbar_wait(&bars->s_full, j & 1);
            tc_fence_after();
            float pr[64];
            {
                uint32_t a[32], b2[32];
                tmem_ld32(tS, a);
                tmem_ld32(tS + 32, b2);
                tmem_wait_ld();
                tc_fence_before();
                mbar_arrive(&bars->s_free);
                if (OOMB_DQ_X2) {
                    const float2 s2 = make_float2(sl2, sl2), nl2 = make_float2(-L2, -L2);
#pragma unroll
                    for (int c = 0; c < 32; c += 2) {
                        const float2 x = fma2(make_float2(__uint_as_float(a[c]), __uint_as_float(a[c + 1])), s2, nl2);
                        const float2 y = fma2(make_float2(__uint_as_float(b2[c]), __uint_as_float(b2[c + 1])), s2, nl2);
                        if (kDqPairN > 0) {
                            const float2 ex = ex2_pair(x, c, kDqPairN), ey = ex2_pair(y, 32 + c, kDqPairN);
                            pr[c] = ex.x;
                            pr[c + 1] = ex.y;
                            pr[32 + c] = ey.x;
                            pr[33 + c] = ey.y;
                        } else {
                            pr[c] = ex2_mix(x.x, c, kDqPolyN);
                            pr[c + 1] = ex2_mix(x.y, c + 1, kDqPolyN);
                            pr[32 + c] = ex2_mix(y.x, 32 + c, kDqPolyN);
                            pr[33 + c] = ex2_mix(y.y, 33 + c, kDqPolyN);
                        }
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const float x = fmaf(__uint_as_float(a[c]), sl2, -L2);
                        pr[c] = ex2_mix(x, c, kDqPolyN);
                    }
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const float x = fmaf(__uint_as_float(b2[c]), sl2, -L2);
                        pr[32 + c] = ex2_mix(x, 32 + c, kDqPolyN);
                    }
                }
            }
            if (lim < 63) {
#pragma unroll
                for (int c = 0; c < 64; ++c) pr[c] = (c <= lim) ? pr[c] : 0.f;
            }
            // ---- dS = P (dP - D), packed bf16 into this group's first 32 dP columns
            mbar_wait(&bars->dp_full, j & 1);
            tc_fence_after();
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) {
                uint32_t d[32];
                tmem_ld32(tDP + c2 * 32, d);
                tmem_wait_ld();
                uint32_t pk[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    if (OOMB_DQ_X2) {
                        const float2 t = add2(make_float2(__uint_as_float(d[2 * u]), __uint_as_float(d[2 * u + 1])),
                                              make_float2(-Dr, -Dr));
                        const float2 v = mul2(make_float2(pr[c2 * 32 + 2 * u], pr[c2 * 32 + 2 * u + 1]), t);
                        pk[u] = pack_bf16(v.x, v.y);
                    } else {
                        pk[u] = pack_bf16(pr[c2 * 32 + 2 * u] * (__uint_as_float(d[2 * u]) - Dr),
                                          pr[c2 * 32 + 2 * u + 1] * (__uint_as_float(d[2 * u + 1]) - Dr));
                    }
                }
                tmem_st16(tDP + c2 * 16, pk);  // below the columns still to be read
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&bars->ds_full);
        }
        // ---- dQ (scaled) leaves TMEM as four [128 x 32] fp32 slices staged in the idle K / V
        // stages (group w: slices 2w, 2w+1), then one TMA tile store each into dq [C][Hq][hd].
        mbar_wait(&bars->dq_done, 0);
        tc_fence_after();
        uint8_t* stage = sK;
#pragma unroll 1
        for (int c = 2 * wg; c < 2 * wg + 2; ++c) {
            if (nb > 0) {
                stage_slice(kDqTmDQ + c * 32 + lane_off, stage + c * kSliceBytes, r, g.scale);
            } else {  // a page-range shard with no key for this tile: dQ = 0 (TMEM was never written)
#pragma unroll
                for (int u = 0; u < 8; ++u) st_slice_f32(stage + c * kSliceBytes, r, u, make_float4(0.f, 0.f, 0.f, 0.f));
            }
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 256);
        if (warp == 4 && lane == 0) {
            for (int c = 0; c < g.hd / 32; ++c)
                tma_store_3d(&tmap_dq, stage + c * kSliceBytes, c * 32, h, z * g.C + qt * kTile);
            bulk_commit();
            bulk_wait_read0();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 3) tmem_dealloc<512>(0);
}

// ===========================================================================
// dK/dV kernel (key-major, persistent)
//
// A work unit is one 128-key block (a past page, or a block of the chunk's own keys) of one kv
// head; its items are the (128-row query tile, q-head of the group) pairs that attend it — the
// query pages that selected the page, or the chunk's tiles from the diagonal on. One CTA per SM
// takes units from an atomic counter in longest-first order (bwd_order_kernel) and overlaps
// consecutive units: the next unit's K/V and first Q/dO tiles load, and its first S^T/dP^T MMAs
// run, while the previous unit finishes and drains its accumulators.
// Per item:
//   S^T = K Q^T, dP^T = V dO^T   SS-MMAs with N = 128 queries (full rate);
//   P^T = exp2(S^T scale log2e - L)  written back IN PLACE of S^T as packed bf16 as soon as
//                                S^T lands, kept in registers for
//   dS^T = P^T (dP^T - D)        written back in place of dP^T;
//   dV += P^T dO, dK += dS^T Q   TS-MMAs (A from TMEM), accumulated over the unit's items.
// Issue order: S(0) dP(0) | dV(0) S(1) dK(0) dP(1) | dV(1) S(2) dK(1) dP(2) | ... — each MMA
// that rewrites S^T / dP^T columns is issued after the MMA that read them, and tcgen05.mma
// operations of one thread execute in issue order.
// Epilogue of a unit: the softmax warps pull dK (scaled) / dV out of TMEM into registers, free
// the accumulators, then stage [128 x 32] fp32 slices in smem for the TMA unit to ADD into the
// fp32 gradient page in L2 (past pages: one owner per (page, kv head, block) per launch, so the
// result is deterministic) or STORE into dk_cur / dv_cur (the chunk's own keys).
// TMEM (all 512 columns, base 0): S^T [0,128) dP^T [128,256) dK [256,384) dV [384,512);
// softmax warpgroup w owns query columns [64w, 64w+64) and packs into its own first 32.
// ===========================================================================
constexpr int kKvStages = 2;
constexpr int kKvK = 0;
constexpr int kKvV = kKvK + kTileBytes;
constexpr int kKvQ = kKvV + kTileBytes;                  // kKvStages stages of [128 x 128]
constexpr int kKvDO = kKvQ + kKvStages * kTileBytes;     // kKvStages stages
constexpr int kKvStage = kKvDO + kKvStages * kTileBytes; // epilogue: one [128 x 32] fp32 slice per warpgroup
constexpr int kKvLD = kKvStage + 2 * kSliceBytes;        // kKvStages stages of {L[128], D[128]} fp32 (TMA bulk)
constexpr int kKvUnitBytes = 160;
constexpr int kKvDesc = kKvLD + kKvStages * 1024;        // 2 unit descriptors
constexpr int kKvBar = kKvDesc + 2 * kKvUnitBytes;
constexpr int kKvSmem = kKvBar + 256;                    // the dynamic smem base is 1024-aligned (checked)
static_assert(kKvSmem <= 232448, "dynamic shared memory above the 227 KB opt-in limit");
constexpr uint32_t kTmS = 0, kTmDP = 128, kTmDK = 256, kTmDV = 384;
// Softmax warpgroups of the dK/dV kernel: each owns kKvCols query columns of every item (2: 64
// columns each; 4: 32 each, half the per-thread exp / dS chain). With 4 the epilogue stays on
// warpgroups 0 / 1 (dK / dV) in two TMEM-load rounds (register budget). Measured: 4 is bitwise
// equal and 2.6 % slower at c3 (the P^T phase only drops 1,388 -> 1,316 clk per item: it is bound
// by the SM's 16 exp2/clk, 1,024 clk for an item's 16K exponentials, not by the per-thread chain).
#ifndef OOMB_KV_WG
#define OOMB_KV_WG 2
#endif
constexpr int kKvWg = OOMB_KV_WG;
static_assert(kKvWg == 2 || kKvWg == 4, "dK/dV softmax warpgroups: 2 or 4");
constexpr int kKvCols = kTile / kKvWg;
constexpr int kKvThreads = 128 + 128 * kKvWg;
constexpr int kKvEpR = kKvWg == 4 ? 2 : 1;  // epilogue TMEM-load rounds
constexpr int kKvEpC = 4 / kKvEpR;          // 32-column slices per round

struct KvBars {
    uint64_t unit_full[2], unit_empty[2];
    uint64_t kv_full, kv_empty;
    uint64_t qdo_full[kKvStages], qdo_empty[kKvStages];
    uint64_t s_full, dp_full, p_full, ds_full;
    uint64_t acc_done, acc_free;
    uint32_t tmem_base;
};

// A work unit as the scheduler publishes it to the MMA and softmax warps.
struct KvUnit {
    uint8_t valid;
    uint8_t past;
    uint8_t has1;  // page size 64: a past unit is two pages of the ascending union, keys [0,64) and [64,128)
    uint8_t n_qps; // past: number of query pages in the list (page size 64: of 128-row query tiles)
    int key0;      // first key of the block (chunk-relative for in-chunk, page-relative for past)
    int n_items;
    int g_kv;
    int kv_row;    // pool tensor-map row of the K/V block (past; page size 64: of the first page)
    int g_row;     // grad-pool tensor-map row (past; page size 64: of the first page)
    int n_valid;   // valid keys of the block (page size 64: of the first page)
    int kv_row1, g_row1, n_valid1;  // page size 64: the second page
    uint64_t qm0, qm1;  // the query pages that selected each page (bit qp)
    uint8_t qps[64];  // past: the query pages that selected the page, ascending (page size 64: query tiles)
};
static_assert(sizeof(KvUnit) <= 120, "unit descriptor");
static_assert(sizeof(KvUnit) <= kKvUnitBytes, "unit descriptor");

// K step ks (16 queries) of a packed P^T / dS^T operand: queries [kKvCols w, kKvCols (w + 1)) of
// warpgroup w sit in the first kKvCols / 2 of its own kKvCols columns.
__host__ __device__ constexpr uint32_t pk_col(int ks) {
    return (ks / (kKvCols / 16)) * kKvCols + (ks % (kKvCols / 16)) * 8;
}

// Items of a unit in order: past units walk (query page of the list, 128-row tile of the page,
// q-head of the group) head-fastest; in-chunk units walk (128-row tile from the key block's
// diagonal on, q-head). Advanced incrementally (no integer division on the per-item path).
struct ItemIter {
    int h, qt, qpi, tile;  // q-head, 128-row query tile, index in the query-page list, tile in the page
    bool diag;
    __device__ __forceinline__ void init(const KvUnit& u, int G, int tpq) {
        h = u.g_kv * G;
        qpi = 0;
        tile = 0;
        if (u.past) {
            qt = u.qps[0] * tpq;
            diag = false;
        } else {
            qt = u.key0 / kTile;
            diag = true;
        }
    }
    __device__ __forceinline__ void next(const KvUnit& u, int G, int tpq) {
        if (++h < (u.g_kv + 1) * G) return;
        h = u.g_kv * G;
        if (!u.past) {
            ++qt;
            diag = false;
            return;
        }
        if (++tile == tpq) {
            tile = 0;
            ++qpi;
            if (qpi < u.n_qps) qt = u.qps[qpi] * tpq;
        } else {
            ++qt;
        }
    }
};

// Decode work index w (through the longest-first order when there is one: unit codes are the chunk's
// own blocks first, then past page blocks; kv head
// fastest) into a unit descriptor.
__device__ void decode_unit(const BwdParams& p, int w, KvUnit& u) {
    const AttnGeom& g = p.g;
    const bool p64 = g.P == kHalf;
    const int n_chunk_blocks = g.chunk_keys ? g.C / kTile : 0, bpp = g.P / kTile;
    const int n_past_units = p64 ? (*p.n_uni + 1) / 2 : *p.n_uni * bpp;
    const int n_units = (n_chunk_blocks + n_past_units) * g.Hkv;
    u.valid = w < n_units;
    u.has1 = 0;
    u.qm0 = u.qm1 = 0ull;
    if (!u.valid) return;
    const int unit = p.order ? p.order[w / g.Hkv] : w / g.Hkv;
    u.g_kv = w % g.Hkv;
    u.n_valid = kTile;
    if (unit < n_chunk_blocks) {
        u.past = 0;
        u.key0 = unit * kTile;
        u.n_items = (n_chunk_blocks - unit) * g.group;
        u.n_qps = 0;
        return;
    }
    const int pu = unit - n_chunk_blocks;
    if (p64) {  // two consecutive pages of the union; items = the 128-row tiles either page is attended by
        u.past = 1;
        u.key0 = 0;
        const int pa = p.uni[2 * pu];
        u.has1 = 2 * pu + 1 < *p.n_uni;
        const int pb = u.has1 ? p.uni[2 * pu + 1] : pa;
        u.qm0 = p.mask[pa];
        u.qm1 = u.has1 ? p.mask[pb] : 0ull;
        const uint64_t any = u.qm0 | u.qm1;
        int k = 0;
        for (int qt = 0; qt < 32; ++qt)
            if ((any >> (2 * qt)) & 3ull) u.qps[k++] = static_cast<uint8_t>(qt);
        u.n_qps = k;
        u.n_items = k * g.group;
        const int64_t nva = g.filled - static_cast<int64_t>(pa) * g.P, nvb = g.filled - static_cast<int64_t>(pb) * g.P;
        u.n_valid = static_cast<int>(nva < 0 ? 0 : (nva > kHalf ? kHalf : nva));
        u.n_valid1 = u.has1 ? static_cast<int>(nvb < 0 ? 0 : (nvb > kHalf ? kHalf : nvb)) : 0;
        const int ka = p.kvslot[pa], ga = p.gslot[pa];
        const int kb = p.kvslot[pb], gb = p.gslot[pb];
        if (ka < 0 || ga < 0 || (u.has1 && (kb < 0 || gb < 0))) {
            atomicOr(p.err, DERR_NOT_RESIDENT);
            u.n_items = 0;
            u.kv_row = u.g_row = u.kv_row1 = u.g_row1 = 0;
            return;
        }
        u.kv_row = (ka * g.Hkv + u.g_kv) * g.P;
        u.g_row = (ga * g.Hkv + u.g_kv) * g.P;
        u.kv_row1 = u.has1 ? (kb * g.Hkv + u.g_kv) * g.P : -2 * kHalf;  // out of bounds: TMA zero fill
        u.g_row1 = u.has1 ? (gb * g.Hkv + u.g_kv) * g.P : 0;
        return;
    }
    const int pid = p.uni[pu / bpp];
    const int sub = pu % bpp;
    u.past = 1;
    u.key0 = sub * kTile;
    const uint64_t m = p.mask[pid];
    int k = 0;
    for (int qp = 0; qp < 64; ++qp)
        if (m & (1ull << qp)) u.qps[k++] = static_cast<uint8_t>(qp);
    u.n_qps = k;
    u.n_items = k * bpp * g.group;
    const int kv_slot = p.kvslot[pid], g_slot = p.gslot[pid];
    const int64_t nv = g.filled - static_cast<int64_t>(pid) * g.P - u.key0;
    u.n_valid = static_cast<int>(nv < 0 ? 0 : (nv > kTile ? kTile : nv));
    if (kv_slot < 0 || g_slot < 0) {  // not resident: report, and do no work for it
        atomicOr(p.err, DERR_NOT_RESIDENT);
        u.n_items = 0;
        u.kv_row = u.g_row = 0;
        return;
    }
    u.kv_row = (kv_slot * g.Hkv + u.g_kv) * g.P + u.key0;
    u.g_row = (g_slot * g.Hkv + u.g_kv) * g.P + u.key0;
}

__global__ void __launch_bounds__(kKvThreads, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                         const __grid_constant__ CUtensorMap tm_kc, const __grid_constant__ CUtensorMap tm_vc,
                         const __grid_constant__ CUtensorMap tm_kp, const __grid_constant__ CUtensorMap tm_vp,
                         const __grid_constant__ CUtensorMap tm_gk, const __grid_constant__ CUtensorMap tm_gv,
                         const __grid_constant__ CUtensorMap tm_dkc, const __grid_constant__ CUtensorMap tm_dvc,
                         BwdParams p, int* work_counter) {
    extern __shared__ __align__(1024) uint8_t smem[];
    KvBars* bars = reinterpret_cast<KvBars*>(smem + kKvBar);
    KvUnit* desc = reinterpret_cast<KvUnit*>(smem + kKvDesc);  // 2 x kKvUnitBytes
    const AttnGeom& g = p.g;
    const bool p64 = g.P == kHalf;
    const int tpq = p64 ? 1 : g.P / kTile;  // page size 64: a past unit lists 128-row query tiles directly
    const int warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023) __trap();  // SW128 operands and the smem budget need a 1 KB-aligned base
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->unit_full[i], 1);
            mbar_init(&bars->unit_empty[i], 1 + 128 * kKvWg);
        }
        mbar_init(&bars->kv_full, 1);
        mbar_init(&bars->kv_empty, 1);
        for (int i = 0; i < kKvStages; ++i) {
            mbar_init(&bars->qdo_full[i], 1);
            mbar_init(&bars->qdo_empty[i], 1);
        }
        mbar_init(&bars->s_full, 1);
        mbar_init(&bars->dp_full, 1);
        mbar_init(&bars->p_full, 128 * kKvWg);
        mbar_init(&bars->ds_full, 128 * kKvWg);
        mbar_init(&bars->acc_done, 1);
        mbar_init(&bars->acc_free, 128 * kKvWg);
        fence_barrier_init();
    }
    if (warp == 3) tmem_alloc<512>(&bars->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (bars->tmem_base != 0) __trap();  // all 512 columns: base column 0 (the constants rely on it)
    uint8_t* sK = smem + kKvK;
    uint8_t* sV = smem + kKvV;
    uint8_t* sQ = smem + kKvQ;
    uint8_t* sDO = smem + kKvDO;

    if (warp == 0) {
        if (lane == 0) {  // scheduler + TMA producer
            int gi = 0;
            KVT(long long w_qe = 0; long long w_kve = 0; long long w_ue = 0;)
            for (int un = 0;; ++un) {
                const int k = un & 1;
                if (un >= 2) KVT_WAIT(w_ue, &bars->unit_empty[k], ((un >> 1) - 1) & 1);
                KvUnit& u = desc[k];
                decode_unit(p, atomicAdd(work_counter, 1), u);
                mbar_arrive(&bars->unit_full[k]);  // release: the descriptor is visible to the waiters
                if (!u.valid) break;
                if (un >= 1) KVT_WAIT(w_kve, &bars->kv_empty, (un - 1) & 1);  // the previous unit's last S / dP
                mbar_expect_tx(&bars->kv_full, 2 * kTileBytes);
                for (int r = 0; r < 2; ++r) {
                    if (u.past && p64) {  // two 64-row pages (pool maps with 64-row boxes)
                        tma_load_2d(sK + r * kRegion, &tm_kp, &bars->kv_full, r * 64, u.kv_row);
                        tma_load_2d(sV + r * kRegion, &tm_vp, &bars->kv_full, r * 64, u.kv_row);
                        tma_load_2d(sK + r * kRegion + kRegion / 2, &tm_kp, &bars->kv_full, r * 64, u.kv_row1);
                        tma_load_2d(sV + r * kRegion + kRegion / 2, &tm_vp, &bars->kv_full, r * 64, u.kv_row1);
                    } else if (u.past) {
                        tma_load_2d(sK + r * kRegion, &tm_kp, &bars->kv_full, r * 64, u.kv_row);
                        tma_load_2d(sV + r * kRegion, &tm_vp, &bars->kv_full, r * 64, u.kv_row);
                    } else {
                        tma_load_3d(sK + r * kRegion, &tm_kc, &bars->kv_full, r * 64, u.g_kv, u.key0);
                        tma_load_3d(sV + r * kRegion, &tm_vc, &bars->kv_full, r * 64, u.g_kv, u.key0);
                    }
                }
                ItemIter it;
                it.init(u, g.group, tpq);
                for (int i = 0; i < u.n_items; ++i, ++gi, it.next(u, g.group, tpq)) {
                    const int st = gi % kKvStages;
                    if (gi >= kKvStages) KVT_WAIT(w_qe, &bars->qdo_empty[st], ((gi / kKvStages) - 1) & 1);
                    mbar_expect_tx(&bars->qdo_full[st], 2 * kTileBytes + 1024);
                    float* ld = reinterpret_cast<float*>(smem + kKvLD) + st * 256;
                    bulk_load(ld, p.Lt + static_cast<int64_t>(it.h) * g.C + it.qt * kTile, 512, &bars->qdo_full[st]);
                    bulk_load(ld + 128, p.Dt + static_cast<int64_t>(it.h) * g.C + it.qt * kTile, 512,
                              &bars->qdo_full[st]);
                    for (int r = 0; r < 2; ++r) {
                        tma_load_3d(sQ + st * kTileBytes + r * kRegion, &tm_q, &bars->qdo_full[st], r * 64, it.h,
                                    it.qt * kTile);
                        tma_load_3d(sDO + st * kTileBytes + r * kRegion, &tm_do, &bars->qdo_full[st], r * 64, it.h,
                                    it.qt * kTile);
                    }
                }
            }
            KVT(trace_value(p.tr, 18, w_qe); trace_value(p.tr, 19, w_kve); trace_value(p.tr, 20, w_ue);)
        }
    } else if (warp == 1) {
        // MMA warp (converged).
        constexpr uint32_t idesc_s = make_idesc_bf16(kTile, kTile, 0, 0);  // [128 keys] x [128 q], K = hd
        // N = hd: at head dim 64 only the 64 real columns (the epilogue never reads the others)
        const uint32_t idesc_g = make_idesc_bf16(kTile, g.hd == 64 ? 64 : kHd, 0, 1);  // [128 keys] x [hd], K = q
        // K = hd contractions: at head dim 64 the k-steps over the zero-padded columns 64-127 would
        // add exact zeros, so they are not issued
        const int nks_hd = g.hd / 16;
        const uint64_t dK = sdesc_k(smem_u32(sK)), dV = sdesc_k(smem_u32(sV));
        const uint64_t dQ = sdesc_k(smem_u32(sQ)), dDO = sdesc_k(smem_u32(sDO));
        const uint64_t dQmn = sdesc_mn(smem_u32(sQ), kRegion), dDOmn = sdesc_mn(smem_u32(sDO), kRegion);
        KVT(long long w_qf = 0; long long w_pf = 0; long long w_dsf = 0; long long w_af = 0; long long w_kvf = 0;)
        auto mma_s = [&](int gi) {
            const int st = gi % kKvStages;
            KVT_WAIT(w_qf, &bars->qdo_full[st], (gi / kKvStages) & 1);
            tc_fence_after();
            const uint64_t so = boff(st * kTileBytes);
            if (nks_hd == kHd / 16) {
#pragma unroll
                for (int ks = 0; ks < kHd / 16; ++ks) umma_ss_w(kTmS, dK + koff(ks, kRegion), dQ + so + koff(ks, kRegion), idesc_s, ks);
            } else {  // head dim 64
#pragma unroll
                for (int ks = 0; ks < kHd / 32; ++ks) umma_ss_w(kTmS, dK + koff(ks, kRegion), dQ + so + koff(ks, kRegion), idesc_s, ks);
            }
            umma_commit_w(&bars->s_full);
        };
        auto mma_dp = [&](int gi) {
            const uint64_t so = boff((gi % kKvStages) * kTileBytes);
            if (nks_hd == kHd / 16) {
#pragma unroll
                for (int ks = 0; ks < kHd / 16; ++ks) umma_ss_w(kTmDP, dV + koff(ks, kRegion), dDO + so + koff(ks, kRegion), idesc_s, ks);
            } else {  // head dim 64
#pragma unroll
                for (int ks = 0; ks < kHd / 32; ++ks) umma_ss_w(kTmDP, dV + koff(ks, kRegion), dDO + so + koff(ks, kRegion), idesc_s, ks);
            }
            umma_commit_w(&bars->dp_full);
        };
        auto mma_dv = [&](int gi, uint32_t first) {
            KVT_WAIT(w_pf, &bars->p_full, gi & 1);
            tc_fence_after();
            const uint64_t so = boff((gi % kKvStages) * kTileBytes);
#pragma unroll
            for (int ks = 0; ks < kTile / 16; ++ks)
                umma_ts_w(kTmDV, kTmS + pk_col(ks), dDOmn + so + mnoff(ks), idesc_g, first | ks);
        };
        auto mma_dk = [&](int gi, uint32_t first) {
            const int st = gi % kKvStages;
            KVT_WAIT(w_dsf, &bars->ds_full, gi & 1);
            tc_fence_after();
            const uint64_t so = boff(st * kTileBytes);
#pragma unroll
            for (int ks = 0; ks < kTile / 16; ++ks)
                umma_ts_w(kTmDK, kTmDP + pk_col(ks), dQmn + so + mnoff(ks), idesc_g, first | ks);
            umma_commit_w(&bars->qdo_empty[st]);
        };
        int gi = 0;
        for (int un = 0;; ++un) {
            const int k = un & 1;
            mbar_wait(&bars->unit_full[k], (un >> 1) & 1);
            const KvUnit& u = desc[k];
            if (!u.valid) break;
            const int n = u.n_items;
            KVT_WAIT(w_kvf, &bars->kv_full, un & 1);
            if (n > 0) {
                mma_s(gi);
                mma_dp(gi);
                if (n == 1) umma_commit_w(&bars->kv_empty);
                for (int i = 0; i < n; ++i) {
                    const uint32_t first = i == 0 ? 0u : 1u;
                    if (i == 0 && un > 0) {  // the previous unit's dK / dV have left TMEM
                        KVT_WAIT(w_af, &bars->acc_free, (un - 1) & 1);
                        tc_fence_after();
                    }
                    mma_dv(gi + i, first);
                    if (i + 1 < n) mma_s(gi + i + 1);   // rewrites S^T after dV(i) read P^T(i)
                    mma_dk(gi + i, first);
                    if (i + 1 < n) {
                        mma_dp(gi + i + 1);  // rewrites dP^T after dK(i) read dS^T(i)
                        if (i + 2 == n) umma_commit_w(&bars->kv_empty);  // last reader of K / V issued
                    }
                }
            } else {
                umma_commit_w(&bars->kv_empty);
            }
            umma_commit_w(&bars->acc_done);
            gi += n;
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->unit_empty[k]);
        }
        KVT(if (lane == 0) {
            trace_value(p.tr, 13, w_qf); trace_value(p.tr, 14, w_pf); trace_value(p.tr, 15, w_dsf);
            trace_value(p.tr, 16, w_af); trace_value(p.tr, 17, w_kvf);
        })
    } else if (warp >= 4) {
        // Warpgroup w: query columns [kKvCols w, kKvCols (w + 1)) of every item; thread = key row (TMEM lane).
        const int quarter = warp & 3, wg = (warp - 4) >> 2;
        const int kr = quarter * 32 + lane;  // key row of the block
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const float sl2 = g.scale * kLog2e;
        const uint32_t tS = kTmS + wg * kKvCols + lane_off, tDP = kTmDP + wg * kKvCols + lane_off;
        uint8_t* stage = smem + kKvStage + (wg & 1) * kSliceBytes;  // epilogue: warpgroups 0 / 1
        const bool issuer = (threadIdx.x & 127) == 0;  // first thread of the warpgroup issues its TMA
        int gi = 0;
        KVT(const long long c_start = clock64(); long long w_uf = 0, w_s0 = 0, w_s = 0, w_dp = 0, w_ad = 0, c_epi = 0,
            c_p = 0, c_ds = 0, n_units = 0, n_items_t = 0;
            if (threadIdx.x == 128) { trace_value(p.tr, 0, smid()); trace_mark(p.tr, 1); })
        for (int un = 0;; ++un) {
            const int k = un & 1;
            KVT_WAIT(w_uf, &bars->unit_full[k], (un >> 1) & 1);
            const KvUnit& u = desc[k];
            if (!u.valid) break;
            const int n = u.n_items;
            KVT(++n_units; n_items_t += n;)
            const bool past = u.past;
            const int key0 = u.key0, g_row = u.g_row, g_kv = u.g_kv;
            // page size 64: key rows [0,64) are the unit's first page, [64,128) its second
            const bool half1 = p64 && past && kr >= kHalf;
            const bool key_ok = p64 && past ? (kr & (kHalf - 1)) < (half1 ? u.n_valid1 : u.n_valid) : kr < u.n_valid;
            const uint64_t qm = half1 ? u.qm1 : u.qm0;
            const int g_row1 = u.g_row1, has1 = u.has1;
            const bool page_full = !(p64 && past) && u.n_valid == kTile;
            ItemIter it;
            it.init(u, g.group, tpq);
            for (int i = 0; i < n; ++i, it.next(u, g.group, tpq)) {
                const int gj = gi + i;
                const int st = gj % kKvStages;
                const uint32_t lrow = smem_u32(smem + kKvLD) + st * 1024 + wg * kKvCols * 4, drow = lrow + 512;
                // visible iff query column c >= lim (causal diagonal: key row <= query row); page size 64:
                // this group's query columns lie in query page 2 qt + wg kKvCols / 64, which may not have
                // chosen the page
                const bool ok = key_ok && (!(p64 && past) || ((qm >> (2 * it.qt + wg * kKvCols / 64)) & 1ull));
                const int lim = ok ? (it.diag ? kr - wg * kKvCols : 0) : 1 << 20;
                const bool masked = it.diag || !page_full;
                mbar_wait(&bars->qdo_full[st], (gj / kKvStages) & 1);  // makes the bulk-copied L / D visible
                // ---- P^T = exp2(S^T sl2 - L): computed as soon as S^T lands, packed in place
                if (i == 0) KVT_WAIT(w_s0, &bars->s_full, gj & 1);
                else KVT_WAIT(w_s, &bars->s_full, gj & 1);
                KVT(const long long cp0 = clock64();)
                tc_fence_after();
                float pr[kKvCols];
#pragma unroll
                for (int c2 = 0; c2 < kKvCols / 32; ++c2) {
                    uint32_t sv[32];
                    tmem_ld32(tS + c2 * 32, sv);
                    tmem_wait_ld();
#pragma unroll
                    for (int c4 = 0; c4 < 8; ++c4) {
                        const float4 l4 = lds128(lrow + (c2 * 32 + c4 * 4) * 4);
                        const int c = c2 * 32 + 4 * c4;
                        if (OOMB_KV_X2) {
                            const float2 s2 = make_float2(sl2, sl2);
                            const float2 x01 = fma2(make_float2(__uint_as_float(sv[4 * c4]), __uint_as_float(sv[4 * c4 + 1])),
                                                    s2, make_float2(-l4.x, -l4.y));
                            const float2 x23 = fma2(make_float2(__uint_as_float(sv[4 * c4 + 2]), __uint_as_float(sv[4 * c4 + 3])),
                                                    s2, make_float2(-l4.z, -l4.w));
                            if (kKvPairN > 0) {
                                const float2 e01 = ex2_pair(x01, c, kKvPairN), e23 = ex2_pair(x23, c + 2, kKvPairN);
                                pr[c + 0] = e01.x;
                                pr[c + 1] = e01.y;
                                pr[c + 2] = e23.x;
                                pr[c + 3] = e23.y;
                            } else {
                                pr[c + 0] = ex2_mix(x01.x, c + 0, kKvPolyN);
                                pr[c + 1] = ex2_mix(x01.y, c + 1, kKvPolyN);
                                pr[c + 2] = ex2_mix(x23.x, c + 2, kKvPolyN);
                                pr[c + 3] = ex2_mix(x23.y, c + 3, kKvPolyN);
                            }
                        } else if (kKvPairN > 0) {
                            const float2 e01 = ex2_pair(make_float2(fmaf(__uint_as_float(sv[4 * c4 + 0]), sl2, -l4.x),
                                                                    fmaf(__uint_as_float(sv[4 * c4 + 1]), sl2, -l4.y)),
                                                        c, kKvPairN);
                            const float2 e23 = ex2_pair(make_float2(fmaf(__uint_as_float(sv[4 * c4 + 2]), sl2, -l4.z),
                                                                    fmaf(__uint_as_float(sv[4 * c4 + 3]), sl2, -l4.w)),
                                                        c + 2, kKvPairN);
                            pr[c + 0] = e01.x;
                            pr[c + 1] = e01.y;
                            pr[c + 2] = e23.x;
                            pr[c + 3] = e23.y;
                        } else {
                            pr[c + 0] = ex2_mix(fmaf(__uint_as_float(sv[4 * c4 + 0]), sl2, -l4.x), c + 0, kKvPolyN);
                            pr[c + 1] = ex2_mix(fmaf(__uint_as_float(sv[4 * c4 + 1]), sl2, -l4.y), c + 1, kKvPolyN);
                            pr[c + 2] = ex2_mix(fmaf(__uint_as_float(sv[4 * c4 + 2]), sl2, -l4.z), c + 2, kKvPolyN);
                            pr[c + 3] = ex2_mix(fmaf(__uint_as_float(sv[4 * c4 + 3]), sl2, -l4.w), c + 3, kKvPolyN);
                        }
                    }
                }
                if (masked) {
#pragma unroll
                    for (int c = 0; c < kKvCols; ++c) pr[c] = (c >= lim) ? pr[c] : 0.f;
                }
#pragma unroll
                for (int c2 = 0; c2 < kKvCols / 32; ++c2) {
                    uint32_t pk[16];
#pragma unroll
                    for (int u2 = 0; u2 < 16; ++u2) pk[u2] = pack_bf16(pr[c2 * 32 + 2 * u2], pr[c2 * 32 + 2 * u2 + 1]);
                    tmem_st16(tS + c2 * 16, pk);  // below the columns still to be read
                }
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(&bars->p_full);
                KVT(c_p += clock64() - cp0;)
                // ---- dS^T = P^T (dP^T - D), packed in place of dP^T
                KVT_WAIT(w_dp, &bars->dp_full, gj & 1);
                KVT(const long long cd0 = clock64();)
                tc_fence_after();
#pragma unroll
                for (int c2 = 0; c2 < kKvCols / 32; ++c2) {
                    uint32_t dv[32];
                    tmem_ld32(tDP + c2 * 32, dv);
                    tmem_wait_ld();
                    uint32_t pk[16];
#pragma unroll
                    for (int c4 = 0; c4 < 8; ++c4) {
                        const float4 d4 = lds128(drow + (c2 * 32 + c4 * 4) * 4);
                        const int c = c2 * 32 + 4 * c4;
                        if (OOMB_KV_X2) {
                            const float2 a = mul2(make_float2(pr[c], pr[c + 1]),
                                                  add2(make_float2(__uint_as_float(dv[4 * c4]), __uint_as_float(dv[4 * c4 + 1])),
                                                       make_float2(-d4.x, -d4.y)));
                            const float2 b = mul2(make_float2(pr[c + 2], pr[c + 3]),
                                                  add2(make_float2(__uint_as_float(dv[4 * c4 + 2]), __uint_as_float(dv[4 * c4 + 3])),
                                                       make_float2(-d4.z, -d4.w)));
                            pk[2 * c4] = pack_bf16(a.x, a.y);
                            pk[2 * c4 + 1] = pack_bf16(b.x, b.y);
                        } else {
                            pk[2 * c4] = pack_bf16(pr[c] * (__uint_as_float(dv[4 * c4]) - d4.x),
                                                   pr[c + 1] * (__uint_as_float(dv[4 * c4 + 1]) - d4.y));
                            pk[2 * c4 + 1] = pack_bf16(pr[c + 2] * (__uint_as_float(dv[4 * c4 + 2]) - d4.z),
                                                       pr[c + 3] * (__uint_as_float(dv[4 * c4 + 3]) - d4.w));
                        }
                    }
                    tmem_st16(tDP + c2 * 16, pk);
                }
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(&bars->ds_full);
                KVT(c_ds += clock64() - cd0;)
            }
            gi += n;
            // ---- epilogue: pull this group's accumulator (dK scaled / dV) into registers, free TMEM
            KVT_WAIT(w_ad, &bars->acc_done, un & 1);
            KVT(const long long ce0 = clock64();)
            tc_fence_after();
            if (wg >= 2) {  // four softmax groups: the epilogue is warpgroups 0 (dK) and 1 (dV)
                mbar_arrive(&bars->acc_free);
                mbar_arrive(&bars->unit_empty[k]);
            } else {
                const uint32_t acc = (wg ? kTmDV : kTmDK) + lane_off;
                const float sc = key_ok ? (wg ? 1.f : g.scale) : 0.f;
                // the fused dM_i read-back: this key row's own-page gradient row in the pool
                const float* rb = nullptr;
                if (n > 0 && !past && p.readback_first >= 0 && key_ok) {
                    const int kk = key0 + kr;
                    const int gs = p.gslot[p.readback_first + kk / g.P];
                    if (gs >= 0)
                        rb = (wg ? p.gv : p.gk) +
                             ((static_cast<size_t>(gs) * g.Hkv + g_kv) * g.P + kk % g.P) * static_cast<size_t>(g.hd);
                }
#pragma unroll
                for (int r = 0; r < kKvEpR; ++r) {
                    uint32_t va[kKvEpC][32];
#pragma unroll
                    for (int c = 0; c < kKvEpC; ++c) tmem_ld32(acc + (r * kKvEpC + c) * 32, va[c]);
                    tmem_wait_ld();
                    if (r == kKvEpR - 1) {
                        tc_fence_before();
                        mbar_arrive(&bars->acc_free);
                    }
                    if (r == 0) mbar_arrive(&bars->unit_empty[k]);  // descriptor fields are in registers
                    if (n > 0) {
                        // ---- [128 x 32] slices through this group's staging buffer into L2 / dk_cur / dv_cur
#pragma unroll
                        for (int c0 = 0; c0 < kKvEpC; ++c0) {
                            const int c = r * kKvEpC + c0;
                            if (c * 32 >= g.hd) break;         // head dim 64: columns 64-127 are zero padding
                            if (issuer) bulk_wait_read0();     // the previous slice has left the staging buffer
                            named_bar_sync(4 + wg, 128);
#pragma unroll
                            for (int u8 = 0; u8 < 8; ++u8) {
                                float4 v4 = make_float4(__fmul_rn(__uint_as_float(va[c0][4 * u8]), sc),
                                                        __fmul_rn(__uint_as_float(va[c0][4 * u8 + 1]), sc),
                                                        __fmul_rn(__uint_as_float(va[c0][4 * u8 + 2]), sc),
                                                        __fmul_rn(__uint_as_float(va[c0][4 * u8 + 3]), sc));
                                if (rb) {
                                    const float4 a4 = __ldg(reinterpret_cast<const float4*>(rb + c * 32) + u8);
                                    v4.x = __fadd_rn(v4.x, a4.x);
                                    v4.y = __fadd_rn(v4.y, a4.y);
                                    v4.z = __fadd_rn(v4.z, a4.z);
                                    v4.w = __fadd_rn(v4.w, a4.w);
                                }
                                st_slice_f32(stage, kr, u8, v4);
                            }
                            fence_proxy_async_smem();
                            named_bar_sync(4 + wg, 128);
                            if (issuer) {
                                if (past && p64) {  // 64-row boxes into each page's gradient block
                                    tma_reduce_add_2d(wg ? &tm_gv : &tm_gk, stage, c * 32, g_row);
                                    if (has1) tma_reduce_add_2d(wg ? &tm_gv : &tm_gk, stage + kSliceBytes / 2, c * 32, g_row1);
                                } else if (past) {
                                    tma_reduce_add_2d(wg ? &tm_gv : &tm_gk, stage, c * 32, g_row);
                                } else {
                                    tma_store_3d(wg ? &tm_dvc : &tm_dkc, stage, c * 32, g_kv, key0);
                                }
                                bulk_commit();
                            }
                        }
                    }
                }
            }
            KVT(c_epi += clock64() - ce0;)
        }
        if (issuer) bulk_wait_read0();
        KVT(if (threadIdx.x == 128) {
            trace_mark(p.tr, 2); trace_value(p.tr, 3, n_units); trace_value(p.tr, 4, n_items_t);
            trace_value(p.tr, 5, w_uf); trace_value(p.tr, 6, w_s0); trace_value(p.tr, 7, w_s);
            trace_value(p.tr, 8, w_dp); trace_value(p.tr, 9, w_ad); trace_value(p.tr, 10, c_epi);
            trace_value(p.tr, 11, c_p); trace_value(p.tr, 12, c_ds); trace_value(p.tr, 21, clock64() - c_start);
        })
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 3) tmem_dealloc<512>(0);
}

}  // namespace


// dQ = sum of the split-K partials in z order (deterministic).
__global__ void dq_split_sum_kernel(const float4* __restrict__ part, int zs, int64_t n4, float4* __restrict__ dq) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float4 a = part[i];
        for (int z = 1; z < zs; ++z) {
            const float4 b = part[z * n4 + i];
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
        dq[i] = a;
    }
}

bool tc_bwd_available() { return true; }

size_t attn_bwd_tc_workspace(const AttnGeom& g, int) {
    const size_t hc = static_cast<size_t>(g.Hq) * g.C * sizeof(float);
    const size_t order = (static_cast<size_t>(g.C / kTile) + static_cast<size_t>(g.max_pages) * bwd_blocks_per_page(g)) * 4;
    return ((2 * hc + 255) & ~size_t(255)) + static_cast<size_t>(g.max_pages) * 12 + 512 + order;
}

void launch_attn_bwd_tc(const AttnGeom& g, const TcPoolMaps& maps, const void* dout, const void* q,
                        const int32_t* sel_off, const int32_t* sel_ids, const int32_t* d_kvslot_layer,
                        const int32_t* d_gslot_layer, float* gkpool, float* gvpool, const void* k_cur,
                        const void* v_cur, const void* out, const float* lse, float* dq, float* dk_cur,
                        float* dv_cur, int* d_err, void* workspace, size_t workspace_bytes, int nnz, int n_pages,
                        cudaStream_t st, cudaStream_t side, cudaEvent_t ev_prep, cudaEvent_t ev_dq, bool join_dq,
                        int readback_first) {
    OOMB_REQUIRE(workspace_bytes >= attn_bwd_tc_workspace(g, nnz), OOMB_ERROR, "bwd workspace too small");
    OOMB_REQUIRE(g.m <= 64, OOMB_CONFIG_ERROR, "tcgen05 backward supports at most 64 query pages per chunk");
    if (first_use_on_device(2)) {
        OOMB_CUDA(cudaFuncSetAttribute(attn_bwd_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDqSmem));
        OOMB_CUDA(cudaFuncSetAttribute(attn_bwd_dkdv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kKvSmem));
    }
    const int num_sms = device_sms();
    BwdWs w = carve(g, workspace);
    ProfScope* prep_scope = new ProfScope(PK_BWD_PREP, st);
    const int64_t rows = static_cast<int64_t>(g.C) * g.Hq;
    // page size 64 pairs union pages per unit: kept in union order
    const bool lpt = OOMB_BWD_LPT && g.P != kHalf;
    bwd_prep_sched_kernel<<<static_cast<unsigned>(1 + (rows + 63) / 64), 1024, 0, st>>>(
        static_cast<const __nv_bfloat16*>(out), static_cast<const __nv_bfloat16*>(dout), lse, g.C, g.Hq, g.hd, w.Dt,
        w.Lt, sel_off, sel_ids, g.m, layer_pages(g), n_pages, w.mask, w.uni, w.n_uni, g.chunk_keys ? g.C / kTile : 0,
        bwd_blocks_per_page(g), std::max(1, g.P / kTile), lpt ? w.order : nullptr, d_err);
    check_launch("bwd_prep_sched_kernel");
    // head dim 64: the 128-wide tiles carry zeros in columns 64-127 (TMA out-of-bounds fill) and the
    // stores of those columns fall outside the tensors (clipped): see launch_attn_fwd_tc4
    const CUtensorMap tq = map_rows_heads(q, g.C, g.Hq, g.hd);
    const CUtensorMap tdo = map_rows_heads(dout, g.C, g.Hq, g.hd);
    const CUtensorMap tkc = map_rows_heads(k_cur, g.C, g.Hkv, g.hd);
    const CUtensorMap tvc = map_rows_heads(v_cur, g.C, g.Hkv, g.hd);
    BwdParams p{g,     sel_off, sel_ids, d_kvslot_layer, d_gslot_layer, gkpool, gvpool, w.Dt, w.Lt, w.mask, w.uni,
                w.n_uni, lpt ? w.order : nullptr, dq, dk_cur, dv_cur, d_err, CtaTrace{}, readback_first};
    delete prep_scope;
    // dQ and dK/dV only read the chunk's inputs and the prep outputs: dQ runs on the pool's side
    // stream, launched first, and the persistent dK/dV CTAs pick up SMs as dQ's last wave drains
    // (and vice versa), so neither kernel's tail leaves SMs idle. join_dq: the caller's stream
    // waits for both; otherwise (OOMB_ATTN_DEFER_DQ) only ev_dq marks dQ's end, and the next
    // chunk's dK/dV may start under this chunk's dQ.
    // The dQ + dK/dV pair as one span on the caller's stream (the two kernels overlap, so their
    // own spans each include time spent sharing the GPU with the other).
    ProfScope* pair_scope = join_dq ? new ProfScope(PK_BWD_PAIR, st) : nullptr;
    OOMB_CUDA(cudaEventRecord(ev_prep, st));
    OOMB_CUDA(cudaStreamWaitEvent(side, ev_prep, 0));
    auto launch_dq = [&] {
        ProfScope s_(PK_BWD_DQ, side);
        const int zs = OOMB_DQ_SPLIT ? attn_tc_splits(g, num_sms) : 1;
        float* part = nullptr;
        const int64_t n = static_cast<int64_t>(g.C) * g.Hq * g.hd;
        if (zs > 1) part = static_cast<float*>(stream_scratch(side, 1, static_cast<size_t>(zs) * n * sizeof(float)));
        const CUtensorMap tdq = map_rows_heads_f32(zs > 1 ? part : dq, static_cast<int64_t>(zs) * g.C, g.Hq, g.hd);
        attn_bwd_dq_kernel<<<dim3(g.Hq, g.C / kTile, zs), 384, kDqSmem, side>>>(tq, tdo, tkc, tvc, maps.kpool,
                                                                                maps.vpool, tdq, p);
        check_launch("attn_bwd_dq_kernel");
        if (zs > 1) {
            dq_split_sum_kernel<<<static_cast<unsigned>(std::min<int64_t>((n / 4 + 255) / 256, 4 * num_sms)), 256, 0,
                                  side>>>(reinterpret_cast<const float4*>(part), zs, n / 4,
                                          reinterpret_cast<float4*>(dq));
            check_launch("dq_split_sum_kernel");
        }
        OOMB_CUDA(cudaEventRecord(ev_dq, side));
    };
    auto launch_dkdv = [&] {
        ProfScope s_(PK_BWD_DKDV, st);
        const int max_union = std::min(nnz, n_pages);
        if (!g.chunk_keys) {  // past-only shard: the chunk's own keys are another shard's
            OOMB_CUDA(cudaMemsetAsync(dk_cur, 0, static_cast<size_t>(g.C) * g.Hkv * g.hd * sizeof(float), st));
            OOMB_CUDA(cudaMemsetAsync(dv_cur, 0, static_cast<size_t>(g.C) * g.Hkv * g.hd * sizeof(float), st));
        }
        const int past_units = g.P == kHalf ? (max_union + 1) / 2 : max_union * (g.P / kTile);
        const int units = ((g.chunk_keys ? g.C / kTile : 0) + past_units) * g.Hkv;
        const int n_ctas = std::max(1, std::min(units, num_sms));
        const CUtensorMap tdkc = map_rows_heads_f32(dk_cur, g.C, g.Hkv, g.hd);
        const CUtensorMap tdvc = map_rows_heads_f32(dv_cur, g.C, g.Hkv, g.hd);
        BwdParams pk = p;
        if (OOMB_KV_TRACE) pk.tr = trace_begin("dkdv", n_ctas, 22);
        attn_bwd_dkdv_kernel<<<n_ctas, kKvThreads, kKvSmem, st>>>(tq, tdo, tkc, tvc, maps.kpool, maps.vpool, maps.gkpool,
                                                            maps.gvpool, tdkc, tdvc, pk, w.n_uni + 1);
        check_launch("attn_bwd_dkdv_kernel");
        if (OOMB_KV_TRACE) trace_end(pk.tr, n_ctas, st);
    };
    if (OOMB_BWD_KV_FIRST) {
        launch_dkdv();
        launch_dq();
    } else {
        launch_dq();
        launch_dkdv();
    }
    {
        if (join_dq) OOMB_CUDA(cudaStreamWaitEvent(st, ev_dq, 0));
        delete pair_scope;

    }
}

}  // namespace oomb
