// SPDX-License-Identifier: Apache-2.0
//
// Paged flash forward, variant 4 — attention.hpp:156-208 on tcgen05 with the key blocks of a
// query tile split between two softmax warpgroups.
//
// One CTA per (128-row query tile, q-head), one CTA per SM, looping over the tile's key blocks
// (its query page's selected pages in list order, then the chunk's causal prefix). Warpgroup w
// owns the blocks j with j % 2 == w: it keeps its own running max m_w, row sum l_w and output
// accumulator O_w (a split-K flash attention), so the two groups' exp work, the S MMAs of one
// group's blocks and the PV MMAs of the other's overlap instead of forming one serial chain.
// At the end O = (O_0 2^(m_0-m) + O_1 2^(m_1-m)) / (l_0 2^(m_0-m) + l_1 2^(m_1-m)), exact.
// The online softmax of each group rescales O_w only when m_w grows by more than 2^8.
//
// S = Q K^T is an SS-MMA with N = 128 (full rate); P is written back into its S buffer as packed
// bf16 and O_w += P V is a TS-MMA. A group's O_w rescale needs PV of its previous block to have
// landed: the commit of S(j) covers every MMA issued before it, PV(j-2) included.
// TMEM (all 512 columns, base 0): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).
// Warp roles (384 threads): w0 Q + K producer, w1 MMA, w2 V producer, w3 TMEM allocator,
// w4..w7 softmax group 0 (even blocks), w8..w11 group 1 (odd blocks); thread = query row.

#include <algorithm>

#include "tc_common.cuh"

namespace oomb {

using namespace tc;

namespace {

#ifndef OOMB_FWD4_KST
#define OOMB_FWD4_KST 3
#endif
constexpr int kKSt = OOMB_FWD4_KST, kVSt = 5 - OOMB_FWD4_KST;  // K / V stages (3 / 2 and 2 / 3 measured equal)
constexpr int kF4Q = 0;
constexpr int kF4K = kF4Q + kTileBytes;
constexpr int kF4V = kF4K + kKSt * kTileBytes;
constexpr int kF4Red = kF4V + kVSt * kTileBytes;  // [2 groups][128 rows] {m, l}
constexpr int kF4Nv = kF4Red + 2 * 128 * 8;       // uint8 valid-key counts of the past blocks
constexpr int kF4NvCap = 8192;
constexpr int kF4Bar = kF4Nv + kF4NvCap;
constexpr int kF4Smem = kF4Bar + 256;
static_assert(kF4Smem <= 232448, "dynamic shared memory above the 227 KB opt-in limit");
constexpr uint32_t kTmS = 0, kTmO = 256;
#ifndef OOMB_FWD4_PCHUNKS
#define OOMB_FWD4_PCHUNKS 2
#endif
// P is published to the MMA warp in kPChunks key chunks: PV starts on the first keys of a block
// while the softmax group is still exponentiating the last ones.
constexpr int kPChunks = OOMB_FWD4_PCHUNKS;
static_assert(kPChunks == 1 || kPChunks == 2 || kPChunks == 4, "P chunks");
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef OOMB_FWD4_POLY
#define OOMB_FWD4_POLY 0  // measured: no gain (the softmax phase is latency-bound, not MUFU-bound)
#endif
constexpr bool kF4Poly = OOMB_FWD4_POLY != 0;
#ifndef OOMB_FWD_SPLIT
#define OOMB_FWD_SPLIT 1  // split-K over key blocks when the grid is small (attn_tc_splits)
#endif
#ifndef OOMB_FWD4_LEAN
#define OOMB_FWD4_LEAN 1  // the FMA-pipe exponential is ex2_lean (one ALU op) rather than ex2_poly
#endif
constexpr bool kF4Lean = OOMB_FWD4_LEAN != 0;
#ifndef OOMB_FWD4_X2
#define OOMB_FWD4_X2 0  // softmax scale-subtract and row sums as packed fp32 pairs
#endif
constexpr bool kF4X2 = OOMB_FWD4_X2 != 0;
#ifndef OOMB_FWD4_PAIR_N
#define OOMB_FWD4_PAIR_N 0  // 1 pair in N of the exponentials as an FMA-pipe packed pair (ex2_lean2);
                            // measured N = 4: 38.54 vs 35.85 ms serialized (slower)
#endif
constexpr int kF4PairN = OOMB_FWD4_PAIR_N;


struct F4Bars {
    uint64_t q_full;
    uint64_t k_full[kKSt], k_empty[kKSt], v_full[kVSt], v_empty[kVSt];
    uint64_t s_full[2], p_full[2][kPChunks], o_done;
    uint32_t tmem_base;
};

struct F4Params {
    AttnGeom g;
    const int32_t* sel_off;
    const int32_t* sel_ids;
    const int32_t* kvslot;
    __nv_bfloat16* out;
    float* lse;
    int* err;
    // split-K over the key blocks (few query tiles, long histories: c1): CTA z of gridDim.z attends
    // blocks [z nb / Z, (z+1) nb / Z) and writes its normalised partial O (fp32) and LSE here; a
    // merge kernel combines them exactly in z order. Null: one split, O / LSE straight to out / lse.
    float* o_part;    // [Z][C][Hq][hd]
    float* lse_part;  // [Z][C][Hq]
};

__global__ void __launch_bounds__(384, 1)
    attn_fwd_tc4_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kc,
                        const __grid_constant__ CUtensorMap tm_vc, const __grid_constant__ CUtensorMap tm_kp,
                        const __grid_constant__ CUtensorMap tm_vp, F4Params p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    F4Bars* bars = reinterpret_cast<F4Bars*>(smem + kF4Bar);
    const AttnGeom& g = p.g;
    const int h = blockIdx.x;
    const int qt = (g.C / kTile) - 1 - static_cast<int>(blockIdx.y);  // longest causal prefix first (LPT)
    const int kvh = h / g.group;
    const bool p64 = g.P == kHalf;  // two query pages per tile, 64-key half blocks (tc_common.cuh)
    const int qp = (qt * kTile) / g.P;
    const int sel_begin = p.sel_off[qp];
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023) __trap();  // SW128 operands need a 1 KB-aligned base
        mbar_init(&bars->q_full, 1);
        for (int i = 0; i < kKSt; ++i) {
            mbar_init(&bars->k_full[i], 1);
            mbar_init(&bars->k_empty[i], 1);
        }
        for (int i = 0; i < kVSt; ++i) {
            mbar_init(&bars->v_full[i], 1);
            mbar_init(&bars->v_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->s_full[i], 1);
            for (int c = 0; c < kPChunks; ++c) mbar_init(&bars->p_full[i][c], 128);
        }
        mbar_init(&bars->o_done, 1);
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
    const int zs = static_cast<int>(gridDim.z), z = static_cast<int>(blockIdx.z);
    const int j0 = static_cast<int>(static_cast<int64_t>(nb_all) * z / zs);  // this split's key blocks
    const int nb = static_cast<int>(static_cast<int64_t>(nb_all) * (z + 1) / zs) - j0;
    uint8_t* sQ = smem + kF4Q;
    uint8_t* sK = smem + kF4K;
    uint8_t* sV = smem + kF4V;

    if (warp == 0 || warp == 2) {
        if (lane == 0) {  // w0: Q + K, w2: V
            const bool is_k = warp == 0;
            const int nst = is_k ? kKSt : kVSt;
            uint8_t* base = is_k ? sK : sV;
            uint64_t* full = is_k ? bars->k_full : bars->v_full;
            uint64_t* empty = is_k ? bars->k_empty : bars->v_empty;
            const CUtensorMap* mp = is_k ? &tm_kp : &tm_vp;
            const CUtensorMap* mc = is_k ? &tm_kc : &tm_vc;
            if (is_k) {
                mbar_expect_tx(&bars->q_full, kTileBytes);
                for (int r = 0; r < 2; ++r) tma_load_3d(sQ + r * kRegion, &tm_q, &bars->q_full, r * 64, h, qt * kTile);
            }
            for (int j = 0; j < nb; ++j) {
                const int st = j % nst;
                if (j >= nst) mbar_wait(&empty[st], ((j / nst) - 1) & 1);
                mbar_expect_tx(&full[st], kTileBytes);
                uint8_t* dst = base + st * kTileBytes;
                const int jb = j0 + j;  // the block's index in the tile's full list
                if (jb < n_past && p64) {  // two 64-row half blocks (pool maps with 64-row boxes)
                    for (int hh = 0; hh < 2; ++hh) {
                        const int row = past_half_row(g, p.sel_ids, p.kvslot, hl, 2 * jb + hh, kvh, is_k ? p.err : nullptr);
                        for (int r = 0; r < 2; ++r)
                            tma_load_2d(dst + r * kRegion + hh * (kRegion / 2), mp, &full[st], r * 64, row);
                    }
                } else if (jb < n_past) {
                    const PastBlock b = past_block(g, p.sel_ids, p.kvslot, sel_begin, jb, kvh, is_k ? p.err : nullptr);
                    for (int r = 0; r < 2; ++r) tma_load_2d(dst + r * kRegion, mp, &full[st], r * 64, b.row);
                } else {
                    for (int r = 0; r < 2; ++r)
                        tma_load_3d(dst + r * kRegion, mc, &full[st], r * 64, kvh, (jb - n_past) * kTile);
                }
            }
        }
    } else if (warp == 1) {
        // MMA warp (converged): S(0) S(1) | PV(0) S(2) | PV(1) S(3) | ... | PV(nb-1)
        constexpr uint32_t idesc_s = make_idesc_bf16(kTile, kTile, 0, 0);  // [128 q] x [128 keys], K = hd
        // N = hd: at head dim 64 only the 64 real columns (the merge never reads the others)
        const uint32_t idesc_o = make_idesc_bf16(kTile, g.hd == 64 ? 64 : kHd, 0, 1);  // [128 q] x [hd], K = keys
        // K = hd contractions: at head dim 64 the k-steps over the zero-padded columns 64-127 would
        // add exact zeros, so they are not issued
        const int nks_hd = g.hd / 16;
        const uint64_t dQ = sdesc_k(smem_u32(sQ));
        const uint64_t dK = sdesc_k(smem_u32(sK));
        const uint64_t dVmn = sdesc_mn(smem_u32(sV), kRegion);
        mbar_wait(&bars->q_full, 0);
        auto mma_s = [&](int j) {
            const int st = j % kKSt, b = j & 1;
            mbar_wait(&bars->k_full[st], (j / kKSt) & 1);
            tc_fence_after();
            const uint64_t so = boff(st * kTileBytes);
            if (nks_hd == kHd / 16) {
#pragma unroll
                for (int ks = 0; ks < kHd / 16; ++ks) umma_ss_w(kTmS + b * 128, dQ + koff(ks, kRegion), dK + so + koff(ks, kRegion), idesc_s, ks);
            } else {  // head dim 64
#pragma unroll
                for (int ks = 0; ks < kHd / 32; ++ks) umma_ss_w(kTmS + b * 128, dQ + koff(ks, kRegion), dK + so + koff(ks, kRegion), idesc_s, ks);
            }
            umma_commit_w(&bars->s_full[b]);
            umma_commit_w(&bars->k_empty[st]);
        };
        auto mma_pv = [&](int j) {
            const int st = j % kVSt, b = j & 1;
            mbar_wait(&bars->v_full[st], (j / kVSt) & 1);
            const uint64_t so = boff(st * kTileBytes);
            const uint32_t first = j < 2 ? 0u : 1u;  // the first block of each group overwrites O_w
            constexpr int kStepsPerChunk = kTile / 16 / kPChunks;
#pragma unroll
            for (int c = 0; c < kPChunks; ++c) {
                mbar_wait(&bars->p_full[b][c], (j >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int i = 0; i < kStepsPerChunk; ++i) {
                    const int ks = c * kStepsPerChunk + i;
                    umma_ts_w(kTmO + b * 128, kTmS + b * 128 + ks * 8, dVmn + so + mnoff(ks), idesc_o, first | ks);
                }
            }
            umma_commit_w(&bars->v_empty[st]);
        };
        if (nb > 0) mma_s(0);
        if (nb > 1) mma_s(1);
        for (int j = 0; j < nb; ++j) {
            mma_pv(j);
            if (j + 2 < nb) mma_s(j + 2);  // S(j+2) rewrites the buffer PV(j) read: issued after it
        }
        umma_commit_w(&bars->o_done);
    } else if (warp >= 4) {
        const int quarter = warp & 3, wg = (warp - 4) >> 2;
        const int r = quarter * 32 + lane;  // query row = TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        uint8_t* nvt = smem + kF4Nv;
        uint16_t* hvt = reinterpret_cast<uint16_t*>(nvt);
        if (p64) stage_half_valid(g, p.sel_ids, hl, hvt, kF4NvCap / 2, threadIdx.x - 128, 256);
        else stage_past_valid(g, p.sel_ids, sel_begin, n_past, nvt, kF4NvCap, threadIdx.x - 128, 256);
        named_bar_sync(3, 256);
        const float sl2 = g.scale * kLog2e;
        const uint32_t tS = kTmS + wg * 128 + lane_off, tO = kTmO + wg * 128 + lane_off;
        float m = -INFINITY;  // this group's running row max (log2 units) that O_w and l are relative to
        float l = 0.f;
        for (int j = wg; j < nb; j += 2) {
            int lo, hi;  // keep key columns c <= lo (c < 64) / c <= hi (c >= 64)
            const int jb = j0 + j;
            if (jb < n_past && p64) {
                lo = half_lim(half_valid(g, p.sel_ids, hl, hvt, kF4NvCap / 2, 2 * jb), r);
                hi = kHalf + half_lim(half_valid(g, p.sel_ids, hl, hvt, kF4NvCap / 2, 2 * jb + 1), r);
            } else {
                lo = (jb < n_past) ? past_valid(g, p.sel_ids, sel_begin, nvt, kF4NvCap, jb) - 1
                                   : ((jb - n_past == qt) ? r : kTile - 1);
                hi = lo;
            }
            mbar_wait(&bars->s_full[wg], (j >> 1) & 1);
            tc_fence_after();
            uint32_t sr[128];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
            tmem_wait_ld();
            if (lo < kHalf - 1 || hi < kTile - 1) {
#pragma unroll
                for (int c = 0; c < kTile; ++c)
                    if (c > (c < kHalf ? lo : hi)) sr[c] = __float_as_uint(-INFINITY);
            }
            float mx8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) mx8[u] = __uint_as_float(sr[u]);
#pragma unroll
            for (int c = 8; c < kTile; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sr[c]));
            const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                   fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
            const float m_new = fmaxf(m, mx);
            bool rescale = false;
            float alpha = 1.f;
            if (m == -INFINITY || m_new > m + kRescaleThreshold) {
                alpha = (m == -INFINITY) ? 0.f : ex2(m - m_new);
                rescale = j >= 2 && m != -INFINITY;
                m = m_new;
            }
            const float m_use = (m == -INFINITY) ? 0.f : m;
            // O_w rescale: PV(j-2) has landed (the commit of S(j) covers it)
            if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll 1
                for (int c = 0; c < 8; ++c) {
                    uint32_t o[16];
                    tmem_ld16(tO + c * 16, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int u = 0; u < 16; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * alpha);
                    tmem_st16(tO + c * 16, o);
                }
            }
            float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            float pe0 = 0.f, pe1 = 0.f;  // kF4X2: the even pair of exponentials, summed with the odd one
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
                uint32_t pk[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    float x0, x1;
                    if (kF4X2) {  // packed fp32 pair: the same two IEEE FMAs in one issue slot
                        const float2 x = fma2(make_float2(__uint_as_float(sr[c4 * 32 + 2 * u]),
                                                          __uint_as_float(sr[c4 * 32 + 2 * u + 1])),
                                              make_float2(sl2, sl2), make_float2(-m_use, -m_use));
                        x0 = x.x;
                        x1 = x.y;
                    } else {
                        x0 = fmaf(__uint_as_float(sr[c4 * 32 + 2 * u]), sl2, -m_use);
                        x1 = fmaf(__uint_as_float(sr[c4 * 32 + 2 * u + 1]), sl2, -m_use);
                    }
                    float e0, e1;
                    if (kF4PairN > 0 && (u % kF4PairN) == kF4PairN - 1) {  // a packed pair on the FMA pipe
                        const float2 e = ex2_lean2(make_float2(x0, x1));
                        e0 = e.x;
                        e1 = e.y;
                    } else {
                        e0 = ex2(x0);
                        // 1 in 4 on the FMA pipe
                        e1 = (kF4Poly && (u & 1)) ? (kF4Lean ? ex2_lean(x1) : ex2_poly(x1)) : ex2(x1);
                    }
                    if (kF4X2 && (u & 1)) {  // row sums as packed pairs too (same additions, same order)
                        const float2 a = add2(make_float2(rs8[(2 * u - 2) & 7], rs8[(2 * u - 1) & 7]),
                                              make_float2(pe0, pe1));
                        const float2 b = add2(make_float2(rs8[(2 * u) & 7], rs8[(2 * u + 1) & 7]), make_float2(e0, e1));
                        rs8[(2 * u - 2) & 7] = a.x;
                        rs8[(2 * u - 1) & 7] = a.y;
                        rs8[(2 * u) & 7] = b.x;
                        rs8[(2 * u + 1) & 7] = b.y;
                    } else if (kF4X2) {
                        pe0 = e0;
                        pe1 = e1;
                    } else {
                        rs8[(2 * u) & 7] += e0;
                        rs8[(2 * u + 1) & 7] += e1;
                    }
                    pk[u] = pack_bf16(e0, e1);
                }
                tmem_st16(tS + c4 * 16, pk);  // P cols [16 c4, 16 c4 + 16): below the S columns still unread
                if ((c4 + 1) % (4 / kPChunks) == 0) {  // publish this chunk of P (and, with chunk 0, the O_w rescale)
                    tmem_wait_st();
                    tc_fence_before();
                    mbar_arrive(&bars->p_full[wg][c4 / (4 / kPChunks)]);
                }
            }
            const float rs = ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
            l = l * alpha + rs;
        }
        // ---- merge the two groups: O = (O_0 a_0 + O_1 a_1) / (l_0 a_0 + l_1 a_1), a_w = 2^(m_w - m)
        float2* red = reinterpret_cast<float2*>(smem + kF4Red);
        red[wg * 128 + r] = make_float2(m, l);
        named_bar_sync(2, 256);
        const float2 o = red[(wg ^ 1) * 128 + r];
        const float m0 = wg ? o.x : m, l0 = wg ? o.y : l, m1 = wg ? m : o.x, l1 = wg ? l : o.y;
        const float mt = fmaxf(m0, m1);
        const float a0 = (l0 > 0.f) ? ex2(m0 - mt) : 0.f, a1 = (l1 > 0.f) ? ex2(m1 - mt) : 0.f;
        const float lt = l0 * a0 + l1 * a1;  // 0 only for a page-range shard that attended no key
        const float s0 = lt > 0.f ? a0 / lt : 0.f, s1 = lt > 0.f ? a1 / lt : 0.f;
        mbar_wait(&bars->o_done, 0);
        tc_fence_after();
        const int t = qt * kTile + r;
        // group w writes output columns [64w, 64w + 64) (head dim 64: group 0 only; columns 64-127
        // of O are the zero padding of the 128-wide tiles, see launch_attn_fwd_tc4)
        __nv_bfloat16* orow = p.out + (static_cast<int64_t>(t) * g.Hq + h) * g.hd + wg * 64;
        float* prow = p.o_part ? p.o_part + ((static_cast<int64_t>(z) * g.C + t) * g.Hq + h) * g.hd + wg * 64 : nullptr;
#pragma unroll 1
        for (int c = 0; c < (wg * 64 < g.hd ? 4 : 0); ++c) {
            uint32_t x0[16], x1[16];
            tmem_ld16(kTmO + wg * 64 + c * 16 + lane_off, x0);
            tmem_ld16(kTmO + 128 + wg * 64 + c * 16 + lane_off, x1);
            tmem_wait_ld();
            float f[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const float v0 = s0 != 0.f ? __uint_as_float(x0[u]) * s0 : 0.f;  // an O_w never written holds
                const float v1 = s1 != 0.f ? __uint_as_float(x1[u]) * s1 : 0.f;  // garbage: never multiply it
                f[u] = v0 + v1;
            }
            if (prow) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    *reinterpret_cast<float4*>(prow + c * 16 + 4 * u) = make_float4(f[4 * u], f[4 * u + 1], f[4 * u + 2], f[4 * u + 3]);
            } else {
                *reinterpret_cast<uint4*>(orow + c * 16) = pack8(f);
                *reinterpret_cast<uint4*>(orow + c * 16 + 8) = pack8(f + 8);
            }
        }
        if (wg == 0) {
            const float L = lt > 0.f ? (mt + __log2f(lt)) * kLn2 : -INFINITY;
            if (p.lse_part) p.lse_part[(static_cast<int64_t>(z) * g.C + t) * g.Hq + h] = L;
            else p.lse[static_cast<int64_t>(t) * g.Hq + h] = L;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 3) tmem_dealloc<512>(0);
}

// Exact merge of the split-K partials, splits in z order (deterministic): LSE = m + ln sum_z
// e^(LSE_z - m), O = sum_z e^(LSE_z - LSE) O_z. One warp per (token, head) row; hd <= 128.
__global__ void fwd_split_merge_kernel(const float* __restrict__ o_part, const float* __restrict__ lse_part, int zs,
                                       int64_t rows, int hd, __nv_bfloat16* __restrict__ out, float* __restrict__ lse) {
    const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    float m = -INFINITY;
    for (int z = 0; z < zs; ++z) m = fmaxf(m, lse_part[z * rows + row]);
    float l = 0.f;
    for (int z = 0; z < zs; ++z) {
        const float x = lse_part[z * rows + row];
        if (x != -INFINITY) l += __expf(x - m);
    }
    const float L = m == -INFINITY ? -INFINITY : m + __logf(l);
    for (int d = lane * 4; d < hd; d += 128) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int z = 0; z < zs; ++z) {
            const float x = lse_part[z * rows + row];
            if (x == -INFINITY) continue;
            const float w = __expf(x - L);
            const float4 o = *reinterpret_cast<const float4*>(o_part + (z * rows + row) * hd + d);
            acc.x += w * o.x;
            acc.y += w * o.y;
            acc.z += w * o.z;
            acc.w += w * o.w;
        }
        __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(out + row * hd + d);
        dst[0] = __floats2bfloat162_rn(acc.x, acc.y);
        dst[1] = __floats2bfloat162_rn(acc.z, acc.w);
    }
    if (lane == 0) lse[row] = L;
}

}  // namespace

// Split count for the forward / dQ kernels. A grid of at most 32 (query tile, head) tiles (c1: 8)
// leaves most of the 148 SMs idle, so each tile's key blocks are split over up to 16 CTAs (at least
// 4 blocks each); larger grids run one CTA per tile. Splitting changes the rounding of the merged
// output, so the rule must give a KV-group shard the same split as the unsharded layer: it does
// whenever a shard still has more than 32 tiles (every BASELINE shape; a split layer of <= 32
// tiles matches within rounding, not bitwise).
int attn_tc_splits(const AttnGeom& g, int num_sms) {
    (void)num_sms;
    if (g.Hq * (g.C / kTile) > 32) return 1;
    const int64_t blocks = (g.filled + kTile - 1) / kTile;  // past keys + this chunk's (an upper bound)
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(16, blocks / 4)));
}

void launch_attn_fwd_tc4(const AttnGeom& g, const TcPoolMaps& maps, const void* q, const int32_t* sel_off,
                         const int32_t* sel_ids, const int32_t* d_kvslot_layer, const void* k_cur, const void* v_cur,
                         void* out, float* lse, int* d_err, cudaStream_t st) {
    if (first_use_on_device(1))
        OOMB_CUDA(cudaFuncSetAttribute(attn_fwd_tc4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kF4Smem));
    // Head dim 64 runs the 128-wide tiles with the upper 64 columns zero: TMA fills the boxes past
    // the tensor's hd columns with zeros, so S = Q K^T is exact and O's upper columns stay 0.
    const CUtensorMap tq = map_rows_heads(q, g.C, g.Hq, g.hd);
    const CUtensorMap tkc = map_rows_heads(k_cur, g.C, g.Hkv, g.hd);
    const CUtensorMap tvc = map_rows_heads(v_cur, g.C, g.Hkv, g.hd);
    const int num_sms = device_sms();
    const int zs = OOMB_FWD_SPLIT ? attn_tc_splits(g, num_sms) : 1;
    const int64_t rows = static_cast<int64_t>(g.C) * g.Hq;
    F4Params p{g, sel_off, sel_ids, d_kvslot_layer, static_cast<__nv_bfloat16*>(out), lse, d_err, nullptr, nullptr};
    if (zs > 1) {  // partials in the stream's scratch: [Z][rows][hd] O, then [Z][rows] LSE
        const size_t ob = static_cast<size_t>(zs) * rows * g.hd * sizeof(float);
        uint8_t* w = static_cast<uint8_t*>(stream_scratch(st, 0, ob + static_cast<size_t>(zs) * rows * sizeof(float)));
        p.o_part = reinterpret_cast<float*>(w);
        p.lse_part = reinterpret_cast<float*>(w + ob);
    }
    attn_fwd_tc4_kernel<<<dim3(g.Hq, g.C / kTile, zs), 384, kF4Smem, st>>>(tq, tkc, tvc, maps.kpool, maps.vpool, p);
    check_launch("attn_fwd_tc4_kernel");
    if (zs > 1) {
        fwd_split_merge_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, st>>>(
            p.o_part, p.lse_part, zs, rows, g.hd, static_cast<__nv_bfloat16*>(out), lse);
        check_launch("fwd_split_merge_kernel");
    }
}

}  // namespace oomb
