// SPDX-License-Identifier: Apache-2.0
//
// Paged flash forward, variant 5 — attention.hpp:156-208 on tcgen05 with THREE S buffers.
//
// One CTA per (128-row query tile, q-head), one CTA per SM, looping over the tile's key blocks
// (its query page's selected pages in list order, then the chunk's causal prefix). The softmax of
// block j cannot start before S(j) lands, and PV(j) cannot start before the softmax has written
// P(j) — with two S buffers S(j+2) is also stuck behind PV(j) (P(j) lives in its buffer), so every
// block pays softmax + PV + S in series. With three buffers S(j+1) and S(j+2) are already in TMEM
// when the softmax finishes block j: the softmax warps run back to back and the tensor pipe only
// waits for P. Two softmax warpgroups (thread = query row) split the 128 key columns of every
// block (64 each), exchange their partial row maxima through smem once per block (both use the
// same online max m), keep partial row sums added at the end, and each rescales / writes its own
// 64 columns of O; O is rescaled only when m grows by more than 2^8.
//
// S = Q K^T is an SS-MMA with N = 128 (full rate); P is written back into its S buffer as packed
// bf16 and O += P V is a TS-MMA.
// TMEM (all 512 columns, base 0): S0 [0,128) S1 [128,256) S2 [256,384) O [384,512).
// Warp roles (384 threads): w0 Q + K producer, w1 MMA, w2 V producer, w3 TMEM allocator,
// w4..w7 softmax group 0 (key / O columns 0..63), w8..w11 group 1 (64..127).

#include "tc_common.cuh"

namespace oomb {

using namespace tc;

namespace {

constexpr int kNS = 3;  // S buffers
constexpr int kKSt = 3, kVSt = 3;
constexpr int kF5Q = 0;
constexpr int kF5K = kF5Q + kTileBytes;
constexpr int kF5V = kF5K + kKSt * kTileBytes;
constexpr int kF5Red = kF5V + kVSt * kTileBytes;  // [2 parities][2 groups][128 rows] partial maxima, then sums
constexpr int kF5Nv = kF5Red + 2 * 2 * 128 * 4;  // uint8 valid-key counts of the past blocks
constexpr int kF5NvCap = 512;                    // blocks beyond it read the selection from global memory
constexpr int kF5Bar = kF5Nv + kF5NvCap;
constexpr int kF5Smem = kF5Bar + 256;
static_assert(kF5Smem <= 232448, "dynamic shared memory above the 227 KB opt-in limit");
constexpr uint32_t kTmS = 0, kTmO = 384;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct F5Bars {
    uint64_t q_full;
    uint64_t k_full[kKSt], k_empty[kKSt], v_full[kVSt], v_empty[kVSt];
    uint64_t s_full[kNS], p_full[kNS], pv_done, o_done;
    uint32_t tmem_base;
};

struct F5Params {
    AttnGeom g;
    const int32_t* sel_off;
    const int32_t* sel_ids;
    const int32_t* kvslot;
    __nv_bfloat16* out;
    float* lse;
    int* err;
};

// K step ks (16 keys) of the packed P operand: keys [64w, 64w+64) of group w sit in the first
// 32 columns of the group's own 64 S columns.
__host__ __device__ constexpr uint32_t p_col(int ks) { return (ks >> 2) * 64 + (ks & 3) * 8; }

__global__ void __launch_bounds__(384, 1)
    attn_fwd_tc5_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kc,
                        const __grid_constant__ CUtensorMap tm_vc, const __grid_constant__ CUtensorMap tm_kp,
                        const __grid_constant__ CUtensorMap tm_vp, F5Params p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    F5Bars* bars = reinterpret_cast<F5Bars*>(smem + kF5Bar);
    const AttnGeom& g = p.g;
    const int h = blockIdx.x;
    const int qt = (g.C / kTile) - 1 - static_cast<int>(blockIdx.y);  // longest causal prefix first (LPT)
    const int kvh = h / g.group;
    const int qp = (qt * kTile) / g.P;
    const int sel_begin = p.sel_off[qp];
    const int n_past = (p.sel_off[qp + 1] - sel_begin) * (g.P / kTile);
    const int nb = n_past + (g.chunk_keys ? qt + 1 : 0);
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
        for (int i = 0; i < kNS; ++i) {
            mbar_init(&bars->s_full[i], 1);
            mbar_init(&bars->p_full[i], 256);
        }
        mbar_init(&bars->pv_done, 1);
        mbar_init(&bars->o_done, 1);
        fence_barrier_init();
    }
    if (warp == 3) tmem_alloc<512>(&bars->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (bars->tmem_base != 0) __trap();  // all 512 columns: base column 0 (the constants rely on it)
    uint8_t* sQ = smem + kF5Q;
    uint8_t* sK = smem + kF5K;
    uint8_t* sV = smem + kF5V;

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
                if (j < n_past) {
                    const PastBlock b = past_block(g, p.sel_ids, p.kvslot, sel_begin, j, kvh, is_k ? p.err : nullptr);
                    for (int r = 0; r < 2; ++r) tma_load_2d(dst + r * kRegion, mp, &full[st], r * 64, b.row);
                } else {
                    for (int r = 0; r < 2; ++r)
                        tma_load_3d(dst + r * kRegion, mc, &full[st], r * 64, kvh, (j - n_past) * kTile);
                }
            }
        }
    } else if (warp == 1) {
        // MMA warp (converged): S(0) S(1) S(2) | PV(0) S(3) | PV(1) S(4) | ... | PV(nb-1)
        constexpr uint32_t idesc_s = make_idesc_bf16(kTile, kTile, 0, 0);  // [128 q] x [128 keys], K = hd
        constexpr uint32_t idesc_o = make_idesc_bf16(kTile, kHd, 0, 1);    // [128 q] x [hd], K = keys
        const uint64_t dQ = sdesc_k(smem_u32(sQ));
        const uint64_t dK = sdesc_k(smem_u32(sK));
        const uint64_t dVmn = sdesc_mn(smem_u32(sV), kRegion);
        mbar_wait(&bars->q_full, 0);
        auto mma_s = [&](int j) {
            const int st = j % kKSt, b = j % kNS;
            mbar_wait(&bars->k_full[st], (j / kKSt) & 1);
            tc_fence_after();
            const uint64_t so = boff(st * kTileBytes);
#pragma unroll
            for (int ks = 0; ks < kHd / 16; ++ks)
                umma_ss_w(kTmS + b * 128, dQ + koff(ks, kRegion), dK + so + koff(ks, kRegion), idesc_s, ks);
            umma_commit_w(&bars->s_full[b]);
            umma_commit_w(&bars->k_empty[st]);
        };
        auto mma_pv = [&](int j) {
            const int st = j % kVSt, b = j % kNS;
            mbar_wait(&bars->p_full[b], (j / kNS) & 1);
            mbar_wait(&bars->v_full[st], (j / kVSt) & 1);
            tc_fence_after();
            const uint64_t so = boff(st * kTileBytes);
            const uint32_t first = j == 0 ? 0u : 1u;
#pragma unroll
            for (int ks = 0; ks < kTile / 16; ++ks)
                umma_ts_w(kTmO, kTmS + b * 128 + p_col(ks), dVmn + so + mnoff(ks), idesc_o, first | ks);
            umma_commit_w(&bars->pv_done);
            umma_commit_w(&bars->v_empty[st]);
        };
        for (int j = 0; j < nb && j < kNS; ++j) mma_s(j);
        for (int j = 0; j < nb; ++j) {
            mma_pv(j);
            if (j + kNS < nb) mma_s(j + kNS);  // S(j+3) rewrites the buffer PV(j) read: issued after it
        }
        umma_commit_w(&bars->o_done);
    } else if (warp >= 4) {
        const int quarter = warp & 3, wg = (warp - 4) >> 2;
        const int r = quarter * 32 + lane;  // query row = TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        float* red = reinterpret_cast<float*>(smem + kF5Red);  // [2][2][128]
        uint8_t* nvt = smem + kF5Nv;
        stage_past_valid(g, p.sel_ids, sel_begin, n_past, nvt, kF5NvCap, threadIdx.x - 128, 256);
        named_bar_sync(3, 256);
        const float sl2 = g.scale * kLog2e;
        const uint32_t tO = kTmO + wg * 64 + lane_off;
        float m = -INFINITY;  // running row max (log2 units) that O and l are relative to
        float l = 0.f;        // this group's partial row sum
        for (int j = 0; j < nb; ++j) {
            const int b = j % kNS, par = j & 1;
            const uint32_t tS = kTmS + b * 128 + wg * 64 + lane_off;
            int lim;  // keep key columns c <= lim of this group's 64
            if (j < n_past) lim = past_valid(g, p.sel_ids, sel_begin, nvt, kF5NvCap, j) - 1 - wg * 64;
            else lim = ((j - n_past == qt) ? r : kTile - 1) - wg * 64;
            mbar_wait(&bars->s_full[b], (j / kNS) & 1);
            tc_fence_after();
            uint32_t sr[64];
            tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
            tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
            tmem_wait_ld();
            if (lim < 63) {
#pragma unroll
                for (int c = 0; c < 64; ++c)
                    if (c > lim) sr[c] = __float_as_uint(-INFINITY);
            }
            float mx8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) mx8[u] = __uint_as_float(sr[u]);
#pragma unroll
            for (int c = 8; c < 64; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sr[c]));
            const float mxg = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                    fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
            red[(par * 2 + wg) * 128 + r] = mxg;  // double-buffered by block parity
            named_bar_sync(2, 256);
            const float mx = fmaxf(mxg, red[(par * 2 + (wg ^ 1)) * 128 + r]) * sl2;
            const float m_new = fmaxf(m, mx);
            bool rescale = false;
            float alpha = 1.f;
            if (m == -INFINITY || m_new > m + kRescaleThreshold) {
                alpha = (m == -INFINITY) ? 0.f : ex2(m - m_new);
                rescale = j > 0 && m != -INFINITY;
                m = m_new;
            }
            const float m_use = (m == -INFINITY) ? 0.f : m;
            float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) {
                uint32_t pk[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const float e0 = ex2(fmaf(__uint_as_float(sr[c2 * 32 + 2 * u]), sl2, -m_use));
                    const float e1 = ex2(fmaf(__uint_as_float(sr[c2 * 32 + 2 * u + 1]), sl2, -m_use));
                    rs8[(2 * u) & 7] += e0;
                    rs8[(2 * u + 1) & 7] += e1;
                    pk[u] = pack_bf16(e0, e1);
                }
                tmem_st16(tS + c2 * 16, pk);  // P packed into the group's first 32 S columns
            }
            // O rescale (this group's 64 columns): PV(j-1) must have landed
            if (__any_sync(0xffffffffu, rescale)) {
                mbar_wait(&bars->pv_done, (j - 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    uint32_t o[16];
                    tmem_ld16(tO + c * 16, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int u = 0; u < 16; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * alpha);
                    tmem_st16(tO + c * 16, o);
                }
            }
            const float rs = ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
            l = l * alpha + rs;
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&bars->p_full[b]);
        }
        // ---- epilogue: l = l_0 + l_1, O / l -> bf16 (this group's 64 columns), lse (natural log);
        // l = 0 only for a page-range shard that attended no key (O never written: zeros, -inf)
        named_bar_sync(2, 256);  // every group is past its last maxima exchange
        red[wg * 128 + r] = l;
        named_bar_sync(2, 256);
        const float lt = l + red[(wg ^ 1) * 128 + r];
        mbar_wait(&bars->o_done, 0);
        tc_fence_after();
        const int t = qt * kTile + r;
        const float inv = lt > 0.f ? 1.f / lt : 0.f;
        __nv_bfloat16* orow = p.out + (static_cast<int64_t>(t) * g.Hq + h) * kHd + wg * 64;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t o[16];
            tmem_ld16(tO + c * 16, o);
            tmem_wait_ld();
            float f[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) f[u] = lt > 0.f ? __uint_as_float(o[u]) * inv : 0.f;
            *reinterpret_cast<uint4*>(orow + c * 16) = pack8(f);
            *reinterpret_cast<uint4*>(orow + c * 16 + 8) = pack8(f + 8);
        }
        if (wg == 0) p.lse[static_cast<int64_t>(t) * g.Hq + h] = lt > 0.f ? (m + __log2f(lt)) * kLn2 : -INFINITY;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 3) tmem_dealloc<512>(0);
}

}  // namespace

void launch_attn_fwd_tc5(const AttnGeom& g, const TcPoolMaps& maps, const void* q, const int32_t* sel_off,
                         const int32_t* sel_ids, const int32_t* d_kvslot_layer, const void* k_cur, const void* v_cur,
                         void* out, float* lse, int* d_err, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        OOMB_CUDA(cudaFuncSetAttribute(attn_fwd_tc5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kF5Smem));
        attr = true;
    }
    const CUtensorMap tq = map_rows_heads(q, g.C, g.Hq, kHd);
    const CUtensorMap tkc = map_rows_heads(k_cur, g.C, g.Hkv, kHd);
    const CUtensorMap tvc = map_rows_heads(v_cur, g.C, g.Hkv, kHd);
    F5Params p{g, sel_off, sel_ids, d_kvslot_layer, static_cast<__nv_bfloat16*>(out), lse, d_err};
    attn_fwd_tc5_kernel<<<dim3(g.Hq, g.C / kTile), 384, kF5Smem, st>>>(tq, tkc, tvc, maps.kpool, maps.vpool, p);
    check_launch("attn_fwd_tc5_kernel");
}

}  // namespace oomb
