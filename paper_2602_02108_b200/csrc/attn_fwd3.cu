// SPDX-License-Identifier: Apache-2.0
//
// Paged flash forward, variant 3 — attention.hpp:156-208 on tcgen05 with every MMA a TS-MMA.
//
// One CTA per (128-row query tile, q-head), one CTA per SM, looping over the tile's key blocks
// (its query page's selected pages in list order, then the chunk's causal prefix). Q is staged
// into TMEM once, so S = Q K^T reads only K from shared memory; P is written back into the S
// columns as packed bf16 and O += P V reads only V. Shared memory then carries the K / V TMA
// stream and one B operand per MMA (~125 B/clk at the tensor rate, under the 128 B/clk port).
//
// S is double buffered: while the softmax warpgroups work on block j, the tensor pipe runs
// S(j+1) and PV(j-1). The two warpgroups split the 128 key columns of each block (64 each);
// they exchange their partial row maxima through shared memory once per block so both use the
// same running max m, and keep partial row sums that are added at the end. O is rescaled only
// when m grows by more than 2^8 (the result is exact either way: O and l stay relative to m).
//
// TMEM (all 512 columns, base 0): Q [0,64) S0 [64,192) S1 [192,320) O [320,448).
// Warp roles (384 threads): w0 K producer, w1 MMA, w2 V producer, w3 TMEM allocator,
// w4..w7 softmax group 0 (key / O columns 0..63), w8..w11 group 1 (64..127).

#include "tc_common.cuh"

namespace oomb {

using namespace tc;

namespace {

constexpr int kKSt = 3, kVSt = 3;  // V stage 2 aliases the Q staging tile (free once Q is in TMEM)
constexpr int kF3Q = 0;
constexpr int kF3K = kF3Q + kTileBytes;
constexpr int kF3V = kF3K + kKSt * kTileBytes;     // V stages 0, 1 (stage 2 = kF3Q)
constexpr int kF3Red = kF3V + 2 * kTileBytes;   // [3][2 groups][128 rows] fp32: maxima by block parity, sums
constexpr int kF3Nv = kF3Red + 3 * 2 * 128 * 4;   // uint8 valid-key counts of the past blocks
constexpr int kF3NvCap = 8192;
constexpr int kF3Bar = kF3Nv + kF3NvCap;
constexpr int kF3Smem = kF3Bar + 256 + 1024;
static_assert(kF3Smem <= 232448, "dynamic shared memory above the 227 KB opt-in limit");
constexpr uint32_t kTmQ = 0, kTmS = 64, kTmO = 320;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef OOMB_FWD_POLY_EVERY
#define OOMB_FWD_POLY_EVERY 0  // measured: the forward is not MUFU-bound; keep every exp2 on MUFU
#endif
constexpr int kPolyEvery = OOMB_FWD_POLY_EVERY;  // 1 in kPolyEvery element pairs use ex2_poly

struct F3Bars {
    uint64_t q_full, q_tmem;
    uint64_t k_full[kKSt], k_empty[kKSt], v_full[kVSt], v_empty[kVSt];
    uint64_t s_full[2], p_full[2], pv_done;
    uint32_t tmem_base;
};

struct F3Params {
    AttnGeom g;
    const int32_t* sel_off;
    const int32_t* sel_ids;
    const int32_t* kvslot;
    __nv_bfloat16* out;
    float* lse;
    int* err;
    CtaTrace tr;
};

// K step ks (16 keys) of the packed P operand: keys [64w, 64w+64) of group w sit in the first
// 32 columns of the group's own 64 S columns.
__host__ __device__ constexpr uint32_t p_col(int ks) { return (ks >> 2) * 64 + (ks & 3) * 8; }

__device__ __forceinline__ void stage_half_row_tmem(const uint8_t* tile, int r, int wg, uint32_t taddr) {
    // columns [64 wg, 64 wg + 64) of a K-major SW128 [128 x 128] tile row -> 32 TMEM columns
#pragma unroll
    for (int c16 = 0; c16 < 2; ++c16) {
        uint32_t v[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = wg * 8 + c16 * 4 + q;  // 16-byte chunk of the row
            const uint4 x =
                *reinterpret_cast<const uint4*>(tile + (c >> 3) * kRegion + r * 128 + (((c & 7) ^ (r & 7)) << 4));
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = x.z;
            v[4 * q + 3] = x.w;
        }
        tmem_st16(taddr + wg * 32 + c16 * 16, v);
    }
}

__global__ void __launch_bounds__(384, 1)
    attn_fwd_tc3_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kc,
                        const __grid_constant__ CUtensorMap tm_vc, const __grid_constant__ CUtensorMap tm_kp,
                        const __grid_constant__ CUtensorMap tm_vp, F3Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    F3Bars* bars = reinterpret_cast<F3Bars*>(smem + kF3Bar);
    const AttnGeom& g = p.g;
    const int h = blockIdx.x;
    const int qt = (g.C / kTile) - 1 - static_cast<int>(blockIdx.y);  // longest causal prefix first (LPT)
    const int kvh = h / g.group;
    const int qp = (qt * kTile) / g.P;
    const int sel_begin = p.sel_off[qp];
    const int n_past = (p.sel_off[qp + 1] - sel_begin) * (g.P / kTile);
    const int nb = n_past + qt + 1;
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        mbar_init(&bars->q_full, 1);
        mbar_init(&bars->q_tmem, 256);
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
            mbar_init(&bars->p_full[i], 256);
        }
        mbar_init(&bars->pv_done, 1);
        fence_barrier_init();
    }
    if (warp == 3) tmem_alloc<512>(&bars->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (bars->tmem_base != 0) __trap();  // all 512 columns: base column 0 (the constants rely on it)
    uint8_t* sQ = smem + kF3Q;
    uint8_t* sK = smem + kF3K;
    uint8_t* sV = smem + kF3V;

    if (warp == 3 && lane == 0 && p.tr.buf && nb > 10) {  // observer: when does s_full of block 9 complete?
        for (int j = 1; j <= 9; j += 2) mbar_wait(&bars->s_full[1], (j >> 1) & 1);
        trace_mark(p.tr, 6);
    }
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
                if (!is_k && j == 2) mbar_wait(&bars->q_tmem, 0);  // V stage 2 reuses the Q staging tile
                mbar_expect_tx(&full[st], kTileBytes);
                uint8_t* dst = (!is_k && st == 2) ? sQ : base + st * kTileBytes;
                if (j < n_past) {
                    const PastBlock b = past_block(g, p.sel_ids, p.kvslot, sel_begin, j, kvh, is_k ? p.err : nullptr);
                    for (int r = 0; r < 2; ++r) tma_load_2d(dst + r * kRegion, mp, &full[st], r * 64, b.row);
                } else {
                    for (int r = 0; r < 2; ++r) tma_load_3d(dst + r * kRegion, mc, &full[st], r * 64, kvh, (j - n_past) * kTile);
                }
            }
        }
    } else if (warp == 1) {
        // MMA warp (converged): S(0) | S(1) PV(0) | S(2) PV(1) | ... | PV(nb-1)
        constexpr uint32_t idesc_s = make_idesc_bf16(kTile, kTile, 0, 0);  // [128 q] x [128 keys], K = hd
        constexpr uint32_t idesc_o = make_idesc_bf16(kTile, kHd, 0, 1);    // [128 q] x [hd], K = keys
        const uint64_t dK = sdesc_k(smem_u32(sK));
        const uint64_t dVmn = sdesc_mn(smem_u32(sV), kRegion);
        const uint64_t dV2mn = sdesc_mn(smem_u32(sQ), kRegion);  // V stage 2 (the Q staging tile)
        mbar_wait(&bars->q_tmem, 0);
        tc_fence_after();
        auto mma_s = [&](int j) {
            const int st = j % kKSt, b = j & 1;
            mbar_wait(&bars->k_full[st], (j / kKSt) & 1);
            if (j == 9 && lane == 0) trace_mark(p.tr, 13);
            tc_fence_after();
            const uint64_t so = boff(st * kTileBytes);
#pragma unroll
            for (int ks = 0; ks < kHd / 16; ++ks)
                umma_ts_w(kTmS + b * 128, kTmQ + ks * 8, dK + so + koff(ks, kRegion), idesc_s, ks);
            umma_commit_w(&bars->s_full[b]);
            umma_commit_w(&bars->k_empty[st]);
        };
        auto mma_pv = [&](int j) {
            const int st = j % kVSt, b = j & 1;
            mbar_wait(&bars->p_full[b], (j >> 1) & 1);
            if (j == 8 && lane == 0) trace_mark(p.tr, 14);
            mbar_wait(&bars->v_full[st], (j / kVSt) & 1);
            if (j == 8 && lane == 0) trace_mark(p.tr, 15);
            tc_fence_after();
            const uint64_t vbase = st == 2 ? dV2mn : dVmn + boff(st * kTileBytes);
            const uint32_t first = j == 0 ? 0u : 1u;
#pragma unroll
            for (int ks = 0; ks < kTile / 16; ++ks)
                umma_ts_w(kTmO, kTmS + b * 128 + p_col(ks), vbase + mnoff(ks), idesc_o, first | ks);
            umma_commit_w(&bars->pv_done);
            umma_commit_w(&bars->v_empty[st]);
        };
        mma_s(0);
        for (int j = 0; j < nb; ++j) {
            const bool tr = j == 8 && lane == 0;
            if (tr) trace_mark(p.tr, 10);
            if (j + 1 < nb) mma_s(j + 1);  // S(j+1) rewrites the buffer PV(j-1) read: issued after it
            if (tr) trace_mark(p.tr, 11);
            mma_pv(j);
            if (tr) trace_mark(p.tr, 12);
        }
    } else if (warp >= 4) {
        const int quarter = warp & 3, wg = (warp - 4) >> 2;
        const int r = quarter * 32 + lane;  // query row = TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        float* red = reinterpret_cast<float*>(smem + kF3Red);  // [2][2][128]
        mbar_wait(&bars->q_full, 0);
        stage_half_row_tmem(sQ, r, wg, kTmQ + lane_off);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars->q_tmem);
        const float sl2 = g.scale * kLog2e;
        uint8_t* nvt = smem + kF3Nv;
        stage_past_valid(g, p.sel_ids, sel_begin, n_past, nvt, kF3NvCap, threadIdx.x - 128, 256);
        named_bar_sync(3, 256);
        float m = -INFINITY;  // running row max (log2 units) that O and l are relative to
        float l = 0.f;        // this group's partial row sum
        for (int j = 0; j < nb; ++j) {
            const int b = j & 1;
            int lim;  // keep key columns c <= lim of this group's 64
            if (j < n_past) {
                lim = past_valid(g, p.sel_ids, sel_begin, nvt, kF3NvCap, j) - 1 - wg * 64;
            } else {
                lim = ((j - n_past == qt) ? r : kTile - 1) - wg * 64;
            }
            const uint32_t tS = kTmS + b * 128 + wg * 64 + lane_off;
            if (j == 9 && threadIdx.x == 128) trace_mark(p.tr, 7);
            mbar_wait(&bars->s_full[b], (j >> 1) & 1);
            const bool tr = (j == 8 || j == 9) && threadIdx.x == 128;
            if (tr) trace_mark(p.tr, j == 8 ? 1 : 5);
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
            // exchange the partial maxima of the two groups (double-buffered by block parity)
            red[(b * 2 + wg) * 128 + r] = mxg;
            if (tr && j == 8) trace_mark(p.tr, 2);
            named_bar_sync(2, 256);
            if (tr && j == 8) trace_mark(p.tr, 3);
            const float mx = fmaxf(mxg, red[(b * 2 + (wg ^ 1)) * 128 + r]) * sl2;
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
#ifdef OOMB_EXP_NOSOFTMAX
            if (true) {
                uint32_t pk[16];
                for (int u = 0; u < 16; ++u) pk[u] = sr[2 * u];
                tmem_st16(tS, pk);
                tmem_st16(tS + 16, pk);
            } else
#endif
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) {
                uint32_t pk[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    // a share of the exponentials runs on the FMA pipe (MUFU is as busy as the tensor core)
                    const float x0 = fmaf(__uint_as_float(sr[c2 * 32 + 2 * u]), sl2, -m_use);
                    const float x1 = fmaf(__uint_as_float(sr[c2 * 32 + 2 * u + 1]), sl2, -m_use);
                    const bool poly = kPolyEvery > 0 && (u % (kPolyEvery > 0 ? kPolyEvery : 1)) == kPolyEvery - 1;
                    const float e0 = poly ? ex2_poly(x0) : ex2(x0);
                    const float e1 = poly ? ex2_poly(x1) : ex2(x1);
                    rs8[(2 * u) & 7] += e0;
                    rs8[(2 * u + 1) & 7] += e1;
                    pk[u] = pack_bf16(e0, e1);
                }
                tmem_st16(tS + c2 * 16, pk);  // P packed into the group's first 32 S columns
            }
            // O rescale: PV(j-1) must have landed (S(j) was issued after it, but completion is
            // what matters for a TMEM read-modify-write)
            if (__any_sync(0xffffffffu, rescale)) {
                mbar_wait(&bars->pv_done, (j - 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    uint32_t o[16];
                    const uint32_t ta = kTmO + wg * 64 + c * 16 + lane_off;
                    tmem_ld16(ta, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int u = 0; u < 16; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * alpha);
                    tmem_st16(ta, o);
                }
            }
            const float rs = ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
            l = l * alpha + rs;
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&bars->p_full[b]);
            if (tr && j == 8) trace_mark(p.tr, 4);
        }
        // ---- epilogue: l = l_0 + l_1, O / l -> bf16 (this group's 64 columns), lse (natural log)
        red[(4 + wg) * 128 + r] = l;  // own buffer: the other group may still read its last maxima
        named_bar_sync(2, 256);
        const float lt = l + red[(4 + (wg ^ 1)) * 128 + r];
        mbar_wait(&bars->pv_done, (nb - 1) & 1);
        tc_fence_after();
        const int t = qt * kTile + r;
        const float inv = 1.f / lt;
        __nv_bfloat16* orow = p.out + (static_cast<int64_t>(t) * g.Hq + h) * kHd + wg * 64;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
            uint32_t o[16];
            tmem_ld16(kTmO + wg * 64 + c * 16 + lane_off, o);
            tmem_wait_ld();
            float f[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) f[u] = __uint_as_float(o[u]) * inv;
            *reinterpret_cast<uint4*>(orow + c * 16) = pack8(f);
            *reinterpret_cast<uint4*>(orow + c * 16 + 8) = pack8(f + 8);
        }
        if (wg == 0) p.lse[static_cast<int64_t>(t) * g.Hq + h] = (m + __log2f(lt)) * kLn2;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 3) tmem_dealloc<512>(0);
}

}  // namespace

void launch_attn_fwd_tc3(const AttnGeom& g, const TcPoolMaps& maps, const void* q, const int32_t* sel_off,
                         const int32_t* sel_ids, const int32_t* d_kvslot_layer, const void* k_cur, const void* v_cur,
                         void* out, float* lse, int* d_err, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        OOMB_CUDA(cudaFuncSetAttribute(attn_fwd_tc3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kF3Smem));
        attr = true;
    }
    const CUtensorMap tq = map_rows_heads(q, g.C, g.Hq, kHd);
    const CUtensorMap tkc = map_rows_heads(k_cur, g.C, g.Hkv, kHd);
    const CUtensorMap tvc = map_rows_heads(v_cur, g.C, g.Hkv, kHd);
    F3Params p{g, sel_off, sel_ids, d_kvslot_layer, static_cast<__nv_bfloat16*>(out), lse, d_err, CtaTrace{}};
    const size_t n_ctas = static_cast<size_t>(g.Hq) * (g.C / kTile);
    p.tr = trace_begin("fwd", n_ctas, 16);
    attn_fwd_tc3_kernel<<<dim3(g.Hq, g.C / kTile), 384, kF3Smem, st>>>(tq, tkc, tvc, maps.kpool, maps.vpool, p);
    check_launch("attn_fwd_tc3_kernel");
    trace_end(p.tr, n_ctas, st);
}

}  // namespace oomb
