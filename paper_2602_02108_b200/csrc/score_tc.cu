// SPDX-License-Identifier: Apache-2.0
//
// tcgen05 page scorer — score_pages (attention.hpp:32-67) for bf16 mode:
//
//   kavg_prep     K_avg = sum * (1/count) (paged_kv.hpp:170-183, fp32 exact), split into
//                 two bf16 planes hi = bf16(K_avg), lo = bf16(K_avg - hi), head-major and
//                 128-padded: [2][Hkv][n_pad][hd]. Every score is q.hi + q.lo accumulated in
//                 fp32 on the tensor cores, so K_avg carries ~16 mantissa bits instead of 8
//                 and the votes stay within ~1e-5 of the fp32 reference — the top-k ids are
//                 then exact wherever the reference's own k-boundary margin exceeds that.
//   score_stats   pass 1, query-major: S = Q K_avg^T per (128-token tile, q-head) over
//                 all candidate blocks; per-row running max / sum of exp (log2 domain).
//   score_vote    pass 2, page-major: S^T = K_avg Q^T per (128-page block, kv group,
//                 group of query pages); each thread owns one page row and sums
//                 exp2(s - m) / l over the tokens of a query page and the group's
//                 q-heads -> per-group partial votes.
//   vote_reduce   vote = sum of the per-group partials in fixed group order, so the
//                 selection is independent of how groups are scheduled (and of how
//                 many GPUs they are sharded over).
// Two exponentials per (token, head, page) triple — the softmax needs normalised
// probabilities before the vote (SURVEY §7 hard part 3).

#include "tc_common.cuh"

namespace oomb {

using namespace tc;

namespace {

#ifndef OOMB_VOTE_QPG
#define OOMB_VOTE_QPG 8
#endif
constexpr int kQpGroup = OOMB_VOTE_QPG;  // query pages per vote CTA (4 / 16 measured no better at c3)
#ifndef OOMB_SCORE_POLY
#define OOMB_SCORE_POLY 4
#endif
constexpr int kScPoly = OOMB_SCORE_POLY;  // 0: every exp2 on MUFU
#ifndef OOMB_STATS_PLANES
#define OOMB_STATS_PLANES 2
#endif
// K_avg planes the stats pass multiplies (2: hi + lo; 1: hi only). The row max only has to be
// consistent between the passes, and the row sum's hi-only error averages out over the
// 128 tokens x G heads a page's vote sums.
constexpr int kStPlanes = OOMB_STATS_PLANES;

__global__ void kavg_prep_kernel(const float* __restrict__ sum, const int32_t* __restrict__ cnt,
                                 const float* __restrict__ kavg_f32, int n, int n_pad, int Hkv, int hd,
                                 __nv_bfloat16* __restrict__ out) {
    const int64_t total = static_cast<int64_t>(Hkv) * n_pad * hd;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int d = static_cast<int>(i % hd);
        const int p = static_cast<int>((i / hd) % n_pad);
        const int h = static_cast<int>(i / (static_cast<int64_t>(hd) * n_pad));
        float v = 0.f;
        if (p < n) {
            const int64_t src = (static_cast<int64_t>(p) * Hkv + h) * hd + d;
            v = kavg_f32 ? kavg_f32[src] : __fmul_rn(sum[src], __fdiv_rn(1.0f, static_cast<float>(cnt[p])));
        }
        const __nv_bfloat16 hi = __float2bfloat16_rn(v);
        out[i] = hi;
        out[total + i] = __float2bfloat16_rn(v - __bfloat162float(hi));
    }
}

struct ScoreParams {
    int C, Hq, Hkv, hd, P, n, n_pad, m;
    float sl2;  // score scale * log2(e)
    float* m2;  // [Hq][C] running max (log2 units)
    float* il;  // [Hq][C] 1 / sum
    float* vote_part;  // [Hkv][m][n]
    int lo_row;        // first row of the lo plane in the K_avg map (= Hkv * kv_stride)
    int kv_stride;     // rows per kv head in a plane (n_pad for kavg_prep's planes, the pool's page capacity
                       // rounded to 128 for the planes the append kernel maintains)
};

// ---------------------------------------------------------------- pass 1
// One CTA per (128-token tile, q-head), looping over all candidate blocks of 128 pages.
// Q is staged into TMEM, so S = Q hi^T + Q lo^T is 16 TS-MMAs per block (smem carries only the
// K_avg planes); S is double buffered. Two softmax warpgroups own page columns [0,64) and
// [64,128) of every block and keep separate online (max, sum) pairs that are merged at the end.
// TMEM: Q [0,64) S0 [64,192) S1 [192,320).
constexpr int kStSt = 3;
constexpr int kStQ = 0;
constexpr int kStK = kStQ + kTileBytes;                 // kStSt stages of {hi, lo} K_avg tiles
constexpr int kStRed = kStK + kStSt * 2 * kTileBytes;   // [2 groups][128] {m, l}
constexpr int kStBar = kStRed + 2 * 128 * 8;
constexpr int kStSmem = kStBar + 256;
static_assert(kStSmem <= 232448, "dynamic shared memory above the 227 KB opt-in limit");
constexpr uint32_t kStTmQ = 0, kStTmS = 64;

struct StatsBars {
    uint64_t q_full, q_tmem;
    uint64_t k_full[kStSt], k_empty[kStSt];
    uint64_t s_full[2], s_free[2];
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(384, 1)
    score_stats_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_ka,
                       ScoreParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    StatsBars* bars = reinterpret_cast<StatsBars*>(smem + kStBar);
    const int h = blockIdx.x, qt = blockIdx.y;
    const int kvh = h / (p.Hq / p.Hkv);
    const int nb = p.n_pad / kTile;
    const int warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023) __trap();
        mbar_init(&bars->q_full, 1);
        mbar_init(&bars->q_tmem, 256);
        for (int i = 0; i < kStSt; ++i) {
            mbar_init(&bars->k_full[i], 1);
            mbar_init(&bars->k_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->s_full[i], 1);
            mbar_init(&bars->s_free[i], 256);
        }
        fence_barrier_init();
    }
    if (warp == 3) tmem_alloc<512>(&bars->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (bars->tmem_base != 0) __trap();
    uint8_t* sQ = smem + kStQ;
    uint8_t* sK = smem + kStK;
    if (warp == 0) {
        if (lane == 0) {  // producer
            mbar_expect_tx(&bars->q_full, kTileBytes);
            for (int r = 0; r < 2; ++r) tma_load_3d(sQ + r * kRegion, &tm_q, &bars->q_full, r * 64, h, qt * kTile);
            for (int j = 0; j < nb; ++j) {
                const int st = j % kStSt;
                if (j >= kStSt) mbar_wait(&bars->k_empty[st], ((j / kStSt) - 1) & 1);
                mbar_expect_tx(&bars->k_full[st], kStPlanes * kTileBytes);
                for (int pl = 0; pl < kStPlanes; ++pl)
                    for (int r = 0; r < 2; ++r)
                        tma_load_2d(sK + (2 * st + pl) * kTileBytes + r * kRegion, &tm_ka, &bars->k_full[st], r * 64,
                                    pl * p.lo_row + kvh * p.kv_stride + j * kTile);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = make_idesc_bf16(kTile, kTile, 0, 0);
        const uint64_t dK = sdesc_k(smem_u32(sK));
        mbar_wait(&bars->q_tmem, 0);
        tc_fence_after();
        for (int j = 0; j < nb; ++j) {
            const int st = j % kStSt, b = j & 1;
            mbar_wait(&bars->k_full[st], (j / kStSt) & 1);
            if (j >= 2) mbar_wait(&bars->s_free[b], ((j - 2) >> 1) & 1);
            tc_fence_after();
#pragma unroll
            for (int pl = 0; pl < kStPlanes; ++pl) {  // S = Q hi^T + Q lo^T
                const uint64_t so = boff((2 * st + pl) * kTileBytes);
#pragma unroll
                for (int ks = 0; ks < kHd / 16; ++ks)
                    umma_ts_w(kStTmS + b * 128, kStTmQ + ks * 8, dK + so + koff(ks, kRegion), idesc, pl | ks);
            }
            umma_commit_w(&bars->s_full[b]);
            umma_commit_w(&bars->k_empty[st]);
        }
    } else if (warp >= 4) {
        const int quarter = warp & 3, wg = (warp - 4) >> 2;
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        mbar_wait(&bars->q_full, 0);
        stage_row_tmem(sQ, kRegion, r, kStTmQ + lane_off);  // both groups write the same values: harmless;
        tmem_wait_st();                                       // group 0 alone would do, but it keeps the
        tc_fence_before();                                    // barrier count uniform
        mbar_arrive(&bars->q_tmem);
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nb; ++j) {
            const int b = j & 1;
            mbar_wait(&bars->s_full[b], (j >> 1) & 1);
            tc_fence_after();
            uint32_t sv[64];
            tmem_ld32(kStTmS + b * 128 + wg * 64 + lane_off, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
            tmem_ld32(kStTmS + b * 128 + wg * 64 + 32 + lane_off, *reinterpret_cast<uint32_t(*)[32]>(&sv[32]));
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(&bars->s_free[b]);
            const int valid = p.n - j * kTile - wg * 64;  // columns >= valid are padding
            if (valid < 64) {
#pragma unroll
                for (int c = 0; c < 64; ++c)
                    if (c >= valid) sv[c] = __float_as_uint(-INFINITY);
            }
            float mx8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) mx8[u] = __uint_as_float(sv[u]);
#pragma unroll
            for (int c = 8; c < 64; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sv[c]));
            const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                   fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * p.sl2;
            const float m_new = fmaxf(m, mx);
            if (m_new == -INFINITY) continue;  // every column so far is padding
            float a8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int c = 0; c < 64; ++c) {  // 1 in kScPoly exponentials on the FMA pipe (MUFU-bound pass)
                const float x = fmaf(__uint_as_float(sv[c]), p.sl2, -m_new);
                a8[c & 7] += (kScPoly > 0 && c % kScPoly == kScPoly - 1) ? ex2_poly4(x) : ex2(x);
            }
            const float acc = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
            l = (m == -INFINITY ? 0.f : l * ex2(m - m_new)) + acc;
            m = m_new;
        }
        // merge the two groups' (max, sum) pairs
        float2* red = reinterpret_cast<float2*>(smem + kStRed);
        red[wg * 128 + r] = make_float2(m, l);
        named_bar_sync(2, 256);
        if (wg == 0) {
            const float2 o = red[128 + r];
            const float mt = fmaxf(m, o.x);
            const float lt = (m == -INFINITY ? 0.f : l * ex2(m - mt)) + (o.x == -INFINITY ? 0.f : o.y * ex2(o.x - mt));
            const int t = qt * kTile + r;
            p.m2[static_cast<int64_t>(h) * p.C + t] = mt;
            p.il[static_cast<int64_t>(h) * p.C + t] = 1.f / lt;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 3) tmem_dealloc<512>(0);
}

// ---------------------------------------------------------------- pass 2
// One CTA per (128-page block, kv group, group of kQpGroup query pages). The block's K_avg hi and
// lo planes are staged into TMEM once, so S^T = hi Q^T + lo Q^T is 16 TS-MMAs per item (item =
// one 128-token tile of one q-head); S^T is double buffered. Thread = page row; the two softmax
// warpgroups own token columns [0,64) / [64,128) and sum exp2(s - m_t) / l_t; their partials are
// added once per query page (all of its tokens and the group's heads) -> per-group partial votes.
// TMEM: hi [0,64) lo [64,128) S^T0 [128,256) S^T1 [256,384).
constexpr int kVoSt = 3;
constexpr int kVoK = 0;                                  // {hi, lo} K_avg tiles (staging)
constexpr int kVoQ = kVoK + 2 * kTileBytes;              // kVoSt stages of Q
constexpr int kVoST = kVoQ + kVoSt * kTileBytes;         // kVoSt stages of {m2[128], 1/l[128]} (TMA bulk)
constexpr int kVoRed = kVoST + kVoSt * 1024;             // [128] partial votes of group 1
constexpr int kVoBar = kVoRed + 512;
constexpr int kVoSmem = kVoBar + 256;
static_assert(kVoSmem <= 232448, "dynamic shared memory above the 227 KB opt-in limit");
constexpr uint32_t kVoTmHi = 0, kVoTmLo = 64, kVoTmS = 128;

struct VoteBars {
    uint64_t ka_full, ka_tmem;
    uint64_t q_full[kVoSt], q_empty[kVoSt];
    uint64_t s_full[2], s_free[2];
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(384, 1)
    score_vote_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_ka,
                      ScoreParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    VoteBars* bars = reinterpret_cast<VoteBars*>(smem + kVoBar);
    const int pb = blockIdx.x, kvh = blockIdx.y;
    const int qp0 = blockIdx.z * kQpGroup;
    const int qp1 = min(p.m, qp0 + kQpGroup);
    const int G = p.Hq / p.Hkv;
    const int tpq = p.P / kTile;  // 128-token tiles per query page
    const int per_qp = G * tpq;
    const int n_items = (qp1 - qp0) * per_qp;
    const int warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023) __trap();
        mbar_init(&bars->ka_full, 1);
        mbar_init(&bars->ka_tmem, 256);
        for (int i = 0; i < kVoSt; ++i) {
            mbar_init(&bars->q_full[i], 1);
            mbar_init(&bars->q_empty[i], 1 + 256);  // MMA done with Q + the softmax warps done with the stats
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->s_full[i], 1);
            mbar_init(&bars->s_free[i], 256);
        }
        fence_barrier_init();
    }
    if (warp == 3) tmem_alloc<512>(&bars->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (bars->tmem_base != 0) __trap();
    uint8_t* sK = smem + kVoK;
    uint8_t* sQ = smem + kVoQ;
    // item i -> (query page, q-head, token tile), query-page major
    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(&bars->ka_full, 2 * kTileBytes);
            for (int pl = 0; pl < 2; ++pl)
                for (int r = 0; r < 2; ++r)
                    tma_load_2d(sK + pl * kTileBytes + r * kRegion, &tm_ka, &bars->ka_full, r * 64,
                                pl * p.lo_row + kvh * p.kv_stride + pb * kTile);
            int qp = qp0, hh = 0, tl = 0;
            for (int i = 0; i < n_items; ++i) {
                const int st = i % kVoSt;
                const int h = kvh * G + hh, tile = qp * tpq + tl;
                if (i >= kVoSt) mbar_wait(&bars->q_empty[st], ((i / kVoSt) - 1) & 1);
                mbar_expect_tx(&bars->q_full[st], kTileBytes + 1024);
                float* stt = reinterpret_cast<float*>(smem + kVoST) + st * 256;
                bulk_load(stt, p.m2 + static_cast<int64_t>(h) * p.C + tile * kTile, 512, &bars->q_full[st]);
                bulk_load(stt + 128, p.il + static_cast<int64_t>(h) * p.C + tile * kTile, 512, &bars->q_full[st]);
                for (int r = 0; r < 2; ++r)
                    tma_load_3d(sQ + st * kTileBytes + r * kRegion, &tm_q, &bars->q_full[st], r * 64, h, tile * kTile);
                if (++tl == tpq) {
                    tl = 0;
                    if (++hh == G) {
                        hh = 0;
                        ++qp;
                    }
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = make_idesc_bf16(kTile, kTile, 0, 0);
        const uint64_t dQ = sdesc_k(smem_u32(sQ));
        mbar_wait(&bars->ka_tmem, 0);
        tc_fence_after();
        for (int i = 0; i < n_items; ++i) {
            const int st = i % kVoSt, b = i & 1;
            mbar_wait(&bars->q_full[st], (i / kVoSt) & 1);
            if (i >= 2) mbar_wait(&bars->s_free[b], ((i - 2) >> 1) & 1);
            tc_fence_after();
            const uint64_t so = boff(st * kTileBytes);
#pragma unroll
            for (int pl = 0; pl < 2; ++pl)  // S^T = hi Q^T + lo Q^T
#pragma unroll
                for (int ks = 0; ks < kHd / 16; ++ks)
                    umma_ts_w(kVoTmS + b * 128, (pl ? kVoTmLo : kVoTmHi) + ks * 8, dQ + so + koff(ks, kRegion), idesc,
                              pl | ks);
            umma_commit_w(&bars->s_full[b]);
            umma_commit_w(&bars->q_empty[st]);
        }
    } else if (warp >= 4) {
        const int quarter = warp & 3, wg = (warp - 4) >> 2;
        const int r = quarter * 32 + lane;  // page row of the block
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const int page = pb * kTile + r;
        mbar_wait(&bars->ka_full, 0);
        stage_row_tmem(sK + wg * kTileBytes, kRegion, r, (wg ? kVoTmLo : kVoTmHi) + lane_off);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars->ka_tmem);
        float* red = reinterpret_cast<float*>(smem + kVoRed);
        float acc4[4] = {0.f, 0.f, 0.f, 0.f};
        int qp = qp0, cnt = 0;
        for (int i = 0; i < n_items; ++i) {
            const int b = i & 1, st = i % kVoSt;
            mbar_wait(&bars->q_full[st], (i / kVoSt) & 1);  // makes the bulk-copied stats visible
            mbar_wait(&bars->s_full[b], (i >> 1) & 1);
            tc_fence_after();
            uint32_t sv[64];
            tmem_ld32(kVoTmS + b * 128 + wg * 64 + lane_off, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
            tmem_ld32(kVoTmS + b * 128 + wg * 64 + 32 + lane_off, *reinterpret_cast<uint32_t(*)[32]>(&sv[32]));
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(&bars->s_free[b]);
            const uint32_t mrow = smem_u32(smem + kVoST) + st * 1024 + wg * 256, lrow = mrow + 512;
#pragma unroll
            for (int c4 = 0; c4 < 16; ++c4) {
                const float4 mm = lds128(mrow + c4 * 16);
                const float4 ll = lds128(lrow + c4 * 16);
                acc4[0] = fmaf(ex2(fmaf(__uint_as_float(sv[c4 * 4 + 0]), p.sl2, -mm.x)), ll.x, acc4[0]);
                acc4[1] = fmaf(ex2(fmaf(__uint_as_float(sv[c4 * 4 + 1]), p.sl2, -mm.y)), ll.y, acc4[1]);
                acc4[2] = fmaf(ex2(fmaf(__uint_as_float(sv[c4 * 4 + 2]), p.sl2, -mm.z)), ll.z, acc4[2]);
                {
                    const float x3 = fmaf(__uint_as_float(sv[c4 * 4 + 3]), p.sl2, -mm.w);
                    acc4[3] = fmaf((kScPoly > 0 && (c4 % (kScPoly > 0 ? kScPoly / 4 + (kScPoly < 4) : 1)) == 0) ? ex2_poly4(x3) : ex2(x3), ll.w, acc4[3]);
                }
            }
            mbar_arrive(&bars->q_empty[st]);  // this stage's stats are consumed (no reuse / parity aliasing)
            if (++cnt == per_qp) {  // every (head, tile) of this query page: add the two groups' partials
                const float a = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
                if (wg == 1) red[r] = a;
                named_bar_sync(2, 256);
                if (wg == 0 && page < p.n) p.vote_part[(static_cast<int64_t>(kvh) * p.m + qp) * p.n + page] = a + red[r];
                named_bar_sync(2, 256);
                acc4[0] = acc4[1] = acc4[2] = acc4[3] = 0.f;
                cnt = 0;
                ++qp;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 3) tmem_dealloc<512>(0);
}

__global__ void vote_reduce_kernel(const float* __restrict__ part, int Hkv, int64_t mn, float* __restrict__ vote) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < mn;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float v = part[i];
        for (int g = 1; g < Hkv; ++g) v += part[g * mn + i];
        vote[i] = v;
    }
}

}  // namespace

bool score_tc_supported(int dtype, int hd, int P, int64_t tokens) {
    return dtype == OOMB_BF16 && hd == kHd && P % kTile == 0 && tokens % kTile == 0 && tokens / P <= 65535;
}

size_t score_tc_workspace(int64_t tokens, int Hq, int Hkv, int64_t n, int P) {
    const int64_t n_pad = (n + kTile - 1) / kTile * kTile;
    const int64_t m = tokens / P;
    return static_cast<size_t>(2 * Hkv * n_pad * kHd * 2) + 2 * static_cast<size_t>(Hq * tokens * 4) +
           static_cast<size_t>(Hkv * m * n * 4) + 4 * 256;
}

void launch_vote_reduce(const float* part, int groups, int64_t mn, float* vote, cudaStream_t st) {
    vote_reduce_kernel<<<static_cast<unsigned>(std::min<int64_t>((mn + 255) / 256, 2048)), 256, 0, st>>>(
        part, groups, mn, vote);
    check_launch("vote_reduce_kernel");
}

void launch_score_tc(const void* q, int64_t tokens, int Hq, int Hkv, int P, const float* kavg_sum,
                     const int32_t* kavg_cnt, const float* kavg_f32, int64_t n, float scale, float* vote,
                     void* ws, cudaStream_t st, bool partial_only, const void* planes_v,
                     int64_t plane_stride) {
    const __nv_bfloat16* planes = static_cast<const __nv_bfloat16*>(planes_v);
    if (first_use_on_device(3)) {
        OOMB_CUDA(cudaFuncSetAttribute(score_stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStSmem));
        OOMB_CUDA(cudaFuncSetAttribute(score_vote_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kVoSmem));
    }
    ProfScope prof_(PK_SCORE, st);
    const int n_pad = static_cast<int>((n + kTile - 1) / kTile * kTile);
    const int m = static_cast<int>(tokens / P);
    uint8_t* w = static_cast<uint8_t*>(ws);
    auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
    __nv_bfloat16* ka = reinterpret_cast<__nv_bfloat16*>(w);
    size_t off = align(static_cast<size_t>(2) * Hkv * n_pad * kHd * 2);
    float* m2 = reinterpret_cast<float*>(w + off);
    off += align(static_cast<size_t>(Hq) * tokens * 4);
    float* il = reinterpret_cast<float*>(w + off);
    off += align(static_cast<size_t>(Hq) * tokens * 4);
    float* part = partial_only ? vote : reinterpret_cast<float*>(w + off);  // [Hkv][m][n]

    // the pool's K_avg planes are kept current by the append kernel (completed pages never change):
    // read them in place; otherwise (fp32 representatives) split K_avg into planes here
    const bool inplace = planes != nullptr && kavg_f32 == nullptr && plane_stride >= n_pad;
    const int kv_stride = inplace ? static_cast<int>(plane_stride) : n_pad;
    if (!inplace) {
        const int64_t tot = static_cast<int64_t>(Hkv) * n_pad * kHd;
        kavg_prep_kernel<<<static_cast<unsigned>(std::min<int64_t>((tot + 255) / 256, 4096)), 256, 0, st>>>(
            kavg_sum, kavg_cnt, kavg_f32, static_cast<int>(n), n_pad, Hkv, kHd, ka);
        check_launch("kavg_prep_kernel");
    }
    CUtensorMap tq = map_rows_heads(q, tokens, Hq, kHd);
    CUtensorMap tka;
    {
        const uint64_t dims[2] = {static_cast<uint64_t>(kHd), 2 * static_cast<uint64_t>(Hkv) * kv_stride};
        const uint64_t strides[1] = {static_cast<uint64_t>(kHd) * 2};
        const uint32_t box[2] = {64, kTile};
        encode_or_throw(&tka, 2, inplace ? const_cast<__nv_bfloat16*>(planes) : ka, dims, strides, box);
    }
    ScoreParams p{static_cast<int>(tokens), Hq, Hkv, kHd, P, static_cast<int>(n), n_pad, m, scale * kLog2e, m2, il,
                  part, Hkv * kv_stride, kv_stride};
    score_stats_kernel<<<dim3(Hq, static_cast<unsigned>(tokens / kTile)), 384, kStSmem, st>>>(tq, tka, p);
    check_launch("score_stats_kernel");
    score_vote_kernel<<<dim3(n_pad / kTile, Hkv, (m + kQpGroup - 1) / kQpGroup), 384, kVoSmem, st>>>(tq, tka, p);
    check_launch("score_vote_kernel");
    if (!partial_only) launch_vote_reduce(part, Hkv, static_cast<int64_t>(m) * n, vote, st);
}

}  // namespace oomb
