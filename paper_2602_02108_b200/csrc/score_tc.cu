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

constexpr int kQpGroup = 8;  // query pages per vote CTA

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

// ---------------------------------------------------------------- pass 1
constexpr int kStQ = 0;
constexpr int kStK = kStQ + kTileBytes;            // 3 stages of {hi, lo} K_avg tiles
constexpr int kStBar = kStK + 3 * 2 * kTileBytes;
constexpr int kStSmem = kStBar + 256 + 1024;

struct StatsBars {
    uint64_t q_full;
    uint64_t k_full[3], k_empty[3];
    uint64_t st_empty[3];  // vote kernel: the compute warps finished reading a stage's stats
    uint64_t s_full[2], s_free[2];
    uint32_t tmem_base;
};

struct ScoreParams {
    int C, Hq, Hkv, hd, P, n, n_pad, m;
    float sl2;  // score scale * log2(e)
    float* m2;  // [Hq][C] running max (log2 units)
    float* il;  // [Hq][C] 1 / sum
    float* vote_part;  // [Hkv][m][n]
    int lo_row;        // first row of the lo plane in the K_avg map (= Hkv * n_pad)
};

__global__ void __launch_bounds__(192, 1)
    score_stats_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_ka,
                       ScoreParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    StatsBars* bars = reinterpret_cast<StatsBars*>(smem + kStBar);
    const int h = blockIdx.x, qt = blockIdx.y;
    const int kvh = h / (p.Hq / p.Hkv);
    const int nb = p.n_pad / kTile;
    const int warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        mbar_init(&bars->q_full, 1);
        for (int i = 0; i < 3; ++i) {
            mbar_init(&bars->k_full[i], 1);
            mbar_init(&bars->k_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->s_full[i], 1);
            mbar_init(&bars->s_free[i], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<256>(&bars->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;
    uint8_t* sQ = smem + kStQ;
    uint8_t* sK = smem + kStK;
    if (warp == 0) {
        if (lane == 0) {  // producer
            mbar_expect_tx(&bars->q_full, kTileBytes);
            for (int r = 0; r < 2; ++r) tma_load_3d(sQ + r * kRegion, &tm_q, &bars->q_full, r * 64, h, qt * kTile);
            for (int j = 0; j < nb; ++j) {
                const int st = j % 3;
                if (j >= 3) mbar_wait(&bars->k_empty[st], ((j - 3) / 3) & 1);
                mbar_expect_tx(&bars->k_full[st], 2 * kTileBytes);
                for (int pl = 0; pl < 2; ++pl)
                    for (int r = 0; r < 2; ++r)
                        tma_load_2d(sK + (2 * st + pl) * kTileBytes + r * kRegion, &tm_ka, &bars->k_full[st], r * 64,
                                    pl * p.lo_row + kvh * p.n_pad + j * kTile);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = make_idesc_bf16(kTile, kTile, 0, 0);
        const uint32_t q_addr = smem_u32(sQ);
        mbar_wait(&bars->q_full, 0);
        for (int j = 0; j < nb; ++j) {
            const int st = j % 3, b = j & 1;
            mbar_wait(&bars->k_full[st], (j / 3) & 1);
            if (j >= 2) mbar_wait(&bars->s_free[b], ((j - 2) >> 1) & 1);
            tc_fence_after();
            if (lane == 0) {
                for (int pl = 0; pl < 2; ++pl) {  // S = Q hi^T + Q lo^T
                    const uint32_t k_addr = smem_u32(sK + (2 * st + pl) * kTileBytes);
                    for (int ks = 0; ks < kHd / 16; ++ks)
                        umma_f16_ss(tmem + b * kTile, desc_k(q_addr, ks, kRegion), desc_k(k_addr, ks, kRegion),
                                    idesc, (pl > 0 || ks > 0) ? 1u : 0u);
                }
                umma_commit(&bars->s_full[b]);
                umma_commit(&bars->k_empty[st]);
            }
            __syncwarp();
        }
    } else {
        const int quarter = warp & 3;  // warps 2..5 -> quarters 2,3,0,1
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nb; ++j) {
            const int b = j & 1;
            mbar_wait(&bars->s_full[b], (j >> 1) & 1);
            tc_fence_after();
            float s[kTile];
#pragma unroll
            for (int c = 0; c < kTile / 16; ++c)
                tmem_ld16(tmem + b * kTile + c * 16 + lane_off, *reinterpret_cast<uint32_t(*)[16]>(&s[c * 16]));
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(&bars->s_free[b]);
            const int valid = p.n - j * kTile;  // columns >= valid are padding
            if (valid < kTile) {
#pragma unroll
                for (int c = 0; c < kTile; ++c)
                    if (c >= valid) s[c] = -INFINITY;
            }
            float mx8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) mx8[u] = s[u];
#pragma unroll
            for (int c = 8; c < kTile; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], s[c]);
            const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                   fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * p.sl2;
            const float m_new = fmaxf(m, mx);
            float a8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int c = 0; c < kTile; ++c) a8[c & 7] += ex2(fmaf(s[c], p.sl2, -m_new));
            const float acc = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
            l = (m == -INFINITY ? 0.f : l * ex2(m - m_new)) + acc;
            m = m_new;
        }
        const int t = qt * kTile + r;
        p.m2[static_cast<int64_t>(h) * p.C + t] = m;
        p.il[static_cast<int64_t>(h) * p.C + t] = 1.f / l;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<256>(tmem);
}

// ---------------------------------------------------------------- pass 2
constexpr int kVoK = 0;
constexpr int kVoQ = kVoK + 2 * kTileBytes;        // K_avg {hi, lo}; then 3 stages of Q
constexpr int kVoST = kVoQ + 3 * kTileBytes;       // 3 stages of {m2[128], 1/l[128]} (TMA bulk)
constexpr int kVoBar = kVoST + 3 * 1024;
constexpr int kVoSmem = kVoBar + 256 + 1024;

__global__ void __launch_bounds__(192, 1)
    score_vote_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_ka,
                      ScoreParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    StatsBars* bars = reinterpret_cast<StatsBars*>(smem + kVoBar);  // q_full = K_avg tile, k_* = Q stages
    const int pb = blockIdx.x, kvh = blockIdx.y;
    const int qp0 = blockIdx.z * kQpGroup;
    const int qp1 = min(p.m, qp0 + kQpGroup);
    const int G = p.Hq / p.Hkv;
    const int tpq = p.P / kTile;  // 128-token tiles per query page
    const int per_qp = G * tpq;
    const int n_items = (qp1 - qp0) * per_qp;
    const int warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        mbar_init(&bars->q_full, 1);
        for (int i = 0; i < 3; ++i) {
            mbar_init(&bars->k_full[i], 1);
            mbar_init(&bars->k_empty[i], 1);
            mbar_init(&bars->st_empty[i], 128);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->s_full[i], 1);
            mbar_init(&bars->s_free[i], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<256>(&bars->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;
    uint8_t* sK = smem + kVoK;
    uint8_t* sQ = smem + kVoQ;
    // item i -> (query page, q-head, token tile)
    auto item = [&](int i, int* qp, int* h, int* tile) {
        *qp = qp0 + i / per_qp;
        const int rem = i % per_qp;
        *h = kvh * G + rem / tpq;
        *tile = (*qp) * tpq + rem % tpq;
    };
    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(&bars->q_full, 2 * kTileBytes);
            for (int pl = 0; pl < 2; ++pl)
                for (int r = 0; r < 2; ++r)
                    tma_load_2d(sK + pl * kTileBytes + r * kRegion, &tm_ka, &bars->q_full, r * 64,
                                pl * p.lo_row + kvh * p.n_pad + pb * kTile);
            for (int i = 0; i < n_items; ++i) {
                const int st = i % 3;
                int qp, h, tile;
                item(i, &qp, &h, &tile);
                if (i >= 3) {
                    mbar_wait(&bars->k_empty[st], ((i - 3) / 3) & 1);
                    // the compute warps read this stage's stats and waited on its k_full phase:
                    // only then may the phase advance again (no parity aliasing)
                    mbar_wait(&bars->st_empty[st], ((i - 3) / 3) & 1);
                }
                mbar_expect_tx(&bars->k_full[st], kTileBytes + 1024);
                float* stt = reinterpret_cast<float*>(smem + kVoST) + st * 256;
                bulk_load(stt, p.m2 + static_cast<int64_t>(h) * p.C + tile * kTile, 512, &bars->k_full[st]);
                bulk_load(stt + 128, p.il + static_cast<int64_t>(h) * p.C + tile * kTile, 512, &bars->k_full[st]);
                for (int r = 0; r < 2; ++r)
                    tma_load_3d(sQ + st * kTileBytes + r * kRegion, &tm_q, &bars->k_full[st], r * 64, h,
                                tile * kTile);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = make_idesc_bf16(kTile, kTile, 0, 0);
        const uint32_t k_addr = smem_u32(sK);
        mbar_wait(&bars->q_full, 0);
        for (int i = 0; i < n_items; ++i) {
            const int st = i % 3, b = i & 1;
            mbar_wait(&bars->k_full[st], (i / 3) & 1);
            if (i >= 2) mbar_wait(&bars->s_free[b], ((i - 2) >> 1) & 1);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t q_addr = smem_u32(sQ + st * kTileBytes);
                for (int pl = 0; pl < 2; ++pl)  // S^T = hi Q^T + lo Q^T
                    for (int ks = 0; ks < kHd / 16; ++ks)
                        umma_f16_ss(tmem + b * kTile, desc_k(k_addr + pl * kTileBytes, ks, kRegion),
                                    desc_k(q_addr, ks, kRegion), idesc, (pl > 0 || ks > 0) ? 1u : 0u);
                umma_commit(&bars->s_full[b]);
                umma_commit(&bars->k_empty[st]);
            }
            __syncwarp();
        }
    } else {
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;  // page row of the block
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const int page = pb * kTile + r;
        float acc4[4] = {0.f, 0.f, 0.f, 0.f};
        for (int i = 0; i < n_items; ++i) {
            const int b = i & 1, st = i % 3;
            int qp, h, tile;
            item(i, &qp, &h, &tile);
            mbar_wait(&bars->k_full[st], (i / 3) & 1);  // makes the bulk-copied stats visible
            mbar_wait(&bars->s_full[b], (i >> 1) & 1);
            tc_fence_after();
            float s[kTile];
#pragma unroll
            for (int c = 0; c < kTile / 16; ++c)
                tmem_ld16(tmem + b * kTile + c * 16 + lane_off, *reinterpret_cast<uint32_t(*)[16]>(&s[c * 16]));
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(&bars->s_free[b]);
            const float* mrow = reinterpret_cast<const float*>(smem + kVoST) + st * 256;
            const float* lrow = mrow + 128;
#pragma unroll
            for (int c4 = 0; c4 < kTile / 4; ++c4) {
                const float4 mm = *reinterpret_cast<const float4*>(mrow + c4 * 4);
                const float4 ll = *reinterpret_cast<const float4*>(lrow + c4 * 4);
                acc4[0] = fmaf(ex2(fmaf(s[c4 * 4 + 0], p.sl2, -mm.x)), ll.x, acc4[0]);
                acc4[1] = fmaf(ex2(fmaf(s[c4 * 4 + 1], p.sl2, -mm.y)), ll.y, acc4[1]);
                acc4[2] = fmaf(ex2(fmaf(s[c4 * 4 + 2], p.sl2, -mm.z)), ll.z, acc4[2]);
                acc4[3] = fmaf(ex2(fmaf(s[c4 * 4 + 3], p.sl2, -mm.w)), ll.w, acc4[3]);
            }
            mbar_arrive(&bars->st_empty[st]);
            if ((i + 1) % per_qp == 0) {  // finished every (head, tile) of this query page
                const float acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
                if (page < p.n) p.vote_part[(static_cast<int64_t>(kvh) * p.m + qp) * p.n + page] = acc;
                acc4[0] = acc4[1] = acc4[2] = acc4[3] = 0.f;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<256>(tmem);
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
                     void* ws, cudaStream_t st, bool partial_only) {
    static bool attr = false;
    if (!attr) {
        OOMB_CUDA(cudaFuncSetAttribute(score_stats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kStSmem));
        OOMB_CUDA(cudaFuncSetAttribute(score_vote_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kVoSmem));
        attr = true;
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

    const int64_t tot = static_cast<int64_t>(Hkv) * n_pad * kHd;
    kavg_prep_kernel<<<static_cast<unsigned>(std::min<int64_t>((tot + 255) / 256, 4096)), 256, 0, st>>>(
        kavg_sum, kavg_cnt, kavg_f32, static_cast<int>(n), n_pad, Hkv, kHd, ka);
    check_launch("kavg_prep_kernel");
    CUtensorMap tq = map_rows_heads(q, tokens, Hq, kHd);
    CUtensorMap tka;
    {
        const uint64_t dims[2] = {static_cast<uint64_t>(kHd), 2 * static_cast<uint64_t>(Hkv) * n_pad};
        const uint64_t strides[1] = {static_cast<uint64_t>(kHd) * 2};
        const uint32_t box[2] = {64, kTile};
        encode_or_throw(&tka, 2, ka, dims, strides, box);
    }
    ScoreParams p{static_cast<int>(tokens), Hq, Hkv, kHd, P, static_cast<int>(n), n_pad, m, scale * kLog2e, m2, il,
                  part, Hkv * n_pad};
    score_stats_kernel<<<dim3(Hq, static_cast<unsigned>(tokens / kTile)), 192, kStSmem, st>>>(tq, tka, p);
    check_launch("score_stats_kernel");
    score_vote_kernel<<<dim3(n_pad / kTile, Hkv, (m + kQpGroup - 1) / kQpGroup), 192, kVoSmem, st>>>(tq, tka, p);
    check_launch("score_vote_kernel");
    if (!partial_only) launch_vote_reduce(part, Hkv, static_cast<int64_t>(m) * n, vote, st);
}

}  // namespace oomb
