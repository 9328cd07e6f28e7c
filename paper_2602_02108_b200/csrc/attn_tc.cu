// SPDX-License-Identifier: Apache-2.0
//
// sm_100a tensor-core kernels of the hot path (bf16 in, fp32 accumulate):
//   * attn_fwd_tc: paged flash forward — attention.hpp:156-208 on tcgen05.
//     One CTA per (128-token query tile, q-head). K/V tiles of 128 keys are
//     fetched by TMA straight out of the paged pool through the page table
//     (one tile coordinate per selected page), then the chunk's causal prefix
//     from k_cur/v_cur. S = Q K^T and O += P V run on tcgen05 with S (double
//     buffered) and O accumulators in TMEM; softmax warps own one row each.
//   * debug_tc_gemm: a single-tile GEMM through the very same TMA / UMMA
//     descriptor builders, used by the tests to validate the bit layouts.
//
// Warp roles (256 threads): w0 = TMA producer for Q and K, w1 = MMA issuer,
// w2 = TMA producer for V, w3 = TMEM allocator, w4..w7 = softmax / epilogue
// (warp w reads TMEM lanes 32*(w%4)..+31, i.e. rows of the tile).

#include "oomb_internal.h"
#include "ptx.cuh"

namespace oomb {

namespace {

constexpr int kTile = 128;                     // query rows per CTA, keys per block
constexpr int kHd = 128;                       // head dim of the tensor-core path
constexpr int kRegion = kTile * 64 * 2;        // one [128 x 64] bf16 SW128 region = 16 KB
constexpr int kTileBytes = 2 * kRegion;        // a [128 x 128] bf16 tile = 32 KB
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kRescaleThreshold = 8.0f;      // log2 units (factor 256) before O is rescaled

// smem map of the forward kernel (all 1024-B aligned)
constexpr int kSmemQ = 0;
constexpr int kSmemK = kSmemQ + kTileBytes;          // 2 stages
constexpr int kSmemV = kSmemK + 2 * kTileBytes;      // 2 stages
constexpr int kSmemP = kSmemV + 2 * kTileBytes;      // 2 buffers
constexpr int kSmemBar = kSmemP + 2 * kTileBytes;    // barriers
constexpr int kFwdSmem = kSmemBar + 256 + 1024;      // + alignment slack

struct FwdBars {
    uint64_t q_full;
    uint64_t k_full[2], k_empty[2];
    uint64_t v_full[2], v_empty[2];
    uint64_t s_full[2], s_free[2];
    uint64_t p_full[2];
    uint64_t pv_done[2];
    uint32_t tmem_base;
};

__device__ __forceinline__ uint4 tc_pack8(const float* e) {
    uint4 pk;
    pk.x = pack_bf16(e[0], e[1]);
    pk.y = pack_bf16(e[2], e[3]);
    pk.z = pack_bf16(e[4], e[5]);
    pk.w = pack_bf16(e[6], e[7]);
    return pk;
}

// Write 8 consecutive bf16 (packed in 4 u32) of row r, 16-byte chunk c (0..15) of a
// K-major SW128 [128 x 128] tile made of two [128 x 64] regions.
__device__ __forceinline__ void st_sw128_chunk(uint8_t* tile, int r, int c, uint4 v) {
    const int region = c >> 3;
    const int cc = c & 7;
    uint8_t* p = tile + region * kRegion + r * 128 + ((cc ^ (r & 7)) << 4);
    *reinterpret_cast<uint4*>(p) = v;
}

__device__ __forceinline__ uint64_t desc_kmajor(uint32_t tile_saddr, int kstep) {
    // kstep of 16 elements: region kstep/4, +32 B inside the 128-B swizzle atom
    return make_sdesc_sw128(tile_saddr + (kstep >> 2) * kRegion + (kstep & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t tile_saddr, int kstep) {
    // B operand [K rows][N] with N split into 64-wide regions (LBO = region stride),
    // 8-row groups at 1024 B (SBO); a K step of 16 rows advances 2048 B.
    return make_sdesc_sw128(tile_saddr + kstep * 2048, kRegion, 1024);
}

}  // namespace

bool tc_supported(const AttnGeom& g, int dtype) {
    return dtype == OOMB_BF16 && g.hd == kHd && g.P % kTile == 0 && g.C % kTile == 0;
}

static void encode_or_throw(CUtensorMap* m, uint32_t rank, const void* base, const uint64_t* dims,
                            const uint64_t* strides, const uint32_t* box) {
    CUresult r = encode_tensor_map(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides,
                                   box, CU_TENSOR_MAP_SWIZZLE_128B);
    if (r != CUDA_SUCCESS) throw Error(OOMB_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

void make_pool_maps(TcPoolMaps& maps, const void* kpool, const void* vpool, int64_t n_slots, const float* gkpool,
                    const float* gvpool, int64_t n_g_slots, int Hkv, int P, int hd) {
    const uint64_t dims[2] = {static_cast<uint64_t>(hd), static_cast<uint64_t>(n_slots) * Hkv * P};
    const uint64_t strides[1] = {static_cast<uint64_t>(hd) * 2};
    const uint32_t box[2] = {64, kTile};
    encode_or_throw(&maps.kpool, 2, kpool, dims, strides, box);
    encode_or_throw(&maps.vpool, 2, vpool, dims, strides, box);
    // fp32 gradient pools: 32-column boxes (128 B rows) for the dK/dV TMA reduce-add epilogue
    const uint64_t gdims[2] = {static_cast<uint64_t>(hd), static_cast<uint64_t>(n_g_slots) * Hkv * P};
    const uint64_t gstrides[1] = {static_cast<uint64_t>(hd) * 4};
    const uint32_t gbox[2] = {32, kTile};
    CUresult r = encode_tensor_map(&maps.gkpool, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(gkpool), gdims,
                                   gstrides, gbox, CU_TENSOR_MAP_SWIZZLE_128B);
    if (r == CUDA_SUCCESS)
        r = encode_tensor_map(&maps.gvpool, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(gvpool), gdims,
                              gstrides, gbox, CU_TENSOR_MAP_SWIZZLE_128B);
    if (r != CUDA_SUCCESS) throw Error(OOMB_CUDA_ERROR, "cuTensorMapEncodeTiled (grad pool) failed: " + std::to_string(r));
    maps.valid = true;
}

// [rows][heads][hd] bf16 tensor viewed as 3-D {hd, heads, rows}; box {64, 1, 128}.
static CUtensorMap map_rows_heads(const void* base, int64_t rows, int heads, int hd) {
    CUtensorMap m;
    const uint64_t dims[3] = {static_cast<uint64_t>(hd), static_cast<uint64_t>(heads), static_cast<uint64_t>(rows)};
    const uint64_t strides[2] = {static_cast<uint64_t>(hd) * 2, static_cast<uint64_t>(heads) * hd * 2};
    const uint32_t box[3] = {64, 1, kTile};
    encode_or_throw(&m, 3, base, dims, strides, box);
    return m;
}

// ===========================================================================
// Forward
// ===========================================================================
struct FwdParams {
    AttnGeom g;
    const int32_t* sel_off;
    const int32_t* sel_ids;
    const int32_t* kvslot;
    __nv_bfloat16* out;
    float* lse;
    int* err;
};

// Key block j of CTA (qt): past blocks first (selected pages in list order, P/128
// blocks each), then the chunk's blocks 0..qt (the last one is the diagonal).
struct BlockInfo {
    bool past;
    int row;      // TMA row coordinate (pool map row, or chunk token)
    int n_valid;  // valid keys in the block (past pages may be partially filled)
    bool diag;
};

__device__ __forceinline__ BlockInfo block_info(const FwdParams& p, int qt, int kvh, int j, int n_past_blocks,
                                                int sel_begin, bool report) {
    const AttnGeom& g = p.g;
    BlockInfo b{};
    if (j < n_past_blocks) {
        const int bpp = g.P / kTile;
        const int pid = p.sel_ids[sel_begin + j / bpp];
        const int sub = j % bpp;
        int slot = (pid >= 0 && pid < g.max_pages) ? p.kvslot[pid] : -1;
        int64_t nv = g.filled - static_cast<int64_t>(pid) * g.P - static_cast<int64_t>(sub) * kTile;
        b.n_valid = static_cast<int>(nv < 0 ? 0 : (nv > kTile ? kTile : nv));
        if (slot < 0) {
            if (report) atomicOr(p.err, (pid >= 0 && pid < g.max_pages) ? DERR_NOT_RESIDENT : DERR_BAD_ID);
            slot = 0;
            b.n_valid = 0;
        }
        b.past = true;
        b.row = (slot * g.Hkv + kvh) * g.P + sub * kTile;
        b.diag = false;
    } else {
        const int cb = j - n_past_blocks;
        b.past = false;
        b.row = cb * kTile;
        b.n_valid = kTile;
        b.diag = cb == qt;
    }
    return b;
}

__global__ void __launch_bounds__(256, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kc,
                       const __grid_constant__ CUtensorMap tm_vc, const __grid_constant__ CUtensorMap tm_kp,
                       const __grid_constant__ CUtensorMap tm_vp, FwdParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    FwdBars* bars = reinterpret_cast<FwdBars*>(smem + kSmemBar);
    const AttnGeom& g = p.g;
    const int h = blockIdx.x;
    const int qt = (g.C / kTile) - 1 - static_cast<int>(blockIdx.y);  // longest causal prefix first (LPT)
    const int kvh = h / g.group;
    const int qp = (qt * kTile) / g.P;
    const int sel_begin = p.sel_off[qp];
    const int n_sel = p.sel_off[qp + 1] - sel_begin;
    const int n_past_blocks = n_sel * (g.P / kTile);
    const int nb = n_past_blocks + qt + 1;
    const int warp = warp_id(), lane = lane_id();

    if (threadIdx.x == 0) {
        mbar_init(&bars->q_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->k_full[i], 1);
            mbar_init(&bars->k_empty[i], 1);
            mbar_init(&bars->v_full[i], 1);
            mbar_init(&bars->v_empty[i], 1);
            mbar_init(&bars->s_full[i], 1);
            mbar_init(&bars->s_free[i], 128);
            mbar_init(&bars->p_full[i], 128);
            mbar_init(&bars->pv_done[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == 3) tmem_alloc<512>(&bars->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;
    const uint32_t tm_s = tmem;          // S buffers: cols [0,128) and [128,256)
    const uint32_t tm_o = tmem + 256;    // O: cols [256,384)
    uint8_t* sQ = smem + kSmemQ;
    uint8_t* sK = smem + kSmemK;
    uint8_t* sV = smem + kSmemV;
    uint8_t* sP = smem + kSmemP;

    if (warp == 0) {
        // ---------------- Q + K producer
        if (lane == 0) {
            tma_prefetch_desc(&tm_q);
            mbar_expect_tx(&bars->q_full, kTileBytes);
            for (int r = 0; r < 2; ++r) tma_load_3d(sQ + r * kRegion, &tm_q, &bars->q_full, r * 64, h, qt * kTile);
            for (int j = 0; j < nb; ++j) {
                const int st = j & 1;
                if (j >= 2) mbar_wait(&bars->k_empty[st], ((j - 2) >> 1) & 1);
                const BlockInfo b = block_info(p, qt, kvh, j, n_past_blocks, sel_begin, true);
                mbar_expect_tx(&bars->k_full[st], kTileBytes);
                uint8_t* dst = sK + st * kTileBytes;
                for (int r = 0; r < 2; ++r) {
                    if (b.past) tma_load_2d(dst + r * kRegion, &tm_kp, &bars->k_full[st], r * 64, b.row);
                    else tma_load_3d(dst + r * kRegion, &tm_kc, &bars->k_full[st], r * 64, kvh, b.row);
                }
            }
        }
    } else if (warp == 2) {
        // ---------------- V producer
        if (lane == 0) {
            for (int j = 0; j < nb; ++j) {
                const int st = j & 1;
                if (j >= 2) mbar_wait(&bars->v_empty[st], ((j - 2) >> 1) & 1);
                const BlockInfo b = block_info(p, qt, kvh, j, n_past_blocks, sel_begin, false);
                mbar_expect_tx(&bars->v_full[st], kTileBytes);
                uint8_t* dst = sV + st * kTileBytes;
                for (int r = 0; r < 2; ++r) {
                    if (b.past) tma_load_2d(dst + r * kRegion, &tm_vp, &bars->v_full[st], r * 64, b.row);
                    else tma_load_3d(dst + r * kRegion, &tm_vc, &bars->v_full[st], r * 64, kvh, b.row);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        constexpr uint32_t idesc_s = make_idesc_bf16(kTile, kTile, 0, 0);   // Q K^T: both K-major
        constexpr uint32_t idesc_o = make_idesc_bf16(kTile, kHd, 0, 1);     // P V: V is MN-major
        const uint32_t q_addr = smem_u32(sQ);
        mbar_wait(&bars->q_full, 0);
        for (int j = 0; j <= nb; ++j) {
            if (j < nb) {
                const int st = j & 1;
                mbar_wait(&bars->k_full[st], (j >> 1) & 1);
                if (j >= 2) mbar_wait(&bars->s_free[st], ((j - 2) >> 1) & 1);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t k_addr = smem_u32(sK + st * kTileBytes);
                    for (int ks = 0; ks < kHd / 16; ++ks)
                        umma_f16_ss(tm_s + st * kTile, desc_kmajor(q_addr, ks), desc_kmajor(k_addr, ks), idesc_s,
                                    ks > 0);
                    umma_commit(&bars->s_full[st]);
                    umma_commit(&bars->k_empty[st]);
                }
                __syncwarp();
            }
            if (j >= 1) {
                const int i = j - 1;
                const int st = i & 1;
                mbar_wait(&bars->p_full[st], (i >> 1) & 1);
                mbar_wait(&bars->v_full[st], (i >> 1) & 1);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t p_addr = smem_u32(sP + st * kTileBytes);
                    const uint32_t v_addr = smem_u32(sV + st * kTileBytes);
                    for (int ks = 0; ks < kTile / 16; ++ks)
                        umma_f16_ss(tm_o, desc_kmajor(p_addr, ks), desc_mnmajor(v_addr, ks), idesc_o,
                                    (i > 0 || ks > 0) ? 1u : 0u);
                    umma_commit(&bars->v_empty[st]);
                    umma_commit(&bars->pv_done[st]);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // ---------------- softmax: thread = one query row
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const float sl2 = g.scale * kLog2e;
        float m = -INFINITY;  // running max (log2 units) that O and l are relative to
        float l = 0.f;
        const int bpp = g.P / kTile;
        // the selection id of past block j is loaded one block ahead (off the critical path)
        int pid_next = n_past_blocks > 0 ? p.sel_ids[sel_begin] : 0;
        for (int j = 0; j < nb; ++j) {
            const int b = j & 1;
            const int pid = pid_next;
            if (j + 1 < n_past_blocks) pid_next = p.sel_ids[sel_begin + (j + 1) / bpp];
            int lim = kTile - 1;  // keep columns c <= lim
            if (j < n_past_blocks) {
                const int64_t nv = g.filled - static_cast<int64_t>(pid) * g.P - static_cast<int64_t>(j % bpp) * kTile;
                lim = static_cast<int>(nv < 0 ? 0 : (nv > kTile ? kTile : nv)) - 1;
            } else if (j - n_past_blocks == qt) {
                lim = r;  // causal diagonal
            }
            const bool need_mask = (j >= n_past_blocks) ? (j - n_past_blocks == qt) : (lim < kTile - 1);
            mbar_wait(&bars->s_full[b], (j >> 1) & 1);
            tc_fence_after();
            uint32_t sr[kTile];
#pragma unroll
            for (int c = 0; c < kTile / 16; ++c)
                tmem_ld16(tm_s + b * kTile + c * 16 + lane_off, *reinterpret_cast<uint32_t(*)[16]>(&sr[c * 16]));
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(&bars->s_free[b]);
            if (need_mask) {
#pragma unroll
                for (int c = 0; c < kTile; ++c)
                    if (c > lim) sr[c] = __float_as_uint(-INFINITY);
            }
            // row max of the raw scores (8 independent chains), scaled once: sl2 > 0
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
                rescale = j > 0 && m != -INFINITY;
                m = m_new;
            }
            const float m_use = (m == -INFINITY) ? 0.f : m;
            // P buffer b was read by PV_{j-2}
            if (j >= 2) mbar_wait(&bars->pv_done[b], ((j - 2) >> 1) & 1);
            uint8_t* pb = sP + b * kTileBytes;
            float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int c = 0; c < kTile / 8; ++c) {
                float e[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    e[u] = ex2(fmaf(__uint_as_float(sr[c * 8 + u]), sl2, -m_use));
                    rs8[u] += e[u];
                }
                uint4 pk;
                pk.x = pack_bf16(e[0], e[1]);
                pk.y = pack_bf16(e[2], e[3]);
                pk.z = pack_bf16(e[4], e[5]);
                pk.w = pack_bf16(e[6], e[7]);
                st_sw128_chunk(pb, r, c, pk);
            }
            // O rescale (warp-collective TMEM access): needs PV_{j-1} complete.
            if (__any_sync(0xffffffffu, rescale)) {
                mbar_wait(&bars->pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int c = 0; c < kHd / 16; ++c) {
                    uint32_t o[16];
                    tmem_ld16(tm_o + c * 16 + lane_off, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int u = 0; u < 16; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * alpha);
                    tmem_st16(tm_o + c * 16 + lane_off, o);
                }
                tmem_wait_st();
            }
            const float rs = ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
            l = l * alpha + rs;
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(&bars->p_full[b]);
        }
        // epilogue: O / l -> bf16, lse (natural log)
        mbar_wait(&bars->pv_done[(nb - 1) & 1], ((nb - 1) >> 1) & 1);
        tc_fence_after();
        const int t = qt * kTile + r;
        const float inv = 1.f / l;
        __nv_bfloat16* orow = p.out + (static_cast<int64_t>(t) * g.Hq + h) * kHd;
#pragma unroll 1
        for (int c = 0; c < kHd / 16; ++c) {
            uint32_t o[16];
            tmem_ld16(tm_o + c * 16 + lane_off, o);
            tmem_wait_ld();
            uint4 a, bq;
            a.x = pack_bf16(__uint_as_float(o[0]) * inv, __uint_as_float(o[1]) * inv);
            a.y = pack_bf16(__uint_as_float(o[2]) * inv, __uint_as_float(o[3]) * inv);
            a.z = pack_bf16(__uint_as_float(o[4]) * inv, __uint_as_float(o[5]) * inv);
            a.w = pack_bf16(__uint_as_float(o[6]) * inv, __uint_as_float(o[7]) * inv);
            bq.x = pack_bf16(__uint_as_float(o[8]) * inv, __uint_as_float(o[9]) * inv);
            bq.y = pack_bf16(__uint_as_float(o[10]) * inv, __uint_as_float(o[11]) * inv);
            bq.z = pack_bf16(__uint_as_float(o[12]) * inv, __uint_as_float(o[13]) * inv);
            bq.w = pack_bf16(__uint_as_float(o[14]) * inv, __uint_as_float(o[15]) * inv);
            *reinterpret_cast<uint4*>(orow + c * 16) = a;
            *reinterpret_cast<uint4*>(orow + c * 16 + 8) = bq;
        }
        p.lse[static_cast<int64_t>(t) * g.Hq + h] = (m + __log2f(l)) * kLn2;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 3) tmem_dealloc<512>(tmem);
}

// ===========================================================================
// Forward, variant 2: two CTAs per SM. Each CTA keeps S and O in 256 TMEM
// columns and writes P (bf16) back into the S columns, so PV runs as a TS-MMA
// (A = P from TMEM, B = V from smem) and smem holds only Q, K and V (96 KB).
// A CTA's own S -> softmax -> PV chain is serial; the co-resident CTA fills the
// tensor pipe while this one runs its softmax.
// ===========================================================================
constexpr int kF2Q = 0;
constexpr int kF2K = kF2Q + kTileBytes;
constexpr int kF2V = kF2K + kTileBytes;
constexpr int kF2Bar = kF2V + kTileBytes;
constexpr int kF2Smem = kF2Bar + 128 + 1024;

struct F2Bars {
    uint64_t q_full, k_full, k_empty, v_full, v_empty, s_full, p_full, pv_done;
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(192, 2)
    attn_fwd_tc2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kc,
                        const __grid_constant__ CUtensorMap tm_vc, const __grid_constant__ CUtensorMap tm_kp,
                        const __grid_constant__ CUtensorMap tm_vp, FwdParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    F2Bars* bars = reinterpret_cast<F2Bars*>(smem + kF2Bar);
    const AttnGeom& g = p.g;
    const int h = blockIdx.x;
    const int qt = (g.C / kTile) - 1 - static_cast<int>(blockIdx.y);
    const int kvh = h / g.group;
    const int qp = (qt * kTile) / g.P;
    const int sel_begin = p.sel_off[qp];
    const int n_past_blocks = (p.sel_off[qp + 1] - sel_begin) * (g.P / kTile);
    const int nb = n_past_blocks + qt + 1;
    const int warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        mbar_init(&bars->q_full, 1);
        mbar_init(&bars->k_full, 1);
        mbar_init(&bars->k_empty, 1);
        mbar_init(&bars->v_full, 1);
        mbar_init(&bars->v_empty, 1);
        mbar_init(&bars->s_full, 1);
        mbar_init(&bars->p_full, 128);
        mbar_init(&bars->pv_done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<256>(&bars->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;
    const uint32_t tm_s = tmem, tm_o = tmem + 128;  // P (bf16x2) overwrites S columns [0, 64)
    uint8_t* sQ = smem + kF2Q;
    uint8_t* sK = smem + kF2K;
    uint8_t* sV = smem + kF2V;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(&bars->q_full, kTileBytes);
            for (int r = 0; r < 2; ++r) tma_load_3d(sQ + r * kRegion, &tm_q, &bars->q_full, r * 64, h, qt * kTile);
            for (int j = 0; j < nb; ++j) {
                const BlockInfo b = block_info(p, qt, kvh, j, n_past_blocks, sel_begin, true);
                if (j >= 1) mbar_wait(&bars->k_empty, (j - 1) & 1);
                mbar_expect_tx(&bars->k_full, kTileBytes);
                for (int r = 0; r < 2; ++r) {
                    if (b.past) tma_load_2d(sK + r * kRegion, &tm_kp, &bars->k_full, r * 64, b.row);
                    else tma_load_3d(sK + r * kRegion, &tm_kc, &bars->k_full, r * 64, kvh, b.row);
                }
                if (j >= 1) mbar_wait(&bars->v_empty, (j - 1) & 1);
                mbar_expect_tx(&bars->v_full, kTileBytes);
                for (int r = 0; r < 2; ++r) {
                    if (b.past) tma_load_2d(sV + r * kRegion, &tm_vp, &bars->v_full, r * 64, b.row);
                    else tma_load_3d(sV + r * kRegion, &tm_vc, &bars->v_full, r * 64, kvh, b.row);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc_s = make_idesc_bf16(kTile, kTile, 0, 0);
        constexpr uint32_t idesc_o = make_idesc_bf16(kTile, kHd, 0, 1);
        const uint32_t q_addr = smem_u32(sQ), k_addr = smem_u32(sK), v_addr = smem_u32(sV);
        mbar_wait(&bars->q_full, 0);
        for (int j = 0; j < nb; ++j) {
            mbar_wait(&bars->k_full, j & 1);
            if (j >= 1) mbar_wait(&bars->pv_done, (j - 1) & 1);  // PV_{j-1} has read P out of the S columns
            tc_fence_after();
            if (lane == 0) {
                for (int ks = 0; ks < kHd / 16; ++ks)
                    umma_f16_ss(tm_s, desc_kmajor(q_addr, ks), desc_kmajor(k_addr, ks), idesc_s, ks > 0);
                umma_commit(&bars->s_full);
                umma_commit(&bars->k_empty);
            }
            __syncwarp();
            mbar_wait(&bars->p_full, j & 1);
            mbar_wait(&bars->v_full, j & 1);
            tc_fence_after();
            if (lane == 0) {
                for (int ks = 0; ks < kTile / 16; ++ks)
                    umma_f16_ts(tm_o, tm_s + ks * 8, desc_mnmajor(v_addr, ks), idesc_o, (j > 0 || ks > 0) ? 1u : 0u);
                umma_commit(&bars->pv_done);
                umma_commit(&bars->v_empty);
            }
            __syncwarp();
        }
    } else {
        const int quarter = warp & 3;  // warps 2..5 -> lane quarters 2,3,0,1
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const float sl2 = g.scale * kLog2e;
        const int bpp = g.P / kTile;
        float m = -INFINITY, l = 0.f;
        int pid_next = n_past_blocks > 0 ? p.sel_ids[sel_begin] : 0;
        for (int j = 0; j < nb; ++j) {
            const int pid = pid_next;
            if (j + 1 < n_past_blocks) pid_next = p.sel_ids[sel_begin + (j + 1) / bpp];
            int lim = kTile - 1;
            if (j < n_past_blocks) {
                const int64_t nv = g.filled - static_cast<int64_t>(pid) * g.P - static_cast<int64_t>(j % bpp) * kTile;
                lim = static_cast<int>(nv < 0 ? 0 : (nv > kTile ? kTile : nv)) - 1;
            } else if (j - n_past_blocks == qt) {
                lim = r;
            }
            mbar_wait(&bars->s_full, j & 1);
            tc_fence_after();
            // pass 1: row max of the raw scores
            float mx8[8] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int c = 0; c < kTile / 32; ++c) {
                uint32_t a[32];
                tmem_ld32(tm_s + c * 32 + lane_off, a);
                tmem_wait_ld();
#pragma unroll
                for (int u = 0; u < 32; ++u) {
                    const float v = (c * 32 + u <= lim) ? __uint_as_float(a[u]) : -INFINITY;
                    mx8[u & 7] = fmaxf(mx8[u & 7], v);
                }
            }
            const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                   fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
            const float m_new = fmaxf(m, mx);
            float alpha = 1.f;
            bool rescale = false;
            if (m == -INFINITY || m_new > m + kRescaleThreshold) {
                alpha = (m == -INFINITY) ? 0.f : ex2(m - m_new);
                rescale = j > 0 && m != -INFINITY;
                m = m_new;
            }
            const float m_use = (m == -INFINITY) ? 0.f : m;
            // O rescale: PV_{j-1} is complete (S_j was issued after it)
            if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll 1
                for (int c = 0; c < kHd / 16; ++c) {
                    uint32_t o[16];
                    tmem_ld16(tm_o + c * 16 + lane_off, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int u = 0; u < 16; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * alpha);
                    tmem_st16(tm_o + c * 16 + lane_off, o);
                }
            }
            // pass 2: P = exp2(s*sl2 - m) packed bf16x2 into S columns [0, 64)
            float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int c = 0; c < kTile / 32; ++c) {
                uint32_t a[32];
                tmem_ld32(tm_s + c * 32 + lane_off, a);
                tmem_wait_ld();
                uint32_t pk[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int c0 = c * 32 + 2 * u;
                    float e0 = ex2(fmaf(__uint_as_float(a[2 * u]), sl2, -m_use));
                    float e1 = ex2(fmaf(__uint_as_float(a[2 * u + 1]), sl2, -m_use));
                    e0 = (c0 <= lim) ? e0 : 0.f;
                    e1 = (c0 + 1 <= lim) ? e1 : 0.f;
                    rs8[(2 * u) & 7] += e0;
                    rs8[(2 * u + 1) & 7] += e1;
                    pk[u] = pack_bf16(e0, e1);
                }
                tmem_st16(tm_s + c * 16 + lane_off, pk);  // P cols [16c, 16c+16) — below S cols still unread
            }
            tmem_wait_st();
            const float rs = ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
            l = l * alpha + rs;
            tc_fence_before();
            mbar_arrive(&bars->p_full);
        }
        mbar_wait(&bars->pv_done, (nb - 1) & 1);
        tc_fence_after();
        const int t = qt * kTile + r;
        const float inv = 1.f / l;
        __nv_bfloat16* orow = p.out + (static_cast<int64_t>(t) * g.Hq + h) * kHd;
#pragma unroll 1
        for (int c = 0; c < kHd / 16; ++c) {
            uint32_t o[16];
            tmem_ld16(tm_o + c * 16 + lane_off, o);
            tmem_wait_ld();
            float f[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) f[u] = __uint_as_float(o[u]) * inv;
            *reinterpret_cast<uint4*>(orow + c * 16) = tc_pack8(f);
            *reinterpret_cast<uint4*>(orow + c * 16 + 8) = tc_pack8(f + 8);
        }
        p.lse[static_cast<int64_t>(t) * g.Hq + h] = (m + __log2f(l)) * kLn2;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<256>(tmem);
}

static int fwd_variant() {
    static int v = [] {
        const char* e = getenv("OOMB_FWD_KERNEL");
        return e ? atoi(e) : 4;  // measured fastest at c3 (variant 5: 175 ms, 3: 165, 4: 157)
    }();
    return v;
}

void launch_attn_fwd_tc(const AttnGeom& g, const TcPoolMaps& maps, const void* q, const int32_t* sel_off,
                        const int32_t* sel_ids, const int32_t* d_kvslot_layer, const void* k_cur, const void* v_cur,
                        void* out, float* lse, int* d_err, cudaStream_t st) {
    ProfScope prof_(PK_FWD, st);
    if (fwd_variant() == 5) {
        launch_attn_fwd_tc5(g, maps, q, sel_off, sel_ids, d_kvslot_layer, k_cur, v_cur, out, lse, d_err, st);
        return;
    }
    if (fwd_variant() == 4 || !g.chunk_keys) {  // variants 4, 5 implement the past-only (range shard) mode
        launch_attn_fwd_tc4(g, maps, q, sel_off, sel_ids, d_kvslot_layer, k_cur, v_cur, out, lse, d_err, st);
        return;
    }
    if (fwd_variant() == 3) {
        launch_attn_fwd_tc3(g, maps, q, sel_off, sel_ids, d_kvslot_layer, k_cur, v_cur, out, lse, d_err, st);
        return;
    }
    static bool attr_set = false;
    if (!attr_set) {
        OOMB_CUDA(cudaFuncSetAttribute(attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem));
        OOMB_CUDA(cudaFuncSetAttribute(attn_fwd_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kF2Smem));
        attr_set = true;
    }
    const CUtensorMap tq = map_rows_heads(q, g.C, g.Hq, kHd);
    const CUtensorMap tkc = map_rows_heads(k_cur, g.C, g.Hkv, kHd);
    const CUtensorMap tvc = map_rows_heads(v_cur, g.C, g.Hkv, kHd);
    FwdParams p{g, sel_off, sel_ids, d_kvslot_layer, static_cast<__nv_bfloat16*>(out), lse, d_err};
    dim3 grid(g.Hq, g.C / kTile);
    if (fwd_variant() == 2) {
        attn_fwd_tc2_kernel<<<grid, 192, kF2Smem, st>>>(tq, tkc, tvc, maps.kpool, maps.vpool, p);
        check_launch("attn_fwd_tc2_kernel");
    } else {
        attn_fwd_tc_kernel<<<grid, 256, kFwdSmem, st>>>(tq, tkc, tvc, maps.kpool, maps.vpool, p);
        check_launch("attn_fwd_tc_kernel");
    }
}

// ===========================================================================
// Descriptor-validation GEMM: one 128 x N tile, K <= 128, single stage.
// mode 0: C = A B^T, A [128][K], B [N][K] (both via TMA, K-major)
// mode 1: C = A B,   A via TMA (K-major), B [K][N] via TMA (MN-major)
// mode 2: C = A B,   A written by threads with the manual SW128 swizzle, B as mode 1
// ===========================================================================
constexpr int kDbgSmem = 32768 + 65536 + 1024 + 1024;

__global__ void __launch_bounds__(128, 1)
    debug_gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                      const __nv_bfloat16* a_raw, float* c, int n, int k, int mode) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;              // K/64 regions of [128 x 64]
    uint8_t* sB = smem + 32768;      // mode 0: K/64 regions of [N x 64]; mode 1/2: N/64 regions of [K x 64]
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 32768 + 65536);
    uint64_t* mma_bar = bar + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(mma_bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(tslot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const bool a_tmem = mode >= 3;  // A operand staged in TMEM columns [256, 256 + K/2)
    if (threadIdx.x == 0) {
        const int a_bytes = (mode == 2 || a_tmem) ? 0 : 128 * k * 2;
        mbar_expect_tx(bar, a_bytes + n * k * 2);
        if (mode != 2 && !a_tmem)
            for (int kb = 0; kb < k / 64; ++kb) tma_load_2d(sA + kb * kRegion, &ta, bar, kb * 64, 0);
        if (mode == 0 || mode == 4)
            for (int kb = 0; kb < k / 64; ++kb) tma_load_2d(sB + kb * n * 128, &tb, bar, kb * 64, 0);
        else
            for (int nb = 0; nb < n / 64; ++nb) tma_load_2d(sB + nb * k * 128, &tb, bar, nb * 64, 0);
    }
    if (mode == 2) {
        const int r = threadIdx.x;
        for (int cidx = 0; cidx < k / 8; ++cidx) {
            const uint4 v = *reinterpret_cast<const uint4*>(a_raw + static_cast<int64_t>(r) * k + cidx * 8);
            const int region = cidx >> 3, cc = cidx & 7;
            *reinterpret_cast<uint4*>(sA + region * kRegion + r * 128 + ((cc ^ (r & 7)) << 4)) = v;
        }
        fence_proxy_async_smem();
    }
    if (a_tmem) {  // row r -> TMEM lane r, bf16 pairs packed per 32-bit column
        const int r = threadIdx.x;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(a_raw + static_cast<int64_t>(r) * k);
        for (int c = 0; c < k / 32; ++c) {
            uint32_t v[16];
            for (int u = 0; u < 16; ++u) v[u] = src[c * 16 + u];
            tmem_st16(tmem + 256 + c * 16 + (static_cast<uint32_t>(warp * 32) << 16), v);
        }
        tmem_wait_st();
        tc_fence_before();
    }
    __syncthreads();
    mbar_wait(bar, 0);
    tc_fence_after();
    if (threadIdx.x == 0) {
        const bool b_kmajor = mode == 0 || mode == 4;
        const uint32_t idesc = make_idesc_bf16(128, n, 0, b_kmajor ? 0 : 1);
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        for (int ks = 0; ks < k / 16; ++ks) {
            const uint64_t ad = make_sdesc_sw128(a0 + (ks >> 2) * kRegion + (ks & 3) * 32, 16, 1024);
            uint64_t bd;
            if (b_kmajor) bd = make_sdesc_sw128(b0 + (ks >> 2) * n * 128 + (ks & 3) * 32, 16, 1024);
            else bd = make_sdesc_sw128(b0 + ks * 2048, k * 128, 1024);
            if (a_tmem) umma_f16_ts(tmem, tmem + 256 + ks * 8, bd, idesc, ks > 0);
            else umma_f16_ss(tmem, ad, bd, idesc, ks > 0);
        }
        umma_commit(mma_bar);
    }
    __syncwarp();
    mbar_wait(mma_bar, 0);
    tc_fence_after();
    const int r = warp * 32 + lane;
    for (int cc = 0; cc < n / 16; ++cc) {
        uint32_t v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cc * 16, v);
        tmem_wait_ld();
        for (int u = 0; u < 16; ++u) c[static_cast<int64_t>(r) * n + cc * 16 + u] = __uint_as_float(v[u]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

void launch_debug_tc_gemm(int mode, const void* a, const void* b, float* c, int m, int n, int k, cudaStream_t st) {
    OOMB_REQUIRE(k <= 128 && mode >= 0 && mode <= 4, OOMB_SHAPE_ERROR, "debug gemm: K <= 128, mode 0..4");
    static bool attr_set = false;
    if (!attr_set) {
        OOMB_CUDA(cudaFuncSetAttribute(debug_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDbgSmem));
        attr_set = true;
    }
    CUtensorMap ta, tb;
    {
        const uint64_t dims[2] = {static_cast<uint64_t>(k), static_cast<uint64_t>(m)};
        const uint64_t strides[1] = {static_cast<uint64_t>(k) * 2};
        const uint32_t box[2] = {64, 128};
        encode_or_throw(&ta, 2, a, dims, strides, box);
    }
    if (mode == 0 || mode == 4) {
        const uint64_t dims[2] = {static_cast<uint64_t>(k), static_cast<uint64_t>(n)};
        const uint64_t strides[1] = {static_cast<uint64_t>(k) * 2};
        const uint32_t box[2] = {64, static_cast<uint32_t>(n)};
        encode_or_throw(&tb, 2, b, dims, strides, box);
    } else {
        const uint64_t dims[2] = {static_cast<uint64_t>(n), static_cast<uint64_t>(k)};
        const uint64_t strides[1] = {static_cast<uint64_t>(n) * 2};
        const uint32_t box[2] = {64, static_cast<uint32_t>(k)};
        encode_or_throw(&tb, 2, b, dims, strides, box);
    }
    debug_gemm_kernel<<<1, 128, kDbgSmem, st>>>(ta, tb, static_cast<const __nv_bfloat16*>(a), c, n, k, mode);
    check_launch("debug_gemm_kernel");
}

}  // namespace oomb
