// SPDX-License-Identifier: Apache-2.0
//
// Shared pieces of the tcgen05 path: shape support, the pool's TMA tensor maps, the forward
// launcher (kernel in attn_fwd4.cu) and debug_tc_gemm — a single-tile GEMM through the very same
// TMA / UMMA descriptor builders, used by the tests to validate the bit layouts (SS and TS forms).

#include "oomb_internal.h"
#include "ptx.cuh"

namespace oomb {

namespace {

constexpr int kTile = 128;                     // query rows per CTA, keys per block
constexpr int kHd = 128;                       // head dim of the tensor-core path
constexpr int kRegion = kTile * 64 * 2;        // one [128 x 64] bf16 SW128 region = 16 KB
constexpr int kHalf = 64;                      // page size 64: one page per TMA box
}  // namespace

// Head dim 128, or 64 on the same 128-wide tiles (upper columns zero, TMA out-of-bounds fill);
// page size a multiple of 128, or 64 (query tiles of two query pages, 64-key half blocks; BASELINE
// configs[0]). Chunks of whole 128-row tiles.
bool tc_supported(const AttnGeom& g, int dtype) {
    return dtype == OOMB_BF16 && (g.hd == kHd || g.hd == 64) && (g.P % kTile == 0 || g.P == kHalf) &&
           g.C % kTile == 0;
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
    const uint32_t rows = P == kHalf ? kHalf : kTile;  // page size 64: one page per box
    const uint32_t box[2] = {64, rows};
    encode_or_throw(&maps.kpool, 2, kpool, dims, strides, box);
    encode_or_throw(&maps.vpool, 2, vpool, dims, strides, box);
    // fp32 gradient pools: 32-column boxes (128 B rows) for the dK/dV TMA reduce-add epilogue
    const uint64_t gdims[2] = {static_cast<uint64_t>(hd), static_cast<uint64_t>(n_g_slots) * Hkv * P};
    const uint64_t gstrides[1] = {static_cast<uint64_t>(hd) * 4};
    const uint32_t gbox[2] = {32, rows};
    CUresult r = encode_tensor_map(&maps.gkpool, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(gkpool), gdims,
                                   gstrides, gbox, CU_TENSOR_MAP_SWIZZLE_128B);
    if (r == CUDA_SUCCESS)
        r = encode_tensor_map(&maps.gvpool, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(gvpool), gdims,
                              gstrides, gbox, CU_TENSOR_MAP_SWIZZLE_128B);
    if (r != CUDA_SUCCESS) throw Error(OOMB_CUDA_ERROR, "cuTensorMapEncodeTiled (grad pool) failed: " + std::to_string(r));
    maps.valid = true;
}


// ===========================================================================
// Forward: the tcgen05 paged flash forward lives in attn_fwd4.cu (key blocks split between two
// softmax warpgroups with their own O accumulators, merged exactly at the end). Earlier designs
// measured at c3 (ms per 1M-token step): one warpgroup + P through smem 237; two CTAs per SM with
// P in TMEM 218; Q in TMEM + column-split groups 165; three S buffers 175; the current split-K 157.
// ===========================================================================
void launch_attn_fwd_tc(const AttnGeom& g, const TcPoolMaps& maps, const void* q, const int32_t* sel_off,
                        const int32_t* sel_ids, const int32_t* d_kvslot_layer, const void* k_cur, const void* v_cur,
                        void* out, float* lse, int* d_err, cudaStream_t st) {
    ProfScope prof_(PK_FWD, st);
    launch_attn_fwd_tc4(g, maps, q, sel_off, sel_ids, d_kvslot_layer, k_cur, v_cur, out, lse, d_err, st);
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
    if (first_use_on_device(4))
        OOMB_CUDA(cudaFuncSetAttribute(debug_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDbgSmem));
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
