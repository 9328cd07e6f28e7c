// SPDX-License-Identifier: Apache-2.0
//
// Shared pieces of the tcgen05 attention kernels: tile geometry, SW128 smem
// layout helpers, UMMA descriptor shortcuts and TMA tensor-map builders.
#pragma once

#include "oomb_internal.h"
#include "ptx.cuh"

namespace oomb {
namespace tc {

constexpr int kTile = 128;               // query rows / keys per block
constexpr int kHd = 128;                 // head dim of the tensor-core path
constexpr int kRegion = kTile * 64 * 2;  // [128 x 64] bf16 SW128 region = 16 KB
constexpr int kTileBytes = 2 * kRegion;  // [128 x 128] bf16 tile = 32 KB
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// 16-byte chunk c (8 bf16) of row r in a K-major SW128 tile made of [rows x 64]
// regions of `region_bytes` each (chunk c lives in region c/8).
__device__ __forceinline__ void st_sw128(uint8_t* tile, int region_bytes, int r, int c, uint4 v) {
    uint8_t* p = tile + (c >> 3) * region_bytes + r * 128 + (((c & 7) ^ (r & 7)) << 4);
    *reinterpret_cast<uint4*>(p) = v;
}

// K-major operand: K step of 16 elements = region kstep/4, +32 B inside the atom.
__device__ __forceinline__ uint64_t desc_k(uint32_t tile, int kstep, int region_bytes) {
    return make_sdesc_sw128(tile + (kstep >> 2) * region_bytes + (kstep & 3) * 32, 16, 1024);
}
// MN-major B operand stored as [K rows][N] in 64-wide N regions (LBO = region stride);
// a K step of 16 rows advances 2048 B.
__device__ __forceinline__ uint64_t desc_mn(uint32_t tile, int kstep, int region_bytes) {
    return make_sdesc_sw128(tile + kstep * 2048, region_bytes, 1024);
}

// Descriptor arithmetic on a precomputed base: the start-address field is the low 14 bits
// (address >> 4) and never carries for shared-memory addresses, so advancing a descriptor
// is one 64-bit add of (byte offset >> 4) — a compile-time constant inside unrolled K loops.
__device__ __forceinline__ uint64_t sdesc_k(uint32_t tile) { return make_sdesc_sw128(tile, 16, 1024); }
__device__ __forceinline__ uint64_t sdesc_mn(uint32_t tile, int region_bytes) {
    return make_sdesc_sw128(tile, region_bytes, 1024);
}
__host__ __device__ constexpr uint64_t koff(int kstep, int region_bytes) {  // K-major K step of 16 elements
    return static_cast<uint64_t>(((kstep >> 2) * region_bytes + (kstep & 3) * 32) >> 4);
}
__host__ __device__ constexpr uint64_t mnoff(int kstep) { return static_cast<uint64_t>((kstep * 2048) >> 4); }
__host__ __device__ constexpr uint64_t boff(int bytes) { return static_cast<uint64_t>(bytes >> 4); }

__device__ __forceinline__ uint4 pack8(const float* e) {
    uint4 pk;
    pk.x = pack_bf16(e[0], e[1]);
    pk.y = pack_bf16(e[2], e[3]);
    pk.z = pack_bf16(e[4], e[5]);
    pk.w = pack_bf16(e[6], e[7]);
    return pk;
}

inline void encode_or_throw(CUtensorMap* m, uint32_t rank, const void* base, const uint64_t* dims,
                            const uint64_t* strides, const uint32_t* box,
                            CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) {
    CUresult r = encode_tensor_map(m, dt, rank, const_cast<void*>(base), dims, strides, box,
                                   CU_TENSOR_MAP_SWIZZLE_128B);
    if (r != CUDA_SUCCESS) throw Error(OOMB_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

// fp32 [rows][heads][hd] tensor viewed as 3-D {hd, heads, rows}; box {32, 1, 128}: the
// 128-B swizzled staging box of the TMA-store epilogues (one 32-column slice of a tile).
inline CUtensorMap map_rows_heads_f32(const void* base, int64_t rows, int heads, int hd) {
    CUtensorMap m;
    const uint64_t dims[3] = {static_cast<uint64_t>(hd), static_cast<uint64_t>(heads), static_cast<uint64_t>(rows)};
    const uint64_t strides[2] = {static_cast<uint64_t>(hd) * 4, static_cast<uint64_t>(heads) * hd * 4};
    const uint32_t box[3] = {32, 1, static_cast<uint32_t>(kTile)};
    encode_or_throw(&m, 3, base, dims, strides, box, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
    return m;
}

// Epilogue staging of fp32 accumulator slices: slice s ([128 rows x 32 fp32] = 16 KB) in the
// TMA SWIZZLE_128B layout, 16-byte unit u (0..7) of row r at r*128 + ((u ^ (r & 7)) << 4).
constexpr int kSliceBytes = kTile * 128;
__device__ __forceinline__ void st_slice_f32(uint8_t* slice, int r, int u, float4 v) {
    *reinterpret_cast<float4*>(slice + r * 128 + ((u ^ (r & 7)) << 4)) = v;
}
// Load 32 accumulator columns of this thread's TMEM lane, scale, and stage them as one slice.
__device__ __forceinline__ void stage_slice(uint32_t taddr, uint8_t* slice, int r, float scale) {
    uint32_t v[32];
    tmem_ld32(taddr, v);
    tmem_wait_ld();
#pragma unroll
    for (int u = 0; u < 8; ++u)
        st_slice_f32(slice, r, u,
                     make_float4(__uint_as_float(v[4 * u]) * scale, __uint_as_float(v[4 * u + 1]) * scale,
                                 __uint_as_float(v[4 * u + 2]) * scale, __uint_as_float(v[4 * u + 3]) * scale));
}

// [rows][heads][hd] bf16 tensor viewed as 3-D {hd, heads, rows}; box {64, 1, box_rows}.
inline CUtensorMap map_rows_heads(const void* base, int64_t rows, int heads, int hd, int box_rows = kTile) {
    CUtensorMap m;
    const uint64_t dims[3] = {static_cast<uint64_t>(hd), static_cast<uint64_t>(heads), static_cast<uint64_t>(rows)};
    const uint64_t strides[2] = {static_cast<uint64_t>(hd) * 2, static_cast<uint64_t>(heads) * hd * 2};
    const uint32_t box[3] = {64, 1, static_cast<uint32_t>(box_rows)};
    encode_or_throw(&m, 3, base, dims, strides, box);
    return m;
}

// Past key block j of a query page: selected page j / bpp, sub-block j % bpp.
struct PastBlock {
    int row;      // pool tensor-map row
    int n_valid;  // valid keys (partially filled pages are masked)
    int pid;
};
__device__ __forceinline__ PastBlock past_block(const AttnGeom& g, const int32_t* sel_ids, const int32_t* kvslot,
                                                int sel_begin, int j, int kvh, int* err) {
    const int bpp = g.P / kTile;
    PastBlock b;
    b.pid = sel_ids[sel_begin + j / bpp];
    const int sub = j % bpp;
    // ids past the layer's last page are a ShapeError in the reference (paged_kv.hpp page range)
    const bool id_ok = b.pid >= 0 && b.pid < g.max_pages && static_cast<int64_t>(b.pid) * g.P < g.filled;
    int slot = id_ok ? kvslot[b.pid] : -1;
    const int64_t nv = g.filled - static_cast<int64_t>(b.pid) * g.P - static_cast<int64_t>(sub) * kTile;
    b.n_valid = static_cast<int>(nv < 0 ? 0 : (nv > kTile ? kTile : nv));
    if (slot < 0) {
        if (err) atomicOr(err, id_ok ? DERR_NOT_RESIDENT : DERR_BAD_ID);
        slot = 0;
        b.n_valid = 0;
    }
    b.row = (slot * g.Hkv + kvh) * g.P + sub * kTile;
    return b;
}

// Stage one 128 x 128 bf16 row of a K-major SW128 tile (two [128 x 64] regions) into 64 TMEM
// columns of this thread's lane (bf16 pairs packed per 32-bit column).
__device__ __forceinline__ void stage_row_tmem(const uint8_t* tile, int region_bytes, int r, uint32_t taddr) {
#pragma unroll
    for (int c16 = 0; c16 < 4; ++c16) {
        uint32_t v[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = c16 * 4 + q;
            const uint4 x = *reinterpret_cast<const uint4*>(tile + (c >> 3) * region_bytes + r * 128 +
                                                             (((c & 7) ^ (r & 7)) << 4));
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = x.z;
            v[4 * q + 3] = x.w;
        }
        tmem_st16(taddr + c16 * 16, v);
    }
}

// Valid keys (0..128) of past key block j of a query page: partially filled pages are masked
// (paged_kv.hpp:295-299). The softmax warps stage these counts into shared memory once per CTA
// so the per-block path never waits on a global load of the selection ids.
__device__ __forceinline__ int past_valid_global(const AttnGeom& g, const int32_t* sel_ids, int sel_begin, int j) {
    const int bpp = g.P / kTile;
    const int pid = sel_ids[sel_begin + j / bpp];
    const int64_t nv = g.filled - static_cast<int64_t>(pid) * g.P - static_cast<int64_t>(j % bpp) * kTile;
    return static_cast<int>(nv < 0 ? 0 : (nv > kTile ? kTile : nv));
}
__device__ __forceinline__ void stage_past_valid(const AttnGeom& g, const int32_t* sel_ids, int sel_begin,
                                                 int n_past, uint8_t* tab, int cap, int tid, int nthr) {
    for (int j = tid; j < n_past && j < cap; j += nthr) tab[j] = static_cast<uint8_t>(past_valid_global(g, sel_ids, sel_begin, j));
}
__device__ __forceinline__ int past_valid(const AttnGeom& g, const int32_t* sel_ids, int sel_begin, const uint8_t* tab,
                                          int cap, int j) {
    return j < cap ? tab[j] : past_valid_global(g, sel_ids, sel_begin, j);
}

// ---------------------------------------------------------------------------------------------
// Page size 64 (BASELINE configs[0]). A 128-row query tile covers query pages 2qt (rows 0-63) and
// 2qt+1 (rows 64-127), and its past keys come as 64-key half blocks, paired into the 128-key blocks
// the kernels consume: when both pages' lists are equal (dense mode, or equal top-k lists) every
// page of the list applies to all 128 rows; otherwise list A's pages (rows 0-63) come first, then
// list B's (rows 64-127). A missing second half (odd count) is an out-of-bounds TMA box (zero
// fill) and is masked. Key visit order does not change the softmax beyond rounding.
// ---------------------------------------------------------------------------------------------
constexpr int kHalf = 64;
struct HalfList {
    int a0, na, b0, nb, same;
    __device__ __forceinline__ int count() const { return same ? na : na + nb; }
    __device__ __forceinline__ int blocks() const { return (count() + 1) >> 1; }
};
// Every thread of the CTA must call it (it contains a barrier).
__device__ __forceinline__ HalfList half_list_sync(const int32_t* off, const int32_t* ids, int qt) {
    HalfList L;
    L.a0 = off[2 * qt];
    L.na = off[2 * qt + 1] - L.a0;
    L.b0 = off[2 * qt + 1];
    L.nb = off[2 * qt + 2] - L.b0;
    int diff = 0;
    if (L.na == L.nb)
        for (int i = threadIdx.x; i < L.na; i += blockDim.x) diff |= ids[L.a0 + i] != ids[L.b0 + i];
    const int any = __syncthreads_or(diff);
    L.same = L.na == L.nb && !any;
    return L;
}
__device__ __forceinline__ int half_page(const HalfList& L, const int32_t* ids, int h, int* rowmask) {
    if (L.same) {
        *rowmask = 3;
        return ids[L.a0 + h];
    }
    if (h < L.na) {
        *rowmask = 1;
        return ids[L.a0 + h];
    }
    *rowmask = 2;
    return ids[L.b0 + h - L.na];
}
// Table entry of half h: valid keys (0..64) | row-half mask << 8 (bit 0: rows 0-63, bit 1: rows 64-127).
__device__ __forceinline__ uint16_t half_entry(const AttnGeom& g, const int32_t* ids, const HalfList& L, int h) {
    if (h >= L.count()) return 0;
    int mask;
    const int pid = half_page(L, ids, h, &mask);
    const int64_t nv = g.filled - static_cast<int64_t>(pid) * g.P;
    if (pid < 0 || pid >= g.max_pages || nv <= 0) return 0;
    return static_cast<uint16_t>((nv > kHalf ? kHalf : nv) | (mask << 8));
}
// Pool tensor-map row of half h for kv head kvh (an out-of-bounds row when absent / not resident).
__device__ __forceinline__ int past_half_row(const AttnGeom& g, const int32_t* ids, const int32_t* kvslot,
                                             const HalfList& L, int h, int kvh, int* err) {
    if (h >= L.count()) return -2 * kHalf;
    int mask;
    const int pid = half_page(L, ids, h, &mask);
    const bool id_ok = pid >= 0 && pid < g.max_pages && static_cast<int64_t>(pid) * g.P < g.filled;
    const int slot = id_ok ? kvslot[pid] : -1;
    if (slot < 0) {
        if (err) atomicOr(err, id_ok ? DERR_NOT_RESIDENT : DERR_BAD_ID);
        return -2 * kHalf;
    }
    return (slot * g.Hkv + kvh) * g.P;
}
__device__ __forceinline__ void stage_half_valid(const AttnGeom& g, const int32_t* ids, const HalfList& L,
                                                 uint16_t* tab, int cap, int tid, int nthr) {
    const int n = L.count();
    for (int h = tid; h < n && h < cap; h += nthr) tab[h] = half_entry(g, ids, L, h);
}
__device__ __forceinline__ uint16_t half_valid(const AttnGeom& g, const int32_t* ids, const HalfList& L,
                                               const uint16_t* tab, int cap, int h) {
    return h < cap ? (h < L.count() ? tab[h] : 0) : half_entry(g, ids, L, h);
}
// Keep-limit of one 64-key half for query row r: keys [0, lim] of the half are visible.
__device__ __forceinline__ int half_lim(uint16_t e, int r) {
    return ((e >> 8) >> (r >> 6)) & 1 ? static_cast<int>(e & 0xff) - 1 : -1;
}

}  // namespace tc
}  // namespace oomb
