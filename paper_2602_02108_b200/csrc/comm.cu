// SPDX-License-Identifier: Apache-2.0
//
// liboomb_comm.so — NCCL exchange steps of the sharded path (include/oomb_comm.h).
//
// Each exchange is an all-gather into a stream-ordered scratch buffer followed by a fixed-order
// combine from liboomb.so (oomb_vote_reduce, oomb_lse_merge), so the result is bitwise identical
// on every rank and does not depend on how NCCL routes the reduction.

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "oomb_comm.h"

struct oomb_comm_s {
    ncclComm_t nccl = nullptr;
    int rank = 0, world = 1, device = 0;
};

namespace {

thread_local std::string g_err;

struct Fail {
    int code;
    std::string msg;
};

void nccl_ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Fail{OOMB_ERROR, std::string(what) + ": " + ncclGetErrorString(r)};
}
void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Fail{OOMB_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e)};
}
void oomb_ok(int st) {
    if (st != OOMB_OK) throw Fail{st, oomb_last_error()};
}
void require(bool ok, int code, const char* msg) {
    if (!ok) throw Fail{code, msg};
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return OOMB_OK;
    } catch (const Fail& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return OOMB_ERROR;
    }
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// Row slices of a [rows] axis over the ranks: rank s owns [off(s), off(s) + len(s)).
struct Slices {
    int64_t chunk, rows;
    int64_t off(int s) const { return std::min<int64_t>(rows, s * chunk); }
    int64_t len(int s) const { return std::min<int64_t>(rows, (s + 1) * chunk) - off(s); }
};
Slices slices(int64_t rows, int world) { return Slices{(rows + world - 1) / world, rows}; }

// Fixed-order sum of `world` packed parts [world][n]: out[i] = ((p0[i] + p1[i]) + p2[i]) + ...
__global__ void ordered_sum_kernel(const float* __restrict__ parts, int world, int64_t n, float* __restrict__ out) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float acc = parts[i];
        for (int r = 1; r < world; ++r) acc = __fadd_rn(acc, parts[static_cast<int64_t>(r) * n + i]);
        out[i] = acc;
    }
}

// Step 1 of a reduce-scatter by row slices: every rank sends slice s of `src` (row_bytes per row)
// to rank s and receives its own slice from every rank, packed in rank order [world][len(me)].
void exchange_slices(oomb_comm_t c, const void* src, size_t row_bytes, const Slices& sl, void* packed,
                     cudaStream_t st) {
    const int me = c->rank;
    const size_t mine = static_cast<size_t>(sl.len(me)) * row_bytes;
    nccl_ok(ncclGroupStart(), "ncclGroupStart");
    for (int s = 0; s < c->world; ++s) {
        const size_t n = static_cast<size_t>(sl.len(s)) * row_bytes;
        if (n) nccl_ok(ncclSend(static_cast<const uint8_t*>(src) + sl.off(s) * row_bytes, n, ncclUint8, s, c->nccl, st),
                       "ncclSend");
        if (mine) nccl_ok(ncclRecv(static_cast<uint8_t*>(packed) + s * mine, mine, ncclUint8, s, c->nccl, st),
                          "ncclRecv");
    }
    nccl_ok(ncclGroupEnd(), "ncclGroupEnd");
}

// Step 3: the all-gather of the owners' slices, in place (each rank broadcasts its slice).
void share_slices(oomb_comm_t c, void* buf, size_t row_bytes, const Slices& sl, cudaStream_t st) {
    nccl_ok(ncclGroupStart(), "ncclGroupStart");
    for (int s = 0; s < c->world; ++s) {
        const size_t n = static_cast<size_t>(sl.len(s)) * row_bytes;
        uint8_t* p = static_cast<uint8_t*>(buf) + sl.off(s) * row_bytes;
        if (n) nccl_ok(ncclBroadcast(p, p, n, ncclUint8, s, c->nccl, st), "ncclBroadcast");
    }
    nccl_ok(ncclGroupEnd(), "ncclGroupEnd");
}

// all-gather `bytes` per rank into a fresh stream-ordered buffer [world][bytes]
void* gather(oomb_comm_t c, const void* src, size_t bytes, cudaStream_t st) {
    void* buf = nullptr;
    cuda_ok(cudaMallocAsync(&buf, bytes * c->world, st), "cudaMallocAsync");
    nccl_ok(ncclAllGather(src, buf, bytes, ncclUint8, c->nccl, st), "ncclAllGather");
    return buf;
}

}  // namespace

extern "C" {

const char* oomb_comm_last_error(void) { return g_err.c_str(); }

int oomb_comm_get_unique_id(uint8_t* id_out) {
    return guard([&] {
        require(id_out != nullptr, OOMB_SHAPE_ERROR, "comm: null id buffer");
        static_assert(sizeof(ncclUniqueId) == OOMB_COMM_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId id;
        nccl_ok(ncclGetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id_out, &id, sizeof id);
    });
}

int oomb_comm_init(const uint8_t* id, int rank, int world, int device, oomb_comm_t* out) {
    return guard([&] {
        require(id != nullptr && out != nullptr, OOMB_SHAPE_ERROR, "comm: null argument");
        require(world >= 1 && rank >= 0 && rank < world, OOMB_CONFIG_ERROR, "comm: rank / world out of range");
        cuda_ok(cudaSetDevice(device), "cudaSetDevice");
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        auto* c = new oomb_comm_s();
        c->rank = rank, c->world = world, c->device = device;
        const ncclResult_t r = ncclCommInitRank(&c->nccl, world, uid, rank);
        if (r != ncclSuccess) {
            delete c;
            nccl_ok(r, "ncclCommInitRank");
        }
        *out = c;
    });
}

int oomb_comm_destroy(oomb_comm_t c) {
    return guard([&] {
        if (!c) return;
        if (c->nccl) nccl_ok(ncclCommDestroy(c->nccl), "ncclCommDestroy");
        delete c;
    });
}

int oomb_comm_rank(oomb_comm_t c, int* rank, int* world) {
    return guard([&] {
        require(c != nullptr, OOMB_STATE_ERROR, "comm: null communicator");
        if (rank) *rank = c->rank;
        if (world) *world = c->world;
    });
}

int oomb_vote_allgather(oomb_comm_t c, const float* partials, int groups_local, int64_t m, int64_t n, float* vote,
                        void* stream) {
    return guard([&] {
        require(c != nullptr, OOMB_STATE_ERROR, "comm: null communicator");
        require(groups_local >= 1 && m >= 0 && n >= 0, OOMB_SHAPE_ERROR, "vote_allgather: bad shape");
        if (m * n == 0) return;
        const size_t bytes = static_cast<size_t>(groups_local) * m * n * sizeof(float);
        void* all = gather(c, partials, bytes, S(stream));  // [world][groups_local][m][n] = global group order
        oomb_ok(oomb_vote_reduce(static_cast<const float*>(all), groups_local * c->world, m, n, vote, stream));
        cuda_ok(cudaFreeAsync(all, S(stream)), "cudaFreeAsync");
    });
}

int oomb_lse_merge_allgather(oomb_comm_t c, const void* o_part, const float* lse_part, int64_t rows, int hd,
                             int dtype, void* out, float* lse, void* stream) {
    return guard([&] {
        require(c != nullptr, OOMB_STATE_ERROR, "comm: null communicator");
        require(rows >= 0 && hd >= 1, OOMB_SHAPE_ERROR, "lse_merge_allgather: bad shape");
        require(dtype == OOMB_BF16 || dtype == OOMB_F32, OOMB_CONFIG_ERROR, "lse_merge_allgather: dtype");
        if (rows == 0) return;
        const size_t ob = static_cast<size_t>(rows) * hd * (dtype == OOMB_BF16 ? 2 : 4);
        void* o_all = gather(c, o_part, ob, S(stream));
        void* l_all = gather(c, lse_part, static_cast<size_t>(rows) * sizeof(float), S(stream));
        oomb_ok(oomb_lse_merge(o_all, static_cast<const float*>(l_all), c->world, rows, hd, dtype, out, lse, stream));
        cuda_ok(cudaFreeAsync(o_all, S(stream)), "cudaFreeAsync");
        cuda_ok(cudaFreeAsync(l_all, S(stream)), "cudaFreeAsync");
    });
}

int oomb_dq_reduce(oomb_comm_t c, const float* dq_part, int64_t count, float* dq, void* stream) {
    return guard([&] {
        require(c != nullptr, OOMB_STATE_ERROR, "comm: null communicator");
        require(count >= 0, OOMB_SHAPE_ERROR, "dq_reduce: bad shape");
        if (count == 0) return;
        void* all = gather(c, dq_part, static_cast<size_t>(count) * sizeof(float), S(stream));
        // rank-ordered sum: the vote reduction's fixed-order kernel over [world][count]
        oomb_ok(oomb_vote_reduce(static_cast<const float*>(all), c->world, 1, count, dq, stream));
        cuda_ok(cudaFreeAsync(all, S(stream)), "cudaFreeAsync");
    });
}

int oomb_allreduce_ordered(oomb_comm_t c, const float* part, int64_t count, float* out, void* stream) {
    return guard([&] {
        require(c != nullptr, OOMB_STATE_ERROR, "comm: null communicator");
        require(count >= 0, OOMB_SHAPE_ERROR, "allreduce_ordered: bad shape");
        if (count == 0) return;
        cudaStream_t st = S(stream);
        if (c->world == 1) {
            if (out != part) cuda_ok(cudaMemcpyAsync(out, part, count * sizeof(float), cudaMemcpyDeviceToDevice, st),
                                     "cudaMemcpyAsync");
            return;
        }
        const Slices sl = slices(count, c->world);
        const int64_t mine = sl.len(c->rank);
        void* packed = nullptr;
        cuda_ok(cudaMallocAsync(&packed, std::max<int64_t>(mine, 1) * c->world * sizeof(float), st), "cudaMallocAsync");
        exchange_slices(c, part, sizeof(float), sl, packed, st);
        if (mine) {
            const unsigned grid = static_cast<unsigned>(std::min<int64_t>((mine + 255) / 256, 148 * 8));
            ordered_sum_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(packed), c->world, mine,
                                                     out + sl.off(c->rank));
            cuda_ok(cudaGetLastError(), "ordered_sum_kernel");
        }
        cuda_ok(cudaFreeAsync(packed, st), "cudaFreeAsync");
        share_slices(c, out, sizeof(float), sl, st);
    });
}

int oomb_lse_merge_ordered(oomb_comm_t c, const void* o_part, const float* lse_part, int64_t rows, int hd, int dtype,
                           void* out, float* lse, void* stream) {
    return guard([&] {
        require(c != nullptr, OOMB_STATE_ERROR, "comm: null communicator");
        require(rows >= 0 && hd >= 1, OOMB_SHAPE_ERROR, "lse_merge_ordered: bad shape");
        require(dtype == OOMB_BF16 || dtype == OOMB_F32, OOMB_CONFIG_ERROR, "lse_merge_ordered: dtype");
        if (rows == 0) return;
        cudaStream_t st = S(stream);
        const size_t ob = static_cast<size_t>(hd) * (dtype == OOMB_BF16 ? 2 : 4);
        const Slices sl = slices(rows, c->world);
        const int64_t mine = sl.len(c->rank);
        void* o_all = nullptr;
        void* l_all = nullptr;
        cuda_ok(cudaMallocAsync(&o_all, std::max<int64_t>(mine, 1) * c->world * ob, st), "cudaMallocAsync");
        cuda_ok(cudaMallocAsync(&l_all, std::max<int64_t>(mine, 1) * c->world * sizeof(float), st), "cudaMallocAsync");
        exchange_slices(c, o_part, ob, sl, o_all, st);
        exchange_slices(c, lse_part, sizeof(float), sl, l_all, st);
        if (mine)
            oomb_ok(oomb_lse_merge(o_all, static_cast<const float*>(l_all), c->world, mine, hd, dtype,
                                   static_cast<uint8_t*>(out) + sl.off(c->rank) * ob, lse + sl.off(c->rank), stream));
        cuda_ok(cudaFreeAsync(o_all, st), "cudaFreeAsync");
        cuda_ok(cudaFreeAsync(l_all, st), "cudaFreeAsync");
        share_slices(c, out, ob, sl, st);
        share_slices(c, lse, sizeof(float), sl, st);
    });
}

int oomb_comm_bytes(int op, int world, int64_t elems, int64_t elem_bytes, int64_t* sent, int64_t* received) {
    return guard([&] {
        require(world >= 1 && elems >= 0 && elem_bytes >= 1, OOMB_SHAPE_ERROR, "comm_bytes: bad shape");
        // per-rank wire bytes of one exchange of an `elems`-element tensor (rank 0's share; the
        // last rank's slice may be shorter)
        const Slices sl = slices(elems, world);
        const int64_t t = elems * elem_bytes, mine = sl.len(0) * elem_bytes;
        int64_t s = 0, r = 0;
        if (op == 0) {  // all-gather of the whole tensor + local fixed-order sum
            s = t * (world - 1);
            r = t * (world - 1);
        } else {        // ordered reduce-scatter by slices + in-place all-gather of the slices
            s = (t - mine) + mine * (world - 1);
            r = mine * (world - 1) + (t - mine);
        }
        if (sent) *sent = world > 1 ? s : 0;
        if (received) *received = world > 1 ? r : 0;
    });
}

}  // extern "C"
