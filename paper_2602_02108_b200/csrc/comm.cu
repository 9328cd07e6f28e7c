// SPDX-License-Identifier: Apache-2.0
//
// liboomb_comm.so — NCCL exchange steps of the sharded path (include/oomb_comm.h).
//
// Each exchange is an all-gather into a stream-ordered scratch buffer followed by a fixed-order
// combine from liboomb.so (oomb_vote_reduce, oomb_lse_merge), so the result is bitwise identical
// on every rank and does not depend on how NCCL routes the reduction.

#include <cuda_runtime.h>
#include <nccl.h>

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

}  // extern "C"
