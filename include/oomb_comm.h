/* SPDX-License-Identifier: Apache-2.0
 *
 * oomb_comm.h — the multi-GPU exchange steps of the path (SURVEY §8 b/e), liboomb_comm.so.
 *
 * One process per GPU; ranks of one node share an NCCL communicator over NVLink/NVSwitch.
 * The reference is single-process ("per-head parallelism permitted only when
 * scatter order is fixed per page"), so every exchange here is deterministic: data are
 * all-gathered and then summed / merged in rank order on every rank, never reduced in an
 * order that depends on the topology.
 *
 *   KV-group sharding   rank r owns a contiguous range of kv groups. Its scorer writes per-group
 *                       partial votes (oomb_score_pages_partial); oomb_vote_allgather sums all
 *                       groups in global group order -> the same vote, hence the same top-k
 *                       selection, on every rank and for every world size.
 *   page-range split    rank r attends its share of each query page's selected pages
 *                       (OOMB_ATTN_PAST_ONLY on r > 0). oomb_lse_merge_allgather merges the
 *                       partial (O_r, LSE_r) exactly; oomb_dq_reduce sums the partial dQ in
 *                       rank order.
 *
 * Statuses are oomb_status (oomb.h); oomb_comm_last_error() holds the message. Buffers are
 * device pointers, `stream` a cudaStream_t as void*. liboomb_comm.so links liboomb.so and NCCL;
 * liboomb.so itself has no NCCL dependency.
 */
#ifndef OOMB_COMM_H_
#define OOMB_COMM_H_

#include <stdint.h>

#include "oomb.h"

#ifdef __cplusplus
extern "C" {
#endif

#define OOMB_COMM_ID_BYTES 128 /* ncclUniqueId */

typedef struct oomb_comm_s* oomb_comm_t;

OOMB_API const char* oomb_comm_last_error(void);
/* Rank 0 creates the id and distributes it out of band (e.g. torch.distributed broadcast). */
OOMB_API int oomb_comm_get_unique_id(uint8_t* id_out);
OOMB_API int oomb_comm_init(const uint8_t* id, int rank, int world, int device, oomb_comm_t* out);
OOMB_API int oomb_comm_destroy(oomb_comm_t comm);
OOMB_API int oomb_comm_rank(oomb_comm_t comm, int* rank, int* world);

/* partials [groups_local][m][n] fp32 of this rank's kv groups -> vote [m][n] fp32 =
 * sum over all ranks' groups in global order (rank-major). Every rank must pass the same
 * groups_local. */
OOMB_API int oomb_vote_allgather(oomb_comm_t comm, const float* partials, int groups_local, int64_t m, int64_t n,
                                 float* vote, void* stream);
/* o_part [rows][hd] (dtype), lse_part [rows] fp32 natural log -> out / lse merged over all ranks:
 * lse = ln sum_r e^{lse_r}, out = sum_r e^{lse_r - lse} o_r (rows = tokens * n_q_heads). */
OOMB_API int oomb_lse_merge_allgather(oomb_comm_t comm, const void* o_part, const float* lse_part, int64_t rows,
                                      int hd, int dtype, void* out, float* lse, void* stream);
/* dq = sum_r dq_part_r in rank order (fp32, count elements). */
OOMB_API int oomb_dq_reduce(oomb_comm_t comm, const float* dq_part, int64_t count, float* dq, void* stream);

/* Proportional variants (each rank moves ~2x the tensor instead of (world-1)x), bitwise equal to the
 * all-gather ones above: the tensor is cut into `world` contiguous row slices; rank s receives slice
 * s of every rank (grouped ncclSend / ncclRecv), combines it in rank order, and broadcasts the
 * combined slice back in place (grouped ncclBroadcast).
 *   oomb_allreduce_ordered: out = sum_r part_r, per element in rank order (dQ, dk_cur / dv_cur of a
 *                           page-range group). out may alias part.
 *   oomb_lse_merge_ordered: the exact (O, LSE) merge of oomb_lse_merge_allgather. */
OOMB_API int oomb_allreduce_ordered(oomb_comm_t comm, const float* part, int64_t count, float* out, void* stream);
OOMB_API int oomb_lse_merge_ordered(oomb_comm_t comm, const void* o_part, const float* lse_part, int64_t rows, int hd,
                                    int dtype, void* out, float* lse, void* stream);
/* Per-rank wire bytes of one exchange of `elems` elements of `elem_bytes` (op 0 = all-gather +
 * local sum, op 1 = the ordered reduce-scatter + all-gather above), for reports. */
OOMB_API int oomb_comm_bytes(int op, int world, int64_t elems, int64_t elem_bytes, int64_t* sent, int64_t* received);

#ifdef __cplusplus
}
#endif

#endif /* OOMB_COMM_H_ */
