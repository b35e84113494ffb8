// Inter-GPU collectives of the distributed eigensolve (one process per GPU). The product
// backend is NCCL (loaded at run time: libnccl.so.2, the torch-bundled one when torch is in
// the process), issued on the context stream. A callback backend exists for the tests this
// environment allows (two processes on ONE GPU, which NCCL refuses): the host application
// supplies the collectives (torch.distributed / gloo in tests), the stream is synchronised
// around every call.
#pragma once
#include <stdint.h>

#include "ctx.h"

struct em_comm {
  int nranks = 1, rank = 0;
  int backend = 0;       // 0 none, 1 NCCL, 2 callbacks
  void* nccl = nullptr;  // ncclComm_t
  em_allreduce_fn allreduce = nullptr;
  em_bcast_fn bcast = nullptr;
  void* user = nullptr;
  int64_t n_allreduce = 0, n_bcast = 0, bytes = 0;  // traffic counters (em_comm_info)
};

namespace em {
extern thread_local em_ctx* g_cur_ctx;  // set at every C ABI entry (capi.cu guarded())
// sum over ranks, in place; no-ops for a single rank
void comm_allreduce_sum(em_ctx* ctx, double* buf, int64_t count);
void comm_bcast(em_ctx* ctx, double* buf, int64_t count, int root);
int comm_unique_id(void* id);
void comm_init_nccl(em_ctx* ctx, int nranks, int rank, const void* id);
void comm_init_callbacks(em_ctx* ctx, int nranks, int rank, em_allreduce_fn ar, em_bcast_fn bc,
                         void* user);
void comm_destroy(em_ctx* ctx);
inline int comm_size(const em_ctx* ctx) { return ctx->comm ? ctx->comm->nranks : 1; }
inline int comm_rank(const em_ctx* ctx) { return ctx->comm ? ctx->comm->rank : 0; }
}  // namespace em
