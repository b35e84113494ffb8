// Communicator of the distributed eigensolve: NCCL (dlopen) or host callbacks (comm.h).
#include "comm.h"

#include <dlfcn.h>
#include <string.h>

namespace em {
thread_local em_ctx* g_cur_ctx = nullptr;
namespace {

// the slice of the NCCL API in use (nccl.h, NCCL >= 2.4)
typedef struct ncclComm* ncclComm_t;
struct NcclUniqueId { char internal[128]; };
constexpr int kNcclFloat64 = 8, kNcclSum = 0;
struct Nccl {
  void* lib = nullptr;
  int (*GetUniqueId)(NcclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, NcclUniqueId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

Nccl* nccl() {
  static Nccl n;
  static bool tried = false;
  if (!tried) {
    tried = true;
    n.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.lib) n.lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (n.lib) {
      auto sym = [&](const char* s) { return dlsym(n.lib, s); };
      n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
      n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
      n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
      n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
      n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(sym("ncclBroadcast"));
      n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
      if (!n.GetUniqueId || !n.CommInitRank || !n.CommDestroy || !n.AllReduce || !n.Broadcast)
        n.lib = nullptr;
    }
  }
  return n.lib ? &n : nullptr;
}

void nccl_check(int rc, const char* what) {
  if (rc == 0) return;
  Nccl* n = nccl();
  const char* msg = (n && n->GetErrorString) ? n->GetErrorString(rc) : "?";
  throw ArgError{std::string(what) + ": NCCL error " + std::to_string(rc) + " (" + msg + ")"};
}

}  // namespace

void comm_allreduce_sum(em_ctx* ctx, double* buf, int64_t count) {
  em_comm* c = ctx->comm;
  if (!c || c->nranks <= 1 || count <= 0) return;
  ++c->n_allreduce;
  c->bytes += count * 8;
  if (c->backend == 1) {
    nccl_check(nccl()->AllReduce(buf, buf, (size_t)count, kNcclFloat64, kNcclSum,
                                 static_cast<ncclComm_t>(c->nccl), ctx->stream),
               "ncclAllReduce");
  } else {
    EM_CK(cudaStreamSynchronize(ctx->stream));
    if (c->allreduce(c->user, buf, count) != 0) throw ArgError{"all-reduce callback failed"};
  }
}

void comm_bcast(em_ctx* ctx, double* buf, int64_t count, int root) {
  em_comm* c = ctx->comm;
  if (!c || c->nranks <= 1 || count <= 0) return;
  ++c->n_bcast;
  c->bytes += count * 8;
  if (c->backend == 1) {
    nccl_check(nccl()->Broadcast(buf, buf, (size_t)count, kNcclFloat64, root,
                                 static_cast<ncclComm_t>(c->nccl), ctx->stream),
               "ncclBroadcast");
  } else {
    EM_CK(cudaStreamSynchronize(ctx->stream));
    if (c->bcast(c->user, buf, count, root) != 0) throw ArgError{"broadcast callback failed"};
  }
}

int comm_unique_id(void* id) {
  Nccl* n = nccl();
  if (!n) throw ArgError{"libnccl.so.2 not found"};
  NcclUniqueId u;
  nccl_check(n->GetUniqueId(&u), "ncclGetUniqueId");
  memcpy(id, &u, sizeof(u));
  return 0;
}

void comm_destroy(em_ctx* ctx) {
  em_comm* c = ctx->comm;
  if (!c) return;
  if (c->backend == 1 && c->nccl) {
    cudaStreamSynchronize(ctx->stream);
    nccl()->CommDestroy(static_cast<ncclComm_t>(c->nccl));
  }
  delete c;
  ctx->comm = nullptr;
}

void comm_init_nccl(em_ctx* ctx, int nranks, int rank, const void* id) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw ArgError{"bad communicator rank / size"};
  Nccl* n = nccl();
  if (!n) throw ArgError{"libnccl.so.2 not found"};
  comm_destroy(ctx);
  NcclUniqueId u;
  memcpy(&u, id, sizeof(u));
  ncclComm_t comm = nullptr;
  nccl_check(n->CommInitRank(&comm, nranks, u, rank), "ncclCommInitRank");
  em_comm* c = new em_comm;
  c->nranks = nranks;
  c->rank = rank;
  c->backend = 1;
  c->nccl = comm;
  ctx->comm = c;
}

void comm_init_callbacks(em_ctx* ctx, int nranks, int rank, em_allreduce_fn ar, em_bcast_fn bc,
                         void* user) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !ar || !bc)
    throw ArgError{"bad communicator rank / size / callbacks"};
  comm_destroy(ctx);
  em_comm* c = new em_comm;
  c->nranks = nranks;
  c->rank = rank;
  c->backend = 2;
  c->allreduce = ar;
  c->bcast = bc;
  c->user = user;
  ctx->comm = c;
}

}  // namespace em
