// A8: counter reduction over NCCL (NVLink 5 / NVSwitch).  The communicator lives in the library
// so the collectives are enqueued on the replay stream; the 128-byte unique id is exchanged by
// the caller (torch.distributed).  libnccl.so.2 is dlopen()ed at run time so the process's copy
// (e.g. the one torch already loaded) is shared and no link-time NCCL dependency exists.
#include <dlfcn.h>

#include <mutex>

#include "saga_internal.cuh"

namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { ncclInt64_ = 4 };
enum { ncclSum_ = 0, ncclMax_ = 2 };

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

Nccl* nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!n.h) n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) return;
    n.getUniqueId = (decltype(n.getUniqueId))dlsym(n.h, "ncclGetUniqueId");
    n.commInitRank = (decltype(n.commInitRank))dlsym(n.h, "ncclCommInitRank");
    n.allReduce = (decltype(n.allReduce))dlsym(n.h, "ncclAllReduce");
    n.commDestroy = (decltype(n.commDestroy))dlsym(n.h, "ncclCommDestroy");
    n.getErrorString = (decltype(n.getErrorString))dlsym(n.h, "ncclGetErrorString");
  });
  return (n.h && n.getUniqueId && n.commInitRank && n.allReduce && n.commDestroy) ? &n : nullptr;
}
}  // namespace

struct saga_comm {
  ncclComm_t comm = nullptr;
  int device = 0, rank = 0, nranks = 1;
};

using saga::set_error;

extern "C" {

saga_status saga_comm_unique_id(void* id128) {
  if (!id128) { set_error("saga_comm_unique_id: NULL"); return SAGA_ERR_INVALID_ARG; }
  Nccl* n = nccl();
  if (!n) { set_error("saga_comm_unique_id: libnccl.so.2 not found"); return SAGA_ERR_NCCL; }
  ncclUniqueId id;
  ncclResult_t r = n->getUniqueId(&id);
  if (r) { set_error("ncclGetUniqueId failed: %s", n->getErrorString ? n->getErrorString(r) : "?"); return SAGA_ERR_NCCL; }
  memcpy(id128, &id, 128);
  return SAGA_OK;
}

saga_status saga_comm_init(const void* id128, int rank, int nranks, int device, saga_comm** out) {
  if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) { set_error("saga_comm_init: bad argument"); return SAGA_ERR_INVALID_ARG; }
  Nccl* n = nccl();
  if (!n) { set_error("saga_comm_init: libnccl.so.2 not found"); return SAGA_ERR_NCCL; }
  SAGA_CK(cudaSetDevice(device));
  ncclUniqueId id;
  memcpy(&id, id128, 128);
  saga_comm* c = new saga_comm();
  c->device = device; c->rank = rank; c->nranks = nranks;
  ncclResult_t r = n->commInitRank(&c->comm, nranks, id, rank);
  if (r) {
    set_error("ncclCommInitRank failed: %s", n->getErrorString ? n->getErrorString(r) : "?");
    delete c;
    return SAGA_ERR_NCCL;
  }
  *out = c;
  return SAGA_OK;
}

saga_status saga_allreduce_counters(saga_comm* c, int64_t* buf_dev, size_t n_elem, int op, saga_stream_t stream) {
  if (!c || (!buf_dev && n_elem) || (op != 0 && op != 1)) { set_error("saga_allreduce_counters: bad argument"); return SAGA_ERR_INVALID_ARG; }
  Nccl* n = nccl();
  if (!n) { set_error("libnccl.so.2 not found"); return SAGA_ERR_NCCL; }
  SAGA_CK(cudaSetDevice(c->device));
  ncclResult_t r = n->allReduce(buf_dev, buf_dev, n_elem, ncclInt64_, op == 0 ? ncclSum_ : ncclMax_, c->comm, (cudaStream_t)stream);
  if (r) { set_error("ncclAllReduce failed: %s", n->getErrorString ? n->getErrorString(r) : "?"); return SAGA_ERR_NCCL; }
  return SAGA_OK;
}

void saga_comm_destroy(saga_comm* c) {
  if (!c) return;
  Nccl* n = nccl();
  if (n && c->comm) n->commDestroy(c->comm);
  delete c;
}

}  // extern "C"
