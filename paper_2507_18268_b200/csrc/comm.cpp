// NCCL transport for the multi-GPU path: 8-24 byte
// allreduces of the PCG sums and grouped send/recv of processor-patch halos.
// libnccl.so.2 is dlopen'ed on first use so the library loads (and the
// single-GPU path runs) without NCCL; if torch already loaded its NCCL the
// same instance is reused (same soname).
#include <dlfcn.h>
#include <nccl.h>

#include "host.h"

namespace lf {

struct Nccl {
  void *h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
  decltype(&ncclCommGetAsyncError) asyncErr = nullptr;
  decltype(&ncclCommSplit) commSplit = nullptr;
};

static Nccl g_nccl;

Nccl *nccl_load() {
  if (g_nccl.h) return &g_nccl;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw Error{LF_ERR_NCCL, std::string("cannot dlopen libnccl.so.2: ") + dlerror()};
#define LF_SYM(field, name)                                                          \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, #name));          \
  if (!g_nccl.field) throw Error{LF_ERR_NCCL, "libnccl missing symbol " #name};
  LF_SYM(getUniqueId, ncclGetUniqueId)
  LF_SYM(commInitRank, ncclCommInitRank)
  LF_SYM(commDestroy, ncclCommDestroy)
  LF_SYM(allReduce, ncclAllReduce)
  LF_SYM(send, ncclSend)
  LF_SYM(recv, ncclRecv)
  LF_SYM(groupStart, ncclGroupStart)
  LF_SYM(groupEnd, ncclGroupEnd)
  LF_SYM(errStr, ncclGetErrorString)
  LF_SYM(asyncErr, ncclCommGetAsyncError)
  LF_SYM(commSplit, ncclCommSplit)
#undef LF_SYM
  g_nccl.h = h;
  return &g_nccl;
}

#define LF_NCCL(x)                                                                   \
  do {                                                                               \
    ncclResult_t r_ = (x);                                                           \
    if (r_ != ncclSuccess)                                                           \
      throw Error{LF_ERR_NCCL, std::string(#x) + ": " + g_nccl.errStr(r_)};          \
  } while (0)

void nccl_unique_id(void *out128) {
  Nccl *n = nccl_load();
  ncclUniqueId id;
  LF_NCCL(n->getUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
}

void *nccl_comm_init(const void *uid128, int nranks, int rank, int device) {
  Nccl *n = nccl_load();
  ncclUniqueId id;
  std::memcpy(&id, uid128, sizeof(id));
  LF_CUDA(cudaSetDevice(device));
  ncclComm_t comm = nullptr;
  LF_NCCL(n->commInitRank(&comm, nranks, id, rank));
  return comm;
}

// a second communicator over the same ranks (the processor-patch halos run
// on it, on their own stream, concurrently with the reductions on the first)
void *nccl_comm_split(void *comm, int rank) {
  ncclComm_t out = nullptr;
  LF_NCCL(g_nccl.commSplit(static_cast<ncclComm_t>(comm), 0, rank, &out, nullptr));
  return out;
}

void nccl_comm_destroy(void *comm) {
  if (comm && g_nccl.h) g_nccl.commDestroy(static_cast<ncclComm_t>(comm));
}

void nccl_allreduce_sum(void *comm, const double *send, double *recv, size_t count, cudaStream_t s) {
  LF_NCCL(g_nccl.allReduce(send, recv, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm), s));
}

void nccl_group_start() { LF_NCCL(g_nccl.groupStart()); }
void nccl_group_end() { LF_NCCL(g_nccl.groupEnd()); }

void nccl_send(void *comm, const double *buf, size_t count, int peer, cudaStream_t s) {
  LF_NCCL(g_nccl.send(buf, count, ncclFloat64, peer, static_cast<ncclComm_t>(comm), s));
}

void nccl_recv(void *comm, double *buf, size_t count, int peer, cudaStream_t s) {
  LF_NCCL(g_nccl.recv(buf, count, ncclFloat64, peer, static_cast<ncclComm_t>(comm), s));
}

void nccl_check_async(void *comm) {
  if (!comm) return;
  ncclResult_t r = ncclSuccess;
  LF_NCCL(g_nccl.asyncErr(static_cast<ncclComm_t>(comm), &r));
  if (r != ncclSuccess && r != ncclInProgress)
    throw Error{LF_ERR_NCCL, std::string("NCCL async error: ") + g_nccl.errStr(r)};
}

}  // namespace lf
