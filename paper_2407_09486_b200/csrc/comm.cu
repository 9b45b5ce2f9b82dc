// comm.cpp -- run-time-loaded NCCL for the fleet-wide threshold statistics.
// Collectives: allreduce of int64 radix histograms (exact, order-independent),
// allgather of per-rank tail counts, rank-ordered allgatherv of score tails
// (grouped broadcasts).  All stream-ordered on the caller's stream.
#include "comm.h"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include "common.cuh"

namespace {

typedef int ncclResult_t;
typedef void *ncclComm_t;
struct ncclUniqueId {
  char internal[128];
};
enum { ncclInt64 = 4, ncclUint64 = 5, ncclFloat64 = 8 };
enum { ncclSum = 0 };

struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Broadcast)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char *(*GetErrorString)(ncclResult_t);
};

Nccl &nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return;
    }
#define SYM(f, name)                                                       \
  n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, name));                   \
  if (!n.f) {                                                              \
    n.why = std::string("missing NCCL symbol ") + name;                    \
    return;                                                                \
  }
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(AllReduce, "ncclAllReduce");
    SYM(AllGather, "ncclAllGather");
    SYM(Broadcast, "ncclBroadcast");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    n.ok = true;
  });
  return n;
}

enova_status nccl_fail(ncclResult_t r, const char *what) {
  enova::set_error(std::string(what) + ": " + nccl().GetErrorString(r));
  return ENOVA_ERR_NCCL;
}

}  // namespace

namespace enova {

enova_status comm_allreduce_u64_sum(enova_comm_t c, const void *send, void *recv, size_t count,
                                    cudaStream_t st) {
  ncclResult_t r = nccl().AllReduce(send, recv, count, ncclUint64, ncclSum, c->nccl, st);
  return r ? nccl_fail(r, "ncclAllReduce") : ENOVA_OK;
}

enova_status comm_allgather_i64(enova_comm_t c, const void *send, void *recv, cudaStream_t st) {
  ncclResult_t r = nccl().AllGather(send, recv, 1, ncclInt64, c->nccl, st);
  return r ? nccl_fail(r, "ncclAllGather") : ENOVA_OK;
}

enova_status comm_allgatherv_f64(enova_comm_t c, const double *local, double *out,
                                 const int64_t *counts, const int64_t *offsets, cudaStream_t st) {
  Nccl &n = nccl();
  ncclResult_t r = n.GroupStart();
  if (r) return nccl_fail(r, "ncclGroupStart");
  for (int q = 0; q < c->world; ++q) {
    if (counts[q] == 0) continue;
    r = n.Broadcast(q == c->rank ? (const void *)local : (const void *)(out + offsets[q]),
                    out + offsets[q], (size_t)counts[q], ncclFloat64, q, c->nccl, st);
    if (r) {
      n.GroupEnd();
      return nccl_fail(r, "ncclBroadcast");
    }
  }
  r = n.GroupEnd();
  return r ? nccl_fail(r, "ncclGroupEnd") : ENOVA_OK;
}

}  // namespace enova

extern "C" {

enova_status enova_comm_unique_id(void *out128) {
  if (!out128) {
    enova::set_error("out128 is NULL");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  Nccl &n = nccl();
  if (!n.ok) {
    enova::set_error(n.why);
    return ENOVA_ERR_NCCL;
  }
  ncclUniqueId id;
  ncclResult_t r = n.GetUniqueId(&id);
  if (r) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(out128, &id, sizeof(id));
  return ENOVA_OK;
}

enova_status enova_comm_create(enova_comm_t *comm, int rank, int world, const void *id128,
                               int device) {
  if (!comm || !id128 || world < 1 || rank < 0 || rank >= world) {
    enova::set_error("invalid comm arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  Nccl &n = nccl();
  if (!n.ok) {
    enova::set_error(n.why);
    return ENOVA_ERR_NCCL;
  }
  ENOVA_CUDA_TRY(cudaSetDevice(device));
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  ncclResult_t r = n.CommInitRank(&c, world, id, rank);
  if (r) return nccl_fail(r, "ncclCommInitRank");
  enova_comm_s *h = new enova_comm_s;
  h->nccl = c;
  h->rank = rank;
  h->world = world;
  h->device = device;
  *comm = h;
  return ENOVA_OK;
}

void enova_comm_destroy(enova_comm_t comm) {
  if (!comm) return;
  if (nccl().ok && comm->nccl) nccl().CommDestroy(comm->nccl);
  delete comm;
}

}  // extern "C"
