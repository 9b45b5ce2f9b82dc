// comm.cu -- collectives of the fleet-wide threshold (comm.h): allreduce of
// uint64 radix histograms (exact, order-independent), allgather of per-rank tail
// counts, allgather of fixed-size fp32 tail slots.  All stream-ordered on the
// caller's stream; NCCL (run-time loaded) or the in-process local backend.
#include "comm.h"

#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <thread>

#include "common.cuh"

namespace {

constexpr double kDefaultCommTimeoutS = 300.0;

typedef int ncclResult_t;
typedef void *ncclComm_t;
struct ncclUniqueId {
  char internal[128];
};
enum { ncclInt64 = 4, ncclUint64 = 5, ncclFloat32 = 7, ncclFloat64 = 8 };
enum { ncclSum = 0 };
enum { ncclSuccess = 0, ncclInProgress = 7 };

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
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *);
  ncclResult_t (*CommAbort)(ncclComm_t);
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
    SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    SYM(CommAbort, "ncclCommAbort");
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

// ------------------------------------------------------------- local ----
constexpr int kMaxLocal = 16;
constexpr size_t kLocalStage = 64 * 1024;   // per-rank reduction scratch (bytes)

struct LocalGroup {
  int world = 0, device = 0, refs = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool broken = false;               // a rank timed out at a rendezvous: the group is dead
  const void *src[kMaxLocal] = {};
  cudaEvent_t ready[kMaxLocal] = {}, done[kMaxLocal] = {};
  void *stage[kMaxLocal] = {};
  std::mutex coop_m;                 // held from comm_coop_begin to comm_coop_end
  cudaEvent_t coop_last = nullptr;   // completion of the previous cooperative launch
  bool coop_recorded = false;
  // host rendezvous of the ranks, bounded by timeout_s: false if a rank did not
  // arrive in time (the group is then broken for every rank)
  bool barrier(double timeout_s) {
    std::unique_lock<std::mutex> l(m);
    if (broken) return false;
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(l, std::chrono::duration<double>(timeout_s),
                                [&] { return gen != g || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

static enova_status local_broken(enova_comm_t c) {
  c->aborted = true;
  set_error("local communicator: a rank did not reach the rendezvous within the timeout");
  return ENOVA_ERR_NCCL;
}

struct LocalSrcs {
  const unsigned long long *p[kMaxLocal];
};

// recv[i] = sum over ranks in rank order (exact: unsigned 64-bit integers)
__global__ void k_local_sum_u64(LocalSrcs s, int world, size_t count,
                                unsigned long long *__restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long v = 0;
    for (int q = 0; q < world; ++q) v += s.p[q][i];
    out[i] = v;
  }
}

// Publish this rank's source, rendezvous, and order this rank's stream after
// every rank's preceding work.
static enova_status local_enter(enova_comm_t c, const void *send, cudaStream_t st) {
  LocalGroup *G = c->local;
  G->src[c->rank] = send;
  ENOVA_CUDA_TRY(cudaEventRecord(G->ready[c->rank], st));
  if (!G->barrier(c->timeout_s)) return local_broken(c);
  for (int q = 0; q < G->world; ++q) ENOVA_CUDA_TRY(cudaStreamWaitEvent(st, G->ready[q], 0));
  return ENOVA_OK;
}

// No rank's later work (which may overwrite its send buffer) starts before
// every rank has finished reading the sources.
static enova_status local_leave(enova_comm_t c, cudaStream_t st) {
  LocalGroup *G = c->local;
  ENOVA_CUDA_TRY(cudaEventRecord(G->done[c->rank], st));
  if (!G->barrier(c->timeout_s)) return local_broken(c);
  for (int q = 0; q < G->world; ++q) ENOVA_CUDA_TRY(cudaStreamWaitEvent(st, G->done[q], 0));
  return ENOVA_OK;
}

static enova_status local_allgather(enova_comm_t c, const void *send, void *recv, size_t bytes,
                                    cudaStream_t st) {
  enova_status r = local_enter(c, send, st);
  if (r) return r;
  LocalGroup *G = c->local;
  for (int q = 0; q < G->world; ++q)
    if (bytes)
      ENOVA_CUDA_TRY(cudaMemcpyAsync(static_cast<char *>(recv) + (size_t)q * bytes, G->src[q],
                                     bytes, cudaMemcpyDeviceToDevice, st));
  return local_leave(c, st);
}

static enova_status local_allreduce_u64(enova_comm_t c, const void *send, void *recv,
                                        size_t count, cudaStream_t st) {
  LocalGroup *G = c->local;
  if (count * 8 > kLocalStage) {
    set_error("local communicator: allreduce larger than its staging buffer");
    return ENOVA_ERR_UNSUPPORTED;
  }
  enova_status r = local_enter(c, send, st);
  if (r) return r;
  LocalSrcs s;
  for (int q = 0; q < kMaxLocal; ++q)
    s.p[q] = static_cast<const unsigned long long *>(q < G->world ? G->src[q] : nullptr);
  unsigned long long *stage = static_cast<unsigned long long *>(G->stage[c->rank]);
  if (count) {
    ENOVA_LAUNCH(k_local_sum_u64, (unsigned)((count + 255) / 256), 256, 0, st, s, G->world, count,
                 stage);
    ENOVA_CUDA_TRY(cudaGetLastError());
  }
  // in-place safe: recv is written only after every rank has read every source
  if ((r = local_leave(c, st))) return r;
  if (count)
    ENOVA_CUDA_TRY(cudaMemcpyAsync(recv, stage, count * 8, cudaMemcpyDeviceToDevice, st));
  return ENOVA_OK;
}

// ------------------------------------------------------------- public ----
static enova_status check_alive(enova_comm_t c) {
  if (c->aborted) {
    set_error("communicator was aborted after an earlier failure or timeout");
    return ENOVA_ERR_NCCL;
  }
  return ENOVA_OK;
}

static void abort_comm(enova_comm_t c) {
  if (!c->aborted && c->nccl && nccl().ok) nccl().CommAbort(c->nccl);
  c->aborted = true;
}

enova_status comm_wait(enova_comm_t c, cudaStream_t st) {
  if (enova_status r = check_alive(c)) return r;
  cudaEvent_t ev;
  ENOVA_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  cudaError_t e = cudaEventRecord(ev, st);
  if (e != cudaSuccess) {
    cudaEventDestroy(ev);
    set_error(std::string("cudaEventRecord: ") + cudaGetErrorString(e));
    return ENOVA_ERR_CUDA;
  }
  const auto t0 = std::chrono::steady_clock::now();
  enova_status out = ENOVA_OK;
  while (true) {
    e = cudaEventQuery(ev);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) {
      set_error(std::string("stream failed while waiting on the communicator: ") +
                cudaGetErrorString(e));
      out = ENOVA_ERR_CUDA;
      break;
    }
    if (c->nccl) {
      ncclResult_t ae = ncclSuccess;
      const ncclResult_t qr = nccl().CommGetAsyncError(c->nccl, &ae);
      if (qr != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress)) {
        set_error(std::string("NCCL asynchronous error: ") +
                  nccl().GetErrorString(qr != ncclSuccess ? qr : ae));
        abort_comm(c);
        out = ENOVA_ERR_NCCL;
        break;
      }
    }
    const double el =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > c->timeout_s) {
      set_error("communicator wait exceeded its timeout (a peer rank is gone or stalled); "
                "communicator aborted");
      abort_comm(c);
      out = ENOVA_ERR_NCCL;
      break;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  cudaEventDestroy(ev);
  return out;
}

enova_status comm_allreduce_u64_sum(enova_comm_t c, const void *send, void *recv, size_t count,
                                    cudaStream_t st) {
  if (enova_status r0 = check_alive(c)) return r0;
  if (c->local) return local_allreduce_u64(c, send, recv, count, st);
  ncclResult_t r = nccl().AllReduce(send, recv, count, ncclUint64, ncclSum, c->nccl, st);
  return r ? nccl_fail(r, "ncclAllReduce") : ENOVA_OK;
}

enova_status comm_allgather_i64(enova_comm_t c, const void *send, void *recv, cudaStream_t st) {
  if (enova_status r0 = check_alive(c)) return r0;
  if (c->local) return local_allgather(c, send, recv, 8, st);
  ncclResult_t r = nccl().AllGather(send, recv, 1, ncclInt64, c->nccl, st);
  return r ? nccl_fail(r, "ncclAllGather") : ENOVA_OK;
}

enova_status comm_allgather_f32(enova_comm_t c, const void *send, void *recv, size_t count,
                                cudaStream_t st) {
  if (enova_status r0 = check_alive(c)) return r0;
  if (c->local) return local_allgather(c, send, recv, count * 4, st);
  ncclResult_t r = nccl().AllGather(send, recv, count, ncclFloat32, c->nccl, st);
  return r ? nccl_fail(r, "ncclAllGather") : ENOVA_OK;
}

enova_status comm_coop_begin(enova_comm_t c, cudaStream_t st) {
  if (!c || !c->local) return ENOVA_OK;
  LocalGroup *G = c->local;
  G->coop_m.lock();
  if (G->coop_recorded) {
    cudaError_t e = cudaStreamWaitEvent(st, G->coop_last, 0);
    if (e != cudaSuccess) {
      G->coop_m.unlock();
      set_error(std::string("cudaStreamWaitEvent: ") + cudaGetErrorString(e));
      return ENOVA_ERR_CUDA;
    }
  }
  return ENOVA_OK;
}

enova_status comm_coop_end(enova_comm_t c, cudaStream_t st) {
  if (!c || !c->local) return ENOVA_OK;
  LocalGroup *G = c->local;
  cudaError_t e = cudaEventRecord(G->coop_last, st);
  G->coop_recorded = (e == cudaSuccess);
  G->coop_m.unlock();
  if (e != cudaSuccess) {
    set_error(std::string("cudaEventRecord: ") + cudaGetErrorString(e));
    return ENOVA_ERR_CUDA;
  }
  return ENOVA_OK;
}

enova_status comm_sum_i64_sync(enova_comm_t c, int64_t in, int64_t *out, void *scratch,
                               cudaStream_t st) {
  unsigned long long v = (unsigned long long)in;
  ENOVA_CUDA_TRY(cudaMemcpyAsync(scratch, &v, 8, cudaMemcpyHostToDevice, st));
  enova_status r = comm_allreduce_u64_sum(c, scratch, scratch, 1, st);
  if (r) return r;
  ENOVA_CUDA_TRY(cudaMemcpyAsync(&v, scratch, 8, cudaMemcpyDeviceToHost, st));
  if ((r = comm_wait(c, st))) return r;
  *out = (int64_t)v;
  return ENOVA_OK;
}

}  // namespace enova

extern "C" {

enova_status enova_comm_set_timeout(enova_comm_t comm, double seconds) {
  if (!comm || !(seconds > 0.0)) {
    enova::set_error("enova_comm_set_timeout: comm required, seconds > 0");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  comm->timeout_s = seconds;
  return ENOVA_OK;
}

enova_status enova_comm_wait(enova_comm_t comm, void *stream) {
  if (!comm) {
    enova::set_error("enova_comm_wait: comm is NULL");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  return enova::comm_wait(comm, static_cast<cudaStream_t>(stream));
}

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
  h->local = nullptr;
  h->rank = rank;
  h->world = world;
  h->device = device;
  h->timeout_s = kDefaultCommTimeoutS;
  h->aborted = false;
  *comm = h;
  return ENOVA_OK;
}

enova_status enova_comm_sum_i64(enova_comm_t comm, int64_t in, int64_t *out, void *stream) {
  if (!comm || !out) {
    enova::set_error("enova_comm_sum_i64: comm and out are required");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  void *scratch = nullptr;
  ENOVA_CUDA_TRY(cudaMalloc(&scratch, 256));
  enova_status r = enova::comm_sum_i64_sync(comm, in, out, scratch, static_cast<cudaStream_t>(stream));
  cudaFree(scratch);
  return r;
}

enova_status enova_comm_create_local(enova_comm_t *comms, int world, int device) {
  if (!comms || world < 1 || world > enova::kMaxLocal) {
    enova::set_error("local communicator: world must be in [1, 16]");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  ENOVA_CUDA_TRY(cudaSetDevice(device));
  enova::LocalGroup *G = new enova::LocalGroup;
  G->world = world;
  G->device = device;
  G->refs = world;
  if (cudaEventCreateWithFlags(&G->coop_last, cudaEventDisableTiming) != cudaSuccess) {
    enova::set_error("local communicator: cudaEventCreate failed");
    return ENOVA_ERR_CUDA;
  }
  for (int q = 0; q < world; ++q) {
    cudaError_t e = cudaEventCreateWithFlags(&G->ready[q], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&G->done[q], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMalloc(&G->stage[q], enova::kLocalStage);
    if (e != cudaSuccess) {
      enova::set_error(std::string("local communicator: ") + cudaGetErrorString(e));
      return ENOVA_ERR_CUDA;   // (leaks the partial group; setup-time failure only)
    }
  }
  for (int q = 0; q < world; ++q) {
    enova_comm_s *h = new enova_comm_s;
    h->nccl = nullptr;
    h->local = G;
    h->rank = q;
    h->world = world;
    h->device = device;
    h->timeout_s = kDefaultCommTimeoutS;
    h->aborted = false;
    comms[q] = h;
  }
  return ENOVA_OK;
}

void enova_comm_destroy(enova_comm_t comm) {
  if (!comm) return;
  if (comm->local) {
    enova::LocalGroup *G = comm->local;
    bool last;
    {
      std::lock_guard<std::mutex> l(G->m);
      last = --G->refs == 0;
    }
    if (last) {
      for (int q = 0; q < G->world; ++q) {
        if (G->ready[q]) cudaEventDestroy(G->ready[q]);
        if (G->done[q]) cudaEventDestroy(G->done[q]);
        if (G->stage[q]) cudaFree(G->stage[q]);
      }
      if (G->coop_last) cudaEventDestroy(G->coop_last);
      delete G;
    }
  } else if (nccl().ok && comm->nccl && !comm->aborted) {
    nccl().CommDestroy(comm->nccl);   // (an aborted communicator is already freed)
  }
  delete comm;
}

}  // extern "C"
