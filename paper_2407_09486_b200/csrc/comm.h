// comm.h -- communicator used only for the fleet-wide threshold (§8e).
// Two backends behind one handle:
//  * NCCL (one process per GPU): resolved at run time with dlopen("libnccl.so.2"),
//    so the library has no link-time dependency and picks up the NCCL that torch
//    already loaded.  Every collective is stream-ordered and graph-capturable.
//  * local: `world` ranks that are host threads of ONE process on one device
//    (enova_comm_create_local).  Collectives rendezvous on the host (a barrier)
//    and move data with stream-ordered device copies / a reduction kernel,
//    ordered across the ranks' streams with events.  It exists so that the
//    multi-rank threshold path (the same kernels and collective sequence as
//    NCCL) can be exercised on a single GPU; it is not graph-capturable.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/enova.h"

namespace enova {
struct LocalGroup;
}

struct enova_comm_s {
  void *nccl;                 // ncclComm_t (NCCL backend), else null
  enova::LocalGroup *local;   // local backend, else null
  int rank, world, device;
  double timeout_s;           // bound of every host-side wait on this communicator
  bool aborted;               // a failure or timeout aborted it: every later call fails
};

namespace enova {
enova_status comm_allreduce_u64_sum(enova_comm_t c, const void *send, void *recv, size_t count,
                                    cudaStream_t st);
// one int64 per rank -> recv[world]
enova_status comm_allgather_i64(enova_comm_t c, const void *send, void *recv, cudaStream_t st);
// count floats per rank -> recv[world][count] (rank order)
enova_status comm_allgather_f32(enova_comm_t c, const void *send, void *recv, size_t count,
                                cudaStream_t st);
// Every cooperative (grid-synchronising) k_pot launch of a local group's ranks
// is bracketed by begin/end: the launches are serialised on the device in host
// enqueue order, so two of them are never co-scheduled on the shared SMs (each
// holds a whole SM; partial co-residency of two spinning grids would deadlock).
// No-ops for NCCL (one rank per device).
enova_status comm_coop_begin(enova_comm_t c, cudaStream_t st);
enova_status comm_coop_end(enova_comm_t c, cudaStream_t st);
// Bounded host wait for everything enqueued on `st` so far: polls the stream and,
// for NCCL, ncclCommGetAsyncError; an asynchronous NCCL error or a wait longer
// than the communicator's timeout aborts the communicator (ncclCommAbort, so no
// rank stays blocked inside a collective) and returns ENOVA_ERR_NCCL.
enova_status comm_wait(enova_comm_t c, cudaStream_t st);
// synchronous sum of one host int64 over the ranks (setup-time use); scratch:
// >= 8 bytes of device memory
enova_status comm_sum_i64_sync(enova_comm_t c, int64_t in, int64_t *out, void *scratch,
                               cudaStream_t st);
}  // namespace enova
