// comm.h -- NCCL communicator used only for the fleet-wide threshold (§8e).
// NCCL is resolved at run time with dlopen("libnccl.so.2"), so the library has
// no link-time dependency and picks up the NCCL that torch already loaded.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/enova.h"

struct enova_comm_s {
  void *nccl;  // ncclComm_t
  int rank, world, device;
};

namespace enova {
enova_status comm_allreduce_u64_sum(enova_comm_t c, const void *send, void *recv, size_t count,
                                    cudaStream_t st);
enova_status comm_allgather_i64(enova_comm_t c, const void *send, void *recv, cudaStream_t st);
// rank-ordered allgatherv of doubles: every rank's local[0..counts[rank]) lands at
// out + offsets[rank]
enova_status comm_allgatherv_f64(enova_comm_t c, const double *local, double *out,
                                 const int64_t *counts, const int64_t *offsets, cudaStream_t st);
}  // namespace enova
