// evaluate.cu -- NEXT-4: point-adjusted detection counts (P/R/F1 of the flags).
//
// "We adopt Precision, Recall and F1-score ... we adopt a point-adjusted
// approach" (citing Huang et al. 2022); the rule as SPEC.md:530-533
// states it (R-21): for each contiguous true-anomaly segment that
// contains at least one predicted point, every point of the segment counts as
// predicted; then P/R/F1 are computed pointwise.
//
// Points are the window end times t in [t_begin, t_begin + nw) of every
// instance: the prediction at t is flag != 0 of the window ending at t, the
// truth is label[t] != 0.  Segments never cross instances and are clipped to
// the evaluated range.  One warp per instance walks the range 32 points at a
// time with ballots: A = truth mask, P = prediction mask; runs of 1-bits of A
// are segments; a run still open at the chunk end carries (length, hit) into
// the next chunk.  Counts are exact integers (int64 atomics), so the result is
// independent of scheduling and of how instances are sharded over GPUs.
#include "common.cuh"

namespace enova {

__global__ void k_point_adjust(const int8_t *__restrict__ labels, int64_t ld_labels,
                               const int8_t *__restrict__ flags, int64_t n_inst, int64_t t_begin,
                               int64_t nw, unsigned long long *__restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t inst = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (inst >= n_inst) return;
  const int8_t *lab = labels + inst * ld_labels + t_begin;
  const int8_t *fl = flags + inst * nw;
  unsigned long long tp = 0, fp = 0, fn = 0, tn = 0;
  unsigned int open_len = 0;   // open segment (carried across chunks)
  bool open_hit = false;
  for (int64_t c0 = 0; c0 < nw; c0 += 32) {
    const int64_t t = c0 + lane;
    const bool in = t < nw;
    const bool a = in && lab[t] != 0;
    const bool p = in && fl[t] != 0;
    const unsigned int A = __ballot_sync(0xffffffffu, a);
    const unsigned int P = __ballot_sync(0xffffffffu, p);
    const unsigned int V = __ballot_sync(0xffffffffu, in);
    fp += __popc(P & ~A);
    tn += __popc(V & ~A & ~P);
    // walk the runs of A (warp-uniform bit arithmetic)
    unsigned int rest = A;
    int pos = 0;   // first bit not yet consumed
    while (pos < 32) {
      if (open_len > 0 && pos == 0) {
        // continuation of the open segment: its leading run starting at bit 0
        const unsigned int run = rest & ~(rest + 1u);   // trailing ones from bit 0
        if (run == 0u) {                                   // segment closed at the chunk boundary
          (open_hit ? tp : fn) += open_len;
          open_len = 0;
          open_hit = false;
          continue;
        }
        open_len += __popc(run);
        open_hit |= (P & run) != 0u;
        rest &= ~run;
        pos = (run == 0xffffffffu) ? 32 : 32 - __clz(run);
        if (pos < 32) {                                    // closed inside this chunk
          (open_hit ? tp : fn) += open_len;
          open_len = 0;
          open_hit = false;
        }
        continue;
      }
      if (rest == 0u) break;
      const int s = __ffs(rest) - 1;                       // next segment start
      const unsigned int from_s = rest >> s;
      const unsigned int ones = from_s & ~(from_s + 1u);   // run length bits at s
      const int len = __popc(ones);
      const unsigned int run = (len == 32) ? 0xffffffffu : (ones << s);
      const bool hit = (P & run) != 0u;
      rest &= ~run;
      const int end = s + len;                             // one past the run
      if (end >= 32) {                                     // open at the chunk end
        open_len = (unsigned int)len;
        open_hit = hit;
        pos = 32;
      } else {
        (hit ? tp : fn) += (unsigned long long)len;
        pos = end;
      }
    }
  }
  if (open_len > 0) (open_hit ? tp : fn) += open_len;
  if (lane == 0) {
    atomicAdd(counts + 0, tp);
    atomicAdd(counts + 1, fp);
    atomicAdd(counts + 2, fn);
    atomicAdd(counts + 3, tn);
  }
}

enova_status point_adjust_counts(const int8_t *labels, int64_t ld_labels, const int8_t *flags,
                                 int64_t n_inst, int64_t t_begin, int64_t nw,
                                 unsigned long long *counts_dev, cudaStream_t st) {
  ENOVA_CUDA_TRY(cudaMemsetAsync(counts_dev, 0, 4 * sizeof(unsigned long long), st));
  if (n_inst == 0 || nw == 0) return ENOVA_OK;
  const int threads = 256;
  const int64_t warps = n_inst;
  const unsigned blocks = (unsigned)((warps * 32 + threads - 1) / threads);
  ENOVA_LAUNCH(k_point_adjust, blocks, threads, 0, st, labels, ld_labels, flags, n_inst, t_begin,
               nw, counts_dev);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

// ---------------------------------------------------------------- NEXT-1 ----
// Stable compaction of the flagged window ids (flags != 0), index order: blocks
// of 1024 flags count, then each block adds up the counts before it (fixed
// order) and scatters with warp ballots.  Feeds enova_explain_windows.
constexpr int kSelBlock = 1024;

__global__ void k_flag_count(const int8_t *__restrict__ flags, int64_t n,
                             unsigned int *__restrict__ counts) {
  const int64_t i = blockIdx.x * (int64_t)kSelBlock + threadIdx.x;
  const int c = __syncthreads_count(i < n && flags[i] != 0);
  if (threadIdx.x == 0) counts[blockIdx.x] = (unsigned int)c;
}

__global__ void k_flag_scatter(const int8_t *__restrict__ flags, int64_t n,
                               const unsigned int *__restrict__ counts, int nblocks,
                               int64_t *__restrict__ ids, long long *__restrict__ total) {
  __shared__ unsigned long long base;
  __shared__ int wsum[kSelBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {   // exclusive prefix of this block (fixed order)
    unsigned long long s = 0, all = 0;
    for (int b = lane; b < nblocks; b += 32) {
      const unsigned long long v = counts[b];
      all += v;
      if (b < (int)blockIdx.x) s += v;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      all += __shfl_xor_sync(0xffffffffu, all, o);
    }
    if (lane == 0) {
      base = s;
      if (blockIdx.x == 0) *total = (long long)all;
    }
  }
  const int64_t i = blockIdx.x * (int64_t)kSelBlock + threadIdx.x;
  const bool f = i < n && flags[i] != 0;
  const unsigned int bal = __ballot_sync(0xffffffffu, f);
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += wsum[w];
  if (f) ids[base + before + __popc(bal & ((1u << lane) - 1u))] = i;
}

enova_status select_flagged(const int8_t *flags, int64_t n, int64_t *ids, long long *count_dev,
                            void *scratch, cudaStream_t st) {
  ENOVA_CUDA_TRY(cudaMemsetAsync(count_dev, 0, sizeof(long long), st));
  if (n == 0) return ENOVA_OK;
  const int64_t nb = (n + kSelBlock - 1) / kSelBlock;
  unsigned int *counts = static_cast<unsigned int *>(scratch);
  ENOVA_LAUNCH(k_flag_count, (unsigned)nb, kSelBlock, 0, st, flags, n, counts);
  ENOVA_LAUNCH(k_flag_scatter, (unsigned)nb, kSelBlock, 0, st, flags, n, counts, (int)nb, ids,
               count_dev);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

size_t select_flagged_scratch_bytes(int64_t n) {
  return align_up((size_t)((n + kSelBlock - 1) / kSelBlock) * 4, 256);
}

}  // namespace enova
