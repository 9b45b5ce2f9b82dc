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

}  // namespace enova
