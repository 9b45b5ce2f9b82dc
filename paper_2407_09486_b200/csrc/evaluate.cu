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
// the evaluated range.  One CTA per instance; each of its 8 warps walks a
// contiguous sub-range 32 points at a time with ballots (A = truth mask,
// P = prediction mask; runs of 1-bits of A are segments; a run still open at a
// chunk end carries (length, hit) into the next chunk); runs touching a
// sub-range boundary are merged in sub-range order by one thread.  Counts are
// exact integers (int64 atomics), so the result is independent of scheduling
// and of how instances are sharded over GPUs.
#include "common.cuh"

namespace enova {

// One CTA per instance, kPaWarps warps; warp w walks the contiguous sub-range
// [w*len, (w+1)*len) of the instance in 32-point ballots.  Segments strictly
// inside a sub-range are counted by that warp; the (possibly continuing) first
// and last runs of every sub-range are left to a fixed-order merge by thread 0.
constexpr int kPaWarps = 8;
constexpr int kPaTile = 1024;   // points per shared-memory tile per warp

struct PaRun {
  unsigned int lead_len, tail_len;   // run touching the sub-range start / end
  int lead_hit, tail_hit, full;      // full: the whole sub-range is one labelled run
};

__global__ void __launch_bounds__(32 * kPaWarps) k_point_adjust(
    const int8_t *__restrict__ labels, int64_t ld_labels, const int8_t *__restrict__ flags,
    int64_t n_inst, int64_t t_begin, int64_t nw, unsigned long long *__restrict__ counts) {
  __shared__ PaRun runs[kPaWarps];
  __shared__ int8_t stl[kPaWarps][kPaTile], stf[kPaWarps][kPaTile];
  __shared__ unsigned long long part[kPaWarps][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t inst = blockIdx.x;
  const int8_t *lab = labels + inst * ld_labels + t_begin;
  const int8_t *fl = flags + inst * nw;
  int64_t sub = (nw + kPaWarps - 1) / kPaWarps;
  sub = (sub + 31) / 32 * 32;
  const int64_t r0 = min(nw, (int64_t)warp * sub), r1 = min(nw, r0 + sub);
  unsigned long long tp = 0, fp = 0, fn = 0, tn = 0;
  unsigned int cur_len = 0;   // the run currently open (carried across chunks)
  bool cur_hit = false, cur_lead = false;   // cur_lead: the open run starts at r0
  PaRun rec{0u, 0u, 0, 0, 0};
  auto finish = [&](bool open_at_end) {     // the open run ends (or reaches r1)
    if (cur_lead) {                         // leading run: merged by thread 0
      rec.lead_len = cur_len;
      rec.lead_hit = cur_hit;
      rec.full = open_at_end ? 1 : 0;
    } else if (open_at_end) {               // trailing run: merged by thread 0
      rec.tail_len = cur_len;
      rec.tail_hit = cur_hit;
    } else {
      (cur_hit ? tp : fn) += cur_len;
    }
    cur_len = 0;
    cur_hit = false;
    cur_lead = false;
  };
  for (int64_t c0 = r0; c0 < r1; c0 += 32) {
    // stage the next kPaTile points of this warp's sub-range in shared memory
    // (all byte loads of a lane in flight at once: one latency per tile)
    const int64_t tile0 = r0 + ((c0 - r0) / kPaTile) * kPaTile;
    if (c0 == tile0) {
      __syncwarp();
#pragma unroll
      for (int k = 0; k < kPaTile / 32; ++k) {
        const int64_t tt = tile0 + k * 32 + lane;
        stl[warp][k * 32 + lane] = (tt < r1) ? lab[tt] : (int8_t)0;
        stf[warp][k * 32 + lane] = (tt < r1) ? fl[tt] : (int8_t)0;
      }
      __syncwarp();
    }
    const int64_t t = c0 + lane;
    const bool in = t < r1;
    const int off = (int)(c0 - tile0) + lane;
    const bool a = in && stl[warp][off] != 0;
    const bool p = in && stf[warp][off] != 0;
    const unsigned int A = __ballot_sync(0xffffffffu, a);
    const unsigned int P = __ballot_sync(0xffffffffu, p);
    const unsigned int V = __ballot_sync(0xffffffffu, in);
    fp += __popc(P & ~A);
    tn += __popc(V & ~A & ~P);
    const int valid_n = (int)min((int64_t)32, r1 - c0);
    int pos = 0;
    while (true) {
      const unsigned int rest = (pos < 32) ? (A >> pos) : 0u;
      if (cur_len > 0 && (rest & 1u) == 0u) finish(false);   // a gap closes the open run
      if (rest == 0u) break;
      const int s = __ffs(rest) - 1;
      const int start = pos + s;
      const unsigned int from = A >> start;
      const unsigned int ones = from & ~(from + 1u);
      const int len = __popc(ones);
      const unsigned int run = (len == 32) ? 0xffffffffu : (ones << start);
      if (cur_len == 0) cur_lead = (c0 + start == r0);
      cur_len += (unsigned int)len;
      cur_hit = cur_hit || ((P & run) != 0u);
      pos = start + len;
      if (pos >= valid_n) break;             // still open at the chunk / sub-range end
    }
  }
  if (cur_len) finish(true);                 // open at r1
  if (lane == 0) {
    runs[warp] = rec;
    part[warp][0] = tp;
    part[warp][1] = fp;
    part[warp][2] = fn;
    part[warp][3] = tn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long T[4] = {0, 0, 0, 0};
    for (int w = 0; w < kPaWarps; ++w)
      for (int k = 0; k < 4; ++k) T[k] += part[w][k];
    // fixed-order merge of the boundary runs
    unsigned long long clen = 0;
    bool chit = false;
    for (int w = 0; w < kPaWarps; ++w) {
      const PaRun r = runs[w];
      if (r.lead_len) {
        clen += r.lead_len;
        chit = chit || r.lead_hit;
        if (r.full) continue;                 // still open
      }
      if (clen) (chit ? T[0] : T[2]) += clen;  // the carried run closed before/at this sub-range
      clen = r.tail_len;
      chit = r.tail_hit;
    }
    if (clen) (chit ? T[0] : T[2]) += clen;
    atomicAdd(counts + 0, T[0]);
    atomicAdd(counts + 1, T[1]);
    atomicAdd(counts + 2, T[2]);
    atomicAdd(counts + 3, T[3]);
  }
}

enova_status point_adjust_counts(const int8_t *labels, int64_t ld_labels, const int8_t *flags,
                                 int64_t n_inst, int64_t t_begin, int64_t nw,
                                 unsigned long long *counts_dev, cudaStream_t st) {
  ENOVA_CUDA_TRY(cudaMemsetAsync(counts_dev, 0, 4 * sizeof(unsigned long long), st));
  if (n_inst == 0 || nw == 0) return ENOVA_OK;
  if (n_inst > 0x7fffffffLL) {
    set_error("too many instances");
    return ENOVA_ERR_UNSUPPORTED;
  }
  ENOVA_LAUNCH(k_point_adjust, (unsigned)n_inst, 32 * kPaWarps, 0, st, labels, ld_labels, flags,
               n_inst, t_begin, nw, counts_dev);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

// ---------------------------------------------------------------- NEXT-1 ----
// Stable compaction of the flagged window ids (flags != 0), index order: blocks
// of 1024 flags count, one small kernel scans the block counts (fixed order,
// O(n) total), then each block scatters with warp ballots.  Feeds
// enova_explain_windows.
constexpr int kSelBlock = 1024;

__global__ void k_flag_count(const int8_t *__restrict__ flags, int64_t n,
                             unsigned int *__restrict__ counts) {
  const int64_t i = blockIdx.x * (int64_t)kSelBlock + threadIdx.x;
  const int c = __syncthreads_count(i < n && flags[i] != 0);
  if (threadIdx.x == 0) counts[blockIdx.x] = (unsigned int)c;
}

// exclusive prefix of the block counts (one CTA, fixed order: each thread sums a
// contiguous span of blocks, then a block-wide scan of the span sums)
__global__ void __launch_bounds__(1024) k_flag_scan(const unsigned int *__restrict__ counts,
                                                    int64_t nblocks,
                                                    unsigned long long *__restrict__ base,
                                                    long long *__restrict__ total) {
  __shared__ unsigned long long wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t per = (nblocks + blockDim.x - 1) / blockDim.x;
  const int64_t b0 = min(nblocks, (int64_t)threadIdx.x * per), b1 = min(nblocks, b0 + per);
  unsigned long long own = 0;
  for (int64_t b = b0; b < b1; ++b) own += counts[b];
  unsigned long long incl = own;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  unsigned long long run = incl - own;
  for (int w = 0; w < warp; ++w) run += wsum[w];
  for (int64_t b = b0; b < b1; ++b) {
    base[b] = run;
    run += counts[b];
  }
  if (threadIdx.x == blockDim.x - 1) *total = (long long)run;
}

__global__ void k_flag_scatter(const int8_t *__restrict__ flags, int64_t n,
                               const unsigned long long *__restrict__ base,
                               int64_t *__restrict__ ids) {
  __shared__ int wsum[kSelBlock / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = blockIdx.x * (int64_t)kSelBlock + threadIdx.x;
  const bool f = i < n && flags[i] != 0;
  const unsigned int bal = __ballot_sync(0xffffffffu, f);
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += wsum[w];
  if (f) ids[base[blockIdx.x] + before + __popc(bal & ((1u << lane) - 1u))] = i;
}

static inline size_t sel_counts_bytes(int64_t nb) { return align_up((size_t)nb * 4, 256); }

enova_status select_flagged(const int8_t *flags, int64_t n, int64_t *ids, long long *count_dev,
                            void *scratch, cudaStream_t st) {
  ENOVA_CUDA_TRY(cudaMemsetAsync(count_dev, 0, sizeof(long long), st));
  if (n == 0) return ENOVA_OK;
  const int64_t nb = (n + kSelBlock - 1) / kSelBlock;
  unsigned int *counts = static_cast<unsigned int *>(scratch);
  unsigned long long *base = reinterpret_cast<unsigned long long *>(
      static_cast<char *>(scratch) + sel_counts_bytes(nb));
  ENOVA_LAUNCH(k_flag_count, (unsigned)nb, kSelBlock, 0, st, flags, n, counts);
  ENOVA_LAUNCH(k_flag_scan, 1, 1024, 0, st, counts, nb, base, count_dev);
  ENOVA_LAUNCH(k_flag_scatter, (unsigned)nb, kSelBlock, 0, st, flags, n, base, ids);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

size_t select_flagged_scratch_bytes(int64_t n) {
  const int64_t nb = (n + kSelBlock - 1) / kSelBlock;
  return sel_counts_bytes(nb) + align_up((size_t)nb * 8, 256);
}

}  // namespace enova
