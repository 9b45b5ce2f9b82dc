// stats.cu -- K1: per-(instance, metric) normalisation statistics (a-1).
//
// "The input metrics are normalized prior to being fed into the VAE"
// (PAPER.md:282); per-dimension z-score with stats from the training horizon
// reused at inference, std floored at 1e-6 (R-4).
//
// One HBM pass, one wave: a persistent grid of one CTA per SM splits the
// flattened (instance, sample) space of the calibration horizon into equal
// contiguous ranges, so every CTA streams the same number of samples whatever
// the fleet shape -- no ragged last wave.  The bytes arrive by bulk copy: a
// producer warp walks the CTA's range as chunks of <= 64 KB inside one instance
// segment and keeps kStatsStages chunks in flight (cp.async.bulk into a shared
// memory ring, mbarrier complete_tx), so the HBM latency is covered without
// register-held loads; 512 consumer threads accumulate from shared memory.
// For each instance SEGMENT of the range the consumers accumulate the SHIFTED
// sums S1 = sum(x - K), S2 = sum((x - K)^2) in fp64, with K = the series' first
// sample (the same shift in every segment, so segment sums simply add), reduce
// them in a fixed order and store them in the instance's contributor slot
// (contributor c = this CTA's index minus the instance's first CTA).  The last
// contributor of an instance (ticket) combines the slots in contributor order:
// mean = K + S1/n, var = S2/n - (S1/n)^2.  With fp32 data and K inside the
// series' range this equals the two-pass fp64 result to ~1e-16 relative, far
// below the fp32 rounding that follows; the result depends on the grid only
// through the contributor split (deterministic for a device).
#include "common.cuh"

namespace enova {

unsigned long long *pair_trace();
// diagnostic %globaltimer stamps of CTA 0 (compiled in with -DENOVA_TRACE only)
__device__ __forceinline__ void k1_stamp(unsigned long long *tr, int slot) {
#ifdef ENOVA_TRACE
  if (tr && blockIdx.x == 0 && slot < 96) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[slot] = t;
  }
#else
  (void)tr;
  (void)slot;
#endif
}

constexpr int kStatsThreads = 512;              // consumers
constexpr int kStatsBlock = kStatsThreads + 32; // + the producer warp
constexpr int kStatsMaxGrid = 512;   // <= 256 SMs x 2 (workspace sizing)
// 3 x 64 KB in flight per SM (same-box ncu, c2: 5 x 32 KB 25.8 us, 10 x 16 KB
// 29.5 us, 3 x 64 KB 23.6 us -- the bytes in flight per SM set the rate)
#ifndef ENOVA_STATS_STAGES
#define ENOVA_STATS_STAGES 3
#endif
#ifndef ENOVA_STATS_CHUNK
#define ENOVA_STATS_CHUNK 65536
#endif
constexpr int kStatsStages = ENOVA_STATS_STAGES;
constexpr int kStatsDefer = 64;   // segments whose ticket / combine wait for finalize()
constexpr uint32_t kStatsChunkBytes = ENOVA_STATS_CHUNK;

// contributors of one instance: a CTA range holds >= floor(N T / nb) >= 64
// samples, so an instance of T samples meets at most ceil(nb / N) + 2 ranges
static inline int64_t stats_max_contrib(int64_t n) {
  return n <= 0 ? 1 : (kStatsMaxGrid + n - 1) / n + 2;
}

// workspace: [0, 256) diag counters | tickets u32[N] | slots f64[N][max_contrib][2][M]
size_t stats_workspace_bytes(int64_t n, int m) {
  if (n < 0) n = 0;
  return 256 + align_up((size_t)n * 4, 256) +
         align_up((size_t)n * stats_max_contrib(n) * 2 * m * sizeof(double), 256);
}

// the CTA whose range [floor(c S / nb), floor((c+1) S / nb)) holds sample x:
// the largest c with floor(c S / nb) <= x, i.e. c = ceil((x+1) nb / S) - 1
__device__ __forceinline__ int64_t cta_of(int64_t x, int64_t S, int nb) {
  return ((x + 1) * nb - 1) / S;
}

// the chunk sequence of a CTA range (walked identically by producer and consumers):
// chunk = [c0, c1) of the flattened space inside instance `inst`, <= cs samples;
// one 64-bit division per range, none per chunk
struct ChunkWalk {
  int64_t pos, r1, T_cal, cs, inst, full_end;
  __device__ __forceinline__ ChunkWalk(int64_t r0, int64_t r1_, int64_t T, int64_t cs_)
      : pos(r0), r1(r1_), T_cal(T), cs(cs_), inst(r0 / T), full_end((r0 / T + 1) * T) {}
  __device__ __forceinline__ bool next(int64_t &c0, int64_t &c1, int64_t &ci) {
    if (pos >= r1) return false;
    if (pos >= full_end) {   // next instance segment
      ++inst;
      full_end += T_cal;
    }
    c0 = pos;
    c1 = min(min(r1, full_end), pos + cs);
    ci = inst;
    pos = c1;
    return true;
  }
};

template <bool kPow2Group>
__global__ void __launch_bounds__(kStatsBlock, 1) k_series_stats(
    const float *__restrict__ X, int64_t ld, int M, int64_t N, int64_t T_cal,
    float *__restrict__ mean_out, float *__restrict__ std_out, unsigned long long *diag,
    unsigned int *ticket, double *slots, int64_t max_contrib, unsigned long long *tr) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[kStatsStages], empty[kStatsStages];
  __shared__ long long dinst[kStatsDefer];   // deferred segments: their instances
  __shared__ int dlast[kStatsDefer];         //   and whether this CTA is the last contributor
  __shared__ int bad_any;
  double *red = reinterpret_cast<double *>(sm + kStatsStages * kStatsChunkBytes);  // [rows][2][M]
  const int G = M / 4;
  const int nslots = kStatsThreads / G;
  const int active = nslots * G;       // consumer threads with a (slot, g)
  const int nb = gridDim.x;
  const int64_t S = N * T_cal;
  const int64_t r0 = (int64_t)blockIdx.x * S / nb, r1 = (int64_t)(blockIdx.x + 1) * S / nb;
  const int64_t cs = max((int64_t)1, (int64_t)(kStatsChunkBytes / (4u * (uint32_t)M)));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < kStatsStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kStatsThreads / 32);
    }
    bad_any = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) k1_stamp(tr, 0);
  if (tid >= kStatsThreads) {
    // ---------------- producer warp: bulk copies, kStatsStages chunks ahead ----------------
    if (lane == 0) {
      ChunkWalk w(r0, r1, T_cal, cs);
      int64_t c0, c1, inst;
      for (int k = 0; w.next(c0, c1, inst); ++k) {
        const int sg = k % kStatsStages;
        if (k >= kStatsStages) mbar_wait(&empty[sg], ((k / kStatsStages) - 1) & 1);
        const int64_t t = c0 - inst * T_cal;
        const uint32_t bytes = (uint32_t)(c1 - c0) * 4u * (uint32_t)M;
        mbar_arrive_expect_tx(&full[sg], bytes);
        bulk_g2s(sm + (size_t)sg * kStatsChunkBytes, X + inst * ld + t * M, bytes, &full[sg]);
        if (k < 24) k1_stamp(tr, 1 + k);
      }
    }
    return;   // the consumers never wait on the producer warp with a CTA barrier
  }
  // ---------------- consumers ----------------
  // finalize(): for every deferred segment (instance inst, this CTA's slot
  // written), the instance's ticket -- an acq_rel RMW at gpu scope after the
  // CTA barrier: it releases this CTA's slot writes (cumulative over the
  // barrier) and, for the last contributor, acquires every other contributor's
  // (no full fences) -- then the last contributor combines the slots in
  // contributor order: mean = K + S1/n, var = S2/n - (S1/n)^2
  int ndef = 0;   // uniform over the consumer threads
  auto finalize = [&]() {
    named_bar_sync(1, kStatsThreads);
    for (int q = tid; q < ndef; q += kStatsThreads) {
      const int64_t inst = dinst[q];
      const int64_t first = cta_of(inst * T_cal, S, nb);
      const int64_t ncontrib = cta_of((inst + 1) * T_cal - 1, S, nb) - first + 1;
      unsigned int old;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                   : "=r"(old)
                   : "l"(ticket + inst)
                   : "memory");
      dlast[q] = (old == (unsigned)ncontrib - 1) ? 1 : 0;
    }
    named_bar_sync(1, kStatsThreads);
    for (int w = tid; w < ndef * M; w += kStatsThreads) {
      const int q = w / M, j = w % M;
      if (!dlast[q]) continue;
      const int64_t inst = dinst[q];
      const int64_t first = cta_of(inst * T_cal, S, nb);
      const int64_t ncontrib = cta_of((inst + 1) * T_cal - 1, S, nb) - first + 1;
      const double *p0 = slots + (size_t)inst * max_contrib * 2 * M;
      double s1 = 0, s2 = 0;
      for (int64_t c = 0; c < ncontrib; ++c) {
        s1 += *(volatile const double *)(p0 + (size_t)c * 2 * M + j);
        s2 += *(volatile const double *)(p0 + (size_t)c * 2 * M + M + j);
      }
      const double n = (double)T_cal;
      const double kj = (double)__ldg(X + inst * ld + j);
      const double m1 = s1 / n;
      double var = s2 / n - m1 * m1;
      if (var < 0) var = 0;
      double sd = sqrt(var);
      if (sd < 1e-6) {
        atomicAdd(diag + 0, 1ull);
        sd = 1e-6;
      }
      mean_out[inst * M + j] = (float)(kj + m1);
      std_out[inst * M + j] = (float)sd;
    }
    named_bar_sync(1, kStatsThreads);   // dinst / dlast are reused
    ndef = 0;
  };
  const int g = tid % G;
  const int slot = tid / G;
  const bool act = tid < active;
  int bad = 0;
  ChunkWalk w(r0, r1, T_cal, cs);
  int64_t c0, c1, ci;
  int k = 0, seg = 0;
  bool have = w.next(c0, c1, ci);
  while (have) {
    const int64_t inst = ci;
    const float4 K = __ldg(reinterpret_cast<const float4 *>(X + inst * ld) + (act ? g : 0));
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, q0 = 0, q1 = 0, q2 = 0, q3 = 0;
    // every chunk of this segment
    do {
      const int sg = k % kStatsStages;
      mbar_wait(&full[sg], (k / kStatsStages) & 1);
      if (tid == 0 && k < 24) k1_stamp(tr, 32 + k);
      const float4 *src = reinterpret_cast<const float4 *>(sm + (size_t)sg * kStatsChunkBytes);
      const int n = (int)(c1 - c0);
      if (act) {
#pragma unroll 4
        for (int t = slot; t < n; t += nslots) {
          const float4 v = src[t * G + g];
          bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
          const double d0 = (double)v.x - K.x, d1 = (double)v.y - K.y, d2 = (double)v.z - K.z,
                       d3 = (double)v.w - K.w;
          a0 += d0; a1 += d1; a2 += d2; a3 += d3;
          q0 = fma(d0, d0, q0); q1 = fma(d1, d1, q1); q2 = fma(d2, d2, q2); q3 = fma(d3, d3, q3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sg]);
      ++k;
      have = w.next(c0, c1, ci);
    } while (have && ci == inst);
    // ---- the segment's sums: fixed-order reduction, contributor slot, ticket ----
    if (tid == 0) k1_stamp(tr, 64 + 2 * min(seg, 7));
    double v8[8] = {a0, a1, a2, a3, q0, q1, q2, q3};
    int nred;   // partial sums per output left in red[] (summed below in index order)
    if (kPow2Group) {
      // G a power of two <= 32 (M in {8, ..., 128}): fixed-order shuffle tree
      // over the slots of a warp (lanes with the same g), one row of red[] per warp
      for (int o = G; o < 32; o <<= 1)
#pragma unroll
        for (int q = 0; q < 8; ++q) v8[q] += __shfl_xor_sync(0xffffffffu, v8[q], o);
      if (lane < G) {
        double *r = red + (size_t)warp * 2 * M;
        r[4 * g + 0] = v8[0]; r[4 * g + 1] = v8[1]; r[4 * g + 2] = v8[2]; r[4 * g + 3] = v8[3];
        r[M + 4 * g + 0] = v8[4]; r[M + 4 * g + 1] = v8[5]; r[M + 4 * g + 2] = v8[6]; r[M + 4 * g + 3] = v8[7];
      }
      nred = kStatsThreads >> 5;
    } else {
      // any G (M a multiple of 4 up to 256): one row of red[] per slot, then a
      // fixed-order pairwise tree over the slots in shared memory (row s += row
      // s + half), so the result does not depend on warp boundaries
      if (act) {
        double *r = red + (size_t)slot * 2 * M;
        r[4 * g + 0] = v8[0]; r[4 * g + 1] = v8[1]; r[4 * g + 2] = v8[2]; r[4 * g + 3] = v8[3];
        r[M + 4 * g + 0] = v8[4]; r[M + 4 * g + 1] = v8[5]; r[M + 4 * g + 2] = v8[6]; r[M + 4 * g + 3] = v8[7];
      }
      int rows = nslots;
      while (rows > 1) {
        const int half = (rows + 1) >> 1;
        named_bar_sync(1, kStatsThreads);
        for (int e = tid; e < (rows - half) * 2 * M; e += kStatsThreads)
          red[e] += red[(size_t)half * 2 * M + e];
        rows = half;
      }
      nred = 1;
    }
    named_bar_sync(1, kStatsThreads);
    const int64_t first = cta_of(inst * T_cal, S, nb);
    const int64_t ncontrib = cta_of((inst + 1) * T_cal - 1, S, nb) - first + 1;
    const int64_t c = blockIdx.x - first;   // contributor index of this CTA
    double *pc = slots + ((size_t)inst * max_contrib + c) * 2 * M;
    for (int e = tid; e < 2 * M; e += kStatsThreads) {   // fixed-order sum over rows
      double sacc = 0;
      for (int q = 0; q < nred; ++q) sacc += red[(size_t)q * 2 * M + e];
      pc[e] = sacc;
    }
    // the tickets and the last contributors' combines of this CTA's segments
    // are deferred to the end of its range (or to a full list): one round of
    // tickets and one of combines instead of two dependent global round trips
    // per segment on the streaming path
    if (tid == 0) dinst[ndef] = inst;
    ++ndef;
    named_bar_sync(1, kStatsThreads);   // red[] is reused by the next segment
    if (ndef == kStatsDefer) finalize();
    if (tid == 0) k1_stamp(tr, 65 + 2 * min(seg, 7));
    ++seg;
  }
  if (ndef) finalize();
  if (bad) atomicOr(&bad_any, 1);
  named_bar_sync(1, kStatsThreads);
  if (tid == 0 && bad_any) atomicAdd(diag + 1, 1ull);   // CTAs with a non-finite sample
  if (tid == 0) k1_stamp(tr, 95);
}

// diag[0] = series whose std was floored, diag[1] = CTAs whose range held a
// non-finite sample (> 0 <=> ENOVA_ERR_NONFINITE).
enova_status compute_stats_async(const enova_series *s, int64_t t_cal_end, float *mean,
                                 float *stdv, unsigned long long *diag_dev, void *ws,
                                 size_t ws_bytes, cudaStream_t st) {
  const int64_t N = s->n_instances;
  const int M = s->n_metrics;
  if (ws_bytes < stats_workspace_bytes(N, M)) {
    set_error("stats workspace too small (size it with enova_stats_workspace_bytes)");
    return ENOVA_ERR_WORKSPACE;
  }
  char *b = static_cast<char *>(ws);
  unsigned long long *diag = diag_dev ? diag_dev : reinterpret_cast<unsigned long long *>(b);
  unsigned int *ticket = reinterpret_cast<unsigned int *>(b + 256);
  double *slots = reinterpret_cast<double *>(b + 256 + align_up((size_t)N * 4, 256));
  int dev = 0, sms = 148;
  ENOVA_CUDA_TRY(cudaGetDevice(&dev));
  ENOVA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // one wave of one CTA per SM, each with an equal share of the N * T_cal
  // samples (at least 64 samples per CTA)
  const int64_t S = N * t_cal_end;
  int64_t nb = sms;
  if (nb > kStatsMaxGrid) nb = kStatsMaxGrid;
  if (nb > S / 64) nb = S / 64;
  if (nb < 1) nb = 1;
  const int G = M / 4;
  const int nslots = kStatsThreads / G;
  if (diag_dev) ENOVA_CUDA_TRY(cudaMemsetAsync(diag_dev, 0, 2 * sizeof(unsigned long long), st));
  ENOVA_CUDA_TRY(cudaMemsetAsync(b, 0, 256 + (size_t)N * 4, st));   // diag (own) + tickets
  const bool pow2 = (G & (G - 1)) == 0 && G <= 32;
  const size_t smem = (size_t)kStatsStages * kStatsChunkBytes +
                      (size_t)(pow2 ? kStatsThreads / 32 : nslots) * 2 * M * sizeof(double);
  auto kern = pow2 ? k_series_stats<true> : k_series_stats<false>;
  ENOVA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ENOVA_LAUNCH(kern, (unsigned)nb, kStatsBlock, smem, st, s->metrics, s->ld_instance, M, N,
               t_cal_end, mean, stdv, diag, ticket, slots, stats_max_contrib(N), pair_trace());
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

enova_status compute_stats(const enova_series *s, int64_t t_cal_end, float *mean, float *stdv,
                           int64_t *n_degenerate, void *ws, size_t ws_bytes, cudaStream_t st) {
  enova_status r = compute_stats_async(s, t_cal_end, mean, stdv, nullptr, ws, ws_bytes, st);
  if (r) return r;
  unsigned long long h[2];
  ENOVA_CUDA_TRY(cudaMemcpyAsync(h, ws, sizeof(h), cudaMemcpyDeviceToHost, st));
  ENOVA_CUDA_TRY(cudaStreamSynchronize(st));
  if (n_degenerate) *n_degenerate = (int64_t)h[0];
  if (h[1]) {
    set_error("non-finite metric value in the calibration horizon");
    return ENOVA_ERR_NONFINITE;
  }
  return ENOVA_OK;
}

}  // namespace enova
