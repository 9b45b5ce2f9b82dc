// threshold.cu -- K3..K5: fleet-wide peaks-over-threshold calibration (a-7..a-9).
//
// "The threshold for detecting anomalies is automatically set using the
// peaks-over-threshold method" (citing Siffer et al. 2017;
// SPEC.md:232-240, 254, 260; R-11..R-13):
//   t   = S_(k), k = floor(q0 n): exact order statistic by a 3-pass radix select
//         over order-preserving uint32 keys of the fp32 scores (11/11/10-bit
//         digits, integer histograms -> all-reduced across ranks, exact);
//   Y   = {s - t : s > t} in fp64, compacted stably in index order (and
//         all-gathered in rank order), so every rank holds the same Y;
//   GPD = maximum likelihood by Grimshaw's reduction: the roots of
//         w(x) = u(x) v(x) - 1 (u = mean 1/(1+xY), v = 1 + mean log1p(xY)) are
//         bracketed on the fixed 64-point grids of both intervals and refined by
//         safeguarded Newton to |step| <= 1e-13 |x|; every root gives
//         gamma = v - 1, sigma = gamma / x, log-likelihood -N (ln sigma + gamma + 1);
//         the exponential candidate (gamma = 0, sigma = Ybar) is always present;
//   z_q = t + sigma/gamma * expm1(-gamma ln(q n / N_t))  (t - sigma ln(.) at gamma = 0).
//
// v3 design: the whole single-GPU threshold is ONE cooperative launch
// (k_pot, one 512-thread CTA per SM) that walks a phase program with grid-wide
// barriers -- histogram pass 0, select + histogram 1, select + histogram 2,
// select + stable compaction, then the fit (Y statistics, grid scan, Newton
// passes, final pass) -- with no host round trip.  With a communicator the same
// kernel runs the phases in four launches separated by the NCCL exchanges
// (histogram all-reduce, tail all-gather).  Every CTA keeps an identical copy of
// the select and fit state and reduces the per-CTA partials itself, in a fixed
// order, after each barrier: the result is deterministic and, because the fit
// partition depends only on N_t and the grid size, identical on every rank and
// for every world size.
#include <math.h>
#include <stddef.h>

#include <vector>

#include "comm.h"
#include "common.cuh"

namespace enova {

constexpr int kBins = 2048;
constexpr int kPotThreads = 512;   // select_digit covers 2048 bins as 512 threads x 4
constexpr int kPotWarps = kPotThreads / 32;
constexpr int kMaxCtas = 256;
constexpr int kMaxWorld = 256;        // ranks of one communicator (fleet threshold)
constexpr int kMaxPts = 128;
constexpr int kMaxSlots = 64;
constexpr int kGrid = 64;
constexpr int kMaxRefinePasses = 60;
constexpr int kMaxStamps = 96;
constexpr int kSums = 6;              // P, L, dP, dL, d2P, d2L per evaluation point
// certification half-width (relative): a certified root lies within 1e-11 |x|
// of the fp64 root of w -- two orders of magnitude inside the z_q parity
// tolerance (1e-9 relative); 5e-14 needed an extra pass on some
// inputs (2M-score mixture: 6 passes -> 5) when w's summation noise near the
// root blurred the sign test
constexpr double kCertRel = 5e-12;

enum { PH_GRID = 0, PH_REFINE = 1, PH_FINAL = 2, PH_DONE = 3, PH_GRID32 = 4, PH_GRIDFIX = 5,
       PH_GRIDBIN = 6, PH_BREFINE = 7 };
// Large tails: before the fp64 (certifying) Halley passes over Y, each bracket's
// root is located by up to kMaxBinRefine Halley passes over the bins (PH_BREFINE:
// w and its derivatives from the binned sums, the iterate kept inside the fp64
// bracket; no sign of a binned w is trusted).  The exact passes then start within
// the binned model's error (~1e-8 relative) of the root: one Halley step lands
// within rounding of it and the next pass certifies it -- two passes over Y
// instead of five from the grid's secant point.
constexpr int kMaxBinRefine = 4;
// a binned Halley step below this (relative) ends the binned passes: the
// iterate it produced is then within the binned model's error of the root
#ifndef ENOVA_BREF_TOL
#define ENOVA_BREF_TOL 1e-10
#endif
constexpr double kBrefTol = ENOVA_BREF_TOL;
// evaluation sums per point of a pass: P, L (+ first and second derivatives)
__device__ __forceinline__ int phase_sums(int phase) {
  return (phase == PH_REFINE || phase == PH_BREFINE) ? kSums : 2;
}
// Large tails (N_t >= kGrid32MinPeaks): the 128-point scan grid is evaluated in
// two passes (PH_GRID32, PH_GRIDBIN) -- points with |x| Ymax <= 1e-3 from six
// fp64 power sums of Y/Ymax (the log1p and 1/(1+t) series, 1e-18 truncation),
// points with x Ymax < -0.9 in fp64 over Y (PH_GRID32, which also bins Y), the
// rest over a log-binned histogram of Y (PH_GRIDBIN): per bin the count, sum and
// sum of squares, each term evaluated at the bin mean with the exact
// second-order correction 1/2 f''(ybar_b) sum (y - ybar_b)^2 -- 2048 bins per
// octave (relative width 3.4e-4), so the remainder is third order (<= 1e-7 of
// the sums even at x Ymax = -0.9) -- and an error bound: a sign is accepted when
// |w| > 1e-6 (|P| + |L| + |P L|), else that point is re-evaluated in fp64 over
// Y (PH_GRIDFIX).  The signs, hence the brackets, are those of the fp64 scan
// wherever the fp64 scan itself resolves them; the binned Halley passes
// (PH_BREFINE) only place the start of the certifying fp64 passes over Y.
constexpr int64_t kGrid32MinPeaks = 100000;
constexpr int kMaxBins = 131072;          // binned grid pass: bins of log2(Y) (x3 int64 each)
constexpr double kBinsPerOctave = 2048.0;
constexpr int kPow = 6;   // power sums of u = Y / Ymax for the series points
constexpr int kMaxPole = 8;      // hybrid pole points (the grid has 7 with x Ymax < -0.9)
constexpr int kPoleList = 96;    // per-warp list of the pass's high Y (flushed when full)
// phase program of k_pot
enum { P_SAMPLE = 0, P_SCAN = 1, P_HIST0 = 2, P_HIST1 = 3, P_HIST2 = 4, P_COMPACT = 5, P_FIT = 6 };
// sampled candidate selection (single GPU, n >= kSampleMinN): P_SAMPLE picks a
// key lo from a strided sample so that >= (1 - q0) + 8 sigma of the scores lie
// at or above it; P_SCAN is the ONE full pass: it counts the keys below lo and
// compacts the others (the candidates, ~2.4% of n) stably into this CTA's
// segment; the radix passes and the peak compaction then read only the
// candidates.  Exact: if the count below lo exceeds k (a sample that
// misjudged the quantile) every CTA falls back to the full passes.
constexpr int kSampleN = 2048;                 // samples per CTA
constexpr int64_t kSampleMinN = int64_t(1) << 22;

// Device-global state of one fit_threshold call.  The first kHeaderBytes of the
// workspace (this struct and histogram 0) are zeroed by one memset per call;
// everything else is initialised by the kernel itself.
struct PotGlobal {
  unsigned int bar_count, bar_gen;   // grid barrier arrivals (bar_gen unused)
  int status;                        // enova_status of the device phases
  int pad0;
  unsigned int prefix, mask;         // radix-select state after the last select
  unsigned long long k_rem;
  float t;
  int pad1;
  long long nt_local, nt_fit;        // peaks of this rank / of the fit (all ranks)
  double gamma, sigma, z_q;
  int method, nroots, converged, overflow;
  long long n_spot;                  // NEXT-2: observations counted by the online SPOT state
  long long nt_refit;                // NEXT-2: N_t at the last (re)fit
  int spot_overflow;                 // NEXT-2: a tick's peaks exceeded the Y capacity (sticky
                                     // until the next calibration fit zeroes the header)
  int pad2;
  int n_stamps, fit_passes;
  unsigned int sample_lo;            // P_SAMPLE's candidate bound (key), read by k_pot_scan
  int pad4;
  int sampled, fit_stamp;            // the last selection ran on the sampled candidates;
                                     // stamp index at the start of the fit (diagnostic)
  unsigned long long stamps[kMaxStamps];   // %globaltimer of CTA 0 at phase boundaries (diagnostic)
  unsigned long long t_first_start, t_last_end;   // over all CTAs (diagnostic)
};

struct FitState {
  int64_t nt, n;
  double t, q, ybar, ymin, ymax;
  int phase, npts, nslots, iters, overflow, converged, nrefine, method, nroots;
  double xs[kMaxPts], w[kMaxPts], L[kMaxPts], dw[kMaxPts], ddw[kMaxPts];
  double P[kMaxPts];          // mean -xY/(1+xY) of the last pass (certification bound)
  // PH_GRID32 / PH_GRIDFIX: the full scan grid, w at its points, how each point
  // is evaluated (0 fp32 certified, 1 series, 2 fp64), evaluation-list <-> grid
  double gx[kMaxPts], gw[kMaxPts], pm[kPow + 1];
  int gmode[kMaxPts], gidx[kMaxPts], ginv[kMaxPts];
  int ngrid, n64, n32, nfix;
  double bin_l0, bin_k;       // PH_GRIDBIN: bin b holds log2(Y) in [l0 + b/k, l0 + (b+1)/k)
  int nbins;
  int triple;                 // REFINE evaluates (x, x(1-d), x(1+d)) per root (certifying)
  int bin_cl;                 // ceil(log2(N_t + 1)): fixed-point headroom of the bin sums
  int use_bins;               // the bins are filled (N_t >= kGrid32MinPeaks): PH_BREFINE first
  int biters, pad_b;          // PH_BREFINE passes run
  // hybrid pole points (x Ymax < -0.9): the Y of bins >= bin_cb (y >~ Ymax / 2,
  // where 1 + x y may approach 0) summed exactly in the PH_GRID32 pass (gP, gL:
  // their mean P and L terms), the bins below bin_cb in PH_GRIDBIN (1 + x y >= ~1/2
  // there: the binned model's accuracy holds); gmode 4 = pole point awaiting its
  // binned part
  int bin_cb, pole_hybrid;
  double gP[kMaxPts], gL[kMaxPts];
  double bdiag[kMaxBinRefine][4];   // diagnostic build (ENOVA_FIT_STAMPS): binned Halley steps
  int bdiag_nr, pad_bd;
  int rdone[kMaxSlots];       // refine slot converged (triple mode)
  double lo[kMaxSlots], hi[kMaxSlots], wlo[kMaxSlots], whi[kMaxSlots];
  int exact[kMaxSlots];
  int refine_idx[kMaxSlots];
  double lfin[kMaxSlots];     // L at a slot's certified root, when the last refine pass evaluated it
  double gamma, sigma, z_q;
};

struct ThrLayout {
  size_t glob, hist, counts, part, nbuf, counts_all, ylocal, yslot, outdev, yall, header, total;
  size_t shist, cand, cand_n;   // sampled selection: sample histograms, candidates, per-CTA counts
  size_t fstate, xsend, xrecv;  // distributed fit (communicator layouts)
  size_t bins;                  // binned passes: [kMaxBins][3] int64 (count, fixed-point sums, see bin_add)
  bool has_bins;
  int64_t cap;
  bool sampled;                 // workspace holds the candidate buffer
};

// world == 0: single-GPU layout.  world >= 1 (communicator): this rank's tail as
// fp32 scores (ylocal, cap), the all-gathered fixed-size slots of every rank
// (yslot, world x cap fp32: a rank never holds more than the global tail, so the
// gather needs no host-side counts), and a device copy of the result.
static inline ThrLayout thr_layout(int64_t n_max, double q0, int world = 0) {
  ThrLayout L;
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o += (b + 255) / 256 * 256; return r; };
  double tail = (1.0 - q0) * (double)n_max;
  if (tail < 0) tail = 0;
  L.cap = (int64_t)ceil(tail) + 16;
  if (L.cap > n_max) L.cap = n_max;
  if (L.cap < 16) L.cap = 16;
  L.glob = take(sizeof(PotGlobal));
  L.shist = take(2 * kBins * 8);                    // sample histograms (zeroed per call)
  L.hist = take(3 * kBins * 8);
  L.header = L.hist + kBins * 8;                    // PotGlobal + sample histograms + histogram 0
  L.counts = take(kMaxCtas * 8);
  L.part = take((size_t)2 * kSums * kMaxPts * kMaxCtas * 8);
  L.nbuf = take(16);
  L.counts_all = take(kMaxWorld * 8);
  L.ylocal = take(world ? (size_t)L.cap * 4 : 0);
  L.yslot = take((size_t)world * (size_t)L.cap * 4);
  L.outdev = take(world ? sizeof(enova_threshold) : 0);
  L.yall = take((size_t)L.cap * 8);
  L.fstate = take(world ? sizeof(FitState) : 0);
  L.xsend = take(world ? (size_t)kSums * kMaxPts * 8 : 0);
  L.xrecv = take((size_t)world * kSums * kMaxPts * 8);
  L.has_bins = L.cap >= kGrid32MinPeaks;
  L.bins = take(L.has_bins ? (size_t)kMaxBins * 3 * 8 : 0);
  // candidates: one segment of ceil(chunk / 4) * 4 scores per CTA (a segment can
  // hold its CTA's whole chunk, so it never overflows)
  L.sampled = (world == 0 && n_max >= kSampleMinN);
  L.cand = take(L.sampled ? ((size_t)n_max + 4u * kMaxCtas) * 4 : 0);
  L.cand_n = take(L.sampled ? (size_t)kMaxCtas * 2 * 8 : 0);
  L.total = o;
  return L;
}

struct PotArgs {
  const float *scores;
  int64_t n_local;          // scores on this rank
  int64_t n;                // scores over all ranks
  unsigned long long k;     // rank of t in the global ascending order
  double q;                 // risk
  PotGlobal *g;
  unsigned long long *hist; // [3][kBins]
  long long *counts;        // [gridDim.x]
  double *part;             // [2][kSums][kMaxPts][kMaxCtas]
  double *ydst;             // single GPU: compaction target Y = s - t (the fit's tail)
  const double *yfit;       // tail the fit runs on (all ranks, rank order)
  float *ylocal;            // communicator: compaction target (raw scores > t), else null
  const float *yslot;       // communicator: gathered [world][cap] slots, else null
  const long long *counts_all;   // communicator: gathered per-rank tail counts
  int world;
  int64_t cap;
  int first, last;          // phase range of this launch
  enova_threshold *out_dev; // optional device copy of the result
  double q0;
  int ycache_cap;           // Y values per CTA held in dynamic shared memory
  const long long *n_dev;   // NEXT-2 refit: n read from device (g->n_spot), else a.n
  unsigned long long *shist; // [2][kBins] sample histograms
  float *cand;              // sampled selection: per-CTA candidate segments, else null
  long long *cand_n;        // [kMaxCtas] candidates, [kMaxCtas] keys below lo, per CTA
  // distributed fit (communicator path): step of this launch (-1: not distributed)
  int dfit_step, dfit_last;
  double *xsend;            // [kSums * kMaxPts] this rank's totals of the step
  const double *xrecv;      // [world][kSums * kMaxPts] gathered totals
  FitState *fstate;         // the fit's state between launches
  unsigned long long *bins; // [kMaxBins][3] binned grid pass (null below kGrid32MinPeaks)
};

__device__ __forceinline__ unsigned int f2key(float f) {
  unsigned int b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(unsigned int k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// grid-wide barrier for a cooperative launch (all CTAs co-resident): a
// monotonically increasing arrival counter (zeroed by the per-call header
// memset, or before each launch of the communicator path).  Barrier number b
// (1-based, counted per CTA in `epoch`) completes when the counter reaches
// b * gridDim.x: one release-add per CTA, then acquire-polls of the same word
// -- no fences, no second hop through a generation flag.
__device__ __forceinline__ void grid_sync(PotGlobal *g, unsigned int &epoch) {
  ++epoch;
  uint32_t ncta;
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncta));
  if (ncta == gridDim.x) {
    // the whole grid is one thread-block cluster (a reduced fit grid of <= 16
    // CTAs): the hardware cluster barrier, release / acquire at cluster scope,
    // orders the global-memory partials like the counter barrier below
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int target = epoch * gridDim.x;
    unsigned int *p = &g->bar_count;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
    unsigned int v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
      if (v >= target) break;
      __nanosleep(16);
    }
  }
  __syncthreads();
}

// diagnostic timestamps (CTA 0, thread 0): the running index lives in shared
// memory -- no global read on the critical path; the stores are fire-and-forget
__shared__ int s_nstamp;
__device__ __forceinline__ void stamp(PotGlobal *g) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const int i = s_nstamp;
    if (i < kMaxStamps - 1) g->stamps[i] = t;
    s_nstamp = i + 1;
  }
}

// contiguous chunk of [0, n) owned by this CTA (multiple of 4 for float4 loads)
__device__ __forceinline__ void score_chunk(int64_t n, int64_t *b0, int64_t *b1) {
  int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  chunk = (chunk + 3) / 4 * 4;
  *b0 = min(n, (int64_t)blockIdx.x * chunk);
  *b1 = min(n, *b0 + chunk);
}

struct SelS {
  unsigned int prefix, mask;
  unsigned long long k_rem;
  float t;
};

// ---------------------------------------------------------------- K3 ----
// Histogram of the digit at `shift` of every key of this CTA's chunk that
// matches the selected prefix; warp-aggregated shared atomics (keys of nearby
// scores share bins), flushed to the global uint64 histogram.  Each thread
// keeps 4 float4 loads in flight.  Pass 2 also counts this CTA's keys above
// the selected 22-bit bucket (*above), so the peak count of the CTA follows
// from its own histogram once the last digit is chosen (no counting pass).
__device__ void hist_pass(const PotArgs &a, const SelS &sel, int pass, unsigned int *h,
                          int *above_smem, const float *src, int64_t len) {
  const int shift = (pass == 0) ? 21 : (pass == 1) ? 10 : 0;
  const int nbins = (pass == 2) ? 1024 : 2048;
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) h[i] = 0;
  if (threadIdx.x == 0) *above_smem = 0;
  __syncthreads();
  const int64_t b0 = 0, b1 = len;
  const unsigned int prefix = sel.prefix, mask = sel.mask;
  const unsigned int bucket_hi = prefix | ~mask;   // pass 2: largest key of the bucket
  int above = 0;
  auto add = [&](float f, bool valid) {
    const unsigned int k = f2key(f);
    const bool hit = valid && ((k & mask) == prefix);
    above += (valid && k > bucket_hi);
    const unsigned int act = __ballot_sync(0xffffffffu, hit);
    if (hit) {
      const unsigned int bin = (k >> shift) & (nbins - 1);
      const unsigned int peers = __match_any_sync(act, bin);
      if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&h[bin], __popc(peers));
    }
  };
  const bool al = (reinterpret_cast<uintptr_t>(src + b0) & 15) == 0;
  int64_t tail0 = b0;
  if (al) {
    const float4 *x4 = reinterpret_cast<const float4 *>(src + b0);
    const int64_t n4 = (b1 - b0) / 4;
    // two register batches of 4 float4 ping-pong: batch k+1 is in flight while
    // batch k is binned (8 x 128-bit loads outstanding per thread)
    const int64_t step = 4 * (int64_t)blockDim.x;
    auto load = [&](float4 (&v)[4], bool (&ok)[4], int64_t i0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * blockDim.x + threadIdx.x;
        ok[u] = i < n4;
        v[u] = ok[u] ? __ldg(x4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto bin = [&](const float4 (&v)[4], const bool (&ok)[4]) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        add(v[u].x, ok[u]);
        add(v[u].y, ok[u]);
        add(v[u].z, ok[u]);
        add(v[u].w, ok[u]);
      }
    };
    float4 va[4], vb[4];
    bool oka[4], okb[4];
    load(va, oka, 0);
    for (int64_t i0 = 0; i0 < n4; i0 += 2 * step) {   // warp-uniform trip count
      load(vb, okb, i0 + step);
      bin(va, oka);
      if (i0 + 2 * step < n4) load(va, oka, i0 + 2 * step);
      bin(vb, okb);
    }
    tail0 = b0 + 4 * n4;
  }
  for (int64_t i0 = tail0; i0 < b1; i0 += blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    add(i < b1 ? __ldg(src + i) : 0.f, i < b1);
  }
  if (pass == 2) {
#pragma unroll
    for (int o = 16; o; o >>= 1) above += __shfl_xor_sync(0xffffffffu, above, o);
    if ((threadIdx.x & 31) == 0 && above) atomicAdd(above_smem, above);
  }
  __syncthreads();
  unsigned long long *gh = a.hist + (size_t)pass * kBins;
  for (int i = threadIdx.x; i < nbins; i += blockDim.x)
    if (h[i]) atomicAdd(gh + i, (unsigned long long)h[i]);
}

// Every CTA reads the (complete) histogram of `pass` and finds the digit that
// holds rank k_rem: 512 threads x 4 bins, block exclusive scan.
__device__ void select_digit(const PotArgs &a, SelS &sel, int pass, unsigned long long *wtot,
                             int *found, const unsigned long long *hist_override = nullptr) {
  const int shift = (pass == 0) ? 21 : (pass == 1) ? 10 : 0;
  const int nbins = (pass == 2) ? 1024 : 2048;
  const unsigned long long *gh = hist_override ? hist_override : a.hist + (size_t)pass * kBins;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long c[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int b = 4 * tid + u;
    c[u] = (b < nbins) ? *(volatile const unsigned long long *)(gh + b) : 0ull;
  }
  const unsigned long long v = c[0] + c[1] + c[2] + c[3];
  unsigned long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long wv = (lane < kPotWarps) ? wtot[lane] : 0ull;
    unsigned long long wi = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kPotWarps) wtot[lane] = wi - wv;
  }
  __syncthreads();
  const unsigned long long k = sel.k_rem;
  unsigned long long before = wtot[warp] + incl - v;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (c[u] && k >= before && k < before + c[u]) {
      found[0] = 4 * tid + u;
      reinterpret_cast<unsigned long long *>(found)[1] = before;
    }
    before += c[u];
  }
  __syncthreads();
  if (tid == 0) {   // sel is shared: one writer (every thread read k before the barrier)
    const unsigned int digit = (unsigned int)found[0];
    const unsigned long long below = reinterpret_cast<unsigned long long *>(found)[1];
    sel.prefix |= digit << shift;
    sel.mask |= (unsigned int)(nbins - 1) << shift;
    sel.k_rem = k - below;
    if (pass == 2) sel.t = key2f(sel.prefix);
  }
  __syncthreads();
}

// ------------------------------------------------------- sampled select ----
// P_SAMPLE: CTA b keys kSampleN evenly spaced scores of its chunk into shared
// memory; two grid-wide histogram levels (top 11 bits, then the next 11 of the
// chosen bucket) locate the sample's order statistic at q0 - delta, delta = 8
// sample standard deviations + 2/S; lo = the lowest key of that 22-bit bucket.
__device__ int64_t sample_total(const PotArgs &a) {   // every CTA's sample size, summed
  int64_t tot = 0;
  const int64_t chunk = ((a.n_local + gridDim.x - 1) / gridDim.x + 3) / 4 * 4;
  for (int b = 0; b < (int)gridDim.x; ++b) {
    const int64_t b0 = min(a.n_local, (int64_t)b * chunk), b1 = min(a.n_local, b0 + chunk);
    tot += min((int64_t)kSampleN, b1 - b0);
  }
  return tot;
}

__device__ void sample_phase(const PotArgs &a, SelS &ssel, unsigned int *h, unsigned int *sk,
                             int &ns_out, unsigned long long *wtot, int *found,
                             unsigned int &epoch, long long *s_tot) {
  int64_t b0, b1;
  score_chunk(a.n_local, &b0, &b1);
  const int64_t len = b1 - b0;
  const int ns = (int)min((int64_t)kSampleN, len);
  // sample j at floor(j len / ns): 32-bit arithmetic when j len < 2^32 (the same
  // integer), the 64-bit division only for chunks above 2M scores
  if (len <= (int64_t)(0xffffffffu / kSampleN)) {
    const uint32_t l32 = (uint32_t)len, n32 = (uint32_t)ns;
    for (int j = threadIdx.x; j < ns; j += blockDim.x)
      sk[j] = f2key(__ldg(a.scores + b0 + (uint32_t)j * l32 / n32));
  } else {
    for (int j = threadIdx.x; j < ns; j += blockDim.x)
      sk[j] = f2key(__ldg(a.scores + b0 + (int64_t)j * len / ns));
  }
  if (threadIdx.x == 0) {
    const int64_t S = sample_total(a);
    const double q0 = a.q0;
    const double delta = 8.0 * sqrt(q0 * (1.0 - q0) / (double)S) + 2.0 / (double)S;
    const double qs = q0 - delta;
    s_tot[0] = qs > 0.0 ? (long long)floor(qs * (double)S) : 0;
    ssel.prefix = 0;
    ssel.mask = 0;
    ssel.k_rem = (unsigned long long)s_tot[0];
  }
  for (int level = 0; level < 2; ++level) {
    const int shift = level == 0 ? 21 : 10;
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < ns; j += blockDim.x) {
      const unsigned int k = sk[j];
      if ((k & ssel.mask) == ssel.prefix) atomicAdd(&h[(k >> shift) & (kBins - 1)], 1u);
    }
    __syncthreads();
    unsigned long long *gh = a.shist + (size_t)level * kBins;
    for (int i = threadIdx.x; i < kBins; i += blockDim.x)
      if (h[i]) atomicAdd(gh + i, (unsigned long long)h[i]);
    grid_sync(a.g, epoch);
    stamp(a.g);
    select_digit(a, ssel, level, wtot, found, gh);
  }
  ns_out = ns;
}

// P_SCAN: the one full pass over this CTA's chunk -- count the keys below lo,
// compact the rest (the candidates) stably (index order) into the CTA's segment
// a.cand + blockIdx.x * seg_cap.  Warp w owns a contiguous sub-range of the
// chunk and streams it with two ping-ponged register batches of 4 x 128-bit
// loads per lane (8 in flight, no CTA barrier in the loop).  Its candidates go
// to its own run: a slice of the shared staging buffer while they fit (plain
// shared-memory stores), else -- after one copy of what the slice holds -- its
// region [w * sub, ...) of the global segment.  When every run stayed in shared
// memory the warps write them straight to their final offsets (coalesced);
// otherwise the runs are moved down in warp order (destination <= source, each
// chunk read before it is written).
//
// Output offsets.  Fast path (lo >= 2^31: lo is the key of a float >= +0, the
// case of every score the detector emits): key(v) >= lo <=> (int)bits(v) >=
// (int)(lo ^ 2^31) for every bit pattern (negative floats and negative NaNs are
// negative ints with keys < 2^31 <= lo; positive NaNs are candidates both ways),
// one integer compare per element; the per-float4 candidate counts of a batch
// (0..4 each) travel packed in the bytes of one word through ONE warp inclusive
// scan (a byte's prefix <= 128), giving every lane its offset in (float4 slot,
// lane, element) = index order.  General path and ragged tails: four ballots per
// float4 on the keys.
#ifndef ENOVA_SCAN_PF
#define ENOVA_SCAN_PF 512
#endif
constexpr int kScanPf = ENOVA_SCAN_PF;   // float4 (multiple of 256): the scan's L2 prefetch distance
__device__ void scan_phase(const PotArgs &a, unsigned int lo, int64_t seg_cap, long long *out_n,
                           float *stage, int stage_cap) {
  __shared__ long long wcount[kPotWarps], wbelow[kPotWarps];
  __shared__ int wspill[kPotWarps];
  int64_t b0, b1;
  score_chunk(a.n_local, &b0, &b1);
  const float *src = a.scores + b0;
  const int64_t len = b1 - b0;
  float *dst = a.cand + (size_t)blockIdx.x * seg_cap;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned int lt = (1u << lane) - 1u;
  // warp sub-ranges: multiples of 4 scores (16 B aligned when the chunk is)
  const int64_t sub = ((len + kPotWarps - 1) / kPotWarps + 3) / 4 * 4;
  const int64_t w0 = min(len, (int64_t)warp * sub), w1 = min(len, w0 + sub);
  unsigned int *wd = reinterpret_cast<unsigned int *>(dst + w0);   // the warp's global region
  const int wcap = stage_cap / kPotWarps;
  unsigned int *ws = reinterpret_cast<unsigned int *>(stage) + (size_t)warp * wcap;   // its smem slice
  bool insm = true;   // warp-uniform: the run is in the smem slice
  long long cnt = 0;  // warp-uniform; the warp's keys below lo = its range - cnt
  // before appending up to `more` candidates: leave the smem slice if they may not fit
  auto reserve = [&](long long more) {
    if (insm && cnt + more > (long long)wcap) {
      for (long long i = lane; i < cnt; i += 32) wd[i] = ws[i];
      __syncwarp();
      insm = false;
    }
  };
  // the leading nv (0..4) elements of q, in index order after the lower lanes'
  auto put4 = [&](const float4 q, int nv) {
    reserve(128);
    const float e4[4] = {q.x, q.y, q.z, q.w};
    bool c[4];
    unsigned int bl[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      c[e] = e < nv && f2key(e4[e]) >= lo;
      bl[e] = __ballot_sync(0xffffffffu, c[e]);
    }
    // lanes below l hold 4 elements each before this lane's first one
    long long o = cnt + __popc(bl[0] & lt) + __popc(bl[1] & lt) + __popc(bl[2] & lt) +
                  __popc(bl[3] & lt);
    unsigned int *out = insm ? ws : wd;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (c[e]) out[o++] = __float_as_uint(e4[e]);
    cnt += __popc(bl[0]) + __popc(bl[1]) + __popc(bl[2]) + __popc(bl[3]);
  };
  const bool al = (reinterpret_cast<uintptr_t>(src + w0) & 15) == 0;
  int64_t tail0 = w0;
  if (al && lo >= 0x80000000u && (w1 - w0) / 4 < 0x40000000) {
    const int lo_i = (int)(lo ^ 0x80000000u);
    const uint4 *x4 = reinterpret_cast<const uint4 *>(src + w0);
    const int nfull = (int)(((w1 - w0) / 4) & ~(int64_t)127);   // full batches of 4 x 32 float4
    unsigned int c32 = 0;   // warp-uniform candidate count (< 2^32: the range is)
    auto ld = [&](uint4 (&v)[4], int i0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(x4 + i0 + u * 32 + lane);
    };
    auto proc = [&](const uint4 (&v)[4]) {
      unsigned int m[4], pk = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        m[u] = ((int)v[u].x >= lo_i ? 1u : 0u) | ((int)v[u].y >= lo_i ? 2u : 0u) |
               ((int)v[u].z >= lo_i ? 4u : 0u) | ((int)v[u].w >= lo_i ? 8u : 0u);
        pk += (unsigned int)__popc(m[u]) << (8 * u);
      }
      unsigned int sc = pk;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned int t = __shfl_up_sync(0xffffffffu, sc, d);
        if (lane >= d) sc += t;
      }
      const unsigned int tot = __shfl_sync(0xffffffffu, sc, 31), ex = sc - pk;
      if (tot == 0) return;   // no candidate in the batch (warp-uniform)
      cnt = c32;
      reserve((long long)(tot & 0xffu) + ((tot >> 8) & 0xffu) + ((tot >> 16) & 0xffu) + (tot >> 24));
      unsigned int b = c32;
      if (insm) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (m[u]) {
            unsigned int *bp = ws + b + ((ex >> (8 * u)) & 0xffu);
            if (m[u] & 1u) *bp++ = v[u].x;
            if (m[u] & 2u) *bp++ = v[u].y;
            if (m[u] & 4u) *bp++ = v[u].z;
            if (m[u] & 8u) *bp = v[u].w;
          }
          b += (tot >> (8 * u)) & 0xffu;
        }
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (m[u]) {
            unsigned int *bp = wd + b + ((ex >> (8 * u)) & 0xffu);
            if (m[u] & 1u) *bp++ = v[u].x;
            if (m[u] & 2u) *bp++ = v[u].y;
            if (m[u] & 4u) *bp++ = v[u].z;
            if (m[u] & 8u) *bp = v[u].w;
          }
          b += (tot >> (8 * u)) & 0xffu;
        }
      }
      c32 = b;
    };
    // L2 prefetch kScanPf float4 ahead of the loads (one bulk prefetch of the
    // warp's next 4 KB per iteration, no registers held): the register batches
    // then mostly hit L2, so the 8 loads in flight per lane cover its latency
    const int64_t n4w = (w1 - w0) / 4;
    auto pf = [&](int64_t i) {
      if (kScanPf > 0 && lane == 0 && i < n4w) {
        const uint32_t bytes = (uint32_t)(min((int64_t)256, n4w - i) * 16);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x4 + i), "r"(bytes) : "memory");
      }
    };
    if (kScanPf > 0)
      for (int64_t i = 0; i < kScanPf; i += 256) pf(i);
    if (nfull > 0) {
      uint4 va[4], vb[4];
      ld(va, 0);
      for (int i0 = 0; i0 < nfull; i0 += 256) {   // warp-uniform trip count
        const bool hb = i0 + 128 < nfull;
        pf((int64_t)i0 + kScanPf);
        if (hb) ld(vb, i0 + 128);
        proc(va);
        if (i0 + 256 < nfull) ld(va, i0 + 256);
        if (hb) proc(vb);
      }
    }
    cnt = c32;
    tail0 = w0 + 4 * (int64_t)nfull;
  } else if (al) {
    const float4 *x4 = reinterpret_cast<const float4 *>(src + w0);
    const int64_t n4 = (w1 - w0) / 4;
    auto ld = [&](float4 (&v)[4], int64_t i0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * 32 + lane;
        v[u] = (i < n4) ? __ldg(x4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto proc = [&](const float4 (&v)[4], int64_t i0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) put4(v[u], (i0 + u * 32 + lane < n4) ? 4 : 0);
    };
    float4 va[4], vb[4];
    ld(va, 0);
    for (int64_t i0 = 0; i0 < n4; i0 += 256) {   // warp-uniform trip count
      ld(vb, i0 + 128);
      proc(va, i0);
      if (i0 + 256 < n4) ld(va, i0 + 256);
      proc(vb, i0 + 128);
    }
    tail0 = w0 + 4 * n4;
  }
  for (int64_t i0 = tail0; i0 < w1; i0 += 128) {   // unaligned or ragged rest
    const int64_t i = i0 + 4 * lane;
    float4 q;
    q.x = i < w1 ? __ldg(src + i) : 0.f;
    q.y = i + 1 < w1 ? __ldg(src + i + 1) : 0.f;
    q.z = i + 2 < w1 ? __ldg(src + i + 2) : 0.f;
    q.w = i + 3 < w1 ? __ldg(src + i + 3) : 0.f;
    put4(q, (int)max((int64_t)0, min((int64_t)4, w1 - i)));
  }
  if (lane == 0) {
    wcount[warp] = cnt;
    wbelow[warp] = (w1 - w0) - cnt;
    wspill[warp] = insm ? 0 : 1;
  }
  __syncthreads();
  long long pos = 0, mypos = 0;
  int spilled = 0;
  for (int w = 0; w < kPotWarps; ++w) {
    if (w == warp) mypos = pos;
    pos += wcount[w];
    spilled |= wspill[w];
  }
  if (!spilled) {
    // every run in shared memory: each warp writes its run at its final offset
    float *to = dst + mypos;
    for (long long i = lane; i < cnt; i += 32) to[i] = __uint_as_float(ws[i]);
  } else {
    // runs -> the global regions [w * sub, ...) first, then one contiguous,
    // index-ordered segment.  Common case (the CTA's candidates fit the staging
    // smem): every warp copies its run to its final offset in shared memory at
    // once, then the CTA writes the segment back.  Otherwise the runs are moved
    // down in warp order, each chunk read before it is written.
    if (insm)
      for (long long i = lane; i < cnt; i += 32) wd[i] = ws[i];
    __syncthreads();   // every run in global memory; the smem slices are free
    if (pos <= (long long)stage_cap) {
      const float *from = dst + (int64_t)warp * sub;
      for (long long i = lane; i < cnt; i += 32) stage[mypos + i] = from[i];
      __syncthreads();
      for (long long i = threadIdx.x; i < pos; i += blockDim.x) dst[i] = stage[i];
    } else {
      long long p2 = wcount[0];
      for (int w = 1; w < kPotWarps; ++w) {
        const long long c = wcount[w];
        const float *from = dst + (int64_t)w * sub;
        float *to = dst + p2;
        for (long long i = 0; i < c; i += blockDim.x) {
          const float v = (i + threadIdx.x < c) ? from[i + threadIdx.x] : 0.f;
          __syncthreads();
          if (i + threadIdx.x < c) to[i + threadIdx.x] = v;
          __syncthreads();
        }
        p2 += c;
      }
    }
  }
  if (threadIdx.x == 0) {
    long long bl = 0;
    for (int w = 0; w < kPotWarps; ++w) bl += wbelow[w];
    out_n[0] = pos;    // candidates of this CTA
    out_n[1] = bl;     // keys below lo
    a.cand_n[blockIdx.x] = pos;
    a.cand_n[kMaxCtas + blockIdx.x] = bl;
  }
  __syncthreads();
}

// The scan as its own (non-cooperative) launch between the sampling launch and
// the selection + fit launch: its register budget is its own (inside the
// phase-program kernel the loop ran at ~1.3 TB/s), same grid and partition.
constexpr int kScanStageBytes = 200 * 1024;   // k_pot_scan's staging smem (51 200 candidates)
__global__ void __launch_bounds__(kPotThreads, 1) k_pot_scan(PotArgs a) {
  extern __shared__ float scan_stage[];
  __shared__ long long n2[2];
  const unsigned int lo = *(volatile unsigned int *)&a.g->sample_lo;
  scan_phase(a, lo, ((a.n_local + gridDim.x - 1) / gridDim.x + 3) / 4 * 4, n2, scan_stage,
             kScanStageBytes / 4);
}

// ---------------------------------------------------------------- K4 ----
// Stable compaction of the peaks Y = s - t (s > t) of this rank in index order.
// The CTA's peak count is known without reading the scores: keys above the
// 22-bit bucket (counted in pass 2) plus its own pass-2 histogram bins above
// the selected digit (h, still in shared memory).  One barrier publishes the
// per-CTA counts; the scatter then keeps 4 float4 loads in flight per thread
// and orders the output by (load slot, thread, element) = index order.
__device__ void compact(const PotArgs &a, const SelS &sel, const unsigned int *h, int above,
                        bool have_hist, int *wcnt, long long *cta_base, unsigned int &epoch,
                        const float *src, int64_t len) {
  const int64_t b0 = 0, b1 = len;
  const float t = sel.t;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c = 0;
  if (have_hist) {
    const unsigned int digit = f2key(t) & 1023u;
    for (int i = (int)digit + 1 + threadIdx.x; i < 1024; i += blockDim.x) c += (int)h[i];
  } else {   // separate launch (communicator path): count by reading the chunk
    above = 0;
    for (int64_t i0 = b0; i0 < b1; i0 += 4 * blockDim.x) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * blockDim.x + threadIdx.x;
        v[u] = (i < b1) ? __ldg(src + i) : -INFINITY;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) c += (v[u] > t);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) wcnt[warp] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = above;
    for (int w = 0; w < kPotWarps; ++w) s += wcnt[w];
    a.counts[blockIdx.x] = s;
  }
  grid_sync(a.g, epoch);
  stamp(a.g);
  if (warp == 0) {   // exclusive prefix of this CTA and the total, fixed order
    long long before = 0, tot = 0;
    for (int b = lane; b < (int)gridDim.x; b += 32) {
      const long long v = *(volatile long long *)(a.counts + b);
      tot += v;
      if (b < (int)blockIdx.x) before += v;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      before += __shfl_xor_sync(0xffffffffu, before, o);
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    if (lane == 0) {
      cta_base[0] = before;
      cta_base[1] = tot;
    }
  }
  __syncthreads();
  long long base = cta_base[0];
  const double td = (double)t;
  const bool al = (reinterpret_cast<uintptr_t>(src + b0) & 15) == 0;
  int *wc = wcnt;   // [4][kPotWarps]
  auto scatter4 = [&](const float (&v)[4][4], const bool (&ok)[4][4]) {
    int cnt[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      cnt[u] = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) cnt[u] += (ok[u][e] && v[u][e] > t);
    }
    int incl[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      incl[u] = cnt[u];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl[u], o);
        if (lane >= o) incl[u] += y;
      }
      if (lane == 31) wc[u * kPotWarps + warp] = incl[u];
    }
    __syncthreads();
    long long off_u = base;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int before_w = 0, all = 0;
      for (int w = 0; w < kPotWarps; ++w) {
        const int vv = wc[u * kPotWarps + w];
        before_w += (w < warp) ? vv : 0;
        all += vv;
      }
      long long o = off_u + before_w + incl[u] - cnt[u];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (ok[u][e] && v[u][e] > t) {
          if (o < a.cap) {
            if (a.ylocal) a.ylocal[o] = v[u][e];
            else a.ydst[o] = (double)v[u][e] - td;
          }
          ++o;
        }
      off_u += all;
    }
    base = off_u;
    __syncthreads();
  };
  int64_t tail0 = b0;
  if (al) {
    const float4 *x4 = reinterpret_cast<const float4 *>(src + b0);
    const int64_t n4 = (b1 - b0) / 4;
    // the next batch's 4 float4 are loaded before this batch is scattered
    const int64_t step = 4 * (int64_t)blockDim.x;
    float4 nq[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = u * blockDim.x + threadIdx.x;
      nq[u] = (i < n4) ? __ldg(x4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int64_t i0 = 0; i0 < n4; i0 += step) {
      float v[4][4];
      bool ok[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * blockDim.x + threadIdx.x;
        const bool g = i < n4;
        const float4 q = nq[u];
        v[u][0] = q.x; v[u][1] = q.y; v[u][2] = q.z; v[u][3] = q.w;
#pragma unroll
        for (int e = 0; e < 4; ++e) ok[u][e] = g;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + step + u * blockDim.x + threadIdx.x;
        nq[u] = (i < n4) ? __ldg(x4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      scatter4(v, ok);
    }
    tail0 = b0 + 4 * n4;
  }
  for (int64_t i0 = tail0; i0 < b1; i0 += 16 * blockDim.x) {   // ragged tail / unaligned
    float v[4][4];
    bool ok[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t i = i0 + (int64_t)u * 4 * blockDim.x + 4 * threadIdx.x + e;
        ok[u][e] = i < b1;
        v[u][e] = ok[u][e] ? __ldg(src + i) : 0.f;
      }
    scatter4(v, ok);
  }
}

// ---------------------------------------------------------------- K5 ----
// Phase machine, run by the whole CTA after each pass (identical in every CTA):
//  GRID  : w at the fixed scan grids -> one slot per sign change (or exact zero),
//          slots in grid order (block prefix count over the points);
//  REFINE: safeguarded Newton on every bracket, one thread per root: w(x), w'(x)
//          from the same pass; the bracket shrinks with the sign of w(x); the
//          Newton iterate is kept if it falls strictly inside the bracket, else
//          the bracket midpoint is used; converged when every step is
//          <= 1e-13 |x| (the oracle bisects to a 2^-60 bracket: both land on the
//          same root of the fp64 w);
//  FINAL : L(x) at the roots -> gamma, sigma, log-likelihood (one thread per
//          root); pick the best; z_q.
__device__ void controller(FitState *f, int *scratch) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int phase = f->phase;   // read by all threads before any write below
  __syncthreads();
  if (phase == PH_GRID32 || phase == PH_GRIDBIN || phase == PH_GRIDFIX) {
    // w at every scan-grid point: series / fp64 (GRID32), certified binned
    // (GRIDBIN), or the fp64 re-evaluations of the uncertain binned points (GRIDFIX)
    const int ng = f->ngrid;
    if (phase == PH_GRID32) {
      if (tid < ng) {
        const int mode = f->gmode[tid];
        if (mode == 1) {
          // series in t = z u, z = x Ymax, u = Y / Ymax (|t| <= 1e-3):
          //   P = sum_m (-1)^m z^m <u^m>,  L = sum_m (-1)^(m+1) z^m <u^m> / m,
          //   P + L = sum_{m>=2} (-1)^m (1 - 1/m) z^m <u^m>  (no O(z) cancellation)
          const double z = f->gx[tid] * f->ymax;
          double P = 0.0, L = 0.0, PL = 0.0, zm = 1.0;
          for (int m = 1; m <= kPow; ++m) {
            zm *= z;
            const double tm = zm * f->pm[m];
            const double sg = (m & 1) ? -1.0 : 1.0;
            P += sg * tm;
            L -= sg * tm / m;
            if (m >= 2) PL += sg * tm * (1.0 - 1.0 / m);
          }
          f->gw[tid] = PL + P * L;
        } else if (mode == 2) {
          if (f->pole_hybrid) {   // the exact high-Y part; the binned part follows
            f->gP[tid] = f->P[f->ginv[tid]];
            f->gL[tid] = f->L[f->ginv[tid]];
            f->gmode[tid] = 4;
          } else {
            f->gw[tid] = f->w[f->ginv[tid]];
          }
        }
      }
      __syncthreads();
      if (tid == 0) {   // the binned points' evaluation list (grid order)
        int nb = 0;
        for (int g = 0; g < ng; ++g)
          if (f->gmode[g] == 0 || f->gmode[g] == 4) {
            f->gidx[nb] = g;
            f->xs[nb] = f->gx[g];
            ++nb;
          }
        f->npts = nb;
        if (nb > 0) f->phase = PH_GRIDBIN;
      }
      __syncthreads();
      if (f->phase == PH_GRIDBIN) return;   // one more pass, over the bins
    } else if (phase == PH_GRIDBIN) {
      if (tid < f->npts) {
        const int g = f->gidx[tid];
        double w = f->w[tid], P = f->P[tid], L = f->L[tid];
        if (f->gmode[g] == 4) {   // pole point: binned low bins + exact high Y
          P += f->gP[g];
          L += f->gL[g];
          w = P + L + P * L;
        }
        f->gw[g] = w;
        // the binned sums carry a third-order remainder <= ~3e-8 of |P| + |L| (bin
        // width 3.4e-4, x Ymax >= -0.9) and fp64 rounding: a 1e-6 bound leaves a
        // 30x margin
        const double bound = 1e-6 * (fabs(P) + fabs(L) + fabs(P * L));
        if (!(fabs(w) > bound)) f->gmode[g] = 3;   // uncertain: fp64 re-evaluation
      }
      __syncthreads();
    }
    if (phase == PH_GRID32 || phase == PH_GRIDBIN) {
      if (tid == 0) {
        int nf = 0;
        for (int g = 0; g < ng; ++g)
          if (f->gmode[g] == 3) {
            f->gidx[nf] = g;
            f->xs[nf] = f->gx[g];
            f->gmode[g] = 2;
            ++nf;
          }
        f->nfix = nf;
        if (nf > 0) {
          f->npts = nf;
          f->phase = PH_GRIDFIX;
        }
      }
      __syncthreads();
      if (f->nfix > 0) return;   // one more (fp64) pass over Y
    } else {
      if (tid < f->nfix) f->gw[f->gidx[tid]] = f->w[tid];
      __syncthreads();
    }
    // the whole grid, in grid order, for the bracket scan
    if (tid < ng) {
      f->xs[tid] = f->gx[tid];
      f->w[tid] = f->gw[tid];
    }
    if (tid == 0) {
      f->npts = ng;
      f->phase = PH_GRID;
    }
    __syncthreads();
    phase = PH_GRID;
  }
  if (phase == PH_GRID) {
    const int npts = f->npts;
    bool ex = false, br = false;
    double xk = 0.0, xk1 = 0.0, wk = 0.0, wk1 = 0.0;
    if (tid < npts) {
      const int j = tid % kGrid;
      xk = f->xs[tid];
      wk = f->w[tid];
      ex = (wk == 0.0);
      if (!ex && j < kGrid - 1) {
        xk1 = f->xs[tid + 1];
        wk1 = f->w[tid + 1];
        br = (wk * wk1 < 0.0);
      }
    }
    const bool has = ex || br;
    const unsigned int bh = __ballot_sync(0xffffffffu, has), bb = __ballot_sync(0xffffffffu, br);
    if (lane == 0 && warp < kMaxPts / 32) {
      scratch[warp] = __popc(bh);
      scratch[8 + warp] = __popc(bb);
    }
    __syncthreads();   // all reads of xs / w done
    int tot_h = 0, tot_b = 0, off_h = 0, off_b = 0;
    for (int w = 0; w < kMaxPts / 32; ++w) {
      tot_h += scratch[w];
      tot_b += scratch[8 + w];
      if (w < warp) {
        off_h += scratch[w];
        off_b += scratch[8 + w];
      }
    }
    const unsigned int lt = (1u << lane) - 1u;
    off_h += __popc(bh & lt);
    off_b += __popc(bb & lt);
    const int ns = min(tot_h, kMaxSlots);
    if (has && off_h < kMaxSlots) {
      f->lo[off_h] = xk;
      f->hi[off_h] = ex ? xk : xk1;
      f->wlo[off_h] = ex ? 0.0 : wk;
      f->whi[off_h] = ex ? 0.0 : wk1;
      f->exact[off_h] = ex ? 1 : 0;
    }
    // refine slots: the bracket slots that fit, in slot order
    int nr = 0;
    {
      // brackets among the first kMaxSlots slots: count those with off_h < kMaxSlots
      const unsigned int bbf = __ballot_sync(0xffffffffu, br && off_h < kMaxSlots);
      if (lane == 0 && warp < kMaxPts / 32) scratch[16 + warp] = __popc(bbf);
      __syncthreads();
      for (int w = 0; w < kMaxPts / 32; ++w) nr += scratch[16 + w];
    }
    const bool triple = 3 * nr <= kMaxPts;
    const bool bref = f->use_bins && nr > 0;   // binned Halley passes first
    if (br && off_h < kMaxSlots) {
      f->refine_idx[off_b] = off_h;
      f->rdone[off_b] = 0;
      double x0 = xk - wk * (xk1 - xk) / (wk1 - wk);   // first iterate: secant point
      if (!(x0 > fmin(xk, xk1) && x0 < fmax(xk, xk1))) x0 = 0.5 * (xk + xk1);
      if (bref) {
        f->xs[off_b] = x0;
      } else if (triple) {
        f->xs[3 * off_b] = x0;
        f->xs[3 * off_b + 1] = x0 * (1.0 - kCertRel);
        f->xs[3 * off_b + 2] = x0 * (1.0 + kCertRel);
      } else {
        f->xs[off_b] = x0;
      }
    }
    __syncthreads();
    if (nr == 0 && tid < ns) f->xs[tid] = f->lo[tid];
    if (tid == 0) {
      f->nslots = ns;
      f->overflow = (tot_h > kMaxSlots) ? 1 : f->overflow;
      f->nrefine = nr;
      f->triple = triple ? 1 : 0;
      f->converged = (nr == 0) ? 1 : 0;
      f->npts = (nr > 0) ? ((triple && !bref) ? 3 * nr : nr) : ns;
      f->phase = (nr > 0) ? (bref ? PH_BREFINE : PH_REFINE) : PH_FINAL;
      f->biters = 0;
    }
    __syncthreads();
    return;
  }
  if (phase == PH_BREFINE) {
    // binned Halley step per bracket, kept inside the (fp64-certified) bracket;
    // after convergence to the binned model (or kMaxBinRefine passes) the
    // iterates start the exact passes
    const int nr = f->nrefine, it = f->biters;
    bool conv = true;
    double xn = 0.0;
    if (tid < nr) {
      const int sidx = f->refine_idx[tid];
      const double x = f->xs[tid], w = f->w[tid], dw = f->dw[tid], ddw = f->ddw[tid];
      const double a = fmin(f->lo[sidx], f->hi[sidx]), b = fmax(f->lo[sidx], f->hi[sidx]);
      const double den = 2.0 * dw * dw - w * ddw;
      xn = (den != 0.0 && isfinite(den)) ? x - 2.0 * w * dw / den : (dw != 0.0 ? x - w / dw : x);
      const bool clamped = !(xn > a && xn < b);
      if (clamped) xn = (xn <= a) ? 0.5 * (x + a) : 0.5 * (x + b);
      conv = fabs(xn - x) <= kBrefTol * fabs(x);
#ifdef ENOVA_FIT_STAMPS   // diagnostic: per pass and root, the relative step (negative if clamped)
      if (it < kMaxBinRefine && tid < 4) f->bdiag[it][tid] = (clamped ? -1.0 : 1.0) * fabs(xn - x) / fabs(x);
      if (tid == 0) f->bdiag_nr = nr;
#endif
    }
    const int all_conv = __syncthreads_and(conv);   // every read of xs / w done
    const bool done = all_conv || it + 1 >= kMaxBinRefine;
    if (tid < nr) {
      if (done && f->triple) {
        f->xs[3 * tid] = xn;
        f->xs[3 * tid + 1] = xn * (1.0 - kCertRel);
        f->xs[3 * tid + 2] = xn * (1.0 + kCertRel);
      } else {
        f->xs[tid] = xn;
      }
    }
    if (tid == 0) {
      f->biters = it + 1;
      if (done) {
        f->phase = PH_REFINE;
        f->npts = f->triple ? 3 * nr : nr;
      }
    }
    __syncthreads();
    return;
  }
  if (phase == PH_REFINE && f->triple) {
    // Halley from the centre point, bracket shrunk with all three points, and
    // certification: opposite signs of w at x(1 -+ d) put the root within
    // 2 d |x| = 1e-11 |x| of x in the SAME pass that found it.
    const int nr = f->nrefine, iters = f->iters;
    bool conv = true, at_centre = true;
    int sidx = 0;
    double xfin = 0.0;
    if (tid < nr) {
      sidx = f->refine_idx[tid];
      const double x = f->xs[3 * tid];
      const double lc = f->L[3 * tid];
      xfin = x;
      if (!f->rdone[tid]) {
        const double w = f->w[3 * tid], dw = f->dw[3 * tid], ddw = f->ddw[3 * tid];
        const double xm = f->xs[3 * tid + 1], wm = f->w[3 * tid + 1];
        const double xp = f->xs[3 * tid + 2], wp = f->w[3 * tid + 2];
        double lo = f->lo[sidx], hi = f->hi[sidx], wlo = f->wlo[sidx];
        bool done = false;
        auto absorb = [&](double xq, double wq) {   // shrink the bracket with an interior point
          if (!(xq > fmin(lo, hi) && xq < fmax(lo, hi))) return;
          if (wq == 0.0) {
            lo = hi = xq;
            xfin = xq;
            done = true;
          } else if ((wq > 0) == (wlo > 0)) {
            lo = xq;
            wlo = wq;
          } else {
            hi = xq;
          }
        };
        absorb(xm, wm);
        absorb(x, w);
        absorb(xp, wp);
        if (!done && (w == 0.0 || wm == 0.0 || wp == 0.0 || ((wm > 0) != (wp > 0)))) {
          done = true;   // certified: a sign change inside [x(1-d), x(1+d)]
          xfin = (w == 0.0) ? x : (wm == 0.0) ? xm : (wp == 0.0) ? xp : x;
        }
        if (!done && lo == hi) {
          done = true;
          xfin = lo;
        }
        f->lo[sidx] = lo;
        f->hi[sidx] = hi;
        f->wlo[sidx] = wlo;
        if (done) {
          f->rdone[tid] = 1;
          f->xs[3 * tid] = xfin;
          at_centre = (xfin == x);
          f->lfin[sidx] = lc;
        } else {
          const double den = 2.0 * dw * dw - w * ddw;
          double xn = (den != 0.0 && isfinite(den)) ? x - 2.0 * w * dw / den
                      : (dw != 0.0 ? x - w / dw : 0.5 * (lo + hi));
          const double a = fmin(lo, hi), b = fmax(lo, hi);
          if (!(xn > a && xn < b) || iters > 20) xn = 0.5 * (lo + hi);   // safeguard: bisect
          f->xs[3 * tid] = xn;
          f->xs[3 * tid + 1] = xn * (1.0 - kCertRel);
          f->xs[3 * tid + 2] = xn * (1.0 + kCertRel);
          conv = false;
        }
      } else {
        f->lfin[sidx] = lc;   // certified in an earlier pass: x is its root, evaluated again
      }
    }
    const int all_conv = __syncthreads_and(conv);
    const bool done = all_conv || iters + 1 >= kMaxRefinePasses;
    // every slot a refined root whose certified x is the centre point this pass
    // evaluated: L at the roots is known, the FINAL pass over Y is skipped
    const bool fused = __syncthreads_and(at_centre) && all_conv && nr == f->nslots;
    if (done) {
      if (tid < nr) f->lo[sidx] = f->xs[3 * tid];
      __syncthreads();
      if (tid < f->nslots) {
        f->xs[tid] = f->lo[tid];
        if (fused) f->L[tid] = f->lfin[tid];
      }
    }
    if (tid == 0) {
      f->iters = iters + 1;
      if (done) {
        f->npts = f->nslots;
        f->phase = PH_FINAL;
        f->converged = all_conv ? 1 : 0;
      }
    }
    __syncthreads();
    if (!fused) return;
    phase = PH_FINAL;   // the candidates' log-likelihoods from the roots' L, now
  }
  if (phase == PH_REFINE) {
    const int nr = f->nrefine, iters = f->iters;
    bool conv = true;
    double xn = 0.0;
    int sidx = 0;
    if (tid < nr) {
      sidx = f->refine_idx[tid];
      const double x = f->xs[tid], w = f->w[tid], dw = f->dw[tid];
      double lo = f->lo[sidx], hi = f->hi[sidx];
      if (w == 0.0) {
        lo = hi = x;
      } else if ((w > 0) == (f->wlo[sidx] > 0)) {
        lo = x;
        f->wlo[sidx] = w;
      } else {
        hi = x;
      }
      f->lo[sidx] = lo;
      f->hi[sidx] = hi;
      xn = (dw != 0.0) ? x - w / dw : 0.5 * (lo + hi);
      const double a = fmin(lo, hi), b = fmax(lo, hi);
      if (!(xn > a && xn < b) || iters > 20) xn = 0.5 * (lo + hi);   // safeguard: bisect
      if (lo == hi) xn = lo;
      conv = fabs(xn - x) <= 1e-13 * fabs(x);
      f->xs[tid] = xn;
    }
    const int all_conv = __syncthreads_and(conv);
    const bool done = all_conv || iters + 1 >= kMaxRefinePasses;
    if (done) {
      // every slot's root estimate is final (exact grid zeros keep lo)
      if (tid < nr) f->lo[sidx] = xn;
      __syncthreads();
      if (tid < f->nslots) f->xs[tid] = f->lo[tid];
    }
    if (tid == 0) {
      f->iters = iters + 1;
      if (done) {
        f->npts = f->nslots;
        f->phase = PH_FINAL;
        f->converged = all_conv ? 1 : 0;
      }
    }
    __syncthreads();
    return;
  }
  if (phase == PH_FINAL) {
    const double N = (double)f->nt;
    const int ns = f->nslots;
    // candidate log-likelihoods, one thread per root (kept in dw / w)
    if (tid < ns) {
      const double x = f->xs[tid];
      const double g = f->L[tid];
      double ll = -INFINITY, sg = 0.0;
      if (x != 0.0 && g != 0.0) {
        sg = g / x;
        if (sg > 0.0) ll = -N * (log(sg) + g + 1.0);
      }
      f->dw[tid] = ll;
      f->w[tid] = sg;
    }
    __syncthreads();
    if (tid == 0) {
      double bg = 0.0, bs = f->ybar, bll = -N * (log(f->ybar) + 1.0);
      int method = 1, nroots = 0;
      for (int s2 = 0; s2 < ns; ++s2) {
        const double ll = f->dw[s2];
        if (!(f->w[s2] > 0.0) || f->xs[s2] == 0.0 || f->L[s2] == 0.0) continue;
        ++nroots;
        const double g = f->L[s2];
        if (ll > bll || (ll == bll && fabs(g) < fabs(bg))) {
          bll = ll;
          bg = g;
          bs = f->w[s2];
          method = 0;
        }
      }
      const double r = f->q * (double)f->n / N;
      const double lr = log(r);
      f->gamma = bg;
      f->sigma = bs;
      f->method = method;
      f->nroots = nroots;
      f->z_q = (bg == 0.0) ? f->t - bs * lr : f->t + (bs / bg) * expm1(-bg * lr);
      f->phase = PH_DONE;
    }
    __syncthreads();
  }
}

// the fixed scan grids of R-13 (same formulas as the oracle), one point per thread
__device__ void setup_grid(FitState *f) {
  const double ymax = f->ymax, ymin = f->ymin, ybar = f->ybar;
  const double a = 1e-12 / ybar;
  const double b = 2.0 * (ybar - ymin) / (ymin * ymin);
  const int k = threadIdx.x;
  if (k < kGrid) {
    const double th = 1e-8 + k * ((1.0 - 2e-8) / (kGrid - 1));
    f->xs[k] = (-1.0 / ymax) * (1.0 - th);
  } else if (k < 2 * kGrid && b > a) {
    const double la = log(a), lb = log(b);
    f->xs[k] = exp(la + (k - kGrid) * ((lb - la) / (kGrid - 1)));
  }
  if (k == 0) {
    f->npts = (b > a) ? 2 * kGrid : kGrid;
    f->phase = PH_GRID;
    f->use_bins = 0;
    f->biters = 0;
  }
  if (f->nt >= kGrid32MinPeaks) {
    __syncthreads();
    if (k == 0) {
      // evaluation list: the fp64 points first, then the fp32 points; series
      // points are not evaluated over Y (power sums)
      const int ng = f->npts;
      int n64 = 0, n32 = 0;
      for (int g = 0; g < ng; ++g) {
        const double z = f->xs[g] * ymax;
        f->gx[g] = f->xs[g];
        f->gmode[g] = (fabs(z) <= 1e-3) ? 1 : (z < -0.9) ? 2 : 0;
        n64 += f->gmode[g] == 2;
        n32 += f->gmode[g] == 0;
      }
      int i64 = 0, i32 = n64;
      for (int g = 0; g < ng; ++g) {
        const int li = f->gmode[g] == 2 ? i64++ : f->gmode[g] == 0 ? i32++ : -1;
        f->ginv[g] = li;
        if (li >= 0) {
          f->gidx[li] = g;
          f->xs[li] = f->gx[g];
        }
      }
      f->ngrid = ng;
      f->n64 = n64;
      f->n32 = n32;
      f->npts = n64;   // PH_GRID32 evaluates the fp64 points; the rest over the bins
      f->phase = PH_GRID32;
      // bins of log2(Y) over [Ymin, Ymax]: kBinsPerOctave per octave, fewer if the
      // range spans more than kMaxBins / kBinsPerOctave octaves
      const double l0 = log2(ymin), oct = fmax(log2(ymax) - l0, 1e-9);
      double bk = kBinsPerOctave;
      if (oct * bk > (double)(kMaxBins - 2)) bk = (double)(kMaxBins - 2) / oct;
      f->bin_l0 = l0;
      f->bin_k = bk;
      f->bin_cl = 64 - __clzll((long long)f->nt);   // N_t < 2^cl
      f->use_bins = 1;
      f->nbins = min(kMaxBins, (int)ceil(oct * bk) + 1);
      // the first bin of the exactly summed high Y: bins from log2(Ymax / 2)
      f->bin_cb = (int)fmin(fmax(floor((log2(ymax) - 1.0 - l0) * bk), 0.0), (double)f->nbins);
      f->pole_hybrid = (n64 <= kMaxPole) ? 1 : 0;
    }
  }
}

// ---- fp64 kernels of the w(x) sums: reciprocal and log1p ----------------
// 1/v: MUFU seed (rcp.approx.ftz.f64) + two Newton steps (rounding-limited).
__device__ __forceinline__ double rcp_nr(double v) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
  double e = fma(-v, r, 1.0);
  r = fma(r, e, r);
  e = fma(-v, r, 1.0);
  return fma(r, e, r);
}

constexpr int kLogTab = 130;      // nodes c_i = 1 + (i - kLogOne)/181, i = 0..128 (+1 pad)
constexpr int kLogOne = 53;       // c_53 = 1 exactly: log(c) = 0, no cancellation near v = 1
constexpr double kLogStep = 181.0;
struct LogTab {
  double inv_c[kLogTab], tlog[kLogTab];   // 1/c_i and -log(1/c_i)
};
__device__ void fill_logtab(LogTab &T) {
  for (int i = threadIdx.x; i < kLogTab; i += blockDim.x) {
    const double c = 1.0 + (double)(i - kLogOne) / kLogStep;
    const double ic = 1.0 / c;
    T.inv_c[i] = ic;
    T.tlog[i] = (i == kLogOne) ? 0.0 : -log(ic);
  }
}

// log1p(u) for u > -1, given v = fl(1 + u) and iv = 1/v:
//   log1p(u) = log(v) + c/v, c = u - (v - 1) the rounding error of v (exact);
//   log(v) = e ln2 + log(c_i) + log1p(r), v = 2^e m, m in [sqrt(1/2), sqrt(2)),
//   c_i the nearest of the nodes 1 + k/181 and r = m/c_i - 1 (|r| < 2^-8,
//   degree-7 alternating series).  Near v = 1 the node is 1 itself, so r = v - 1
//   exactly and the result keeps full relative accuracy for tiny |u|.  One
//   branch-free path (about 2 ulp measured against long-double log1p).
__device__ __forceinline__ double log1p_fast(double u, double v, double iv, const LogTab &T) {
  const double c = u - (v - 1.0);
  int hi = __double2hiint(v);
  const int lo = __double2loint(v);
  int e = (hi >> 20) - 1023;
  hi = (hi & 0x000fffff) | 0x3ff00000;
  if (hi > 0x3ff6a09e) {   // m > sqrt(2): halve
    hi -= 0x00100000;
    ++e;
  }
  const double m = __hiloint2double(hi, lo);
  int idx = __double2int_rd(fma(m - 1.0, kLogStep, kLogOne + 0.5));
  idx = min(max(idx, 0), kLogTab - 2);
  const double r = fma(m, T.inv_c[idx], -1.0);
  double p = -0.125;
  p = fma(p, r, 1.0 / 7.0);
  p = fma(p, r, -1.0 / 6.0);
  p = fma(p, r, 0.2);
  p = fma(p, r, -0.25);
  p = fma(p, r, 1.0 / 3.0);
  p = fma(p, r, -0.5);
  p = fma(p, r, 1.0);
  constexpr double kLn2Hi = 6.93147180369123816490e-01, kLn2Lo = 1.90821492927058770002e-10;
  const double ed = (double)e;
  return fma(ed, kLn2Hi, T.tlog[idx]) + fma(ed, kLn2Lo, fma(p, r, c * iv));
}

// Sums over this CTA's slice of Y of P = -xY/(1+xY), L = log1p(xY) and, for
// the REFINE passes, their x-derivatives dP = -Y r^2, dL = Y r, d2P = 2 Y^2 r^3,
// d2L = -Y^2 r^2 (r = 1/(1+xY)), for up to 4 points x per warp item.
template <bool kDeriv>
__device__ __forceinline__ void eval_bundle(const double *Y, int64_t s0, int64_t s1,
                                            const double (&x)[4], int nu,
                                            double (&acc)[4][kSums], const LogTab &T) {
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int k = 0; k < kSums; ++k) acc[u][k] = 0.0;
  for (int64_t i = s0 + (threadIdx.x & 31); i < s1; i += 32) {
    const double y = Y[i];   // shared-memory copy (or global: coherent load, not .nc)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u < nu) {
        const double xy = x[u] * y;
        const double v = 1.0 + xy;
        const double r = rcp_nr(v);
        acc[u][0] -= xy * r;
        acc[u][1] += log1p_fast(xy, v, r, T);
        if (kDeriv) {
          const double yr = y * r;
          const double yr2 = yr * yr;
          acc[u][2] -= yr * r;
          acc[u][3] += yr;
          acc[u][4] = fma(2.0 * yr2, r, acc[u][4]);
          acc[u][5] -= yr2;
        }
      }
    }
  }
  constexpr int nk = kDeriv ? kSums : 2;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int k = 0; k < nk; ++k)
#pragma unroll
      for (int o = 16; o; o >>= 1) acc[u][k] += __shfl_xor_sync(0xffffffffu, acc[u][k], o);
}

// ---- the log2(Y) bins: deterministic fixed-point sums ----------------------
// Bin b of log2(Y) has the reference point r_b = 2^(l0 + (b + 1/2)/k) and keeps
// the count, sum (y - r_b) and sum (y - r_b)^2 of its values as int64 fixed point
// (integer atomics: exact and order-free, so every run -- and every rank of a
// replicated fit -- sees the same bin sums bit for bit).  |y - r_b| < 2^(E_b - 8)
// (E_b = the exponent of r_b; a bin is < 2^-9.4 r_b wide for any k >= 475, the
// smallest k a float range can need) and a bin holds <= N_t < 2^cl values, so
// the scales 2^(69 - cl - E_b) and 2^(77 - cl - 2 E_b) keep every sum below 2^61
// while quantising y - r_b at ~2^(cl - 69) of y (~4e-15 at N_t = 2M).
__device__ __forceinline__ double pow2i(int k) {   // 2^k, -1022 <= k <= 1023
  return __hiloint2double((k + 1023) << 20, 0);
}
__device__ __forceinline__ double bin_ref(double l0, double bk, int b) {
  return exp2(l0 + ((double)b + 0.5) / bk);
}
__device__ __forceinline__ int exp_of(double v) {   // unbiased exponent of a normal v > 0
  return ((__double2hiint(v) >> 20) & 0x7ff) - 1023;
}
__device__ __forceinline__ void bin_add(unsigned long long *bins, int bi, double y, double l0,
                                        double bk, int cl) {
  const double rb = bin_ref(l0, bk, bi);
  const int E = exp_of(rb);
  const double d = y - rb;   // exact (Sterbenz: y and r_b within a factor 2)
  const long long dq = __double2ll_rn(d * pow2i(69 - cl - E));
  const long long qq = __double2ll_rn((d * d) * pow2i(77 - cl - 2 * E));
  atomicAdd(bins + 3 * bi, 1ull);
  atomicAdd(bins + 3 * bi + 1, (unsigned long long)dq);
  atomicAdd(bins + 3 * bi + 2, (unsigned long long)qq);
}

// PH_GRIDBIN / PH_BREFINE: sums of the P and L terms of up to 4 points over
// this CTA's bins (lanes over bins): per bin n f(x m) + 1/2 f''(x m) x^2 S2 with m
// the bin mean and S2 = sum (y - m)^2 -- f = log1p, f'' = -1/(1+u)^2; P's term
// -u/(1+u), its second derivative 2/(1+u)^3.  kDeriv (PH_BREFINE) adds the
// x-derivatives of the sums at zeroth order in the bin spread (sum y and sum y^2
// exact, 1/(1 + x y) taken at the bin mean): they only steer the binned Halley
// steps, never a sign or a certified value.
template <bool kDeriv>
__device__ __forceinline__ void eval_bins(const unsigned long long *bins, int j0, int j1,
                                          const double (&x)[4], int nu,
                                          double (&acc)[4][kSums], const LogTab &T, double l0,
                                          double bk, int cl, unsigned pole_mask = 0u, int cb = 0) {
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int k = 0; k < kSums; ++k) acc[u][k] = 0.0;
  // this CTA's bins b = blockIdx.x + j gridDim.x, j in [j0, j1) (lanes over j)
  for (int j = j0 + (threadIdx.x & 31); j < j1; j += 32) {
    const int b = (int)blockIdx.x + j * (int)gridDim.x;
    const long long cnt = (long long)__ldcg(bins + 3 * b);
    if (cnt == 0) continue;
    const double n = (double)cnt;
    const double rb = bin_ref(l0, bk, b);
    const int E = exp_of(rb);
    const double sd = (double)(long long)__ldcg(bins + 3 * b + 1) * pow2i(E + cl - 69);
    const double qd = (double)(long long)__ldcg(bins + 3 * b + 2) * pow2i(2 * E + cl - 77);
    const double dm = sd / n;
    const double m = rb + dm;
    const double s2 = fmax(qd - sd * dm, 0.0);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u < nu && !(((pole_mask >> u) & 1u) && b >= cb)) {   // pole points: bins < cb only
        const double xm = x[u] * m;
        const double v = 1.0 + xm;
        const double r = rcp_nr(v);
        const double c2 = x[u] * x[u] * r * r * s2;   // x^2 S2 / (1 + x m)^2
        acc[u][0] = fma(n, -xm * r, fma(c2, r, acc[u][0]));
        acc[u][1] = fma(n, log1p_fast(xm, v, r, T), fma(-0.5, c2, acc[u][1]));
        if (kDeriv) {
          const double sy = n * m, sy2 = fma(n * m, m, s2);   // sum y, sum y^2
          const double r2 = r * r;
          acc[u][2] -= sy * r2;
          acc[u][3] += sy * r;
          acc[u][4] = fma(2.0 * sy2, r2 * r, acc[u][4]);
          acc[u][5] -= sy2 * r2;
        }
      }
    }
  }
  constexpr int nk = kDeriv ? kSums : 2;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int k = 0; k < nk; ++k)
#pragma unroll
      for (int o = 16; o; o >>= 1) acc[u][k] += __shfl_xor_sync(0xffffffffu, acc[u][k], o);
}

struct FitShared {
  FitState f;
  LogTab tab;
  int scratch[32];
  double sred[kMaxPts][kSums];   // per warp item partial sums [slice * npts + pt][k]
  double powp[kPotWarps][kPow];  // PH_GRID32: per-warp power sums of Y / Ymax
  double plist[kPotWarps][kPoleList];   // PH_GRID32: the warp's high Y awaiting evaluation
  double pacc[kPotWarps][kMaxPole][2];  // PH_GRID32: per-warp exact P, L sums of the pole points
  double red[kSums][kMaxPts];    // grid totals after the barrier
};

// Communicator path: the fit's Y is every rank's tail in rank order -- the
// order a single GPU's stable compaction of the concatenated scores produces,
// so the threshold is bit-identical for every world size -- built from the
// gathered fixed-size slots.  Every CTA derives the rank offsets itself and
// writes exactly the slice [c0, c1) that fit() assigns it: no grid barrier.
// Returns N_t (> cap if any rank overflowed its slot: ENOVA_ERR_WORKSPACE).
__device__ int64_t pack_tails(const PotArgs &a, long long *s_off) {
  if (threadIdx.x == 0) {
    long long o = 0;
    bool bad = false;
    for (int r = 0; r < a.world; ++r) {
      const long long c = *(volatile const long long *)(a.counts_all + r);
      s_off[r] = o;
      bad = bad || c > a.cap || c < 0;
      o += bad ? 0 : c;
    }
    s_off[a.world] = (bad || o > a.cap) ? a.cap + 1 : o;
  }
  __syncthreads();
  const int64_t nt = s_off[a.world];
  if (blockIdx.x == 0 && threadIdx.x == 0) a.g->nt_fit = nt;
  if (nt < 10 || nt > a.cap) return nt;
  const int nb = gridDim.x;
  const int64_t chunk = (nt + nb - 1) / nb;
  const int64_t c0 = min(nt, (int64_t)blockIdx.x * chunk), c1 = min(nt, c0 + chunk);
  const double td = (double)*(volatile float *)&a.g->t;
  double *Y = const_cast<double *>(a.yfit);
  for (int r = 0; r < a.world; ++r) {
    const int64_t lo = max(c0, (int64_t)s_off[r]), hi = min(c1, (int64_t)s_off[r + 1]);
    const float *src = a.yslot + (size_t)r * (size_t)a.cap;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
      Y[i] = (double)src[i - s_off[r]] - td;
  }
  __syncthreads();
  return nt;
}

// ---- the fit's building blocks (shared by the one-launch fit and the
// distributed per-pass launches) ----

// this CTA's slice [c0, c1) of a tail of nt values
__device__ __forceinline__ void fit_slice(int64_t nt, int64_t &c0, int64_t &c1) {
  const int nb = gridDim.x;
  const int64_t chunk = (nt + nb - 1) / nb;
  c0 = min(nt, (int64_t)blockIdx.x * chunk);
  c1 = min(nt, c0 + chunk);
}

// Y statistics of this CTA's slice -> partial buffer rows 0..2 (sum, min, max);
// stages the slice in shared memory when it fits.  src = the fp64 tail.
__device__ void fit_stats_partials(const PotArgs &a, FitShared &S, const double *src, int64_t c0,
                                   int64_t c1, bool cached, double *ycache) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s = 0.0, mn = INFINITY, mx = -INFINITY;
  for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
    const double y = src[i];   // written by this kernel / launch: coherent load
    if (cached) ycache[i - c0] = y;
    s += y;
    mn = fmin(mn, y);
    mx = fmax(mx, y);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    S.sred[warp][0] = s;
    S.sred[warp][1] = mn;
    S.sred[warp][2] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ts = 0.0, tmn = INFINITY, tmx = -INFINITY;
    for (int w = 0; w < kPotWarps; ++w) {
      ts += S.sred[w][0];
      tmn = fmin(tmn, S.sred[w][1]);
      tmx = fmax(tmx, S.sred[w][2]);
    }
    a.part[0 * kMaxCtas + blockIdx.x] = ts;
    a.part[1 * kMaxCtas + blockIdx.x] = tmn;
    a.part[2 * kMaxCtas + blockIdx.x] = tmx;
  }
}

// the binned grid pass's histogram starts empty: every CTA zeroes its slice
// (first written after the next grid barrier)
__device__ __forceinline__ void zero_bins(unsigned long long *bins) {
  if (!bins) return;
  const int n = kMaxBins * 3;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    bins[i] = 0ull;
}

// grid totals of the statistics partials (fixed order; warp 0 of every CTA)
__device__ void fit_stats_totals(const PotArgs &a, double &ts, double &tmn, double &tmx) {
  const int lane = threadIdx.x & 31, nb = gridDim.x;
  ts = 0.0;
  tmn = INFINITY;
  tmx = -INFINITY;
  for (int b = lane; b < nb; b += 32) {
    ts += *(volatile double *)(a.part + b);
    tmn = fmin(tmn, *(volatile double *)(a.part + kMaxCtas + b));
    tmx = fmax(tmx, *(volatile double *)(a.part + 2 * kMaxCtas + b));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    ts += __shfl_xor_sync(0xffffffffu, ts, o);
    tmn = fmin(tmn, __shfl_xor_sync(0xffffffffu, tmn, o));
    tmx = fmax(tmx, __shfl_xor_sync(0xffffffffu, tmx, o));
  }
}

// one evaluation pass over this CTA's slice at the points of f (list order):
// CTA partials per (k, point) -> pw ([kSums][kMaxPts][kMaxCtas])
__device__ void fit_eval_partials(FitShared &S, const double *Y, int64_t c0, int64_t c1,
                                  double *pw, unsigned long long *bins) {
  FitState &f = S.f;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int phase = f.phase;
  const int npts = f.npts;
  const bool deriv = (phase == PH_REFINE);
  const bool mixed = (phase == PH_GRID32);
  const bool binned = (phase == PH_GRIDBIN || phase == PH_BREFINE);
  const int nk = phase_sums(phase);
  // PH_GRIDBIN: the list points over this CTA's slice of the bins, not over Y
  // (bins dealt round-robin: CTA b takes bins b, b + grid, ... -- the occupied
  // bins cluster in a few octaves, so contiguous slices left most CTAs idle)
  if (binned) {
    c0 = 0;
    c1 = (f.nbins - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  }
  // bundles of 4 list points (PH_GRID32: the fp64 points; the rest of the grid
  // is evaluated over the bins).  Warp items = (bundle, Y slice); the points are
  // spread evenly over the bundles (a refine pass's 6 points: 3 + 3, not 4 + 2)
  // (PH_GRID32 with hybrid pole points: no warp items -- the pole points' exact
  // high-Y part is summed in the mixed loop below)
  const bool hybrid = mixed && f.pole_hybrid;
#ifndef ENOVA_AB_NOPOLE   // diagnostic A/B only (results invalid without the pole points)
  const int n64 = mixed ? (hybrid ? 0 : f.n64) : npts;
#else
  const int n64 = mixed ? 0 : npts;
#endif
  const int nA = (n64 + 3) / 4;
  const int sA = (nA >= kPotWarps) ? 1 : kPotWarps / max(nA, 1);
  const int items = nA * sA;
  for (int it = warp; it < items; it += kPotWarps) {
    const int bnd = it % nA, sl = it / nA;
    const int slices = sA;
    const int64_t len = c1 - c0;
    const int64_t s0 = c0 + len * sl / slices, s1 = c0 + len * (sl + 1) / slices;
    const int base = bnd * n64 / nA, nu = (bnd + 1) * n64 / nA - base;
    double x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = (u < nu) ? f.xs[base + u] : 0.0;
    double acc[4][kSums];
    if (deriv)
      eval_bundle<true>(Y, s0, s1, x, nu, acc, S.tab);
    else if (phase == PH_BREFINE)
      eval_bins<true>(bins, (int)s0, (int)s1, x, nu, acc, S.tab, f.bin_l0, f.bin_k, f.bin_cl);
    else if (binned) {
      unsigned pm = 0u;   // PH_GRIDBIN list points that are hybrid pole points
      for (int u = 0; u < nu; ++u) pm |= (f.gmode[f.gidx[base + u]] == 4 ? 1u : 0u) << u;
      eval_bins<false>(bins, (int)s0, (int)s1, x, nu, acc, S.tab, f.bin_l0, f.bin_k, f.bin_cl,
                       pm, f.bin_cb);
    }
    else
      eval_bundle<false>(Y, s0, s1, x, nu, acc, S.tab);
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (u < nu)
#pragma unroll
          for (int k = 0; k < kSums; ++k) S.sred[sl * npts + base + u][k] = acc[u][k];
    }
  }
  if (mixed) {   // power sums of u = Y / Ymax for the series points (fp64, fixed order)
                 // and the bins of log2(Y) for PH_GRIDBIN (count, sum, sum of squares)
    const double iy = 1.0 / f.ymax;
    const float l0f = (float)f.bin_l0, bkf = (float)f.bin_k;
    const int nbn = f.nbins;
    double q[kPow];
#pragma unroll
    for (int m = 0; m < kPow; ++m) q[m] = 0.0;
    const int np = hybrid ? f.n64 : 0, cb = f.bin_cb;
    const unsigned lt = (1u << lane) - 1u;
    for (int i = lane; i < 2 * kMaxPole; i += 32) (&S.pacc[warp][0][0])[i] = 0.0;
    __syncwarp();
    double *lst = S.plist[warp];
    int cnt = 0;   // warp-uniform: high Y in the warp's list
    // the list's contributions to every pole point (list order; lanes over items,
    // fixed xor tree, added to the warp's sums in flush order)
    auto flush = [&]() {
      for (int u = 0; u < np; ++u) {
        const double x = f.xs[u];
        double aP = 0.0, aL = 0.0;
        for (int j = lane; j < cnt; j += 32) {
          const double yv = lst[j];
          const double xy = x * yv, v = 1.0 + xy, r = rcp_nr(v);
          aP -= xy * r;
          aL += log1p_fast(xy, v, r, S.tab);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          aP += __shfl_xor_sync(0xffffffffu, aP, o);
          aL += __shfl_xor_sync(0xffffffffu, aL, o);
        }
        if (lane == 0) {
          S.pacc[warp][u][0] += aP;
          S.pacc[warp][u][1] += aL;
        }
      }
      __syncwarp();
      cnt = 0;
    };
    // thread (warp, lane) takes i = c0 + tid + k blockDim as before (power-sum order
    // unchanged); the warp-uniform trip count lets the warp ballot its high Y
    for (int64_t i0 = c0 + (int64_t)warp * 32; i0 < c1; i0 += blockDim.x) {
      const int64_t i = i0 + lane;
      const bool ok = i < c1;
      const double y = ok ? Y[i] : 0.0;
      int bi = -1;
      if (ok) {
        const double u = y * iy;
        double pw_ = u;
#pragma unroll
        for (int m = 0; m < kPow; ++m) {
          q[m] += pw_;
          pw_ *= u;
        }
        float lg;
        asm("lg2.approx.f32 %0, %1;" : "=f"(lg) : "f"((float)y));
        bi = min(max(__float2int_rd((lg - l0f) * bkf), 0), nbn - 1);
#ifndef ENOVA_AB_NOBIN   // diagnostic A/B only (results invalid without the bins)
        bin_add(bins, bi, y, f.bin_l0, f.bin_k, f.bin_cl);
#else
        if (bi == -7) bin_add(bins, bi, y, f.bin_l0, f.bin_k, f.bin_cl);
#endif
      }
      const bool hi = np > 0 && bi >= cb;
      const unsigned bal = __ballot_sync(0xffffffffu, hi);
      if (bal) {
        if (cnt + 32 > kPoleList) flush();
        if (hi) lst[cnt + __popc(bal & lt)] = y;
        __syncwarp();
        cnt += __popc(bal);
      }
    }
    if (cnt) flush();
#pragma unroll
    for (int m = 0; m < kPow; ++m) {
#pragma unroll
      for (int o = 16; o; o >>= 1) q[m] += __shfl_xor_sync(0xffffffffu, q[m], o);
      if (lane == 0) S.powp[warp][m] = q[m];
    }
  }
  __syncthreads();
  if (mixed && threadIdx.x < kPow) {   // CTA partial power sums -> partial row 2
    double sp = 0.0;
    for (int w = 0; w < kPotWarps; ++w) sp += S.powp[w][threadIdx.x];
    pw[((size_t)2 * kMaxPts + threadIdx.x) * kMaxCtas + blockIdx.x] = sp;
  }
  // CTA partial per (k, point): slices summed in order (hybrid PH_GRID32: the
  // pole points' exact high-Y sums, warps summed in order)
  for (int i = threadIdx.x; i < nk * npts; i += blockDim.x) {
    const int k = i / npts, pt = i % npts;
    double s = 0.0;
    if (hybrid) {
      for (int w = 0; w < kPotWarps; ++w) s += S.pacc[w][pt][k];
    } else {
      for (int sl = 0; sl < sA; ++sl) s += S.sred[sl * npts + pt][k];
    }
    pw[((size_t)k * kMaxPts + pt) * kMaxCtas + blockIdx.x] = s;
  }
}

// grid totals of one pass (after the barrier), fixed order: one warp per
// (k, point), 4 items in flight per warp -> S.red
__device__ void fit_eval_totals(FitShared &S, const double *pw) {
  FitState &f = S.f;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nb = gridDim.x;
  const int npts = f.npts;
  const bool mixed = (f.phase == PH_GRID32);
  const int nk = phase_sums(f.phase);
  constexpr int kJ = (kMaxCtas + 31) / 32;
  const int nitems = nk * npts + (mixed ? kPow : 0);   // + the power sums (row 2)
  for (int i0 = 4 * warp; i0 < nitems; i0 += 4 * kPotWarps) {
    double v[4][kJ];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + q;
      const bool extra = i >= nk * npts;
      const int k = extra ? 2 : i / npts, pt = extra ? i - nk * npts : i % npts;
      const double *src = pw + ((size_t)k * kMaxPts + pt) * kMaxCtas;
#pragma unroll
      for (int j = 0; j < kJ; ++j) {
        const int b = lane + 32 * j;
        v[q][j] = (i < nitems && b < nb) ? *(volatile const double *)(src + b) : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double sum = 0.0;
#pragma unroll
      for (int j = 0; j < kJ; ++j) sum += v[q][j];
#pragma unroll
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const int i = i0 + q;
      if (lane == 0 && i < nitems) {
        if (i >= nk * npts) S.red[2][i - nk * npts] = sum;
        else S.red[i / npts][i % npts] = sum;
      }
    }
  }
}

// means of the pass totals in S.red -> w (and derivatives) at the list points,
// then the controller (next points, roots, candidates, z_q)
__device__ void fit_finish_pass(FitShared &S) {
  FitState &f = S.f;
  const int npts = f.npts;
  const bool deriv = phase_sums(f.phase) == kSums;
  const bool mixed = (f.phase == PH_GRID32);
  const double N = (double)f.nt;
  if (threadIdx.x < npts) {
    const int pt = threadIdx.x;
    const double Pm = S.red[0][pt] / N, Lm = S.red[1][pt] / N;
    f.w[pt] = Pm + Lm + Pm * Lm;
    f.L[pt] = Lm;
    f.P[pt] = Pm;
    if (deriv) {
      const double dPm = S.red[2][pt] / N, dLm = S.red[3][pt] / N;
      const double d2Pm = S.red[4][pt] / N, d2Lm = S.red[5][pt] / N;
      f.dw[pt] = dPm + dLm + dPm * Lm + Pm * dLm;
      f.ddw[pt] = d2Pm + d2Lm + d2Pm * Lm + 2.0 * dPm * dLm + Pm * d2Lm;
    }
  }
  if (mixed && threadIdx.x == 0)
    for (int m = 1; m <= kPow; ++m) f.pm[m] = S.red[2][m - 1] / N;   // mean u^m
  __syncthreads();
  controller(&f, S.scratch);
}

// the fit's result -> PotGlobal (CTA 0, thread 0)
__device__ void fit_publish(const PotArgs &a, const FitState &f) {
  PotGlobal *g = a.g;
#ifdef ENOVA_FIT_STAMPS   // diagnostic: the binned Halley steps into the stamp slots 72..88
  for (int i = 0; i < kMaxBinRefine * 4; ++i)
    g->stamps[72 + i] = (unsigned long long)__double_as_longlong((&f.bdiag[0][0])[i]);
  g->stamps[88] = (unsigned long long)f.bdiag_nr;
#endif
  g->gamma = f.gamma;
  g->sigma = f.sigma;
  g->z_q = f.z_q;
  g->method = f.method;
  g->nroots = f.nroots;
  g->overflow = f.overflow;
  g->converged = f.converged;
  g->fit_passes = f.iters;
  int st = ENOVA_OK;
  if (f.overflow) st = ENOVA_ERR_UNSUPPORTED;
  else if (!f.converged) st = ENOVA_ERR_UNSUPPORTED;
  g->status = st;
}

// f's run-wide fields from the Y statistics
__device__ void fit_init_state(const PotArgs &a, FitState &f, int64_t nt, double ts, double tmn,
                               double tmx) {
  f.nt = nt;
  f.n = a.n_dev ? *(volatile const long long *)a.n_dev : a.n;
  f.t = (double)*(volatile float *)&a.g->t;
  f.q = a.q;
  f.overflow = 0;
  f.converged = 0;
  f.iters = 0;
  f.phase = PH_GRID;
  f.ybar = ts / (double)nt;
  f.ymin = tmn;
  f.ymax = tmx;
}

__device__ void fit(const PotArgs &a, FitShared &S, unsigned int &epoch, const int64_t nt) {
  FitState &f = S.f;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (nt < 10 || nt > a.cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
      a.g->status = (nt < 10) ? ENOVA_ERR_TOO_FEW_EXCEEDANCES : ENOVA_ERR_WORKSPACE;
    return;   // uniform over the grid
  }
  int64_t c0, c1;
  fit_slice(nt, c0, c1);
  // this CTA's slice of Y is staged in shared memory by the Y-statistics pass
  // (every later pass reads it from there); global reads if it does not fit
  extern __shared__ double ycache[];
  const bool cached = (c1 - c0) <= (int64_t)a.ycache_cap;
  const double *Y = cached ? (const double *)ycache - c0 : a.yfit;
  fill_logtab(S.tab);   // first read after the next barrier

  // ---- Ybar, Ymin, Ymax (pass 0, partial buffer 0) ----
  fit_stats_partials(a, S, a.yfit, c0, c1, cached, ycache);
  if (nt >= kGrid32MinPeaks) zero_bins(a.bins);
  grid_sync(a.g, epoch);
  stamp(a.g);
  if (warp == 0) {
    double ts, tmn, tmx;
    fit_stats_totals(a, ts, tmn, tmx);
    if (lane == 0) fit_init_state(a, f, nt, ts, tmn, tmx);
  }
  __syncthreads();
  setup_grid(&f);
  __syncthreads();

  // ---- evaluation passes (partials double-buffered: one barrier per pass) ----
  for (int pass = 1;; ++pass) {
    if (f.phase == PH_DONE) break;
    double *pw = a.part + (size_t)(pass & 1) * kSums * kMaxPts * kMaxCtas;
    fit_eval_partials(S, Y, c0, c1, pw, a.bins);
    stamp(a.g);
    grid_sync(a.g, epoch);
    stamp(a.g);
    fit_eval_totals(S, pw);
    __syncthreads();
#ifdef ENOVA_FIT_STAMPS
    stamp(a.g);
#endif
    fit_finish_pass(S);
#ifdef ENOVA_FIT_STAMPS
    stamp(a.g);
#endif
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) fit_publish(a, f);
}

// ---- distributed fit (SURVEY §8e "distributed-fit variant") ----
// Each rank fits on its OWN tail only: one launch per evaluation pass; between
// launches the ranks' pass totals (this rank's CTA partials summed in CTA
// order) are all-gathered and every rank sums them in rank order, so every
// rank sees the same totals, runs the same controller and ends with the same
// z_q (bit-identical across ranks; across world sizes equal up to the fp64
// summation order, like the replicated fit across grid sizes).
//   step 0: this rank's Y = raw tail - t (fp64), its statistics -> xsend
//   step s >= 1: combine the gathered totals (stats at s = 1), finish the pass
//   (controller), evaluate the next pass over the local tail -> xsend
// f persists in global memory between launches (CTA 0 stores, all CTAs load).
constexpr int kDfitLen = kSums * kMaxPts;   // doubles per rank per exchange

__device__ void fstate_copy(FitState *dst, const FitState *src) {
  const int n = (int)(sizeof(FitState) / 8);
  const long long *s = reinterpret_cast<const long long *>(src);
  long long *d = reinterpret_cast<long long *>(dst);
  for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = *(volatile const long long *)(s + i);
}

__device__ void dfit_step(const PotArgs &a, FitShared &S, unsigned int &epoch) {
  FitState &f = S.f;
  PotGlobal *g = a.g;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ntl = *(volatile long long *)&g->nt_local;   // this rank's peaks
  int64_t c0, c1;
  fit_slice(ntl, c0, c1);
  extern __shared__ double ycache[];
  const bool cached = (c1 - c0) <= (int64_t)a.ycache_cap;
  double *Yl = a.ydst;   // this rank's fp64 tail
  if (a.dfit_step == 0) {
    const double td = (double)*(volatile float *)&g->t;
    for (int64_t i = c0 + threadIdx.x; i < c1 && ntl <= a.cap; i += blockDim.x)
      Yl[i] = (double)a.ylocal[i] - td;
    __syncthreads();
    fit_stats_partials(a, S, Yl, c0, c1, false, ycache);
    zero_bins(a.bins);
    grid_sync(g, epoch);
    if (blockIdx.x == 0 && warp == 0) {
      double ts, tmn, tmx;
      fit_stats_totals(a, ts, tmn, tmx);
      if (lane == 0) {
        a.xsend[0] = ts;
        a.xsend[1] = tmn;
        a.xsend[2] = tmx;
        a.xsend[3] = (double)ntl;
      }
    }
    return;
  }
  // ---- s >= 1: the gathered totals of the previous exchange ----
  if (a.dfit_step == 1) {
    if (threadIdx.x == 0) {
      double ts = 0.0, tmn = INFINITY, tmx = -INFINITY;
      long long nt = 0;
      bool over = false;   // a rank's tail overflowed its workspace (same on every rank)
      for (int r = 0; r < a.world; ++r) {   // rank order
        const double *x = a.xrecv + (size_t)r * kDfitLen;
        ts += x[0];
        tmn = fmin(tmn, x[1]);
        tmx = fmax(tmx, x[2]);
        nt += (long long)x[3];
        over = over || x[3] > (double)a.cap;
      }
      f.nt = over ? 0 : nt;
      if (!over && nt >= 10) fit_init_state(a, f, nt, ts, tmn, tmx);
      else f.phase = PH_DONE;
      if (blockIdx.x == 0) {
        g->nt_fit = nt;
        if (f.nt < 10) g->status = over ? ENOVA_ERR_WORKSPACE : ENOVA_ERR_TOO_FEW_EXCEEDANCES;
      }
    }
    __syncthreads();
    if (f.nt < 10) {
      if (blockIdx.x == 0) {   // later steps see PH_DONE
        const int n = (int)(sizeof(FitState) / 8);
        const long long *src = reinterpret_cast<const long long *>(&f);
        long long *dst = reinterpret_cast<long long *>(a.fstate);
        for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
      }
      return;
    }
    fill_logtab(S.tab);
    setup_grid(&f);
    __syncthreads();
  } else {
    fstate_copy(&f, a.fstate);
    __syncthreads();
    if (f.phase == PH_DONE || f.nt < 10) return;   // converged in an earlier step
    fill_logtab(S.tab);
    // S.red = the ranks' pass totals summed in rank order
    const int npts = f.npts;
    const bool mixed = (f.phase == PH_GRID32);
    const int nk = phase_sums(f.phase);
    for (int i = threadIdx.x; i < nk * npts + (mixed ? kPow : 0); i += blockDim.x) {
      const bool extra = i >= nk * npts;
      const int k = extra ? 2 : i / npts, pt = extra ? i - nk * npts : i % npts;
      double sum = 0.0;
      for (int r = 0; r < a.world; ++r) sum += a.xrecv[(size_t)r * kDfitLen + k * kMaxPts + pt];
      S.red[k][pt] = sum;
    }
    __syncthreads();
    fit_finish_pass(S);
    __syncthreads();
  }
  if (f.phase == PH_DONE) {
    if (blockIdx.x == 0 && threadIdx.x == 0) fit_publish(a, f);
  } else {
    // the next pass over this rank's tail
    const double *Y = Yl;
    if (cached) {
      for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) ycache[i - c0] = Yl[i];
      Y = (const double *)ycache - c0;
    }
    __syncthreads();
    double *pw = a.part;
    fit_eval_partials(S, Y, c0, c1, pw, a.bins);
    grid_sync(g, epoch);
    if (blockIdx.x == 0) {
      fit_eval_totals(S, pw);
      __syncthreads();
      const int npts = f.npts;
      const bool mixed = (f.phase == PH_GRID32);
      const int nk = phase_sums(f.phase);
      for (int i = threadIdx.x; i < nk * npts + (mixed ? kPow : 0); i += blockDim.x) {
        const bool extra = i >= nk * npts;
        const int k = extra ? 2 : i / npts, pt = extra ? i - nk * npts : i % npts;
        a.xsend[k * kMaxPts + pt] = S.red[k][pt];
      }
      if (a.dfit_last && threadIdx.x == 0) g->status = ENOVA_ERR_UNSUPPORTED;   // not converged
    }
  }
  if (blockIdx.x == 0) {   // the state the next step finishes from
    __syncthreads();
    const int n = (int)(sizeof(FitState) / 8);
    const long long *src = reinterpret_cast<const long long *>(&f);
    long long *dst = reinterpret_cast<long long *>(a.fstate);
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  }
}

union PotShared {
  struct {
    unsigned int h[kBins];
    unsigned int sk[kSampleN];   // P_SAMPLE: this CTA's sample keys
  } s;
  FitShared fit;
};

__global__ void __launch_bounds__(kPotThreads, 1) k_pot(PotArgs a) {
  __shared__ PotShared sh;
  __shared__ SelS sel;
  __shared__ unsigned long long wtot[kPotWarps];
  __shared__ long long found[2];
  __shared__ long long cta_base[2];
  __shared__ int wcnt[4 * kPotWarps];
  __shared__ int above;
  __shared__ long long s_off[kMaxWorld + 1];
  __shared__ SelS ssel;            // sampled selection state
  __shared__ long long s_tot[2];
  __shared__ int cmode;            // 1: the radix passes run on the candidates
  __shared__ long long my_n[2];    // this CTA's candidates / keys below lo
  PotGlobal *g = a.g;
  unsigned int epoch = 0;   // grid barriers passed in this launch
  bool spot_skip = false;
  bool spot_full = false;   // SPOT refit on a truncated peak set: report, do not fit
  if (threadIdx.x == 0) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (blockIdx.x == 0) {
      g->stamps[kMaxStamps - 1] = t0;
      s_nstamp = g->n_stamps;
    }
    atomicMax(&g->t_first_start, ~t0);   // stored complemented: max(~t) = ~min(t)
  }
  if (threadIdx.x == 0) {
    cmode = 0;
    if (a.first <= P_HIST0) {
      sel.prefix = 0;
      sel.mask = 0;
      sel.k_rem = a.k;
      sel.t = 0.f;
    } else {
      sel.prefix = g->prefix;
      sel.mask = g->mask;
      sel.k_rem = g->k_rem;
      sel.t = g->t;
    }
  }
  __syncthreads();
  // the slice the radix passes and the compaction read: this CTA's candidate
  // segment (sampled selection) or its chunk of the scores
  const int64_t seg_cap = a.cand ? ((a.n_local + gridDim.x - 1) / gridDim.x + 3) / 4 * 4 : 0;
  auto slice = [&](const float *&src, int64_t &len) {
    if (cmode) {
      src = a.cand + (size_t)blockIdx.x * seg_cap;
      len = my_n[0];
    } else {
      int64_t b0, b1;
      score_chunk(a.n_local, &b0, &b1);
      src = a.scores + b0;
      len = b1 - b0;
    }
  };
  for (int ph = a.first; ph <= a.last; ++ph) {
    if (ph > a.first) grid_sync(g, epoch);
    stamp(g);
    if (ph == P_SAMPLE) {
      int ns = 0;
      sample_phase(a, ssel, sh.s.h, sh.s.sk, ns, wtot, reinterpret_cast<int *>(found), epoch, s_tot);
      if (blockIdx.x == 0 && threadIdx.x == 0) g->sample_lo = ssel.prefix;
    } else if (ph == P_SCAN) {
      // the candidates were compacted by k_pot_scan (previous launch): this
      // CTA's counts
      if (threadIdx.x == 0) {
        my_n[0] = *(volatile long long *)(a.cand_n + blockIdx.x);
        my_n[1] = *(volatile long long *)(a.cand_n + kMaxCtas + blockIdx.x);
      }
      // every CTA: keys below lo over the grid (fixed order) -> candidate mode
      // iff the k-th order statistic is among the candidates
      if (threadIdx.x == 0) {
        long long below = 0;
        for (int b = 0; b < (int)gridDim.x; ++b)
          below += *(volatile long long *)(a.cand_n + kMaxCtas + b);
        cmode = (unsigned long long)below <= a.k ? 1 : 0;
        if (cmode) sel.k_rem = a.k - (unsigned long long)below;
        if (blockIdx.x == 0) g->sampled = cmode;
      }
      __syncthreads();
      // P_HIST0 follows without a barrier of its own: it reads only this CTA's
      // segment (written above) and its histogram was zeroed by the header memset
      ph = P_HIST0;
      const float *src;
      int64_t len;
      slice(src, len);
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * kBins; i += gridDim.x * blockDim.x)
        a.hist[kBins + i] = 0ull;
      hist_pass(a, sel, 0, sh.s.h, &above, src, len);
    } else if (ph == P_HIST0) {
      // zero what is not covered by the per-call header memset (first used
      // after the next barrier)
      unsigned long long *h12 = a.hist + kBins;
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * kBins;
           i += gridDim.x * blockDim.x)
        h12[i] = 0ull;
      const float *src;
      int64_t len;
      slice(src, len);
      hist_pass(a, sel, 0, sh.s.h, &above, src, len);
    } else if (ph == P_HIST1 || ph == P_HIST2) {
      const float *src;
      int64_t len;
      slice(src, len);
      select_digit(a, sel, ph - P_HIST1, wtot, reinterpret_cast<int *>(found));
      hist_pass(a, sel, ph - P_HIST0, sh.s.h, &above, src, len);
    } else if (ph == P_COMPACT) {
      const float *src;
      int64_t len;
      slice(src, len);
      select_digit(a, sel, 2, wtot, reinterpret_cast<int *>(found));
      compact(a, sel, sh.s.h, above, a.first < P_COMPACT, wcnt, cta_base, epoch, src, len);
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        g->t = sel.t;
        g->nt_local = cta_base[1];
        g->nt_fit = cta_base[1];
        if (cta_base[1] > a.cap) g->status = ENOVA_ERR_WORKSPACE;
      }
    } else if (ph == P_FIT) {
      if (blockIdx.x == 0 && threadIdx.x == 0) g->fit_stamp = s_nstamp - 1;
      // SPOT refit with no peak added since the last fit: the model is unchanged
      // (the cited Algorithm 1 refits only when a peak arrives) -- keep the threshold
      spot_full = a.n_dev && *(volatile int *)&g->spot_overflow != 0;
      spot_skip = !spot_full && a.n_dev &&
                  *(volatile long long *)&g->nt_fit == *(volatile long long *)&g->nt_refit;
      if (!spot_skip && !spot_full) {
        if (a.dfit_step >= 0) {
          dfit_step(a, sh.fit, epoch);
        } else {
          const int64_t nt = a.yslot ? pack_tails(a, s_off)
                                     : (int64_t)*(volatile long long *)&g->nt_fit;
          fit(a, sh.fit, epoch, nt);
        }
      }
    }
  }
  stamp(g);
  if (threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    atomicMax(&g->t_last_end, t1);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    g->n_stamps = s_nstamp;
    if (a.last < P_COMPACT) {
      g->prefix = sel.prefix;
      g->mask = sel.mask;
      g->k_rem = sel.k_rem;
    }
    if (a.last == P_FIT && !a.n_dev) g->n_spot = a.n;   // SPOT state starts at the calibration
    if (a.last == P_FIT && !spot_skip && !spot_full) g->nt_refit = g->nt_fit;
    if (spot_full) g->status = ENOVA_ERR_WORKSPACE;
    if (a.last == P_FIT && a.out_dev && !spot_skip) {
      enova_threshold *o = a.out_dev;
      const int st = g->status;
      o->init_quantile = a.q0;
      o->risk_q = a.q;
      o->t = (double)g->t;
      o->gamma = g->gamma;
      o->sigma = g->sigma;
      o->z_q = (st == ENOVA_OK) ? g->z_q : __longlong_as_double(0x7ff8000000000000ll);
      o->n = a.n_dev ? *(volatile const long long *)a.n_dev : a.n;
      o->n_peaks = g->nt_fit;
      o->method = g->method;
      o->reserved = st;
    }
  }
}

// ------------------------------------------------------------- driver ----
constexpr int kMaxYCacheBytes = 160 * 1024;

// Grid of the next fits (0 = one CTA per SM) and their cluster size: the step
// orchestration (step.cu) runs a reduced fit grid next to the detection scores.
// The result depends on the grid only through the fit's summation order
// (deterministic for a given grid, within the parity tolerance of any other).
static thread_local int g_pot_ctas = 0, g_pot_cluster = 0;
void set_pot_grid(int ctas, int cluster) {
  g_pot_ctas = ctas;
  g_pot_cluster = cluster;
}

static enova_status launch_pot(const PotArgs &a, int nb, cudaStream_t st, bool reset_barrier = false) {
  if (a.first == P_SAMPLE && a.last > P_SAMPLE) {
    // sampled selection: sampling launch -> k_pot_scan -> selection + fit launch
    PotArgs s1 = a;
    s1.last = P_SAMPLE;
    enova_status r = launch_pot(s1, nb, st, reset_barrier);
    if (r) return r;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb);
    cfg.blockDim = dim3(kPotThreads);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    if (g_pot_cluster > 1 && nb % g_pot_cluster == 0) {
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)g_pot_cluster;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
    }
    static bool scan_attr[64] = {};
    int dv = 0;
    ENOVA_CUDA_TRY(cudaGetDevice(&dv));
    if (dv < 0 || dv >= 64 || !scan_attr[dv]) {
      ENOVA_CUDA_TRY(cudaFuncSetAttribute((const void *)k_pot_scan,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          kScanStageBytes));
      ENOVA_CUDA_TRY(cudaFuncSetAttribute((const void *)k_pot_scan,
                                          cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      if (dv >= 0 && dv < 64) scan_attr[dv] = true;
    }
    cfg.dynamicSmemBytes = kScanStageBytes;
    count_launch();
    ENOVA_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_pot_scan, a));
    PotArgs s3 = a;
    s3.first = P_SCAN;
    return launch_pot(s3, nb, st, true);
  }
  PotArgs c = a;
  static bool attr_set[64] = {};   // per device (function attributes are per context)
  int dev = 0;
  ENOVA_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    ENOVA_CUDA_TRY(cudaFuncSetAttribute((const void *)k_pot,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        kMaxYCacheBytes));
    // a reduced fit grid may be ONE cluster of up to 16 CTAs (grid_sync)
    ENOVA_CUDA_TRY(cudaFuncSetAttribute((const void *)k_pot,
                                        cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  // the fit partitions N_t <= cap peaks into nb contiguous slices
  const int64_t per_cta = (a.cap + nb - 1) / nb;
  const int64_t cap_vals = per_cta < kMaxYCacheBytes / 8 ? per_cta : kMaxYCacheBytes / 8;
  c.ycache_cap = (int)cap_vals;
  size_t dyn = (a.first <= P_FIT && a.last >= P_FIT) ? (size_t)cap_vals * 8 : 0;
  if (dyn == 0) c.ycache_cap = 0;
  if (reset_barrier) ENOVA_CUDA_TRY(cudaMemsetAsync(&a.g->bar_count, 0, sizeof(unsigned int), st));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb);
  cfg.blockDim = dim3(kPotThreads);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  int na = 1;
  if (g_pot_cluster > 1 && nb % g_pot_cluster == 0) {
    // whole TPCs: the CTAs of a reduced fit grid take SM pairs, so a concurrent
    // CTA-pair score launch keeps every other TPC
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = (unsigned)g_pot_cluster;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    na = 2;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  count_launch();
  ENOVA_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_pot, c));
  return ENOVA_OK;
}

static int pot_grid() {
  if (g_pot_ctas > 0) return g_pot_ctas < kMaxCtas ? g_pot_ctas : kMaxCtas;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms < kMaxCtas ? sms : kMaxCtas;
}

static PotArgs make_args(const float *scores, int64_t n_local, int64_t n, double q0, double q,
                         char *b, const ThrLayout &L, bool comm) {
  PotArgs a;
  a.scores = scores;
  a.n_local = n_local;
  a.n = n;
  a.k = (unsigned long long)floor(q0 * (double)n);
  a.q = q;
  a.q0 = q0;
  a.g = reinterpret_cast<PotGlobal *>(b + L.glob);
  a.hist = reinterpret_cast<unsigned long long *>(b + L.hist);
  a.counts = reinterpret_cast<long long *>(b + L.counts);
  a.part = reinterpret_cast<double *>(b + L.part);
  a.ydst = reinterpret_cast<double *>(b + L.yall);
  a.yfit = reinterpret_cast<const double *>(b + L.yall);
  a.ylocal = comm ? reinterpret_cast<float *>(b + L.ylocal) : nullptr;
  a.yslot = comm ? reinterpret_cast<const float *>(b + L.yslot) : nullptr;
  a.counts_all = comm ? reinterpret_cast<const long long *>(b + L.counts_all) : nullptr;
  a.world = 0;
  a.cap = L.cap;
  a.shist = reinterpret_cast<unsigned long long *>(b + L.shist);
  a.cand = (!comm && L.sampled) ? reinterpret_cast<float *>(b + L.cand) : nullptr;
  a.cand_n = (!comm && L.sampled) ? reinterpret_cast<long long *>(b + L.cand_n) : nullptr;
  // single GPU with a large score vector: the sampled one-pass selection
  a.first = (a.cand && scores && n_local >= kSampleMinN) ? P_SAMPLE : P_HIST0;
  a.last = P_FIT;
  a.out_dev = nullptr;
  a.n_dev = nullptr;
  a.dfit_step = -1;
  a.dfit_last = 0;
  a.xsend = comm ? reinterpret_cast<double *>(b + L.xsend) : nullptr;
  a.xrecv = comm ? reinterpret_cast<const double *>(b + L.xrecv) : nullptr;
  a.fstate = comm ? reinterpret_cast<FitState *>(b + L.fstate) : nullptr;
  a.bins = L.has_bins ? reinterpret_cast<unsigned long long *>(b + L.bins) : nullptr;
  return a;
}

static enova_status check_k(int64_t n, double q0) {
  if (n <= 0) {
    set_error("no scores");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  const int64_t k = (int64_t)floor(q0 * (double)n);
  if (k < 0 || k >= n) {
    set_error("init_quantile out of range");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  return ENOVA_OK;
}

static enova_status status_error(int st) {
  switch (st) {
    case ENOVA_OK: return ENOVA_OK;
    case ENOVA_ERR_TOO_FEW_EXCEEDANCES:
      set_error("fewer than 10 exceedances above the initial threshold");
      break;
    case ENOVA_ERR_WORKSPACE: set_error("peak count exceeds workspace capacity"); break;
    case ENOVA_ERR_UNSUPPORTED:
      set_error("GPD fit: more than 64 Grimshaw roots or root refinement did not converge");
      break;
    default: set_error("threshold fit failed"); break;
  }
  return (enova_status)st;
}

static enova_status launch_pot_comm(const PotArgs &a, int nb, cudaStream_t st, bool reset,
                                    enova_comm_t comm) {
  enova_status r = comm_coop_begin(comm, st);
  if (r) return r;
  r = launch_pot(a, nb, st, reset);
  const enova_status r2 = comm_coop_end(comm, st);
  return r ? r : r2;
}

// Communicator path, stream-ordered and free of host synchronisation (so it can
// be captured in a CUDA graph with the NCCL calls): the phases of k_pot run as
// separate cooperative launches with the collectives between them --
//   HIST0 | allreduce h0 | HIST1 | allreduce h1 | HIST2 | allreduce h2 | COMPACT |
//   allgather tail counts + allgather fixed-size tail slots | FIT (pack + fit).
// n: the global score count (sum of n_local over ranks, same on every rank).
enova_status fit_threshold_comm_async(const float *scores, int64_t n_local, int64_t n, double q0,
                                      double q, enova_comm_t comm, enova_threshold *out_dev,
                                      void *ws, size_t ws_bytes, int64_t n_global_max,
                                      cudaStream_t st) {
  char *b = static_cast<char *>(ws);
  if (comm->world > kMaxWorld) {
    set_error("communicator larger than 256 ranks");
    return ENOVA_ERR_UNSUPPORTED;
  }
  const ThrLayout L = thr_layout(n_global_max, q0, comm->world);
  if (ws_bytes < L.total) {
    set_error("threshold workspace too small (size it with the communicator's world size)");
    return ENOVA_ERR_WORKSPACE;
  }
  enova_status r = check_k(n, q0);
  if (r) return r;
  if (n > n_global_max || n_local > n) {
    set_error("total score count exceeds n_global_max used to size the workspace");
    return ENOVA_ERR_WORKSPACE;
  }
  PotArgs a = make_args(scores, n_local, n, q0, q, b, L, true);
  a.world = comm->world;
  const int nb = pot_grid();
  ENOVA_CUDA_TRY(cudaMemsetAsync(b, 0, L.header, st));
  for (int p = P_HIST0; p <= P_HIST2; ++p) {
    a.first = a.last = p;
    if ((r = launch_pot_comm(a, nb, st, p > P_HIST0, comm))) return r;
    r = comm_allreduce_u64_sum(comm, a.hist + (size_t)(p - P_HIST0) * kBins,
                               a.hist + (size_t)(p - P_HIST0) * kBins, (size_t)kBins, st);
    if (r) return r;
  }
  a.first = a.last = P_COMPACT;
  if ((r = launch_pot_comm(a, nb, st, true, comm))) return r;
  r = comm_allgather_i64(comm, &a.g->nt_local, b + L.counts_all, st);
  if (r) return r;
  r = comm_allgather_f32(comm, a.ylocal, b + L.yslot, (size_t)L.cap, st);
  if (r) return r;
  a.first = a.last = P_FIT;
  a.out_dev = out_dev;
  return launch_pot_comm(a, nb, st, true, comm);
}

// Distributed fit (SURVEY §8e variant): the same selection phases, then each
// rank fits on its own tail -- no tail gather -- with one cooperative launch per
// fit step and an all-gather of the ranks' pass totals (6 KB per rank) between
// steps (dfit_step above).  A fixed launch sequence (graph-capturable): step 0
// + kDfitSteps steps; steps after convergence exit at once.
constexpr int kDfitSteps = 16;
enova_status fit_threshold_dist_async(const float *scores, int64_t n_local, int64_t n, double q0,
                                      double q, enova_comm_t comm, enova_threshold *out_dev,
                                      void *ws, size_t ws_bytes, int64_t n_global_max,
                                      cudaStream_t st) {
  char *b = static_cast<char *>(ws);
  if (comm->world > kMaxWorld) {
    set_error("communicator larger than 256 ranks");
    return ENOVA_ERR_UNSUPPORTED;
  }
  const ThrLayout L = thr_layout(n_global_max, q0, comm->world);
  if (ws_bytes < L.total) {
    set_error("threshold workspace too small (size it with the communicator's world size)");
    return ENOVA_ERR_WORKSPACE;
  }
  enova_status r = check_k(n, q0);
  if (r) return r;
  if (n > n_global_max || n_local > n) {
    set_error("total score count exceeds n_global_max used to size the workspace");
    return ENOVA_ERR_WORKSPACE;
  }
  PotArgs a = make_args(scores, n_local, n, q0, q, b, L, true);
  a.world = comm->world;
  const int nb = pot_grid();
  ENOVA_CUDA_TRY(cudaMemsetAsync(b, 0, L.header, st));
  for (int p = P_HIST0; p <= P_HIST2; ++p) {
    a.first = a.last = p;
    if ((r = launch_pot_comm(a, nb, st, p > P_HIST0, comm))) return r;
    r = comm_allreduce_u64_sum(comm, a.hist + (size_t)(p - P_HIST0) * kBins,
                               a.hist + (size_t)(p - P_HIST0) * kBins, (size_t)kBins, st);
    if (r) return r;
  }
  a.first = a.last = P_COMPACT;
  if ((r = launch_pot_comm(a, nb, st, true, comm))) return r;
  a.first = a.last = P_FIT;
  for (int step = 0; step <= kDfitSteps; ++step) {
    a.dfit_step = step;
    a.dfit_last = step == kDfitSteps;
    a.out_dev = a.dfit_last ? out_dev : nullptr;
    if ((r = launch_pot_comm(a, nb, st, true, comm))) return r;
    if (step < kDfitSteps) {
      r = comm_allgather_f32(comm, reinterpret_cast<const float *>(a.xsend), b + L.xrecv,
                             (size_t)2 * kSums * kMaxPts, st);
      if (r) return r;
    }
  }
  return ENOVA_OK;
}

// Host syncs: single GPU one (the result).  With a communicator one more (the
// global score count, all-reduced) before the stream-ordered path above.
enova_status fit_threshold(const float *scores, int64_t n_local, double q0, double q,
                           enova_comm_t comm, enova_threshold *out, void *ws, size_t ws_bytes,
                           int64_t n_global_max, cudaStream_t st) {
  char *b = static_cast<char *>(ws);
  const ThrLayout L = thr_layout(n_global_max, q0, comm ? comm->world : 0);
  if (ws_bytes < L.total) {
    set_error(comm ? "threshold workspace too small (size it with the communicator's world size)"
                   : "threshold workspace too small");
    return ENOVA_ERR_WORKSPACE;
  }
  enova_status r;
  if (comm) {
    int64_t n = 0;
    if ((r = comm_sum_i64_sync(comm, n_local, &n, b + L.nbuf, st))) return r;
    enova_threshold *od = reinterpret_cast<enova_threshold *>(b + L.outdev);
    if ((r = fit_threshold_comm_async(scores, n_local, n, q0, q, comm, od, ws, ws_bytes,
                                      n_global_max, st)))
      return r;
    ENOVA_CUDA_TRY(cudaMemcpyAsync(out, od, sizeof(*out), cudaMemcpyDeviceToHost, st));
    if ((r = comm_wait(comm, st))) return r;   // bounded: a dead peer -> ENOVA_ERR_NCCL
    if ((r = status_error(out->reserved))) return r;
    out->reserved = 0;
    return ENOVA_OK;
  }
  const int64_t n = n_local;
  r = check_k(n, q0);
  if (r) return r;
  if (n > n_global_max) {
    set_error("total score count exceeds n_global_max used to size the workspace");
    return ENOVA_ERR_WORKSPACE;
  }
  PotArgs a = make_args(scores, n_local, n, q0, q, b, L, false);
  ENOVA_CUDA_TRY(cudaMemsetAsync(b, 0, L.header, st));
  if ((r = launch_pot(a, pot_grid(), st))) return r;
  PotGlobal hg;
  ENOVA_CUDA_TRY(cudaMemcpyAsync(&hg, a.g, sizeof(hg), cudaMemcpyDeviceToHost, st));
  ENOVA_CUDA_TRY(cudaStreamSynchronize(st));
  if ((r = status_error(hg.status))) return r;
  out->init_quantile = q0;
  out->risk_q = q;
  out->t = (double)hg.t;
  out->gamma = hg.gamma;
  out->sigma = hg.sigma;
  out->z_q = hg.z_q;
  out->n = n;
  out->n_peaks = hg.nt_fit;
  out->method = hg.method;
  out->reserved = 0;
  return ENOVA_OK;
}

// Stream-ordered single-GPU variant: no host synchronisation; the result (and
// its status in out_dev->reserved) is written to device memory by the kernel.
enova_status fit_threshold_async(const float *scores, int64_t n, double q0, double q,
                                 enova_threshold *out_dev, void *ws, size_t ws_bytes,
                                 int64_t n_global_max, cudaStream_t st) {
  char *b = static_cast<char *>(ws);
  const ThrLayout L = thr_layout(n_global_max, q0);
  if (ws_bytes < L.total) {
    set_error("threshold workspace too small");
    return ENOVA_ERR_WORKSPACE;
  }
  enova_status r = check_k(n, q0);
  if (r) return r;
  if (n > n_global_max) {
    set_error("score count exceeds n_global_max used to size the workspace");
    return ENOVA_ERR_WORKSPACE;
  }
  PotArgs a = make_args(scores, n, n, q0, q, b, L, false);
  a.out_dev = out_dev;
  ENOVA_CUDA_TRY(cudaMemsetAsync(b, 0, L.header, st));
  return launch_pot(a, pot_grid(), st);
}

size_t threshold_workspace_bytes(int64_t n_max, double q0, int world) {
  return thr_layout(n_max, q0, world).total;
}

// diagnostic: byte offsets of PotGlobal.n_stamps / .stamps in the threshold workspace
int64_t pot_sampled_offset() { return (int64_t)offsetof(PotGlobal, sampled); }
int64_t pot_fit_stamp_offset() { return (int64_t)offsetof(PotGlobal, fit_stamp); }

void pot_stamp_offsets(int64_t *n_off, int64_t *st_off) {
  *n_off = (int64_t)offsetof(PotGlobal, n_stamps);
  *st_off = (int64_t)offsetof(PotGlobal, stamps);
}

// ---------------------------------------------------------------- NEXT-2 ----
// Online SPOT (Siffer et al. 2017, cited by PAPER.md:297 for the POT threshold;
// DESIGN.md R-23) on the single-GPU threshold workspace left by a calibration
// fit: Y (the peaks) stays at L.yall, N_t in g->nt_fit, t in g->t, the count of
// non-anomalous observations in g->n_spot.  A tick's scores are flagged against
// the current z_q (enova_detect*), then k_spot_append adds every NON-anomalous
// score above t to Y in index order (anomalies are never used to update the
// model) and counts the non-anomalous observations; a refit re-runs the fit
// phase of k_pot on the grown Y with n read from the device.
__global__ void __launch_bounds__(1024) k_spot_append(const float *__restrict__ scores,
                                                      const int8_t *__restrict__ flags, int64_t n,
                                                      PotGlobal *g, double *__restrict__ Y,
                                                      int64_t cap) {
  // one CTA; thread i owns the contiguous span [i*per, (i+1)*per): count its
  // peaks, block-exclusive scan (fixed order), then write them in index order
  __shared__ long long wpk[32], wna[32];
  __shared__ long long base_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t b0 = min(n, (int64_t)threadIdx.x * per), b1 = min(n, b0 + per);
  const float t = *(volatile float *)&g->t;
  const double td = (double)t;
  long long pk = 0, na = 0;
  for (int64_t i = b0; i < b1; ++i) {
    const bool normal = flags[i] == 0;
    na += normal;
    pk += normal && scores[i] > t;
  }
  long long incl = pk;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  long long nas = na;
#pragma unroll
  for (int o = 16; o; o >>= 1) nas += __shfl_xor_sync(0xffffffffu, nas, o);
  if (lane == 31) wpk[warp] = incl;
  if (lane == 0) wna[warp] = nas;
  if (threadIdx.x == 0) base_s = *(volatile long long *)&g->nt_fit;
  __syncthreads();
  long long before = incl - pk;
  for (int w = 0; w < warp; ++w) before += wpk[w];
  long long idx = base_s + before;
  for (int64_t i = b0; i < b1 && idx < cap; ++i) {
    const float sv = scores[i];
    if (flags[i] == 0 && sv > t) Y[idx++] = (double)sv - td;
  }
  if (threadIdx.x == 0) {
    long long tp = 0, tn = 0;
    for (int w = 0; w < nw; ++w) {
      tp += wpk[w];
      tn += wna[w];
    }
    g->n_spot += tn;
    long long nt = base_s + tp;
    if (nt > cap) {   // peaks beyond the capacity are lost: the next refit reports
      g->spot_overflow = 1;   // ENOVA_ERR_WORKSPACE instead of fitting a truncated Y
      nt = cap;
    }
    g->nt_fit = nt;
  }
}

enova_status spot_update(const float *scores, const int8_t *flags, int64_t n, void *ws,
                         size_t ws_bytes, int64_t n_global_max, double q0, cudaStream_t st) {
  const ThrLayout L = thr_layout(n_global_max, q0);
  if (ws_bytes < L.total) {
    set_error("threshold workspace too small");
    return ENOVA_ERR_WORKSPACE;
  }
  char *b = static_cast<char *>(ws);
  if (n == 0) return ENOVA_OK;
  ENOVA_LAUNCH(k_spot_append, 1, 1024, 0, st, scores, flags, n,
               reinterpret_cast<PotGlobal *>(b + L.glob), reinterpret_cast<double *>(b + L.yall),
               L.cap);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

enova_status spot_refit(double q, enova_threshold *out_dev, void *ws, size_t ws_bytes,
                        int64_t n_global_max, double q0, cudaStream_t st) {
  const ThrLayout L = thr_layout(n_global_max, q0);
  if (ws_bytes < L.total) {
    set_error("threshold workspace too small");
    return ENOVA_ERR_WORKSPACE;
  }
  char *b = static_cast<char *>(ws);
  PotArgs a = make_args(nullptr, 0, 0, q0, q, b, L, false);
  a.first = a.last = P_FIT;
  a.out_dev = out_dev;
  a.n_dev = &a.g->n_spot;
  return launch_pot(a, pot_grid(), st, true);
}

}  // namespace enova
