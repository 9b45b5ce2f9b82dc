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
//         k-section (bisection when S = 1) to a 2^-60 bracket; every root gives
//         gamma = v - 1, sigma = gamma / x, log-likelihood -N (ln sigma + gamma + 1);
//         the exponential candidate (gamma = 0, sigma = Ybar) is always present;
//   z_q = t + sigma/gamma * expm1(-gamma ln(q n / N_t))  (t - sigma ln(.) at gamma = 0).
// All reductions use a fixed block partition and a fixed combine order, so the
// result is deterministic and identical on every rank.
#include <math.h>

#include <vector>


#include "comm.h"
#include "common.cuh"

namespace enova {

constexpr int kBins = 2048;
constexpr int kSelThreads = 1024;
constexpr int kCompactBlocks = 1184;  // 8 per SM
constexpr int kCompactThreads = 256;
constexpr int kFitBlocks = 592;   // 4 per SM; blocks beyond ceil(N_t/256) only join the ticket
constexpr int kFitThreads = 256;
constexpr int kMaxPts = 128;
constexpr int kMaxSlots = 64;
constexpr int kGrid = 64;

enum { PH_GRID = 0, PH_REFINE = 1, PH_FINAL = 2, PH_DONE = 3 };

struct SelState {
  unsigned int prefix, mask;
  unsigned long long k_rem;
  float t;
  int pad;
};

struct FitState {
  int64_t nt, n;
  double t, q, ybar, ymin, ymax;
  int phase, npts, nslots, S, iters, overflow;
  unsigned int counter, pad;
  double xs[kMaxPts], w[kMaxPts], L[kMaxPts], dw[kMaxPts];
  double lo[kMaxSlots], hi[kMaxSlots], wlo[kMaxSlots], whi[kMaxSlots];
  int converged;
  int exact[kMaxSlots];
  int refine_idx[kMaxSlots];   // slot of the k-th refined bracket
  int nrefine;
  // result
  double gamma, sigma, z_q;
  int method, nroots;
};

struct ThrLayout {
  size_t hist, sel, fit, partials, counts, counts_all, nbuf, ylocal, yall, total;
  int64_t cap;
};

static inline ThrLayout thr_layout(int64_t n_max, double q0) {
  ThrLayout L;
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o += (b + 255) / 256 * 256; return r; };
  double tail = (1.0 - q0) * (double)n_max;
  if (tail < 0) tail = 0;
  L.cap = (int64_t)ceil(tail) + 16;
  if (L.cap > n_max) L.cap = n_max;
  if (L.cap < 16) L.cap = 16;
  L.hist = take(kBins * 8);
  L.sel = take(sizeof(SelState));
  L.fit = take(sizeof(FitState));
  L.partials = take((size_t)kFitBlocks * (8 * kMaxPts + 4) * 8);
  L.counts = take((kCompactBlocks + 1) * 8);
  L.counts_all = take(1024 * 8);
  L.nbuf = take(16);
  L.ylocal = take((size_t)L.cap * 8);
  L.yall = take((size_t)L.cap * 8);
  L.total = o;
  return L;
}

__device__ __forceinline__ unsigned int f2key(float f) {
  unsigned int b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(unsigned int k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// ---------------------------------------------------------------- K3 ----
__global__ void k_sel_init(SelState *s, unsigned long long k) {
  s->prefix = 0;
  s->mask = 0;
  s->k_rem = k;
  s->t = 0.f;
}

__global__ void k_hist(const float *__restrict__ x, int64_t n, const SelState *__restrict__ sel,
                       unsigned long long *__restrict__ hist, int shift, int nbins) {
  __shared__ unsigned int h[kBins];
  for (int i = threadIdx.x; i < nbins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const unsigned int prefix = sel->prefix, mask = sel->mask;
  const int64_t n4 = n / 4;
  const float4 *x4 = reinterpret_cast<const float4 *>(x);
  const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto add = [&](float f) {
    unsigned int k = f2key(f);
    if ((k & mask) == prefix) atomicAdd(&h[(k >> shift) & (nbins - 1)], 1u);
  };
  if (aligned) {
    for (int64_t i = i0; i < n4; i += stride) {
      float4 v = __ldg(x4 + i);
      add(v.x); add(v.y); add(v.z); add(v.w);
    }
    for (int64_t i = 4 * n4 + i0; i < n; i += stride) add(__ldg(x + i));
  } else {
    for (int64_t i = i0; i < n; i += stride) add(__ldg(x + i));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nbins; i += blockDim.x)
    if (h[i]) atomicAdd(hist + i, (unsigned long long)h[i]);
}

// one block of 1024 threads, 2 bins per thread: find the digit holding rank k_rem
__global__ void k_select(unsigned long long *__restrict__ hist, SelState *__restrict__ sel,
                         int shift, int nbins) {
  __shared__ unsigned long long warp_tot[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long c0 = 0, c1 = 0;
  if (2 * tid < nbins) c0 = hist[2 * tid];
  if (2 * tid + 1 < nbins) c1 = hist[2 * tid + 1];
  unsigned long long v = c0 + c1, incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long wv = warp_tot[lane], wi = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    warp_tot[lane] = wi - wv;  // exclusive warp offsets
  }
  __syncthreads();
  const unsigned long long before = warp_tot[warp] + incl - v;  // exclusive prefix of bin 2*tid
  const unsigned long long k = sel->k_rem;
  __syncthreads();
  int digit = -1;
  unsigned long long below = 0;
  if (c0 && k >= before && k < before + c0) {
    digit = 2 * tid;
    below = before;
  } else if (c1 && k >= before + c0 && k < before + c0 + c1) {
    digit = 2 * tid + 1;
    below = before + c0;
  }
  if (digit >= 0) {
    sel->prefix |= (unsigned int)digit << shift;
    sel->mask |= (unsigned int)(nbins - 1) << shift;
    sel->k_rem = k - below;
    if (shift == 0) sel->t = key2f(sel->prefix);
  }
  __syncthreads();
  if (2 * tid < nbins) hist[2 * tid] = 0;
  if (2 * tid + 1 < nbins) hist[2 * tid + 1] = 0;
}

// ---------------------------------------------------------------- K4 ----
__device__ __forceinline__ void chunk_of(int64_t n, int64_t *b0, int64_t *b1) {
  int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  chunk = (chunk + 255) / 256 * 256;
  *b0 = min(n, (int64_t)blockIdx.x * chunk);
  *b1 = min(n, *b0 + chunk);
}

__global__ void k_count_peaks(const float *__restrict__ x, int64_t n,
                              const SelState *__restrict__ sel,
                              long long *__restrict__ counts) {
  __shared__ int wsum[32];
  int64_t b0, b1;
  chunk_of(n, &b0, &b1);
  const double t = (double)sel->t;
  int c = 0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) c += ((double)__ldg(x + i) > t);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += wsum[w];
    counts[blockIdx.x] = s;
  }
}

// exclusive scan of nblk (<= 2048) counts in place; total at counts[nblk].
// One block of 1024 threads, two counts per thread (warp shuffles + warp totals).
__global__ void k_scan_counts(long long *counts, int nblk) {
  __shared__ long long warp_tot[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long c0 = (2 * tid < nblk) ? counts[2 * tid] : 0;
  long long c1 = (2 * tid + 1 < nblk) ? counts[2 * tid + 1] : 0;
  long long v = c0 + c1, incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    long long wv = warp_tot[lane], wi = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    warp_tot[lane] = wi - wv;
    if (lane == 31) counts[nblk] = wi;
  }
  __syncthreads();
  const long long before = warp_tot[warp] + incl - v;
  if (2 * tid < nblk) counts[2 * tid] = before;
  if (2 * tid + 1 < nblk) counts[2 * tid + 1] = before + c0;
}

__global__ void k_scatter_peaks(const float *__restrict__ x, int64_t n,
                                const SelState *__restrict__ sel,
                                const long long *__restrict__ offsets, double *__restrict__ Y,
                                int64_t cap) {
  __shared__ int woff[kCompactThreads / 32 + 1];
  int64_t b0, b1;
  chunk_of(n, &b0, &b1);
  const double t = (double)sel->t;
  long long base = offsets[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t i0 = b0; i0 < b1; i0 += blockDim.x) {
    int64_t i = i0 + threadIdx.x;
    double s = (i < b1) ? (double)__ldg(x + i) : 0.0;
    bool f = (i < b1) && (s > t);
    unsigned int bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) woff[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int w = 0; w < nw; ++w) {
        int c = woff[w];
        woff[w] = run;
        run += c;
      }
      woff[nw] = run;
    }
    __syncthreads();
    if (f) {
      const long long o = base + woff[warp] + __popc(bal & ((1u << lane) - 1u));
      if (o < cap) Y[o] = s - t;
    }
    base += woff[nw];
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K5 ----
__device__ bool last_block_done(unsigned int *counter) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int ticket = atomicAdd(counter, 1u);
    last = (ticket == gridDim.x - 1);
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

template <typename T, typename Op>
__device__ T block_reduce(T v, Op op, T *scratch) {
  // fixed-order tree: warp xor-shuffle, then warp totals in order
  for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  T r = scratch[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = op(r, scratch[w]);
  return r;
}

__device__ void setup_grid(FitState *f) {
  // the fixed scan grids of R-13 (same formulas as the oracle)
  const double ymax = f->ymax, ymin = f->ymin, ybar = f->ybar;
  for (int k = 0; k < kGrid; ++k) {
    double th = 1e-8 + k * ((1.0 - 2e-8) / (kGrid - 1));
    f->xs[k] = (-1.0 / ymax) * (1.0 - th);
  }
  double a = 1e-12 / ybar;
  double b = 2.0 * (ybar - ymin) / (ymin * ymin);
  int np = kGrid;
  if (b > a) {
    double la = log(a), lb = log(b);
    for (int k = 0; k < kGrid; ++k) f->xs[kGrid + k] = exp(la + k * ((lb - la) / (kGrid - 1)));
    np = 2 * kGrid;
  }
  f->npts = np;
  f->phase = PH_GRID;
}

// Phase machine run by the last block of each evaluation launch.
//  GRID  : w at the fixed scan grids -> one slot per sign change (or exact zero);
//  REFINE: safeguarded Newton on every bracket: w(x), w'(x) from the same pass;
//          the bracket shrinks with the sign of w(x); the Newton iterate is kept
//          if it falls strictly inside the bracket, else the bracket midpoint is
//          used; converged when every step is <= 1e-13 |x| (the oracle bisects
//          to a 2^-60 bracket: both land on the same root of the fp64 w);
//  FINAL : L(x) at the roots -> gamma, sigma, log-likelihood; pick; z_q.
__device__ void controller(FitState *f) {
  if (f->phase == PH_GRID) {
    int ns = 0;
    auto push = [&](double lo, double hi, double wlo, double whi, int exact) {
      if (ns >= kMaxSlots) {
        f->overflow = 1;
        return;
      }
      f->lo[ns] = lo;
      f->hi[ns] = hi;
      f->wlo[ns] = wlo;
      f->whi[ns] = whi;
      f->exact[ns] = exact;
      ++ns;
    };
    for (int g = 0; g * kGrid < f->npts; ++g) {
      const double *x = f->xs + g * kGrid;
      const double *w = f->w + g * kGrid;
      for (int k = 0; k < kGrid - 1; ++k) {
        if (w[k] == 0.0)
          push(x[k], x[k], 0.0, 0.0, 1);
        else if (w[k] * w[k + 1] < 0.0)
          push(x[k], x[k + 1], w[k], w[k + 1], 0);
      }
      if (w[kGrid - 1] == 0.0) push(x[kGrid - 1], x[kGrid - 1], 0.0, 0.0, 1);
    }
    f->nslots = ns;
    int nr = 0;
    for (int s = 0; s < ns; ++s)
      if (!f->exact[s]) f->refine_idx[nr++] = s;
    f->nrefine = nr;
    f->converged = 0;
    if (nr > 0) {
      for (int r = 0; r < nr; ++r) {   // first iterate: secant (regula falsi) point
        const int s = f->refine_idx[r];
        const double lo = f->lo[s], hi = f->hi[s];
        double x0 = lo - f->wlo[s] * (hi - lo) / (f->whi[s] - f->wlo[s]);
        if (!(x0 > fmin(lo, hi) && x0 < fmax(lo, hi))) x0 = 0.5 * (lo + hi);
        f->xs[r] = x0;
      }
      f->npts = nr;
      f->phase = PH_REFINE;
    } else {
      f->phase = PH_FINAL;
      f->converged = 1;
      for (int s = 0; s < ns; ++s) f->xs[s] = f->lo[s];
      f->npts = ns;
    }
    return;
  }
  if (f->phase == PH_REFINE) {
    bool all_conv = true;
    for (int r = 0; r < f->nrefine; ++r) {
      const int s = f->refine_idx[r];
      const double x = f->xs[r], w = f->w[r], dw = f->dw[r];
      double lo = f->lo[s], hi = f->hi[s];
      if (w == 0.0) {
        lo = hi = x;
      } else if ((w > 0) == (f->wlo[s] > 0)) {
        lo = x;
        f->wlo[s] = w;
      } else {
        hi = x;
      }
      f->lo[s] = lo;
      f->hi[s] = hi;
      double xn = (dw != 0.0) ? x - w / dw : 0.5 * (lo + hi);
      const double a = fmin(lo, hi), b = fmax(lo, hi);
      if (!(xn > a && xn < b) || f->iters > 20) xn = 0.5 * (lo + hi);   // safeguard: bisect
      if (lo == hi) xn = lo;
      if (!(fabs(xn - x) <= 1e-13 * fabs(x))) all_conv = false;
      f->xs[r] = xn;
    }
    if (all_conv) {
      // every slot's root estimate is final (exact grid zeros keep lo)
      for (int r = 0; r < f->nrefine; ++r) f->lo[f->refine_idx[r]] = f->xs[r];
      for (int s = 0; s < f->nslots; ++s) f->xs[s] = f->lo[s];
      f->npts = f->nslots;
      f->phase = PH_FINAL;
      f->converged = 1;
    }
    return;
  }
  if (f->phase == PH_FINAL) {
    const double N = (double)f->nt;
    double bg = 0.0, bs = f->ybar, bll = -N * (log(f->ybar) + 1.0);
    int method = 1, nroots = 0;
    for (int s = 0; s < f->nslots; ++s) {
      const double x = f->xs[s];
      const double g = f->L[s];
      if (x == 0.0 || g == 0.0) continue;
      const double sg = g / x;
      if (!(sg > 0.0)) continue;
      ++nroots;
      const double ll = -N * (log(sg) + g + 1.0);
      if (ll > bll || (ll == bll && fabs(g) < fabs(bg))) {
        bll = ll;
        bg = g;
        bs = sg;
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
}

// K5 as ONE cooperative launch (one CTA per SM, grid-wide barriers): every CTA
// keeps an identical copy of the fit state in shared memory and, after each
// grid barrier, reduces the per-CTA partial sums itself in a fixed order and
// runs the same controller -- so no host round trips, no extra broadcast
// barrier, and a deterministic result.
//   phase 0: Ybar, Ymin, Ymax -> scan grids;  then per pass: evaluate
//   P = mean(-xY/(1+xY)), L = mean(log1p(xY)) (+ dP = mean(-Y/(1+xY)^2),
//   dL = mean(Y/(1+xY)) for Newton) at the state's points; controller.
constexpr int kCoopThreads = 256;

// grid-wide barrier for a cooperative launch (all CTAs co-resident): one arrival
// per CTA on a global ticket, the last one bumps the generation word.
__device__ __forceinline__ void grid_barrier(unsigned int *count, unsigned int *gen,
                                             unsigned int nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g = *(volatile unsigned int *)gen;
    __threadfence();
    const unsigned int ticket = atomicAdd(count, 1u);
    if (ticket == nb - 1) {
      *(volatile unsigned int *)count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*(volatile unsigned int *)gen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}
constexpr int kMaxRefinePasses = 60;

__device__ __forceinline__ void coop_reduce_points(FitState &f, const double *part, int nb,
                                                   int npts, bool deriv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double N = (double)f.nt;
  const int nk = deriv ? 4 : 2;
  for (int pt = warp; pt < npts; pt += kCoopThreads / 32) {
    double a[4] = {0, 0, 0, 0};
    for (int b = lane; b < nb; b += 32)
      for (int k = 0; k < nk; ++k) a[k] += part[((size_t)k * kMaxPts + pt) * kFitBlocks + b];
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
      for (int k = 0; k < 4; ++k) a[k] += __shfl_xor_sync(0xffffffffu, a[k], o);
    if (lane == 0) {
      const double Pm = a[0] / N, Lm = a[1] / N, dPm = a[2] / N, dLm = a[3] / N;
      f.w[pt] = Pm + Lm + Pm * Lm;
      f.L[pt] = Lm;
      f.dw[pt] = dPm + dLm + dPm * Lm + Pm * dLm;
    }
  }
}

__global__ void __launch_bounds__(kCoopThreads, 1)
    k_fit_coop(const double *__restrict__ Y, FitState *gf, double *__restrict__ part,
               const long long *nt_dev, int64_t n, const SelState *sel, double q) {
  __shared__ FitState f;
  unsigned int *bar_count = &gf->counter, *bar_gen = &gf->pad;
  __shared__ double wS[4][kCoopThreads / 32][kMaxPts];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = gridDim.x;
  if (threadIdx.x == 0) {
    f.nt = *nt_dev;
    f.n = n;
    f.t = (double)sel->t;
    f.q = q;
    f.overflow = 0;
    f.converged = 0;
    f.iters = 0;
    f.phase = PH_GRID;
  }
  __syncthreads();
  const int64_t nt = f.nt;
  const int64_t chunk = (nt + nb - 1) / nb;
  const int64_t b0 = min(nt, (int64_t)blockIdx.x * chunk), b1 = min(nt, b0 + chunk);

  // ---- Ybar, Ymin, Ymax ----
  {
    double s = 0.0, mn = INFINITY, mx = -INFINITY;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      const double y = Y[i];
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
      wS[0][warp][0] = s;
      wS[1][warp][0] = mn;
      wS[2][warp][0] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double ts = 0.0, tmn = INFINITY, tmx = -INFINITY;
      for (int w = 0; w < kCoopThreads / 32; ++w) {
        ts += wS[0][w][0];
        tmn = fmin(tmn, wS[1][w][0]);
        tmx = fmax(tmx, wS[2][w][0]);
      }
      part[blockIdx.x] = ts;
      part[kFitBlocks + blockIdx.x] = tmn;
      part[2 * kFitBlocks + blockIdx.x] = tmx;
    }
    grid_barrier(bar_count, bar_gen, nb);
    if (warp == 0) {
      double ts = 0.0, tmn = INFINITY, tmx = -INFINITY;
      for (int b = lane; b < nb; b += 32) {
        ts += part[b];
        tmn = fmin(tmn, part[kFitBlocks + b]);
        tmx = fmax(tmx, part[2 * kFitBlocks + b]);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        ts += __shfl_xor_sync(0xffffffffu, ts, o);
        tmn = fmin(tmn, __shfl_xor_sync(0xffffffffu, tmn, o));
        tmx = fmax(tmx, __shfl_xor_sync(0xffffffffu, tmx, o));
      }
      if (lane == 0) {
        f.ybar = ts / (double)nt;
        f.ymin = tmn;
        f.ymax = tmx;
        setup_grid(&f);
      }
    }
    __syncthreads();
  }

  // ---- evaluation passes (partials double-buffered: one barrier per pass) ----
  for (int pass = 0; pass < kMaxRefinePasses + 3; ++pass) {
    double *pw = part + 4 * kFitBlocks + (size_t)(pass & 1) * 4 * kMaxPts * kFitBlocks;
    const int phase = f.phase;
    if (phase == PH_DONE) break;
    const int npts = f.npts;
    const bool deriv = (phase == PH_REFINE);
    if (npts > 0) {
      for (int q0 = 0; q0 < npts; q0 += 4) {
        double P[4] = {0, 0, 0, 0}, L[4] = {0, 0, 0, 0}, dP[4] = {0, 0, 0, 0},
               dL[4] = {0, 0, 0, 0};
        double x[4];
        int nu = min(4, npts - q0);
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = (u < nu) ? f.xs[q0 + u] : 0.0;
        for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
          const double y = Y[i];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (u < nu) {
              const double xy = x[u] * y;
              const double r = 1.0 / (1.0 + xy);
              P[u] -= xy * r;
              L[u] += log1p(xy);
              if (deriv) {
                const double yr = y * r;
                dL[u] += yr;
                dP[u] -= yr * r;
              }
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
          for (int o = 16; o; o >>= 1) {
            P[u] += __shfl_xor_sync(0xffffffffu, P[u], o);
            L[u] += __shfl_xor_sync(0xffffffffu, L[u], o);
            dP[u] += __shfl_xor_sync(0xffffffffu, dP[u], o);
            dL[u] += __shfl_xor_sync(0xffffffffu, dL[u], o);
          }
        }
        if (lane == 0) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < nu) {
              wS[0][warp][q0 + u] = P[u];
              wS[1][warp][q0 + u] = L[u];
              wS[2][warp][q0 + u] = dP[u];
              wS[3][warp][q0 + u] = dL[u];
            }
        }
      }
      __syncthreads();
      const int nk = deriv ? 4 : 2;
      for (int i = threadIdx.x; i < nk * npts; i += blockDim.x) {
        const int k = i / npts, pt = i % npts;
        double sum = 0.0;
        for (int w = 0; w < kCoopThreads / 32; ++w) sum += wS[k][w][pt];
        pw[((size_t)k * kMaxPts + pt) * kFitBlocks + blockIdx.x] = sum;
      }
    }
    grid_barrier(bar_count, bar_gen, nb);
    if (npts > 0) coop_reduce_points(f, pw, nb, npts, deriv);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (phase == PH_REFINE && ++f.iters >= kMaxRefinePasses && f.phase == PH_REFINE) {
        // not converged: keep the current iterates, mark, and finish
        for (int r = 0; r < f.nrefine; ++r) f.lo[f.refine_idx[r]] = f.xs[r];
        controller(&f);
        if (f.phase == PH_REFINE) {
          for (int s2 = 0; s2 < f.nslots; ++s2) f.xs[s2] = f.lo[s2];
          f.npts = f.nslots;
          f.phase = PH_FINAL;
        }
      } else {
        controller(&f);
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    gf->nt = f.nt;
    gf->gamma = f.gamma;
    gf->sigma = f.sigma;
    gf->z_q = f.z_q;
    gf->method = f.method;
    gf->nroots = f.nroots;
    gf->overflow = f.overflow;
    gf->converged = f.converged;
    gf->phase = f.phase;
  }
}


// ------------------------------------------------------------- driver ----
// Host syncs: single GPU 2 (after the grid scan: N_t, iteration count; at the
// end: the result).  With a communicator 2 more (global n; tail counts for the
// rank-ordered allgatherv).
enova_status fit_threshold(const float *scores, int64_t n_local, double q0, double q,
                           enova_comm_t comm, enova_threshold *out, void *ws, size_t ws_bytes,
                           int64_t n_global_max, cudaStream_t st) {
  char *b = static_cast<char *>(ws);
  const ThrLayout L = thr_layout(n_global_max, q0);
  if (ws_bytes < L.total) {
    set_error("threshold workspace too small");
    return ENOVA_ERR_WORKSPACE;
  }
  unsigned long long *nbuf = reinterpret_cast<unsigned long long *>(b + L.nbuf);
  unsigned long long *hist = reinterpret_cast<unsigned long long *>(b + L.hist);
  SelState *sel = reinterpret_cast<SelState *>(b + L.sel);
  FitState *fit = reinterpret_cast<FitState *>(b + L.fit);
  double *partials = reinterpret_cast<double *>(b + L.partials);
  long long *counts = reinterpret_cast<long long *>(b + L.counts);
  long long *counts_all = reinterpret_cast<long long *>(b + L.counts_all);
  double *ylocal = reinterpret_cast<double *>(b + L.ylocal);
  double *yall = reinterpret_cast<double *>(b + L.yall);
  long long *nt_dev = counts + kCompactBlocks;  // total written by k_scan_counts

  // global n
  int64_t n = n_local;
  if (comm) {
    unsigned long long hn = (unsigned long long)n_local;
    ENOVA_CUDA_TRY(cudaMemcpyAsync(nbuf, &hn, 8, cudaMemcpyHostToDevice, st));
    enova_status s = comm_allreduce_u64_sum(comm, nbuf, nbuf, 1, st);
    if (s) return s;
    ENOVA_CUDA_TRY(cudaMemcpyAsync(&hn, nbuf, 8, cudaMemcpyDeviceToHost, st));
    ENOVA_CUDA_TRY(cudaStreamSynchronize(st));
    n = (int64_t)hn;
  }
  if (n <= 0) {
    set_error("no scores");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (n > n_global_max) {
    set_error("total score count exceeds n_global_max used to size the workspace");
    return ENOVA_ERR_WORKSPACE;
  }
  const int64_t k = (int64_t)floor(q0 * (double)n);
  if (k < 0 || k >= n) {
    set_error("init_quantile out of range");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }

  // K3: radix select of the k-th smallest key (3 digit passes, exact)
  ENOVA_CUDA_TRY(cudaMemsetAsync(hist, 0, kBins * 8, st));
  ENOVA_LAUNCH(k_sel_init, 1, 1, 0, st, sel, (unsigned long long)k);
  const int shifts[3] = {21, 10, 0};
  const int nbins[3] = {2048, 2048, 1024};
  int hblocks = (int)((n_local + 4095) / 4096);   // ~8 keys per thread
  if (hblocks < 1) hblocks = 1;
  if (hblocks > 148 * 4) hblocks = 148 * 4;
  for (int pass = 0; pass < 3; ++pass) {
    if (n_local > 0)
      ENOVA_LAUNCH(k_hist, hblocks, 512, 0, st, scores, n_local, sel, hist, shifts[pass],
                   nbins[pass]);
    if (comm) {
      enova_status s = comm_allreduce_u64_sum(comm, hist, hist, (size_t)nbins[pass], st);
      if (s) return s;
    }
    ENOVA_LAUNCH(k_select, 1, kSelThreads, 0, st, hist, sel, shifts[pass], nbins[pass]);
  }

  // K4: stable compaction of the peaks (bounded by the workspace capacity)
  double *ydst = comm ? ylocal : yall;
  if (n_local > 0) {
    ENOVA_LAUNCH(k_count_peaks, kCompactBlocks, kCompactThreads, 0, st, scores, n_local, sel,
                 counts);
    ENOVA_LAUNCH(k_scan_counts, 1, 1024, 0, st, counts, kCompactBlocks);
    ENOVA_LAUNCH(k_scatter_peaks, kCompactBlocks, kCompactThreads, 0, st, scores, n_local, sel,
                 counts, ydst, L.cap);
  } else {
    ENOVA_CUDA_TRY(cudaMemsetAsync(nt_dev, 0, 8, st));
  }
  ENOVA_CUDA_TRY(cudaGetLastError());
  if (comm) {
    enova_status s = comm_allgather_i64(comm, nt_dev, counts_all, st);
    if (s) return s;
    std::vector<int64_t> hc(comm->world), off(comm->world);
    ENOVA_CUDA_TRY(cudaMemcpyAsync(hc.data(), counts_all, 8 * comm->world,
                                   cudaMemcpyDeviceToHost, st));
    ENOVA_CUDA_TRY(cudaStreamSynchronize(st));
    int64_t tot = 0;
    for (int r = 0; r < comm->world; ++r) {
      off[r] = tot;
      if (hc[r] > L.cap) {
        set_error("peak count exceeds workspace capacity");
        return ENOVA_ERR_WORKSPACE;
      }
      tot += hc[r];
    }
    if (tot > L.cap) {
      set_error("peak count exceeds workspace capacity");
      return ENOVA_ERR_WORKSPACE;
    }
    s = comm_allgatherv_f64(comm, ylocal, yall, hc.data(), off.data(), st);
    if (s) return s;
    long long tl = tot;
    ENOVA_CUDA_TRY(cudaMemcpyAsync(nbuf + 1, &tl, 8, cudaMemcpyHostToDevice, st));
    nt_dev = reinterpret_cast<long long *>(nbuf + 1);
  }

  // K5: GPD fit (replicated, deterministic).  N_t is read back once so every fit
  // launch is sized to the tail (few blocks -> cheap last-block tickets).
  int64_t nt_h = 0;
  {
    long long v = 0;
    ENOVA_CUDA_TRY(cudaMemcpyAsync(&v, nt_dev, 8, cudaMemcpyDeviceToHost, st));
    ENOVA_CUDA_TRY(cudaStreamSynchronize(st));
    nt_h = v;
  }
  if (nt_h > L.cap) {
    set_error("peak count exceeds workspace capacity");
    return ENOVA_ERR_WORKSPACE;
  }
  if (nt_h < 10) {
    set_error("fewer than 10 exceedances above the initial threshold");
    return ENOVA_ERR_TOO_FEW_EXCEEDANCES;
  }
  {
    int dev = 0, sms = 148;
    ENOVA_CUDA_TRY(cudaGetDevice(&dev));
    ENOVA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int nb = sms < kFitBlocks ? sms : kFitBlocks;
    const int64_t need = (nt_h + 63) / 64;   // >= 64 peaks per CTA
    if (need < nb) nb = (int)(need < 1 ? 1 : need);
    const double *Yc = yall;
    FitState *fc = fit;
    double *pc = partials;
    const long long *ntc = nt_dev;
    int64_t nc = n;
    const SelState *sc = sel;
    double qc = q;
    void *args[] = {(void *)&Yc, (void *)&fc, (void *)&pc, (void *)&ntc,
                    (void *)&nc, (void *)&sc, (void *)&qc};
    ENOVA_CUDA_TRY(cudaMemsetAsync(&fit->counter, 0, sizeof(unsigned int), st));
    count_launch();
    ENOVA_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_fit_coop, dim3(nb),
                                               dim3(kCoopThreads), args, 0, st));
  }
  struct {
    int overflow, converged;
  } hh;
  ENOVA_CUDA_TRY(cudaMemcpyAsync(&hh.overflow, &fit->overflow, 4, cudaMemcpyDeviceToHost, st));
  ENOVA_CUDA_TRY(cudaMemcpyAsync(&hh.converged, &fit->converged, 4, cudaMemcpyDeviceToHost, st));
  struct {
    double gamma, sigma, z_q;
    int method, nroots;
  } res;
  ENOVA_CUDA_TRY(cudaMemcpyAsync(&res, &fit->gamma, sizeof(res), cudaMemcpyDeviceToHost, st));
  float t = 0.f;
  ENOVA_CUDA_TRY(cudaMemcpyAsync(&t, &sel->t, 4, cudaMemcpyDeviceToHost, st));
  ENOVA_CUDA_TRY(cudaStreamSynchronize(st));
  if (hh.overflow) {
    set_error("more than 64 Grimshaw roots");
    return ENOVA_ERR_UNSUPPORTED;
  }
  if (!hh.converged) {
    set_error("GPD root refinement did not converge");
    return ENOVA_ERR_UNSUPPORTED;
  }
  out->init_quantile = q0;
  out->risk_q = q;
  out->t = (double)t;
  out->gamma = res.gamma;
  out->sigma = res.sigma;
  out->z_q = res.z_q;
  out->n = n;
  out->n_peaks = nt_h;
  out->method = res.method;
  out->reserved = 0;
  return ENOVA_OK;
}

size_t threshold_workspace_bytes(int64_t n_max, double q0) { return thr_layout(n_max, q0).total; }

}  // namespace enova
