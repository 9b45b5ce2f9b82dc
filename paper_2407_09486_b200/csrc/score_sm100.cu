// score_sm100.cu -- K2: fused window scorer on 5th-generation tensor cores.
//
// One CTA scores a tile of 128 consecutive windows of one instance (a-2..a-6):
//
//   stage   : the tile's 128+W-1 raw fp32 samples are read once (coalesced
//             128-bit loads), normalised z = (X - mean)/std in fp32, clamped to
//             +-1e4 and rounded to fp16 (R-4, R-17), and stored as fp16 "planes"
//             of 8 metrics per sample (16 B per sample per plane).
//   GEMM1   : h_pre = X_win W1^T as an implicit-GEMM conv1d over the window taps.
//             The window matrix is never materialised: for K-chunk pair
//             (tau, plane) the A operand is a shared-memory descriptor whose start
//             is plane + (tau)*16 B -- consecutive windows are consecutive rows of
//             the K-major no-swizzle canonical layout (rows 16 B apart, SBO = 128 B,
//             LBO = plane stride, or 16 B when M = 8 pairs taps tau, tau+1).
//             tcgen05.mma kind::f16 M=128 N=H K=16 per step, fp32 accumulate in
//             TMEM; W1's fp16 image streams through a 4-stage bulk-copy ring.
//   epi 1   : h = tanh(h_pre + b1) (fp32), split h = hi + lo (two fp16) -> smem.
//   GEMM2   : [mu | lv] = (h_hi + h_lo) [Wmu | Wlv]^T  (two passes, one accumulator)
//   epi 2   : score = 1/2 sum(mu^2 + expm1(lv) - lv)  (R-6);
//             mu = hi + lo -> smem.
//   GEMM3   : a3_pre = (mu_hi + mu_lo) W3^T
//   epi 3   : MD = (sum_k x_k - w_bar . tanh(a3_pre + b3) - b_bar) / D  (R-8,
//             column-sum identity of the linear output layer), flag (R-9, R-10).
//
// Two CTAs share an SM (<= ~95 KB smem, 256 TMEM columns each) so one CTA's
// epilogue overlaps the other's GEMM1.
#include <stdlib.h>
#include <string.h>

#include <atomic>

#include "common.cuh"
#include "layout.h"

namespace enova {

struct ScoreParams {
  const float *X;
  int64_t ld, n_inst, t_begin, nw;  // nw = t_end - t_begin
  const float *mean, *stdv;
  int W, M, P, D, Z, NS, tiles_per_inst, nsteps;
  const uint8_t *w1img, *headsimg, *w3img;
  const float *b1, *bml, *b3, *wbar;
  const double *bbar;
  float *scores, *md;
  int8_t *flags;
  double z_q;
  const double *z_q_dev;   // device threshold (enova_detect_async); overrides z_q
};

constexpr int kRows = 128;       // windows per tile (UMMA M)
constexpr int kStageSteps = 4;   // K=16 MMA steps per ring stage
constexpr int kStages = 4;       // ring depth

template <int H, int ZP>
struct ScoreSmem {
  static constexpr int N2 = 2 * ZP;
  static constexpr uint32_t kStepBytes = 32 * H;                 // one K=16 step of W1
  static constexpr uint32_t kStageBytes = kStageSteps * kStepBytes;
  static constexpr uint32_t kRingBytes = kStages * kStageBytes;
  static constexpr uint32_t kHBytes = kRows * H * 2;             // one of h_hi / h_lo
  static constexpr uint32_t kRegion = kRingBytes > 2 * kHBytes ? kRingBytes : 2 * kHBytes;
  static constexpr uint32_t kHeadsBytes = N2 * H * 2;
  static constexpr uint32_t kW3Bytes = H * 16 * 2;
  static constexpr uint32_t kMuBytes = kRows * 16 * 2;           // one of mu_hi / mu_lo
  static constexpr uint32_t kTmemCols = (H + N2) <= 32 ? 32 : (H + N2) <= 64 ? 64
                                      : (H + N2) <= 128 ? 128 : 256;
  // offsets (planes first; their size depends on W, M at run time)
  __host__ __device__ static uint32_t planes_bytes(int P, int NS) { return (uint32_t)(P * NS * 16); }
  __host__ __device__ static uint32_t off_ssum(int P, int NS) { return (planes_bytes(P, NS) + 127) / 128 * 128; }
  __host__ __device__ static uint32_t off_region(int P, int NS) {
    return (off_ssum(P, NS) + NS * 4 + 1023) / 1024 * 1024;
  }
  __host__ __device__ static uint32_t off_heads(int P, int NS) { return off_region(P, NS) + kRegion; }
  __host__ __device__ static uint32_t off_w3(int P, int NS) { return off_heads(P, NS) + kHeadsBytes; }
  __host__ __device__ static uint32_t off_mu(int P, int NS) { return off_w3(P, NS) + kW3Bytes; }
  __host__ __device__ static uint32_t off_bars(int P, int NS) { return off_mu(P, NS) + 2 * kMuBytes; }
  __host__ __device__ static uint32_t total(int P, int NS) { return off_bars(P, NS) + 8 * (2 * kStages + 2) + 16; }
};

__device__ __forceinline__ float kl_term(float mu, float lv) {
  // mu^2 + (e^lv - 1 - lv); the bracket by series for |lv| < 0.5 (no cancellation)
  float f;
  if (fabsf(lv) < 0.5f) {
    float p = 1.f / 362880.f;
    p = fmaf(p, lv, 1.f / 40320.f);
    p = fmaf(p, lv, 1.f / 5040.f);
    p = fmaf(p, lv, 1.f / 720.f);
    p = fmaf(p, lv, 1.f / 120.f);
    p = fmaf(p, lv, 1.f / 24.f);
    p = fmaf(p, lv, 1.f / 6.f);
    p = fmaf(p, lv, 0.5f);
    f = lv * lv * p;
  } else {
    f = expm1f(lv) - lv;
  }
  return fmaf(mu, mu, f);
}

template <int H, int ZP>
__global__ void __launch_bounds__(128, 2) k_score(const ScoreParams p) {
  using S = ScoreSmem<H, ZP>;
  constexpr int N2 = S::N2;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int P = p.P, NS = p.NS, M = p.M, W = p.W;

  uint8_t *planes = smem;
  float *ssum = reinterpret_cast<float *>(smem + S::off_ssum(P, NS));
  uint8_t *region = smem + S::off_region(P, NS);   // W1 ring, later h_hi | h_lo
  uint8_t *heads = smem + S::off_heads(P, NS);
  uint8_t *w3s = smem + S::off_w3(P, NS);
  uint8_t *mus = smem + S::off_mu(P, NS);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + S::off_bars(P, NS));
  uint64_t *empty = full + kStages;
  uint64_t *wbar_img = empty + kStages;
  uint64_t *mma_bar = wbar_img + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(mma_bar + 1);

  const int64_t inst = blockIdx.x / p.tiles_per_inst;
  const int64_t r0 = (int64_t)(blockIdx.x % p.tiles_per_inst) * kRows;
  const int nrows = (int)min((int64_t)kRows, p.nw - r0);
  const int64_t s0 = p.t_begin - (W - 1) + r0;     // first sample of the tile
  const int ns_valid = nrows + W - 1;
  const int n_stages_total = (p.nsteps + kStageSteps - 1) / kStageSteps;

  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    mbar_init(wbar_img, 1);
    mbar_init(mma_bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, S::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // ---- producer: weight images (heads, W3 once; W1 through the ring) ----
  if (warp == 1 && lane == 0) {
    mbar_arrive_expect_tx(wbar_img, S::kHeadsBytes + S::kW3Bytes);
    bulk_g2s(heads, p.headsimg, S::kHeadsBytes, wbar_img);
    bulk_g2s(w3s, p.w3img, S::kW3Bytes, wbar_img);
    for (int g = 0; g < kStages && g < n_stages_total; ++g) {
      int steps = min(kStageSteps, p.nsteps - g * kStageSteps);
      uint32_t bytes = steps * S::kStepBytes;
      mbar_arrive_expect_tx(full + g, bytes);
      bulk_g2s(region + g * S::kStageBytes, p.w1img + (size_t)g * S::kStageBytes, bytes, full + g);
    }
  }

  // ---- stage normalised fp16 samples into planes ----
  {
    const int G = M >> 2;  // float4 per sample
    const float *Xi = p.X + inst * p.ld;
    const float *mi = p.mean + inst * M;
    const float *si = p.stdv + inst * M;
    for (int e = tid; e < NS * G; e += blockDim.x) {
      int t = e / G, g = e - t * G;
      uint2 packed = make_uint2(0u, 0u);
      if (t < ns_valid) {
        float4 v = __ldg(reinterpret_cast<const float4 *>(Xi + (s0 + t) * M) + g);
        float4 mu = __ldg(reinterpret_cast<const float4 *>(mi) + g);
        float4 sd = __ldg(reinterpret_cast<const float4 *>(si) + g);
        float z0 = __fdiv_rn(__fsub_rn(v.x, mu.x), sd.x);
        float z1 = __fdiv_rn(__fsub_rn(v.y, mu.y), sd.y);
        float z2 = __fdiv_rn(__fsub_rn(v.z, mu.z), sd.z);
        float z3 = __fdiv_rn(__fsub_rn(v.w, mu.w), sd.w);
        z0 = fminf(fmaxf(z0, -1e4f), 1e4f);
        z1 = fminf(fmaxf(z1, -1e4f), 1e4f);
        z2 = fminf(fmaxf(z2, -1e4f), 1e4f);
        z3 = fminf(fmaxf(z3, -1e4f), 1e4f);
        packed.x = pack_half2(__float2half_rn(z0), __float2half_rn(z1));
        packed.y = pack_half2(__float2half_rn(z2), __float2half_rn(z3));
      }
      int j0 = 4 * g;  // first metric of this float4
      uint8_t *dst = planes + (size_t)(j0 >> 3) * NS * 16 + (size_t)t * 16 + (j0 & 7) * 2;
      *reinterpret_cast<uint2 *>(dst) = packed;
    }
  }
  __syncthreads();
  // per-sample sums s_t = sum_j x_{t,j} (fp32, j ascending) for the MD window sums
  for (int t = tid; t < NS; t += blockDim.x) {
    float s = 0.f;
    for (int pl = 0; pl < P; ++pl) {
      const __half *row = reinterpret_cast<const __half *>(planes + (size_t)pl * NS * 16 + t * 16);
#pragma unroll
      for (int e = 0; e < 8; ++e) s += __half2float(row[e]);
    }
    ssum[t] = s;
  }
  fence_proxy_async_smem();
  __syncthreads();

  // ---- GEMM1 (warp 0 issues, one elected lane) ----
  const uint32_t idesc1 = make_idesc_f16(128, H);
  const uint32_t planes_a = smem_u32(planes);
  const uint32_t plane_bytes = (uint32_t)NS * 16;
  if (warp == 0) {
    for (int q = 0; q < p.nsteps; ++q) {
      const int g = q / kStageSteps, st = g % kStages, u = g / kStages;
      if (q % kStageSteps == 0) {
        mbar_wait(full + st, u & 1);
        tc_fence_after();
      }
      if (lane == 0) {
        const int c0 = 2 * q;
        const int tau0 = c0 / P, p0 = c0 - tau0 * P;
        const uint32_t a_addr = planes_a + p0 * plane_bytes + tau0 * 16;
        const uint32_t a_lbo = (P >= 2) ? plane_bytes : 16u;
        const uint64_t adesc = make_sdesc(a_addr, a_lbo, 128);
        const uint32_t b_addr =
            smem_u32(region + st * S::kStageBytes + (q % kStageSteps) * S::kStepBytes);
        const uint64_t bdesc = make_sdesc(b_addr, 16 * H, 128);
        mma_f16_ss(tmem, adesc, bdesc, idesc1, q > 0 ? 1u : 0u);
        if (q % kStageSteps == kStageSteps - 1 || q == p.nsteps - 1) mma_commit(empty + st);
        if (q == p.nsteps - 1) mma_commit(mma_bar);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    for (int g = kStages; g < n_stages_total; ++g) {
      const int st = g % kStages, u = g / kStages;
      mbar_wait(empty + st, (u - 1) & 1);
      if (lane == 0) {
        int steps = min(kStageSteps, p.nsteps - g * kStageSteps);
        uint32_t bytes = steps * S::kStepBytes;
        mbar_arrive_expect_tx(full + st, bytes);
        bulk_g2s(region + st * S::kStageBytes, p.w1img + (size_t)g * S::kStageBytes, bytes,
                 full + st);
      }
      __syncwarp();
    }
  }

  // ---- epilogue 1: h = tanh(acc + b1) -> hi/lo fp16, K-major canonical A images ----
  mbar_wait(mma_bar, 0);
  tc_fence_after();
  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
  uint8_t *h_hi = region;
  uint8_t *h_lo = region + S::kHBytes;
#pragma unroll 1
  for (int c = 0; c < H; c += 32) {
    float v[32];
    tmem_ld32(lane_addr + c, v);
    tmem_wait_ld();
#pragma unroll
    for (int e8 = 0; e8 < 32; e8 += 8) {
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        float h0 = tanhf(v[e8 + e] + __ldg(p.b1 + c + e8 + e));
        float h1 = tanhf(v[e8 + e + 1] + __ldg(p.b1 + c + e8 + e + 1));
        __half a0 = __float2half_rn(h0), a1 = __float2half_rn(h1);
        __half b0 = __float2half_rn(h0 - __half2float(a0));
        __half b1 = __float2half_rn(h1 - __half2float(a1));
        hi[e >> 1] = pack_half2(a0, a1);
        lo[e >> 1] = pack_half2(b0, b1);
      }
      const size_t off = kmajor_step_offset(tid, c + e8, kRows);
      *reinterpret_cast<uint4 *>(h_hi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4 *>(h_lo + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();

  // ---- GEMM2: heads ----
  if (warp == 0) {
    mbar_wait(wbar_img, 0);
    tc_fence_after();
    if (lane == 0) {
      const uint32_t idesc2 = make_idesc_f16(128, N2);
      const uint32_t hb = smem_u32(heads);
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        const uint32_t ab = smem_u32(pass == 0 ? h_hi : h_lo);
        for (int s = 0; s < H / 16; ++s) {
          uint64_t ad = make_sdesc(ab + s * (32 * kRows), 16 * kRows, 128);
          uint64_t bd = make_sdesc(hb + s * (32 * N2), 16 * N2, 128);
          mma_f16_ss(tmem + H, ad, bd, idesc2, (pass | s) ? 1u : 0u);
        }
      }
      mma_commit(mma_bar);
    }
    __syncwarp();
  }

  // ---- epilogue 2: KL score; mu -> hi/lo fp16 ----
  mbar_wait(mma_bar, 1);
  tc_fence_after();
  float score;
  {
    float v[N2];
    if constexpr (N2 == 32) {
      tmem_ld32(lane_addr + H, v);
    } else {
      tmem_ld16(lane_addr + H, v);
    }
    tmem_wait_ld();
    float acc = 0.f;
    float mu[16];
#pragma unroll
    for (int z = 0; z < 16; ++z) mu[z] = 0.f;
#pragma unroll
    for (int z = 0; z < ZP; ++z) {
      if (z < p.Z) {
        float m = v[z] + __ldg(p.bml + z);
        float l = v[ZP + z] + __ldg(p.bml + ZP + z);
        mu[z] = m;
        acc += kl_term(m, l);
      }
    }
    score = fmaxf(0.5f * acc, 0.f);
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int z = 0; z < 16; z += 2) {
      __half a0 = __float2half_rn(mu[z]), a1 = __float2half_rn(mu[z + 1]);
      __half b0 = __float2half_rn(mu[z] - __half2float(a0));
      __half b1 = __float2half_rn(mu[z + 1] - __half2float(a1));
      hi[z >> 1] = pack_half2(a0, a1);
      lo[z >> 1] = pack_half2(b0, b1);
    }
    uint8_t *mu_hi = mus, *mu_lo = mus + S::kMuBytes;
    *reinterpret_cast<uint4 *>(mu_hi + kmajor_step_offset(tid, 0, kRows)) =
        make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4 *>(mu_hi + kmajor_step_offset(tid, 8, kRows)) =
        make_uint4(hi[4], hi[5], hi[6], hi[7]);
    *reinterpret_cast<uint4 *>(mu_lo + kmajor_step_offset(tid, 0, kRows)) =
        make_uint4(lo[0], lo[1], lo[2], lo[3]);
    *reinterpret_cast<uint4 *>(mu_lo + kmajor_step_offset(tid, 8, kRows)) =
        make_uint4(lo[4], lo[5], lo[6], lo[7]);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();

  // ---- GEMM3: decoder hidden layer (reuses the GEMM1 accumulator columns) ----
  if (warp == 0) {
    tc_fence_after();
    if (lane == 0) {
      const uint32_t idesc3 = make_idesc_f16(128, H);
      const uint32_t bd_addr = smem_u32(w3s);
      mma_f16_ss(tmem, make_sdesc(smem_u32(mus), 16 * kRows, 128), make_sdesc(bd_addr, 16 * H, 128),
                 idesc3, 0u);
      mma_f16_ss(tmem, make_sdesc(smem_u32(mus + S::kMuBytes), 16 * kRows, 128),
                 make_sdesc(bd_addr, 16 * H, 128), idesc3, 1u);
      mma_commit(mma_bar);
    }
    __syncwarp();
  }

  // ---- epilogue 3: MD by the column-sum identity; flag ----
  mbar_wait(mma_bar, 0);
  tc_fence_after();
  float dot = 0.f;
#pragma unroll 1
  for (int c = 0; c < H; c += 32) {
    float v[32];
    tmem_ld32(lane_addr + c, v);
    tmem_wait_ld();
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      float a3 = tanhf(v[e] + __ldg(p.b3 + c + e));
      dot = fmaf(__ldg(p.wbar + c + e), a3, dot);
    }
  }
  float sx = 0.f;
  for (int tau = 0; tau < W; ++tau) sx += ssum[tid + tau];
  const float mdv = (sx - dot - (float)(*p.bbar)) / (float)p.D;

  if (tid < nrows) {
    const int64_t o = inst * p.nw + r0 + tid;
    if (p.scores) p.scores[o] = score;
    if (p.md) p.md[o] = mdv;
    if (p.flags) {
      const double zq = p.z_q_dev ? __ldg(p.z_q_dev) : p.z_q;
      p.flags[o] = ((double)score > zq) ? (mdv >= 0.f ? 1 : -1) : 0;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, S::kTmemCols);
}

template <int H, int ZP>
static enova_status launch_score_t(const ScoreParams &p, cudaStream_t st) {
  using S = ScoreSmem<H, ZP>;
  const uint32_t smem = S::total(p.P, p.NS);
  auto kern = k_score<H, ZP>;
  ENOVA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int64_t grid = p.n_inst * p.tiles_per_inst;
  if (grid <= 0) return ENOVA_OK;
  if (grid > 0x7fffffffLL) {
    set_error("too many tiles for one launch");
    return ENOVA_ERR_UNSUPPORTED;
  }
  ENOVA_LAUNCH(kern, (unsigned)grid, 128, smem, st, p);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

bool pair_path_ok(const DetLayout &L);
enova_status launch_score_pair(const enova_series *s, const DetLayout &L, const void *det_ws,
                               float *scores, float *md, int8_t *flags, double z_q,
                               const double *z_q_dev, cudaStream_t st);

bool rows_path_ok(const DetLayout &L);
enova_status launch_score_rows(const enova_series *s, const DetLayout &L, const void *det_ws,
                               float *scores, float *md, int8_t *flags, double z_q,
                               const double *z_q_dev, cudaStream_t st);

// Kernel choice by shape:
//  * few windows per instance (nw <= kRowModeMaxWindows, e.g. a streaming tick):
//    the instance-batched row kernel (128 independent windows per tile);
//  * else the weight-stationary CTA-pair kernel whenever half of W1 fits in
//    shared memory (all BASELINE configs), else the W1-streaming kernel.
// enova_set_score_kernel(1 | 2 | 3) forces the stream / pair / rows kernel
// (diagnostic, for A/B and parity tests; "rows" only where the row kernel
// supports the shape); 0 restores the choice by shape.
constexpr int64_t kRowModeMaxWindows = 16;
static std::atomic<int> g_forced_kernel{0};   // 0 auto, 1 stream, 2 pair, 3 rows
void set_forced_kernel(int k) { g_forced_kernel.store(k, std::memory_order_relaxed); }
static int forced_kernel() { return g_forced_kernel.load(std::memory_order_relaxed); }

enova_status launch_score(const enova_series *s, const DetLayout &L, const void *det_ws,
                          float *scores, float *md, int8_t *flags, double z_q, const double *z_q_dev,
                          cudaStream_t st) {
  const int f = forced_kernel();
  const int64_t nw = s->t_end - s->t_begin;
  if (rows_path_ok(L) && (f == 3 || (f == 0 && nw <= kRowModeMaxWindows)))
    return launch_score_rows(s, L, det_ws, scores, md, flags, z_q, z_q_dev, st);
  if (f != 1 && pair_path_ok(L))
    return launch_score_pair(s, L, det_ws, scores, md, flags, z_q, z_q_dev, st);
  ScoreParams p{};
  const uint8_t *b = static_cast<const uint8_t *>(det_ws);
  p.X = s->metrics;
  p.ld = s->ld_instance;
  p.n_inst = s->n_instances;
  p.t_begin = s->t_begin;
  p.nw = s->t_end - s->t_begin;
  p.mean = s->norm_mean;
  p.stdv = s->norm_std;
  p.W = L.W;
  p.M = L.M;
  p.P = L.P;
  p.D = L.D;
  p.Z = L.Z;
  p.NS = (kRows + L.W - 1 + 7) / 8 * 8;
  p.tiles_per_inst = (int)((p.nw + kRows - 1) / kRows);
  p.nsteps = L.D / 16;
  p.w1img = b + L.off_w1;
  p.headsimg = b + L.off_heads;
  p.w3img = b + L.off_w3;
  p.b1 = reinterpret_cast<const float *>(b + L.off_b1);
  p.bml = reinterpret_cast<const float *>(b + L.off_bml);
  p.b3 = reinterpret_cast<const float *>(b + L.off_b3);
  p.wbar = reinterpret_cast<const float *>(b + L.off_wbar);
  p.bbar = reinterpret_cast<const double *>(b + L.off_bbar);
  p.scores = scores;
  p.md = md;
  p.flags = flags;
  p.z_q = z_q;
  p.z_q_dev = z_q_dev;
  if (p.nw <= 0) return ENOVA_OK;
  switch (L.H * 100 + L.ZP) {
    case 3208: return launch_score_t<32, 8>(p, st);
    case 3216: return launch_score_t<32, 16>(p, st);
    case 6408: return launch_score_t<64, 8>(p, st);
    case 6416: return launch_score_t<64, 16>(p, st);
    case 12808: return launch_score_t<128, 8>(p, st);
    case 12816: return launch_score_t<128, 16>(p, st);
  }
  set_error("unsupported (H, Z)");
  return ENOVA_ERR_UNSUPPORTED;
}

}  // namespace enova
