// score_rows_sm100.cu -- K2 rows: instance-batched window scorer for ranges with
// few windows per instance -- above all the streaming tick (a-10, P:309
// "executed in streaming computing framework"), where every instance
// contributes exactly one window (the one ending at the newest sample).
//
// The windowed kernels (score_pair_sm100.cu, score_sm100.cu) tile 128
// consecutive windows of ONE instance and exploit the Hankel overlap (each
// sample staged once); with one window per instance they would fill 1 of 128
// MMA rows.  Here the 128 rows of a tile are 128 independent windows
// (row g of the range -> instance g / nw, window g mod nw), so no row is wasted:
//
//   staging : thread r owns row r for the whole tile.  Per K-step q it reads the
//             16 raw fp32 values 16q..16q+15 of its flattened window (the window
//             is W*M contiguous floats), normalises and rounds them exactly as
//             the windowed kernels do (R-4, R-17), and writes them into a ring
//             of K-step A images (128 rows x 16 fp16, K-major canonical, 4 KB);
//             raw loads run kRPF K-steps ahead in registers.
//   GEMM1   : tcgen05.mma cta_group::1 kind::f16 M=128 N=H K=16 per step, A from
//             the ring, B = W1's back-to-back K-step image streamed through a
//             4-stage bulk-copy ring; the TMEM accumulator starts from zero.
//   epilogue: E1 (tanh(acc + b1) -> h hi/lo), GEMM2 (heads), E2 (KL, mu hi/lo),
//             GEMM3 (decoder, from zero in the GEMM1 columns), E3 (MD by the
//             column-sum identity with tanh(acc + b3), flag) -- the same
//             element-wise arithmetic (epilogue.cuh)
//             and the same window-sum association as the windowed CTA-pair
//             kernel, so a streamed window scores bit-identically to the same
//             window scored in a batch.
//
// Envelope: M in {8, 16} (a K-step holds whole samples), H in {32, 64, 128}.
#include <type_traits>

#include "common.cuh"
#include "epilogue.cuh"
#include "layout.h"

namespace enova {

struct RowParams {
  const float *X;
  int64_t ld, t_begin, nw, n_rows;
  const float *mean, *stdv;
  int W, M, D, Z, nsteps;
  const uint8_t *w1img, *headsimg, *w3img;
  const float *b1, *bml, *b3, *wbar;
  const double *bbar;
  float *scores, *md;
  int8_t *flags;
  double z_q;
  const double *z_q_dev;
  // NEXT-1 explain mode: rows are gathered window ids, outputs per metric
  const int64_t *rows;          // [n_rows] window ids g = instance * nw + (t - t_begin)
  int64_t n_win;                // explain mode: ids outside [0, n_win) are invalid (NaN rows)
  const float *wbarm, *bbarm;   // [M][H], [M] per-metric column sums of W_dec2, b_dec2
  float *md_metric;             // [n_rows][M]
};

constexpr int kRR = 128;                 // rows per tile (UMMA M)
constexpr int kRWStageSteps = 4;         // W1 ring: K-steps per stage
constexpr int kRWStages = 4;             // W1 ring depth (row kernel)
constexpr int kMaxWStages = 8;           // RowBars capacity (the stream kernel's W1 ring)
constexpr int kRAStages = 16;            // A ring depth (one K-step each)
constexpr uint32_t kRAStepBytes = kRR * 16 * 2;   // 4 KB
constexpr int kRowThreads = 128;         // thread = row
constexpr int kRThreads = kRowThreads + 64;       // + MMA issuer warp + W1 producer warp
constexpr int kRMmaWarp = 4, kRProdWarp = 5;
constexpr int kRPF = 8;                  // K-steps of raw samples in flight per thread

struct RowBars {
  uint64_t w_full[kMaxWStages], w_empty[kMaxWStages], a_full[kRAStages], a_empty[kRAStages];
  uint64_t wimg, g1_done, h_full, g2_done, mu_full, g3_done;
  uint64_t e3_done;   // split epilogue (stream kernel): the helpers' E3 partials are in smem
  uint64_t e2_done;   // split epilogue, ZP = 16: the helpers' KL terms z = 8..15 are in smem
  uint32_t tmem_slot, pad;
};

struct RowLayoutSm {
  uint32_t region, astage, heads, w3, mubuf, vec, wbarm, bars, total, w_stage_bytes, tmem_cols;
};

__host__ __device__ inline RowLayoutSm row_smem_layout(int H, int ZP,
                                                       uint32_t a_ring_bytes = kRAStages * kRAStepBytes,
                                                       int w_stages = kRWStages,
                                                       int w_stage_steps = kRWStageSteps) {
  RowLayoutSm L;
  uint32_t o = 0;
  auto take = [&](uint32_t b, uint32_t a) {
    o = (o + a - 1) / a * a;
    const uint32_t r = o;
    o += b;
    return r;
  };
  L.w_stage_bytes = (uint32_t)w_stage_steps * 32 * H;
  const uint32_t ring = (uint32_t)w_stages * L.w_stage_bytes, hb = 2u * kRR * H * 2;
  L.region = take(ring > hb ? ring : hb, 1024);      // W1 ring, then h hi | lo
  L.astage = take(a_ring_bytes, 1024);
  L.heads = take((uint32_t)2 * ZP * H * 2, 128);
  L.w3 = take((uint32_t)H * 16 * 2, 128);
  L.mubuf = take(2u * kRR * 16 * 2, 128);
  L.vec = take((3u * H + 2u * ZP) * 4, 16);           // b1 | b3 | w_bar | [bmu | blv]
  L.wbarm = take(16u * H * 4, 16);                     // explain mode: per-metric w_bar [M<=16][H]
  L.bars = take(sizeof(RowBars), 16);
  L.total = o;
  const uint32_t cols = (uint32_t)(H + 2 * ZP);
  L.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : 256;
  return L;
}

// window-sum accumulator with the windowed kernels' association (score_pair:
// s_t per sample; 8-sample block sums ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7));
// blocks alternately into acc0 / acc1 while a 16-sample pair of blocks fits,
// a leftover block into acc0, leftover samples one by one into acc1)
struct WinSum {
  float sprev, p01, a0, p45, acc0, acc1;
  __device__ __forceinline__ void init() { sprev = p01 = a0 = p45 = acc0 = acc1 = 0.f; }
  __device__ __forceinline__ void push(int tau, float s, int W8, int nb2) {
    if (tau >= W8) {
      acc1 += s;
      return;
    }
    const int k = tau & 7;
    if ((k & 1) == 0) {
      sprev = s;
      return;
    }
    const float pr = sprev + s;
    if (k == 1) {
      p01 = pr;
    } else if (k == 3) {
      a0 = p01 + pr;
    } else if (k == 5) {
      p45 = pr;
    } else {
      const float bs = a0 + (p45 + pr);
      const int b = tau >> 3;
      if (b < nb2 && (b & 1)) acc1 += bs;
      else acc0 += bs;
    }
  }
};

// E1 (encoder tanh -> h hi/lo), E2 (KL score,
// mu hi/lo), E3 (MD by the column-sum identity, flag) for one row of a row
// tile -- the CTA-pair kernel's element-wise arithmetic (epilogue.cuh) in the
// same association.  Row threads of warps 0-3; GEMM2/GEMM3 are issued by the
// MMA warp between the h_full / mu_full arrivals and the g2_done / g3_done
// commits of RowBars.
// kPart: 0 = the whole epilogue of the row; 1 / 2 = the row thread / its helper
// thread (a warp of the same TMEM lane quadrant) of a split epilogue: E1 over
// the first / second half of the H columns (element-wise: any split is
// bit-identical), E2 by the row thread only, E3's four interleaved fma chains
// (columns k mod 4) as chains 0, 1 / 2, 3 with the helper's (d2 + d3) passed
// through shared memory (e3part, e3_done) -- the same operations in the same
// order as kPart 0, so the split epilogue is bit-identical to the whole one.
template <int H, int ZP, class Bars, class SxFn, int kPart = 0>
__device__ __forceinline__ void rows_epilogue(uint32_t tmem, int warp, int lane, int r, int64_t row,
                                              bool valid, SxFn &&sx_fn, uint8_t *region,
                                              uint8_t *mubuf, const float *b1cs,
                                              const float *b3s, const float *wbs,
                                              const float *bmls, Bars &B, int Z, int D,
                                              const double *bbar, float *scores, float *md_out,
                                              int8_t *flags, double z_q, const double *z_q_dev,
                                              unsigned long long *tr = nullptr,
                                              const float *wbarm_s = nullptr,
                                              const float *xsum = nullptr,
                                              const float *bbarm = nullptr, float *md_metric = nullptr,
                                              int M = 0, int W = 0, float *e3part = nullptr,
                                              float *e2part = nullptr) {
  auto stamp = [&](int slot) {   // diagnostic; compiled in with -DENOVA_TRACE only
#ifdef ENOVA_TRACE
    if (tr && r == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tr[slot] = t;
    }
#else
    (void)slot;
    (void)tr;
#endif
  };
    // ---- E1: h = tanh(acc + b1) -> hi/lo fp16 A images ----
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    mbar_wait_sleep(&B.g1_done, 0, 256);   // (the K loop: long; polling would slow its warps)
    stamp(6);
    tc_fence_after();
    constexpr int kC0 = kPart == 2 ? H / 2 : 0, kC1 = kPart == 1 ? H / 2 : H;
#pragma unroll 1
    for (int c16 = kC0; c16 < kC1; c16 += 16) {
      float v[16], bc[16];
      tmem_ld16(lane_addr + c16, v);
      lds16(b1cs + c16, bc);
      tmem_wait_ld();
#pragma unroll
      for (int e8 = 0; e8 < 16; e8 += 8) {
        uint32_t hi[4], lo[4];
        e1_tanh_split8_b(v + e8, bc + e8, hi, lo);   // acc = W1 x (from zero)
        const size_t off = kmajor_step_offset(r, c16 + e8, kRR);
        *reinterpret_cast<uint4 *>(region + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4 *>(region + kRR * H * 2 + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
    tmem_wait_st();
    fence_proxy_async_smem();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&B.h_full);
    stamp(7);
    if constexpr (kPart == 2 && ZP == 16) {
      // helper: E2 for z = 8..15 -- the KL terms into e2part (the row thread sums
      // all 16 in z order), mu's hi / lo pairs of that K half into the GEMM3 image
      mbar_wait_sleep(&B.g2_done, 0, 32);
      tc_fence_after();
      float vm[8], vl[8];
      tmem_ld8(lane_addr + H + 8, vm);
      tmem_ld8(lane_addr + H + ZP + 8, vl);
      tmem_wait_ld();
      float mz[8];
#pragma unroll
      for (int z = 0; z < 8; ++z) {
        const float m = vm[z] + bmls[8 + z];
        const float t = kl_term2(m, vl[z] + bmls[ZP + 8 + z]);
        mz[z] = 8 + z < Z ? m : 0.f;
        e2part[z * kRR + r] = 8 + z < Z ? t : 0.f;
      }
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int z = 0; z < 8; z += 2) {
        const uint32_t hp = cvt_pack_f16x2(mz[z], mz[z + 1]);
        const float2 hf = __half22float2(*reinterpret_cast<const __half2 *>(&hp));
        hi[z >> 1] = hp;
        lo[z >> 1] = cvt_pack_f16x2(mz[z] - hf.x, mz[z + 1] - hf.y);
      }
      const size_t off1 = kmajor_step_offset(r, 8, kRR);
      *reinterpret_cast<uint4 *>(mubuf + off1) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4 *>(mubuf + kRR * 32 + off1) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&B.mu_full);
        mbar_arrive(&B.e2_done);
      }
    }
    if constexpr (kPart == 2) {
      // helper: E3 chains 2, 3 -> e3part
      mbar_wait_sleep(&B.g3_done, 0, 32);
      tc_fence_after();
      float d2 = 0.f, d3 = 0.f;
#pragma unroll 1
      for (int c32 = 0; c32 < H; c32 += 32) {
        float v[32];
        tmem_ld16(lane_addr + c32, *reinterpret_cast<float(*)[16]>(&v[0]));
        tmem_ld16(lane_addr + c32 + 16, *reinterpret_cast<float(*)[16]>(&v[16]));
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
          const float4 ww = *reinterpret_cast<const float4 *>(wbs + c32 + k);
          const float4 bb = *reinterpret_cast<const float4 *>(b3s + c32 + k);
          d2 = fmaf(ww.z, tanh_mufu(v[k + 2] + bb.z), d2);
          d3 = fmaf(ww.w, tanh_mufu(v[k + 3] + bb.w), d3);
        }
      }
      e3part[r] = d2 + d3;
      __syncwarp();
      if (lane == 0) mbar_arrive(&B.e3_done);
      return;
    }

    // ---- E2: KL score; mu -> hi/lo fp16 ----
    mbar_wait_sleep(&B.g2_done, 0, kPart ? 32 : 64);
    stamp(8);
    tc_fence_after();
    float score;
    {
      const uint32_t hacc = lane_addr + H;
      float vm[ZP], vl[ZP];
      if constexpr (ZP == 16) {
        tmem_ld16(hacc, vm);
        tmem_ld16(hacc + ZP, vl);
      } else {
        tmem_ld8(hacc, vm);
        tmem_ld8(hacc + ZP, vl);
      }
      tmem_wait_ld();
      stamp(12);
      // every term first (branch-free: independent chains the scheduler can
      // interleave), then the sum in z order (the same additions as before:
      // + 0.f for z >= Z leaves kl unchanged, kl >= +0)
      // (split, ZP = 16: this thread takes z = 0..7, its helper z = 8..15)
      constexpr int kZ1 = (kPart == 1 && ZP == 16) ? 8 : ZP;
      float mz[ZP], tz[ZP];
#pragma unroll
      for (int z = 0; z < kZ1; ++z) {
        const float m = vm[z] + bmls[z];
        const float t = kl_term2(m, vl[z] + bmls[ZP + z]);
        mz[z] = z < Z ? m : 0.f;
        tz[z] = z < Z ? t : 0.f;
      }
      uint32_t hi[8], lo[8];
#pragma unroll
      for (int z = 0; z < kZ1; z += 2) {
        const float m2[2] = {mz[z], mz[z + 1]};
        const uint32_t hp = cvt_pack_f16x2(m2[0], m2[1]);
        const float2 hf = __half22float2(*reinterpret_cast<const __half2 *>(&hp));
        hi[z >> 1] = hp;
        lo[z >> 1] = cvt_pack_f16x2(m2[0] - hf.x, m2[1] - hf.y);
      }
      const size_t off0 = kmajor_step_offset(r, 0, kRR);
      *reinterpret_cast<uint4 *>(mubuf + off0) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4 *>(mubuf + kRR * 32 + off0) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      if constexpr (ZP == 16 && kZ1 == ZP) {
        const size_t off1 = kmajor_step_offset(r, 8, kRR);
        *reinterpret_cast<uint4 *>(mubuf + off1) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
        *reinterpret_cast<uint4 *>(mubuf + kRR * 32 + off1) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
      }
      stamp(13);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      stamp(14);
      if (lane == 0) mbar_arrive(&B.mu_full);
      if constexpr (kZ1 < ZP) {   // the helper's terms, then the sum in z order
        mbar_wait(&B.e2_done, 0);
#pragma unroll
        for (int z = kZ1; z < ZP; ++z) tz[z] = e2part[(z - kZ1) * kRR + r];
      }
      float kl = 0.f;
#pragma unroll
      for (int z = 0; z < ZP; ++z) kl += tz[z];
      score = fmaxf(0.5f * kl, 0.f);
    }
    stamp(9);

    // ---- E3: MD by the column-sum identity; flag ----
    const float sx = sx_fn();   // window sum (may be computed here, off the E1 path)
    mbar_wait_sleep(&B.g3_done, 0, kPart ? 32 : 64);
    stamp(10);
    tc_fence_after();
    float d4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
    for (int c32 = 0; c32 < H; c32 += 32) {
      float v[32];
      tmem_ld16(lane_addr + c32, *reinterpret_cast<float(*)[16]>(&v[0]));
      tmem_ld16(lane_addr + c32 + 16, *reinterpret_cast<float(*)[16]>(&v[16]));
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        const float4 ww = *reinterpret_cast<const float4 *>(wbs + c32 + k);
        const float4 bb = *reinterpret_cast<const float4 *>(b3s + c32 + k);
        d4[0] = fmaf(ww.x, tanh_mufu(v[k] + bb.x), d4[0]);   // acc = W3 mu (from zero)
        d4[1] = fmaf(ww.y, tanh_mufu(v[k + 1] + bb.y), d4[1]);
        if constexpr (kPart == 0) {
          d4[2] = fmaf(ww.z, tanh_mufu(v[k + 2] + bb.z), d4[2]);
          d4[3] = fmaf(ww.w, tanh_mufu(v[k + 3] + bb.w), d4[3]);
        }
      }
    }
    float d23;
    if constexpr (kPart == 1) {
      mbar_wait(&B.e3_done, 0);
      d23 = e3part[r];
    } else {
      d23 = d4[2] + d4[3];
    }
    const float dot = (d4[0] + d4[1]) + d23;
    const float mdv = (sx - dot - (float)(*bbar)) / (float)D;
    if (wbarm_s) {
      // NEXT-1: per-metric mean difference MD_j = (sum_tau x_{tau,j} - w_bar_j . a3 -
      // b_bar_j) / W with w_bar_j = sum_tau W_dec2[tau M + j, :] (the column-sum
      // identity per metric; MD = mean_j MD_j).  Accurate tanh here (explain path).
      float dm[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) dm[j] = 0.f;
#pragma unroll 1
      for (int c16 = 0; c16 < H; c16 += 16) {
        float v[16];
        tmem_ld16(lane_addr + c16, v);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float a3 = tanh_2mufu(v[k] + b3s[c16 + k]);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < M) dm[j] = fmaf(wbarm_s[j * H + c16 + k], a3, dm[j]);
        }
      }
      if (valid) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < M) md_metric[row * M + j] = (xsum[j] - dm[j] - __ldg(bbarm + j)) / (float)W;
      }
    }
    if (valid) {
      if (scores) scores[row] = score;
      if (md_out) md_out[row] = mdv;
      if (flags) {
        const double zq = z_q_dev ? __ldg(z_q_dev) : z_q;
        flags[row] = ((double)score > zq) ? (mdv >= 0.f ? 1 : -1) : 0;
      }
    }
    stamp(11);
}

template <int H, int ZP, int M, bool kExplain>
__global__ void __launch_bounds__(kRThreads, 1) k_score_rows(const RowParams p) {
  constexpr int N2 = 2 * ZP;
  extern __shared__ __align__(1024) uint8_t smem[];
  const RowLayoutSm SL = row_smem_layout(H, ZP);
  float *wbarm_s = reinterpret_cast<float *>(smem + SL.wbarm);
  if (kExplain)
    for (int i = threadIdx.x; i < M * H; i += blockDim.x) wbarm_s[i] = p.wbarm[i];
  uint8_t *region = smem + SL.region;
  uint8_t *astage = smem + SL.astage;
  uint8_t *heads = smem + SL.heads;
  uint8_t *w3s = smem + SL.w3;
  uint8_t *mubuf = smem + SL.mubuf;
  RowBars &B = *reinterpret_cast<RowBars *>(smem + SL.bars);
  float *b1s = reinterpret_cast<float *>(smem + SL.vec);
  float *b3s = b1s + H;
  float *wbs = b3s + H;
  float *bmls = wbs + H;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t row0 = (int64_t)blockIdx.x * kRR;
  const int n_wstages = (p.nsteps + kRWStageSteps - 1) / kRWStageSteps;

  if (tid == 0) {
    for (int i = 0; i < kRWStages; ++i) {
      mbar_init(&B.w_full[i], 1);
      mbar_init(&B.w_empty[i], 1);
    }
    for (int i = 0; i < kRAStages; ++i) {
      mbar_init(&B.a_full[i], kRowThreads / 32);
      mbar_init(&B.a_empty[i], 1);
    }
    mbar_init(&B.wimg, 1);
    mbar_init(&B.g1_done, 1);
    mbar_init(&B.h_full, kRowThreads / 32);
    mbar_init(&B.g2_done, 1);
    mbar_init(&B.mu_full, kRowThreads / 32);
    mbar_init(&B.g3_done, 1);
    fence_mbar_init();
  }
  for (int i = tid; i < H; i += blockDim.x) {
    b1s[i] = __fmul_rn(p.b1[i], kTwoLog2e);   // E1 exponent bias (GEMM1 starts from zero)
    b3s[i] = p.b3[i];
    wbs[i] = p.wbar[i];
  }
  for (int i = tid; i < N2; i += blockDim.x) bmls[i] = p.bml[i];
  for (int i = tid; i < (int)(2 * kRR * 16 * 2 / 16); i += blockDim.x)   // mu K-half 1 = 0 if ZP = 8
    reinterpret_cast<uint4 *>(mubuf)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tmem_alloc(&B.tmem_slot, SL.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem_slot;

  if (warp == kRProdWarp) {
    // ---------------- W1 ring producer (+ heads / W3 images once) ----------------
    if (lane == 0) {
      const uint32_t hb = (uint32_t)N2 * H * 2, w3b = (uint32_t)H * 16 * 2;
      mbar_arrive_expect_tx(&B.wimg, hb + w3b);
      bulk_g2s(heads, p.headsimg, hb, &B.wimg);
      bulk_g2s(w3s, p.w3img, w3b, &B.wimg);
      for (int g = 0; g < n_wstages; ++g) {
        const int st = g % kRWStages, u = g / kRWStages;
        if (g >= kRWStages) mbar_wait(&B.w_empty[st], (u - 1) & 1);
        const int steps = min(kRWStageSteps, p.nsteps - g * kRWStageSteps);
        const uint32_t bytes = (uint32_t)steps * 32 * H;
        mbar_arrive_expect_tx(&B.w_full[st], bytes);
        bulk_g2s(region + st * SL.w_stage_bytes, p.w1img + (size_t)g * SL.w_stage_bytes, bytes,
                 &B.w_full[st]);
      }
    }
  } else if (warp == kRMmaWarp) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc1 = make_idesc_f16(128, H);
    const uint32_t aa = smem_u32(astage), ra = smem_u32(region);
    // one iteration per W1 stage, its K-steps unrolled (straight-line waits and
    // commits: see k_stream_rows)
    const int n_groups = (p.nsteps + kRWStageSteps - 1) / kRWStageSteps;
    for (int g = 0; g < n_groups; ++g) {
      const int st = g % kRWStages;
      mbar_wait(&B.w_full[st], (g / kRWStages) & 1);
      const int steps = min(kRWStageSteps, p.nsteps - g * kRWStageSteps);
#pragma unroll
      for (int j = 0; j < kRWStageSteps; ++j) {
        if (j < steps) {
          const int q = g * kRWStageSteps + j, a = q % kRAStages;
          mbar_wait(&B.a_full[a], (q / kRAStages) & 1);
          tc_fence_after();
          const uint64_t ad = make_sdesc(aa + a * kRAStepBytes, kRR * 16, 128);
          const uint64_t bd = make_sdesc(ra + st * SL.w_stage_bytes + j * 32 * H, 16 * H, 128);
          mma_f16_warp(tmem, ad, bd, idesc1, q > 0 ? 1u : 0u);
          mma_commit_warp(&B.a_empty[a]);
        }
      }
      mma_commit_warp(&B.w_empty[st]);
    }
    mma_commit_warp(&B.g1_done);
    // heads GEMM2: [mu | lv] = (h_hi + h_lo) [Wmu | Wlv]^T, accumulator at column H
    mbar_wait(&B.wimg, 0);
    mbar_wait(&B.h_full, 0);
    tc_fence_after();
    if (lane == 0) {
      const uint32_t idesc2 = make_idesc_f16(128, N2);
      const uint32_t hb = smem_u32(heads);
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        const uint32_t ab = smem_u32(region) + (uint32_t)pass * (kRR * H * 2);
        for (int s = 0; s < H / 16; ++s) {
          const uint64_t ad = make_sdesc(ab + s * (32 * kRR), 16 * kRR, 128);
          const uint64_t bd = make_sdesc(hb + s * (32 * N2), 16 * N2, 128);
          mma_f16_ss(tmem + H, ad, bd, idesc2, (pass | s) ? 1u : 0u);
        }
      }
      mma_commit(&B.g2_done);
    }
    __syncwarp();
    // decoder GEMM3 into the GEMM1 columns (re-armed with b3 by E1)
    mbar_wait(&B.mu_full, 0);
    tc_fence_after();
    if (lane == 0) {
      const uint32_t idesc3 = make_idesc_f16(128, H);
      const uint64_t bd = make_sdesc(smem_u32(w3s), 16 * H, 128);
      mma_f16_ss(tmem, make_sdesc(smem_u32(mubuf), 16 * kRR, 128), bd, idesc3, 0u);
      mma_f16_ss(tmem, make_sdesc(smem_u32(mubuf) + kRR * 16 * 2, 16 * kRR, 128), bd, idesc3, 1u);
      mma_commit(&B.g3_done);
    }
    __syncwarp();
  } else {
    // ---------------- row threads: staging, then the epilogues ----------------
    const int r = tid;
    const int64_t row = row0 + r;
    const bool valid = row < p.n_rows;
    const int64_t gid_in = kExplain ? (valid ? __ldg(p.rows + row) : 0) : row;   // window id
    // explain mode: an id outside the series' windows is scored as window 0
    // (in-bounds loads) and its outputs are overwritten with NaN below
    const bool id_ok = !kExplain || (gid_in >= 0 && gid_in < p.n_win);
    const int64_t gid = id_ok ? gid_in : 0;
    const int64_t inst = valid ? gid / p.nw : 0;
    const int64_t wi = valid ? gid - inst * p.nw : 0;
    float xsum[kExplain ? M : 1];
#pragma unroll
    for (int j = 0; j < (kExplain ? M : 1); ++j) xsum[j] = 0.f;
    float mu[M], sd[M], rc[M];
#pragma unroll
    for (int j = 0; j < M; j += 4) {
      const float4 a = __ldg(reinterpret_cast<const float4 *>(p.mean + inst * M + j));
      const float4 b = __ldg(reinterpret_cast<const float4 *>(p.stdv + inst * M + j));
      mu[j] = a.x; mu[j + 1] = a.y; mu[j + 2] = a.z; mu[j + 3] = a.w;
      sd[j] = b.x; sd[j + 1] = b.y; sd[j + 2] = b.z; sd[j + 3] = b.w;
    }
#pragma unroll
    for (int j = 0; j < M; ++j) rc[j] = __frcp_rn(sd[j]);
    const int W8 = p.W & ~7, nb2 = 2 * (W8 / 16);
    WinSum ws;
    ws.init();
    const float *src = p.X + inst * p.ld + (p.t_begin + wi - (p.W - 1)) * M;
    float4 buf[kRPF][4];
#pragma unroll
    for (int u = 0; u < kRPF; ++u)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        buf[u][k] = (valid && u < p.nsteps)
                        ? __ldg(reinterpret_cast<const float4 *>(src + 16 * u) + k)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
    uint8_t *arow = astage + (r >> 3) * 128 + (r & 7) * 16;
    for (int q0 = 0; q0 < p.nsteps; q0 += kRPF) {
#pragma unroll
      for (int u = 0; u < kRPF; ++u) {
        const int q = q0 + u;
        if (q < p.nsteps) {
          float x[16];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            x[4 * k] = buf[u][k].x; x[4 * k + 1] = buf[u][k].y;
            x[4 * k + 2] = buf[u][k].z; x[4 * k + 3] = buf[u][k].w;
          }
          // refill this slot with K-step q + kRPF (consumed kRPF steps later)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            buf[u][k] = (valid && q + kRPF < p.nsteps)
                            ? __ldg(reinterpret_cast<const float4 *>(src + 16 * (q + kRPF)) + k)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
          uint32_t pk[8];
          float xr[16];
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const int j0 = e % M, j1 = (e + 1) % M;
            const float z0 = fminf(fmaxf(div_rn(__fsub_rn(x[e], mu[j0]), sd[j0], rc[j0]), -1e4f), 1e4f);
            const float z1 = fminf(fmaxf(div_rn(__fsub_rn(x[e + 1], mu[j1]), sd[j1], rc[j1]), -1e4f), 1e4f);
            const uint32_t h2 = valid ? cvt_pack_f16x2(z0, z1) : 0u;
            pk[e >> 1] = h2;
            const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&h2));
            xr[e] = f.x;
            xr[e + 1] = f.y;
            if constexpr (kExplain) {   // per-metric window sums, tau ascending
              xsum[j0] += f.x;
              xsum[j1] += f.y;
            }
          }
          const int a = q % kRAStages;
          if (q >= kRAStages) mbar_wait(&B.a_empty[a], ((q / kRAStages) - 1) & 1);
          uint8_t *dst = arow + a * kRAStepBytes;
          *reinterpret_cast<uint4 *>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4 *>(dst + kRR * 16) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&B.a_full[a]);
          // per-sample sums s_t (fp16 values, the windowed kernels' association)
          float pg[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) pg[k] = (xr[4 * k] + xr[4 * k + 1]) + (xr[4 * k + 2] + xr[4 * k + 3]);
          if constexpr (M == 16) {
            ws.push(q, (pg[0] + pg[1]) + (pg[2] + pg[3]), W8, nb2);
          } else {   // M == 8: two samples per K-step
            ws.push(2 * q, pg[0] + pg[1], W8, nb2);
            ws.push(2 * q + 1, pg[2] + pg[3], W8, nb2);
          }
        }
      }
    }
    const float sx = ws.acc0 + ws.acc1;

    rows_epilogue<H, ZP>(tmem, warp, lane, r, row, valid, [&]() { return sx; }, region, mubuf,
                         b1s, b3s, wbs, bmls, B,
                         p.Z, p.D, p.bbar, p.scores, p.md, p.flags, p.z_q, p.z_q_dev, nullptr,
                         kExplain ? wbarm_s : nullptr, kExplain ? xsum : nullptr, p.bbarm,
                         p.md_metric, M, p.W);
    if (kExplain && valid && !id_ok) {   // same thread wrote the row: program order
      const float qnan = __int_as_float(0x7fc00000);
      if (p.scores) p.scores[row] = qnan;
      if (p.md) p.md[row] = qnan;
#pragma unroll
      for (int j = 0; j < M; ++j) p.md_metric[row * M + j] = qnan;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, SL.tmem_cols);
}

template <int H, int ZP, int M, bool kExplain>
static enova_status launch_rows_t(const RowParams &p, cudaStream_t st) {
  const RowLayoutSm SL = row_smem_layout(H, ZP);
  auto kern = k_score_rows<H, ZP, M, kExplain>;
  static thread_local int cached_dev = -1;
  int dev = 0;
  ENOVA_CUDA_TRY(cudaGetDevice(&dev));
  if (dev != cached_dev) {
    ENOVA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SL.total));
    cached_dev = dev;
  }
  const int64_t tiles = (p.n_rows + kRR - 1) / kRR;
  if (tiles <= 0) return ENOVA_OK;
  if (tiles > 0x7fffffffLL) {
    set_error("too many rows for one launch");
    return ENOVA_ERR_UNSUPPORTED;
  }
  ENOVA_LAUNCH(kern, (unsigned)tiles, kRThreads, SL.total, st, p);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

bool rows_path_ok(const DetLayout &L) {
  return (L.M == 8 || L.M == 16) && row_smem_layout(L.H, L.ZP).total <= 227 * 1024;
}

template <bool kExplain>
static enova_status dispatch_rows(const DetLayout &L, const RowParams &p, cudaStream_t st) {
  switch (L.M * 10000 + L.H * 100 + L.ZP) {
    case 83208: return launch_rows_t<32, 8, 8, kExplain>(p, st);
    case 83216: return launch_rows_t<32, 16, 8, kExplain>(p, st);
    case 86408: return launch_rows_t<64, 8, 8, kExplain>(p, st);
    case 86416: return launch_rows_t<64, 16, 8, kExplain>(p, st);
    case 92808: return launch_rows_t<128, 8, 8, kExplain>(p, st);
    case 92816: return launch_rows_t<128, 16, 8, kExplain>(p, st);
    case 163208: return launch_rows_t<32, 8, 16, kExplain>(p, st);
    case 163216: return launch_rows_t<32, 16, 16, kExplain>(p, st);
    case 166408: return launch_rows_t<64, 8, 16, kExplain>(p, st);
    case 166416: return launch_rows_t<64, 16, 16, kExplain>(p, st);
    case 172808: return launch_rows_t<128, 8, 16, kExplain>(p, st);
    case 172816: return launch_rows_t<128, 16, 16, kExplain>(p, st);
  }
  set_error("unsupported (M, H, Z) for the row kernel");
  return ENOVA_ERR_UNSUPPORTED;
}

static RowParams row_params(const enova_series *s, const DetLayout &L, const void *det_ws) {
  RowParams p{};
  const uint8_t *b = static_cast<const uint8_t *>(det_ws);
  p.X = s->metrics;
  p.ld = s->ld_instance;
  p.t_begin = s->t_begin;
  p.nw = s->t_end - s->t_begin;
  p.n_rows = s->n_instances * p.nw;
  p.mean = s->norm_mean;
  p.stdv = s->norm_std;
  p.W = L.W;
  p.M = L.M;
  p.D = L.D;
  p.Z = L.Z;
  p.nsteps = L.D / 16;
  p.w1img = b + L.off_w1;
  p.headsimg = b + L.off_heads;
  p.w3img = b + L.off_w3;
  p.b1 = reinterpret_cast<const float *>(b + L.off_b1);
  p.bml = reinterpret_cast<const float *>(b + L.off_bml);
  p.b3 = reinterpret_cast<const float *>(b + L.off_b3);
  p.wbar = reinterpret_cast<const float *>(b + L.off_wbar);
  p.bbar = reinterpret_cast<const double *>(b + L.off_bbar);
  p.wbarm = reinterpret_cast<const float *>(b + L.off_wbarm);
  p.bbarm = reinterpret_cast<const float *>(b + L.off_bbarm);
  return p;
}

enova_status launch_score_rows(const enova_series *s, const DetLayout &L, const void *det_ws,
                               float *scores, float *md, int8_t *flags, double z_q,
                               const double *z_q_dev, cudaStream_t st) {
  RowParams p = row_params(s, L, det_ws);
  p.scores = scores;
  p.md = md;
  p.flags = flags;
  p.z_q = z_q;
  p.z_q_dev = z_q_dev;
  if (p.nw <= 0 || p.n_rows == 0) return ENOVA_OK;
  return dispatch_rows<false>(L, p, st);
}

// NEXT-1: explain the windows whose ids are listed in rows_dev (g = instance *
// nw + (t - t_begin) within the series range): per-metric MD plus the window's
// score and MD (bit-identical to the batch kernels), one row each.
enova_status launch_explain_rows(const enova_series *s, const DetLayout &L, const void *det_ws,
                                 const int64_t *rows_dev, int64_t n_rows, float *md_metric,
                                 float *scores, float *md, cudaStream_t st) {
  RowParams p = row_params(s, L, det_ws);
  p.n_rows = n_rows;
  p.rows = rows_dev;
  p.n_win = s->n_instances * p.nw;
  p.md_metric = md_metric;
  p.scores = scores;
  p.md = md;
  if (n_rows == 0) return ENOVA_OK;
  return dispatch_rows<true>(L, p, st);
}

// =====================================================================
// Ingest-normalised streaming ring (a-10 fast path; include/enova.h
// enova_stream_*).  Each new sample is normalised ONCE on ingest with the frozen
// calibration statistics (R-4) -- exactly the windowed kernels'
// arithmetic: x = fp16_RN(clamp(RN((X - mean) / std), +-1e4)) -- and kept as
// fp16 in a mirror ring [N][2W][M] (the W samples of the window ending at tick
// k are contiguous: slots (k+1) mod W ..) next to its fp32 sample sum
// s = sum_j x_j (the windowed kernels' association) in [N][2W].  A tick needs
// no normalisation: the GEMM1 A operand of 4 K-steps for 128 instances is ONE
// 16 KB bulk copy of the tile's contiguous range of the tiled canonical ring
// (below), consumed by no-swizzle K-major UMMA descriptors, so the kernel is a
// bulk-copy -> tcgen05 pipeline plus the shared epilogue.
// =====================================================================

// The fp16 ring is TILED in the UMMA's no-swizzle K-major canonical layout:
//   [tile of 128 instances][2W slots][M/8 halves][128 rows][8 fp16]
// so one slot of one tile is M/8 contiguous 2 KB half-blocks, and the A
// operand of ANY run of K-steps of a tile's windows is ONE contiguous range (a
// window = slots [s0, s0 + W) of the mirror ring; K-step q = half-blocks
// s0 M/8 + 2q, +1): the stream kernel moves it with plain 16 KB bulk copies
// instead of 2-D TMA boxes of 128 scattered 128-B rows (which paced the K loop
// at ~0.65 us per 4 K-steps).  The fp32 sample-sum ring stays [N][pitch]; its
// pitch is padded off a power of two (consecutive instances on different DRAM
// channels).
__host__ __device__ inline int64_t sums_pitch(int W) { return (int64_t)2 * W + 8; }
__host__ __device__ inline size_t stream_elem(int64_t i, int s, int j, int W, int M) {
  return ((((size_t)(i >> 7) * 2 * W + s) * (size_t)(M >> 3) + (size_t)(j >> 3)) << 10) +
         ((size_t)(i & 127) << 3) + (size_t)(j & 7);
}
size_t stream_sums_offset(int64_t n, int W, int M) {
  const size_t tiles = (size_t)((n + 127) / 128);
  return align_up(tiles * 128 * 2 * W * M * 2, 256);
}
size_t stream_ring_bytes(int64_t n, int W, int M) {
  return stream_sums_offset(n, W, M) + (size_t)n * sums_pitch(W) * 4;
}

template <int G>
__global__ void k_stream_push(__half *__restrict__ ring16, float *__restrict__ sums, int64_t n,
                              int W, const float *__restrict__ sample,
                              const float *__restrict__ mean, const float *__restrict__ stdv,
                              int64_t tick) {
  constexpr int M = 4 * G;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int slot = (int)(tick % W);
  const float4 *xs = reinterpret_cast<const float4 *>(sample + i * M);
  const float4 *ms = reinterpret_cast<const float4 *>(mean + i * M);
  const float4 *ss = reinterpret_cast<const float4 *>(stdv + i * M);
  float pg[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    __half *r0 = ring16 + stream_elem(i, slot, 4 * g, W, M);       // tiled canonical layout
    __half *r1 = ring16 + stream_elem(i, slot + W, 4 * g, W, M);   // the mirror slot
    const float4 v = __ldg(xs + g), mu = __ldg(ms + g), sd = __ldg(ss + g);
    const float z0 = fminf(fmaxf(div_rn(__fsub_rn(v.x, mu.x), sd.x, __frcp_rn(sd.x)), -1e4f), 1e4f);
    const float z1 = fminf(fmaxf(div_rn(__fsub_rn(v.y, mu.y), sd.y, __frcp_rn(sd.y)), -1e4f), 1e4f);
    const float z2 = fminf(fmaxf(div_rn(__fsub_rn(v.z, mu.z), sd.z, __frcp_rn(sd.z)), -1e4f), 1e4f);
    const float z3 = fminf(fmaxf(div_rn(__fsub_rn(v.w, mu.w), sd.w, __frcp_rn(sd.w)), -1e4f), 1e4f);
    uint2 pk;
    pk.x = cvt_pack_f16x2(z0, z1);
    pk.y = cvt_pack_f16x2(z2, z3);
    *reinterpret_cast<uint2 *>(r0) = pk;
    *reinterpret_cast<uint2 *>(r1) = pk;
    const float2 f01 = __half22float2(*reinterpret_cast<const __half2 *>(&pk.x));
    const float2 f23 = __half22float2(*reinterpret_cast<const __half2 *>(&pk.y));
    pg[g] = (f01.x + f01.y) + (f23.x + f23.y);
  }
  // balanced tree over the G groups (= the windowed kernels' lane xor tree)
#pragma unroll
  for (int w = 1; w < G; w <<= 1)
#pragma unroll
    for (int k = 0; k + w < G; k += 2 * w) pg[k] = pg[k] + pg[k + w];
  sums[(size_t)i * sums_pitch(W) + slot] = pg[0];
  sums[(size_t)i * sums_pitch(W) + slot + W] = pg[0];
}

enova_status stream_push(void *ring, int64_t n, int W, int M, const float *sample,
                         const float *mean, const float *stdv, int64_t tick, cudaStream_t st) {
  if (n == 0) return ENOVA_OK;
  __half *r16 = static_cast<__half *>(ring);
  float *sums = reinterpret_cast<float *>(static_cast<uint8_t *>(ring) + stream_sums_offset(n, W, M));
  const int threads = 128;
  const unsigned blocks = (unsigned)((n + threads - 1) / threads);
  switch (M) {
    case 8: ENOVA_LAUNCH(k_stream_push<2>, blocks, threads, 0, st, r16, sums, n, W, sample, mean, stdv, tick); break;
    case 16: ENOVA_LAUNCH(k_stream_push<4>, blocks, threads, 0, st, r16, sums, n, W, sample, mean, stdv, tick); break;
    case 32: ENOVA_LAUNCH(k_stream_push<8>, blocks, threads, 0, st, r16, sums, n, W, sample, mean, stdv, tick); break;
    case 64: ENOVA_LAUNCH(k_stream_push<16>, blocks, threads, 0, st, r16, sums, n, W, sample, mean, stdv, tick); break;
    default: set_error("stream ring: M must be 8, 16, 32 or 64"); return ENOVA_ERR_UNSUPPORTED;
  }
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

// A ring of the stream kernel: stages of kSAK K-steps = one bulk copy of the
// tile's contiguous canonical-layout range (kSAK x [2 halves][128 rows][16 B]);
// the W1 ring's stages hold the same kSAK K-steps.
#ifndef ENOVA_SAK
#define ENOVA_SAK 8
#endif
constexpr int kSAK = ENOVA_SAK;
// A group needs one A and one W1 stage: the two rings get the same depth, as
// deep as shared memory allows (192 KB in flight per SM; with the MMA warp's
// straight-line group loop a 4-K-step group takes ~410 cycles, the 4 MMAs' own cost).
constexpr int kSAStages = 24 / kSAK;
constexpr int kSWStages = kSAStages;   // the stream kernel's W1 ring
static_assert(kSWStages <= kMaxWStages && kSAStages <= kRAStages, "RowBars capacity");
constexpr int kSAWarp = 6;                        // A producer warp
constexpr int kSHelperWarp0 = 7;                  // warps 7-10: epilogue helpers (TMEM quadrant warp & 3)
constexpr int kSThreads = kRThreads + 32 + kRowThreads;
// the helpers' E3 partials reuse the GEMM3 A image (mubuf): GEMM3 has completed
// (g3_done) before any helper writes
__device__ __forceinline__ float *e3part_of(uint8_t *smem, const RowLayoutSm &SL) {
  return reinterpret_cast<float *>(smem + SL.mubuf);
}
// the helpers' KL terms z = 8..15 ([8][128] floats) in the explain-only w_bar
// region, unused by the stream kernel
__device__ __forceinline__ float *e2part_of(uint8_t *smem, const RowLayoutSm &SL) {
  return reinterpret_cast<float *>(smem + SL.wbarm);
}
constexpr uint32_t kSAStageBytes = kRR * 32 * kSAK;

struct StreamParams {
  const float *sums;        // [N][2W] fp32 sample sums
  int64_t n, tick;
  int W, M, D, Z, nsteps;
  const uint8_t *w1img, *headsimg, *w3img;
  const float *b1, *bml, *b3, *wbar;
  const double *bbar;
  float *scores, *md;
  int8_t *flags;
  const double *z_q_dev;
  unsigned long long *trace;   // diagnostic timeline of CTA 0 (NULL normally)
  // fused ingest (enova_stream_step): push sample [N][M] of `tick` before scoring
  const float *sample, *mean, *stdv;
  __half *ring16;
  float *sums_w;
};

// Window sum of one row computed by a whole warp with coalesced loads: lane l
// holds s_{l + 32c}; 8-sample block sums by xor-shuffles (the ((s0+s1)+(s2+s3)) +
// ((s4+s5)+(s6+s7)) tree), then the WinSum chains (blocks alternately into acc0 /
// acc1, a leftover block into acc0, leftover samples into acc1) evaluated
// redundantly by every lane -- the same association as WinSum::push.
template <int NC>
__device__ __forceinline__ float warp_window_sum(const float (&v)[NC], int W) {
  const int lane = threadIdx.x & 31;
  const int W8 = W & ~7, nb2 = 2 * (W8 / 16), nblk = W8 / 8;
  float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    float b = v[c];
    b += __shfl_xor_sync(0xffffffffu, b, 1);
    b += __shfl_xor_sync(0xffffffffu, b, 2);
    b += __shfl_xor_sync(0xffffffffu, b, 4);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int blk = 4 * c + q;
      const float bs = __shfl_sync(0xffffffffu, b, 8 * q);
      if (blk < nblk) {
        if (blk < nb2 && (blk & 1)) acc1 += bs;
        else acc0 += bs;
      }
    }
  }
  for (int tau = W8; tau < W; ++tau) {   // leftover samples (W % 8), in order
    float src = v[0];
#pragma unroll
    for (int c = 1; c < NC; ++c)
      if ((tau >> 5) == c) src = v[c];
    acc1 += __shfl_sync(0xffffffffu, src, tau & 31);
  }
  (void)lane;
  return acc0 + acc1;
}

// ingest of one instance's new sample (k_stream_push's arithmetic, G float4 groups)
template <int G>
__device__ __forceinline__ void stream_push_one(const StreamParams &p, int64_t i) {
  constexpr int M = 4 * G;
  const int W = p.W;
  const int slot = (int)(p.tick % W);
  const float4 *xs = reinterpret_cast<const float4 *>(p.sample + i * M);
  const float4 *ms = reinterpret_cast<const float4 *>(p.mean + i * M);
  const float4 *ss = reinterpret_cast<const float4 *>(p.stdv + i * M);
  float pg[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    __half *r0 = p.ring16 + stream_elem(i, slot, 4 * g, W, M);
    __half *r1 = p.ring16 + stream_elem(i, slot + W, 4 * g, W, M);
    const float4 v = __ldg(xs + g), mu = __ldg(ms + g), sd = __ldg(ss + g);
    const float z0 = fminf(fmaxf(div_rn(__fsub_rn(v.x, mu.x), sd.x, __frcp_rn(sd.x)), -1e4f), 1e4f);
    const float z1 = fminf(fmaxf(div_rn(__fsub_rn(v.y, mu.y), sd.y, __frcp_rn(sd.y)), -1e4f), 1e4f);
    const float z2 = fminf(fmaxf(div_rn(__fsub_rn(v.z, mu.z), sd.z, __frcp_rn(sd.z)), -1e4f), 1e4f);
    const float z3 = fminf(fmaxf(div_rn(__fsub_rn(v.w, mu.w), sd.w, __frcp_rn(sd.w)), -1e4f), 1e4f);
    uint2 pk;
    pk.x = cvt_pack_f16x2(z0, z1);
    pk.y = cvt_pack_f16x2(z2, z3);
    *reinterpret_cast<uint2 *>(r0) = pk;
    *reinterpret_cast<uint2 *>(r1) = pk;
    const float2 f01 = __half22float2(*reinterpret_cast<const __half2 *>(&pk.x));
    const float2 f23 = __half22float2(*reinterpret_cast<const __half2 *>(&pk.y));
    pg[g] = (f01.x + f01.y) + (f23.x + f23.y);
  }
#pragma unroll
  for (int w = 1; w < G; w <<= 1)
#pragma unroll
    for (int k = 0; k + w < G; k += 2 * w) pg[k] = pg[k] + pg[k + w];
  p.sums_w[(size_t)i * sums_pitch(W) + slot] = pg[0];
  p.sums_w[(size_t)i * sums_pitch(W) + slot + W] = pg[0];
}

template <int H, int ZP>
__global__ void __launch_bounds__(kSThreads, 1) k_stream_rows(const StreamParams p) {
  constexpr int N2 = 2 * ZP;
  extern __shared__ __align__(1024) uint8_t smem[];
  const RowLayoutSm SL = row_smem_layout(H, ZP, kSAStages * kSAStageBytes, kSWStages, kSAK);
  uint8_t *region = smem + SL.region;
  uint8_t *astage = smem + SL.astage;
  uint8_t *heads = smem + SL.heads;
  uint8_t *w3s = smem + SL.w3;
  uint8_t *mubuf = smem + SL.mubuf;
  RowBars &B = *reinterpret_cast<RowBars *>(smem + SL.bars);
  float *b1s = reinterpret_cast<float *>(smem + SL.vec);
  float *b3s = b1s + H;
  float *wbs = b3s + H;
  float *bmls = wbs + H;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t row0 = (int64_t)blockIdx.x * kRR;
  const int W = p.W;
  const int woff = (int)((p.tick + 1) % W);   // oldest sample's slot of the window ending at tick
  unsigned long long *tr = (blockIdx.x == 0) ? p.trace : nullptr;
  auto stamp = [&](int slot) {   // diagnostic; compiled in with -DENOVA_TRACE only
#ifdef ENOVA_TRACE
    if (tr) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tr[slot] = t;
    }
#else
    (void)slot;
    (void)tr;
#endif
  };
  if (tid == 0) stamp(0);

  // 1. barrier initialisation, then the producers start at once (they need
  //    nothing else); the consumers (rows, their helpers, the MMA warp) load the
  //    biases and allocate TMEM meanwhile and meet at their own named barrier
  if (tid == 0) {
    for (int i = 0; i < kSWStages; ++i) {
      mbar_init(&B.w_full[i], 1);
      mbar_init(&B.w_empty[i], 1);
    }
    for (int i = 0; i < kSAStages; ++i) {
      mbar_init(&B.a_full[i], 1);   // the producer's expect_tx (the bulk copy completes the bytes)
      mbar_init(&B.a_empty[i], 1);
    }
    mbar_init(&B.wimg, 1);
    mbar_init(&B.g1_done, 1);
    mbar_init(&B.h_full, 2 * kRowThreads / 32);   // row warps + helper warps (E1 halves)
    mbar_init(&B.g2_done, 1);
    mbar_init(&B.mu_full, (ZP == 16 ? 2 : 1) * kRowThreads / 32);   // + the helpers' E2 half
    mbar_init(&B.g3_done, 1);
    mbar_init(&B.e3_done, kRowThreads / 32);
    mbar_init(&B.e2_done, kRowThreads / 32);
    fence_mbar_init();
  }
  __syncthreads();
  const int n_groups = (p.nsteps + kSAK - 1) / kSAK;

  if (warp == kRProdWarp) {
    // ---------------- producer: heads / W3 images, W1 ring (bulk copies) ----------------
    if (lane == 0) {
      const uint32_t hb = (uint32_t)N2 * H * 2, w3b = (uint32_t)H * 16 * 2;
      mbar_arrive_expect_tx(&B.wimg, hb + w3b);
      bulk_g2s(heads, p.headsimg, hb, &B.wimg);
      bulk_g2s(w3s, p.w3img, w3b, &B.wimg);
      for (int g = 0; g < n_groups; ++g) {
        const int st = g % kSWStages;
        if (g >= kSWStages) mbar_wait_sleep(&B.w_empty[st], ((g / kSWStages) - 1) & 1, 64);
        const int steps = min(kSAK, p.nsteps - g * kSAK);
        const uint32_t bytes = (uint32_t)steps * 32 * H;
        mbar_arrive_expect_tx(&B.w_full[st], bytes);
        bulk_g2s(region + st * SL.w_stage_bytes, p.w1img + (size_t)g * SL.w_stage_bytes, bytes,
                 &B.w_full[st]);
        if (g < 16) stamp(56 + g);
      }
    }
  } else if (warp == kSAWarp) {
    // ---------------- A producer: one bulk copy (kSAK K-steps x 128 instances) per group ----------------
    // The window's newest sample is its last K-step (last group): only that
    // group waits for this tick's fused pushes; the older groups stream while
    // the row threads ingest.
    const uint8_t *tsrc = reinterpret_cast<const uint8_t *>(p.ring16) +
                          (((size_t)blockIdx.x * 2 * W + woff) * (size_t)(p.M >> 3) << 11);
    for (int g = 0; g < n_groups; ++g) {
      if (g == n_groups - 1 && p.sample) named_bar_sync_na(5, kRowThreads + 32);
      if (lane == 0) {
        const int a = g % kSAStages;
        if (g >= kSAStages) mbar_wait_sleep(&B.a_empty[a], ((g / kSAStages) - 1) & 1, 64);
        const uint32_t bytes = (uint32_t)min(kSAK, p.nsteps - g * kSAK) * 4096u;
        mbar_arrive_expect_tx(&B.a_full[a], bytes);
        bulk_g2s(astage + a * kSAStageBytes, tsrc + (size_t)g * kSAStageBytes, bytes, &B.a_full[a]);
        if (g < 20) stamp(16 + g);
        if (g == 0) stamp(1);
        if (g == n_groups - 1) stamp(2);
      }
      __syncwarp();
    }
  } else {
    // ---------------- consumers: biases, TMEM ----------------
    constexpr int kCons = kSThreads - 64;   // rows, MMA warp, helpers
    const int ctid = warp < kRProdWarp ? tid : tid - 64;
    for (int i = ctid; i < H; i += kCons) {
      b1s[i] = __fmul_rn(p.b1[i], kTwoLog2e);   // E1 exponent bias (GEMM1 starts from zero)
      b3s[i] = p.b3[i];
      wbs[i] = p.wbar[i];
    }
    for (int i = ctid; i < N2; i += kCons) bmls[i] = p.bml[i];
    for (int i = ctid; i < (int)(2 * kRR * 16 * 2 / 16); i += kCons)
      reinterpret_cast<uint4 *>(mubuf)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tmem_alloc(&B.tmem_slot, SL.tmem_cols);
    tc_fence_before();
    named_bar_sync_na(6, kCons);
    tc_fence_after();
    const uint32_t tmem = B.tmem_slot;

    if (warp == kRMmaWarp) {
      // ---------------- MMA issuer ----------------
      const uint32_t idesc1 = make_idesc_f16(128, H);
      const uint32_t aa = smem_u32(astage), ra = smem_u32(region);
      // one iteration per group (its kSAK MMAs unrolled): waits, MMAs, commits in
      // straight-line code.  A loop over K-steps with the waits at j == 0 and the
      // commits at j == kSAK - 1 paced the rings at ~1200 cycles per group instead
      // of ~410 (tools/ubench_c4.cu, k_bis V1 vs V3)
      for (int g = 0; g < n_groups; ++g) {
        const int a = g % kSAStages, st = g % kSWStages;
        mbar_wait(&B.a_full[a], (g / kSAStages) & 1);
        if (lane == 0 && g < 20) stamp(36 + g);
        mbar_wait(&B.w_full[st], (g / kSWStages) & 1);
        if (lane == 0 && g < 16) stamp(72 + g);
        tc_fence_after();
        const int steps = min(kSAK, p.nsteps - g * kSAK);
#pragma unroll
        for (int j = 0; j < kSAK; ++j) {
          if (j < steps) {
            // K-step j of the stage: [2 halves (LBO 2 KB)][16 row groups (SBO 128 B)][8 rows][16 B]
            const uint64_t ad = make_sdesc(aa + a * kSAStageBytes + j * 4096, 2048, 128);
            const uint64_t bd = make_sdesc(ra + st * SL.w_stage_bytes + j * 32 * H, 16 * H, 128);
            mma_f16_warp(tmem, ad, bd, idesc1, (g | j) ? 1u : 0u);
          }
        }
        if (lane == 0 && g == 0) stamp(3);
        mma_commit_warp(&B.a_empty[a]);
        mma_commit_warp(&B.w_empty[st]);
      }
      if (lane == 0) stamp(4);
      mma_commit_warp(&B.g1_done);
      // (the E-chain waits back off: a spinning MMA warp takes issue slots from
      // the row warp that shares its SM sub-partition)
      mbar_wait(&B.wimg, 0);
#ifdef ENOVA_MMA_SPIN
      mbar_wait(&B.h_full, 0);
#else
      mbar_wait_sleep(&B.h_full, 0, 32);
#endif
      tc_fence_after();
      if (lane == 0) {
        const uint32_t idesc2 = make_idesc_f16(128, N2);
        const uint32_t hb = smem_u32(heads);
#pragma unroll 1
        for (int pass = 0; pass < 2; ++pass) {
          const uint32_t ab = smem_u32(region) + (uint32_t)pass * (kRR * H * 2);
          for (int s = 0; s < H / 16; ++s) {
            const uint64_t ad = make_sdesc(ab + s * (32 * kRR), 16 * kRR, 128);
            const uint64_t bd = make_sdesc(hb + s * (32 * N2), 16 * N2, 128);
            mma_f16_ss(tmem + H, ad, bd, idesc2, (pass | s) ? 1u : 0u);
          }
        }
        mma_commit(&B.g2_done);
      }
      __syncwarp();
#ifdef ENOVA_MMA_SPIN
      mbar_wait(&B.mu_full, 0);
#else
      mbar_wait_sleep(&B.mu_full, 0, 32);
#endif
      tc_fence_after();
      if (lane == 0) {
        const uint32_t idesc3 = make_idesc_f16(128, H);
        const uint64_t bd = make_sdesc(smem_u32(w3s), 16 * H, 128);
        mma_f16_ss(tmem, make_sdesc(smem_u32(mubuf), 16 * kRR, 128), bd, idesc3, 0u);
        mma_f16_ss(tmem, make_sdesc(smem_u32(mubuf) + kRR * 16 * 2, 16 * kRR, 128), bd, idesc3, 1u);
        mma_commit(&B.g3_done);
      }
      __syncwarp();
    } else if (warp >= kSHelperWarp0) {
      // ---------------- helpers: the second E1 half and E3 chains 2, 3 of the rows of their quadrant ----------------
      const int q4 = warp & 3, r = q4 * 32 + lane;
      auto no_sx = []() -> float { return 0.f; };
      rows_epilogue<H, ZP, RowBars, decltype(no_sx) &, 2>(
          tmem, q4, lane, r, row0 + r, row0 + r < p.n, no_sx, region, mubuf, b1s, b3s, wbs, bmls, B,
          p.Z, p.D, p.bbar, nullptr, nullptr, nullptr, 0.0, nullptr, nullptr, nullptr, nullptr,
          nullptr, nullptr, 0, 0, e3part_of(smem, SL), e2part_of(smem, SL));
    } else {
      // ---------------- row threads: the fused ingest, window sums, the epilogues ----------------
      const int r = tid;
      const int64_t row = row0 + r;
      const bool valid = row < p.n;
      if (p.sample) {   // fused ingest of this tick's sample, visible to the bulk copies (async proxy)
        if (valid) {
          switch (p.M) {
            case 8: stream_push_one<2>(p, row); break;
            case 16: stream_push_one<4>(p, row); break;
            case 32: stream_push_one<8>(p, row); break;
            default: stream_push_one<16>(p, row); break;
          }
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");   // pushes -> the bulk copies
        __syncwarp();   // reconverge after the per-row push
        named_bar_arrive(5, kRowThreads + 32);   // the A producer syncs before the last group
      }
      const int W8 = W & ~7, nb2 = 2 * (W8 / 16);
      WinSum ws;
      ws.init();
      // window sums: each thread prefetches its row's W per-sample sums as aligned
      // float4 (W <= 64: 17 x 16 B covering [woff, woff + W), issued now, in flight
      // while the A groups stream) and folds them in WinSum order before E3
      const bool pre = W <= 64;
      const int wsh = woff & 3;   // uniform over the CTA
      float4 sv4[17];
      if (pre) {
        const float4 *sp4 = reinterpret_cast<const float4 *>(
            p.sums + (size_t)(valid ? row : 0) * sums_pitch(W) + (woff - wsh));
#pragma unroll
        for (int k = 0; k < 17; ++k)
          sv4[k] = (valid && 4 * k < wsh + W) ? __ldg(sp4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      // (reduced only before E3, where MD needs it: off the E1 / E2 critical path)
      auto sx_fn = [&]() -> float {
        float sx = 0.f;
        if (pre && valid) {
          auto fold = [&](auto shift_c) {
            constexpr int sh = decltype(shift_c)::value;
#pragma unroll
            for (int tau = 0; tau < 64; ++tau) {
              if (tau < W) {
                const int e = tau + sh;
                const float4 q = sv4[e >> 2];
                const float v = (e & 3) == 0 ? q.x : (e & 3) == 1 ? q.y : (e & 3) == 2 ? q.z : q.w;
                ws.push(tau, v, W8, nb2);
              }
            }
          };
          switch (wsh) {
            case 0: fold(std::integral_constant<int, 0>{}); break;
            case 1: fold(std::integral_constant<int, 1>{}); break;
            case 2: fold(std::integral_constant<int, 2>{}); break;
            default: fold(std::integral_constant<int, 3>{}); break;
          }
          sx = ws.acc0 + ws.acc1;
        } else if (valid) {   // long windows: per-thread loads (the association of WinSum)
          const float *sp = p.sums + (size_t)row * sums_pitch(W) + woff;
          for (int tau = 0; tau < W; ++tau) ws.push(tau, __ldg(sp + tau), W8, nb2);
          sx = ws.acc0 + ws.acc1;
        }
        return sx;
      };
      // the window sum is folded now, while GEMM1 runs (the rows wait for it anyway)
      const float sx_pre = sx_fn();
      auto sx_get = [sx_pre]() -> float { return sx_pre; };
      if (r == 0) stamp(5);
      rows_epilogue<H, ZP, RowBars, decltype(sx_get) &, 1>(
          tmem, warp, lane, r, row, valid, sx_get, region, mubuf, b1s, b3s, wbs, bmls, B, p.Z, p.D,
          p.bbar, p.scores, p.md, p.flags, 0.0, p.z_q_dev, tr, nullptr, nullptr, nullptr, nullptr, 0,
          0, e3part_of(smem, SL), e2part_of(smem, SL));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(B.tmem_slot, SL.tmem_cols);
}

unsigned long long *pair_trace();
enova_status stream_detect(const void *ring, int64_t n, int64_t tick, const DetLayout &L,
                           const void *det_ws, const double *z_q_dev, int8_t *flags, float *scores,
                           float *md, cudaStream_t st, const float *sample = nullptr,
                           const float *mean = nullptr, const float *stdv = nullptr);


template <int H, int ZP>
static enova_status launch_stream_t(const StreamParams &p, cudaStream_t st) {
  const RowLayoutSm SL = row_smem_layout(H, ZP, kSAStages * kSAStageBytes, kSWStages, kSAK);
  auto kern = k_stream_rows<H, ZP>;
  static thread_local int cached_dev = -1;
  int dev = 0;
  ENOVA_CUDA_TRY(cudaGetDevice(&dev));
  if (dev != cached_dev) {
    ENOVA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SL.total));
    cached_dev = dev;
  }
  const int64_t tiles = (p.n + kRR - 1) / kRR;
  if (tiles > 0x7fffffffLL) {
    set_error("too many instances for one launch");
    return ENOVA_ERR_UNSUPPORTED;
  }
  ENOVA_LAUNCH(kern, (unsigned)tiles, kSThreads, SL.total, st, p);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

enova_status stream_detect(const void *ring, int64_t n, int64_t tick, const DetLayout &L,
                           const void *det_ws, const double *z_q_dev, int8_t *flags, float *scores,
                           float *md, cudaStream_t st, const float *sample,
                           const float *mean, const float *stdv) {
  if (n == 0) return ENOVA_OK;
  const int W = L.W, M = L.M;
  StreamParams p{};
  const uint8_t *b = static_cast<const uint8_t *>(det_ws);
  p.sums = reinterpret_cast<const float *>(static_cast<const uint8_t *>(ring) +
                                           stream_sums_offset(n, W, M));
  p.n = n;
  p.tick = tick;
  p.W = W;
  p.M = M;
  p.D = L.D;
  p.Z = L.Z;
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
  p.z_q_dev = z_q_dev;
  p.trace = pair_trace();
  p.sample = sample;
  p.mean = mean;
  p.stdv = stdv;
  p.ring16 = const_cast<__half *>(static_cast<const __half *>(ring));
  p.sums_w = const_cast<float *>(p.sums);
  switch (L.H * 100 + L.ZP) {
    case 3208: return launch_stream_t<32, 8>(p, st);
    case 3216: return launch_stream_t<32, 16>(p, st);
    case 6408: return launch_stream_t<64, 8>(p, st);
    case 6416: return launch_stream_t<64, 16>(p, st);
    case 12808: return launch_stream_t<128, 8>(p, st);
    case 12816: return launch_stream_t<128, 16>(p, st);
  }
  set_error("unsupported (H, Z)");
  return ENOVA_ERR_UNSUPPORTED;
}

enova_status stream_step(void *ring, int64_t n, int64_t tick, const DetLayout &L,
                         const void *det_ws, const float *sample, const float *mean,
                         const float *stdv, const double *z_q_dev, int8_t *flags, float *scores,
                         float *md, cudaStream_t st) {
  return stream_detect(ring, n, tick, L, det_ws, z_q_dev, flags, scores, md, st, sample, mean, stdv);
}

}  // namespace enova
