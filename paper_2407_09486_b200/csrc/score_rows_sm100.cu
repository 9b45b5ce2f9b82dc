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
//             4-stage bulk-copy ring; the TMEM accumulator is pre-loaded with b1.
//   epilogue: E1 (tanh -> h hi/lo), GEMM2 (heads), E2 (KL, mu hi/lo), GEMM3
//             (decoder, accumulator re-armed with b3), E3 (MD by the column-sum
//             identity, flag) -- the same element-wise arithmetic (epilogue.cuh)
//             and the same window-sum association as the windowed CTA-pair
//             kernel, so a streamed window scores bit-identically to the same
//             window scored in a batch.
//
// Envelope: M in {8, 16} (a K-step holds whole samples), H in {32, 64, 128}.
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
};

constexpr int kRR = 128;                 // rows per tile (UMMA M)
constexpr int kRWStageSteps = 4;         // W1 ring: K-steps per stage
constexpr int kRWStages = 8;             // W1 ring depth
constexpr int kRAStages = 8;             // A ring depth (one K-step each)
constexpr uint32_t kRAStepBytes = kRR * 16 * 2;   // 4 KB
constexpr int kRowThreads = 128;         // thread = row
constexpr int kRThreads = kRowThreads + 64;       // + MMA issuer warp + W1 producer warp
constexpr int kRMmaWarp = 4, kRProdWarp = 5;
constexpr int kRPF = 8;                  // K-steps of raw samples in flight per thread

struct RowBars {
  uint64_t w_full[kRWStages], w_empty[kRWStages], a_full[kRAStages], a_empty[kRAStages];
  uint64_t wimg, g1_done, h_full, g2_done, mu_full, g3_done;
  uint32_t tmem_slot, pad;
};

struct RowLayoutSm {
  uint32_t region, astage, heads, w3, mubuf, vec, bars, total, w_stage_bytes, tmem_cols;
};

__host__ __device__ inline RowLayoutSm row_smem_layout(int H, int ZP) {
  RowLayoutSm L;
  uint32_t o = 0;
  auto take = [&](uint32_t b, uint32_t a) {
    o = (o + a - 1) / a * a;
    const uint32_t r = o;
    o += b;
    return r;
  };
  L.w_stage_bytes = (uint32_t)kRWStageSteps * 32 * H;
  const uint32_t ring = kRWStages * L.w_stage_bytes, hb = 2u * kRR * H * 2;
  L.region = take(ring > hb ? ring : hb, 1024);      // W1 ring, then h hi | lo
  L.astage = take(kRAStages * kRAStepBytes, 1024);
  L.heads = take((uint32_t)2 * ZP * H * 2, 128);
  L.w3 = take((uint32_t)H * 16 * 2, 128);
  L.mubuf = take(2u * kRR * 16 * 2, 128);
  L.vec = take((3u * H + 2u * ZP) * 4, 16);           // b1 | b3 | w_bar | [bmu | blv]
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

template <int H, int ZP, int M>
__global__ void __launch_bounds__(kRThreads, 1) k_score_rows(const RowParams p) {
  constexpr int N2 = 2 * ZP;
  extern __shared__ __align__(1024) uint8_t smem[];
  const RowLayoutSm SL = row_smem_layout(H, ZP);
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
    b1s[i] = p.b1[i];
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

  if (warp < 4) {
    // GEMM1 accumulator of this row pre-loaded with b1 (GEMM1 accumulates on top)
    const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16);
    tmem_fill_cols<H>(la, b1s);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

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
    for (int q = 0; q < p.nsteps; ++q) {
      const int a = q % kRAStages, g = q / kRWStageSteps, st = g % kRWStages;
      mbar_wait(&B.a_full[a], (q / kRAStages) & 1);
      if (q % kRWStageSteps == 0) mbar_wait(&B.w_full[st], (g / kRWStages) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint64_t ad = make_sdesc(aa + a * kRAStepBytes, kRR * 16, 128);
        const uint64_t bd = make_sdesc(
            ra + st * SL.w_stage_bytes + (q % kRWStageSteps) * 32 * H, 16 * H, 128);
        mma_f16_ss(tmem, ad, bd, idesc1, 1u);
        mma_commit(&B.a_empty[a]);
        if (q % kRWStageSteps == kRWStageSteps - 1 || q == p.nsteps - 1) mma_commit(&B.w_empty[st]);
        if (q == p.nsteps - 1) mma_commit(&B.g1_done);
      }
      __syncwarp();
    }
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
      mma_f16_ss(tmem, make_sdesc(smem_u32(mubuf), 16 * kRR, 128), bd, idesc3, 1u);
      mma_f16_ss(tmem, make_sdesc(smem_u32(mubuf) + kRR * 16 * 2, 16 * kRR, 128), bd, idesc3, 1u);
      mma_commit(&B.g3_done);
    }
    __syncwarp();
  } else {
    // ---------------- row threads: staging, then the epilogues ----------------
    const int r = tid;
    const int64_t row = row0 + r;
    const bool valid = row < p.n_rows;
    const int64_t inst = valid ? row / p.nw : 0;
    const int64_t wi = valid ? row - inst * p.nw : 0;
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

    // ---- E1: h = tanh(acc) -> hi/lo fp16 A images; re-arm acc with b3 ----
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    mbar_wait(&B.g1_done, 0);
    tc_fence_after();
#pragma unroll 1
    for (int c16 = 0; c16 < H; c16 += 16) {
      float v[16];
      tmem_ld16(lane_addr + c16, v);
      tmem_wait_ld();
      tmem_fill_cols<16>(lane_addr + c16, b3s + c16);
#pragma unroll
      for (int e8 = 0; e8 < 16; e8 += 8) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const float h0 = tanh_2mufu(v[e8 + k]);
          const float h1 = tanh_2mufu(v[e8 + k + 1]);
          float a0, r0, a1, r1;
          split_unit(h0, a0, r0);
          split_unit(h1, a1, r1);
          hi[k >> 1] = cvt_pack_f16x2(a0, a1);
          lo[k >> 1] = cvt_pack_f16x2(r0, r1);
        }
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

    // ---- E2: KL score; mu -> hi/lo fp16 ----
    mbar_wait(&B.g2_done, 0);
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
      float kl = 0.f;
      uint32_t hi[8], lo[8];
#pragma unroll
      for (int z = 0; z < ZP; z += 2) {
        float m2[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          float m = 0.f;
          if (z + u < p.Z) {
            m = vm[z + u] + bmls[z + u];
            kl += kl_term2(m, vl[z + u] + bmls[ZP + z + u]);
          }
          m2[u] = m;
        }
        const uint32_t hp = cvt_pack_f16x2(m2[0], m2[1]);
        const float2 hf = __half22float2(*reinterpret_cast<const __half2 *>(&hp));
        hi[z >> 1] = hp;
        lo[z >> 1] = cvt_pack_f16x2(m2[0] - hf.x, m2[1] - hf.y);
      }
      const size_t off0 = kmajor_step_offset(r, 0, kRR);
      *reinterpret_cast<uint4 *>(mubuf + off0) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4 *>(mubuf + kRR * 32 + off0) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      if constexpr (ZP == 16) {
        const size_t off1 = kmajor_step_offset(r, 8, kRR);
        *reinterpret_cast<uint4 *>(mubuf + off1) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
        *reinterpret_cast<uint4 *>(mubuf + kRR * 32 + off1) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
      }
      score = fmaxf(0.5f * kl, 0.f);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&B.mu_full);

    // ---- E3: MD by the column-sum identity; flag ----
    mbar_wait(&B.g3_done, 0);
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
        d4[0] = fmaf(ww.x, tanh_mufu(v[k]), d4[0]);
        d4[1] = fmaf(ww.y, tanh_mufu(v[k + 1]), d4[1]);
        d4[2] = fmaf(ww.z, tanh_mufu(v[k + 2]), d4[2]);
        d4[3] = fmaf(ww.w, tanh_mufu(v[k + 3]), d4[3]);
      }
    }
    const float dot = (d4[0] + d4[1]) + (d4[2] + d4[3]);
    const float mdv = (sx - dot - (float)(*p.bbar)) / (float)p.D;
    if (valid) {
      if (p.scores) p.scores[row] = score;
      if (p.md) p.md[row] = mdv;
      if (p.flags) {
        const double zq = p.z_q_dev ? __ldg(p.z_q_dev) : p.z_q;
        p.flags[row] = ((double)score > zq) ? (mdv >= 0.f ? 1 : -1) : 0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, SL.tmem_cols);
}

template <int H, int ZP, int M>
static enova_status launch_rows_t(const RowParams &p, cudaStream_t st) {
  const RowLayoutSm SL = row_smem_layout(H, ZP);
  auto kern = k_score_rows<H, ZP, M>;
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

enova_status launch_score_rows(const enova_series *s, const DetLayout &L, const void *det_ws,
                               float *scores, float *md, int8_t *flags, double z_q,
                               const double *z_q_dev, cudaStream_t st) {
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
  p.scores = scores;
  p.md = md;
  p.flags = flags;
  p.z_q = z_q;
  p.z_q_dev = z_q_dev;
  if (p.nw <= 0 || p.n_rows == 0) return ENOVA_OK;
  switch (L.M * 10000 + L.H * 100 + L.ZP) {
    case 83208: return launch_rows_t<32, 8, 8>(p, st);
    case 83216: return launch_rows_t<32, 16, 8>(p, st);
    case 86408: return launch_rows_t<64, 8, 8>(p, st);
    case 86416: return launch_rows_t<64, 16, 8>(p, st);
    case 92808: return launch_rows_t<128, 8, 8>(p, st);
    case 92816: return launch_rows_t<128, 16, 8>(p, st);
    case 163208: return launch_rows_t<32, 8, 16>(p, st);
    case 163216: return launch_rows_t<32, 16, 16>(p, st);
    case 166408: return launch_rows_t<64, 8, 16>(p, st);
    case 166416: return launch_rows_t<64, 16, 16>(p, st);
    case 172808: return launch_rows_t<128, 8, 16>(p, st);
    case 172816: return launch_rows_t<128, 16, 16>(p, st);
  }
  set_error("unsupported (M, H, Z) for the row kernel");
  return ENOVA_ERR_UNSUPPORTED;
}

}  // namespace enova
