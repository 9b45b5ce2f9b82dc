// layout.h -- host/device description of the prepared-detector image (K0) and
// of the score kernel's shared-memory plan.
#pragma once
#include <stddef.h>
#include <stdint.h>

#include "../../include/enova.h"

namespace enova {

struct DetLayout {
  int W, M, H, Z;
  int ZP;   // latent padded to 8 or 16 (mu and lv halves of the heads GEMM)
  int N2;   // heads GEMM N = 2 * ZP
  int D;    // W * M
  int P;    // fp16 planes of 8 metrics per sample (M / 8)
  size_t off_w1, off_heads, off_w3;        // fp16 canonical UMMA B images
  size_t off_b1, off_bml, off_b3, off_wbar; // fp32 vectors
  size_t off_bbar;                           // fp64 scalar
  size_t off_wbarm, off_bbarm;               // NEXT-1: per-metric column sums [M][H] fp32, [M] fp32
  // CTA-pair (cta_group::2) images: rank r holds B rows [r*N/2, (r+1)*N/2)
  size_t off_w1p, off_headsp, off_w3p;
  bool pair_ok;                              // W1 half fits in shared memory
  size_t total;
};

// Returns false if the detector is outside the fast-path envelope.
static inline bool det_layout(int W, int M, int H, int Z, DetLayout *L) {
  // M / 4 metric groups must be a power of two: the staging threads of the
  // score kernels map (sample, group) by shifts and reduce a sample's groups with
  // an xor-shuffle tree (M = 48 was accepted before round 2 and scored wrongly)
  if (!(M == 8 || M == 16 || M == 32 || M == 64)) return false;
  if (W < 2 || W > 256 || (W % 2) != 0) return false;
  if (!(H == 32 || H == 64 || H == 128)) return false;
  if (Z < 1 || Z > 16) return false;
  L->W = W; L->M = M; L->H = H; L->Z = Z;
  L->ZP = Z <= 8 ? 8 : 16;
  L->N2 = 2 * L->ZP;
  L->D = W * M;
  L->P = M / 8;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 255) / 256 * 256; return r; };
  L->off_w1 = take((size_t)H * L->D * 2);
  L->off_heads = take((size_t)L->N2 * H * 2);
  L->off_w3 = take((size_t)H * 16 * 2);
  L->off_b1 = take((size_t)H * 4);
  L->off_bml = take((size_t)L->N2 * 4);
  L->off_b3 = take((size_t)H * 4);
  L->off_wbar = take((size_t)H * 4);
  L->off_bbar = take(8);
  L->off_wbarm = take((size_t)M * H * 4);
  L->off_bbarm = take((size_t)M * 4);
  L->off_w1p = take((size_t)H * L->D * 2);
  L->off_headsp = take((size_t)L->N2 * H * 2);
  L->off_w3p = take((size_t)H * 16 * 2);
  L->pair_ok = ((size_t)(H / 2) * L->D * 2) <= 128 * 1024;
  L->total = o;
  return true;
}

// Byte offset of element (n, k) of a K-major, no-swizzle canonical operand
// image whose K extent is split in 16-wide MMA steps laid out back to back:
//   step q = k / 16 occupies 32*N bytes; inside it [k-half (2)][n-group][8 rows][8 el].
__host__ __device__ static inline size_t kmajor_step_offset(int n, int k, int N) {
  int q = k >> 4, kk = k & 15;
  return (size_t)q * 32 * N + (size_t)(kk >> 3) * 16 * N + (size_t)(n >> 3) * 128 +
         (size_t)(n & 7) * 16 + (size_t)(kk & 7) * 2;
}

// Pair image: B rows split in two halves of N/2 (one per CTA of a cta_group::2
// pair); each half is a back-to-back K-step image with N/2 rows.
__host__ __device__ static inline size_t pair_offset(int n, int k, int N, int K) {
  const int half = N / 2;
  const int r = n / half, nl = n - r * half;
  return (size_t)r * half * K * 2 + kmajor_step_offset(nl, k, half);
}

}  // namespace enova
