// ubench_scan.cu -- diagnostic: throughput of one streaming pass over 100M fp32
// scores on one CTA (512 threads) per SM, with and without the warp-level
// stable compaction of the k_pot scan phase (not part of the library).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <cuda_runtime.h>

__host__ __device__ __forceinline__ unsigned f2key(float f) {
  unsigned b; memcpy(&b, &f, 4);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

template <int MODE>   // 0 count only, 1 warp compaction (shuffle scan), 2 ballot compaction
__global__ void __launch_bounds__(512, 1) k_scan(const float *s, int64_t n, unsigned lo, float *dst,
                                                 long long *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t chunk = ((n + gridDim.x - 1) / gridDim.x + 3) / 4 * 4;
  const int64_t b0 = min(n, (int64_t)blockIdx.x * chunk), b1 = min(n, b0 + chunk);
  const int64_t len = b1 - b0;
  const int64_t sub = ((len + 15) / 16 + 3) / 4 * 4;
  const int64_t w0 = min(len, warp * sub), w1 = min(len, w0 + sub);
  const float4 *x4 = reinterpret_cast<const float4 *>(s + b0 + w0);
  float *wd = dst + b0 + w0;
  const int64_t n4 = (w1 - w0) / 4;
  long long cnt = 0, below = 0;
  float4 a[4], b[4];
  auto ld = [&](float4 (&v)[4], int64_t i0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * 32 + lane;
      v[u] = i < n4 ? __ldg(x4 + i) : make_float4(-1e30f, -1e30f, -1e30f, -1e30f);
    }
  };
  auto proc = [&](const float4 (&v)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float e4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
      bool c[4];
      int k = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) { c[e] = f2key(e4[e]) >= lo; k += c[e]; }
      below += 4 - k;
      if (MODE == 1) {
        int incl = k;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        long long o = cnt + incl - k;
#pragma unroll
        for (int e = 0; e < 4; ++e) if (c[e]) wd[o++] = e4[e];
        cnt += __shfl_sync(0xffffffffu, incl, 31);
      } else if (MODE == 2) {
        // four ballots (one per element slot): candidates before lane l's element e =
        // popc of lower lanes in all four ballots + own earlier elements
        unsigned bl[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) bl[e] = __ballot_sync(0xffffffffu, c[e]);
        const unsigned lt = (1u << lane) - 1u;
        int before = __popc(bl[0] & lt) + __popc(bl[1] & lt) + __popc(bl[2] & lt) + __popc(bl[3] & lt);
        long long o = cnt + before;
#pragma unroll
        for (int e = 0; e < 4; ++e) if (c[e]) wd[o++] = e4[e];
        cnt += __popc(bl[0]) + __popc(bl[1]) + __popc(bl[2]) + __popc(bl[3]);
      }
    }
  };
  ld(a, 0);
  for (int64_t i0 = 0; i0 < n4; i0 += 256) {
    ld(b, i0 + 128);
    proc(a);
    ld(a, i0 + 256);
    proc(b);
  }
  if (lane == 0) atomicAdd((unsigned long long *)out, (unsigned long long)(below + cnt));
}

int main() {
  const int64_t n = 100000000;
  float *s, *d;
  long long *o;
  cudaMalloc(&s, n * 4);
  cudaMalloc(&d, n * 4);
  cudaMalloc(&o, 8);
  // scores: ramp pattern, 2.4% above lo
  float *h = (float *)malloc(n * 4);
  for (int64_t i = 0; i < n; ++i) h[i] = (float)((i * 2654435761ull) % 1000000) * 1e-4f;
  cudaMemcpy(s, h, n * 4, cudaMemcpyHostToDevice);
  const unsigned lo = f2key(97.6f) ;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  void *flush;
  cudaMalloc(&flush, 256 << 20);
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      cudaMemset(flush, r, 256 << 20);
      cudaEventRecord(e0);
      if (mode == 0) k_scan<0><<<sms, 512>>>(s, n, lo, d, o);
      if (mode == 1) k_scan<1><<<sms, 512>>>(s, n, lo, d, o);
      if (mode == 2) k_scan<2><<<sms, 512>>>(s, n, lo, d, o);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("mode %d (%s): %.1f us  %.2f TB/s\n", mode,
           mode == 0 ? "count" : mode == 1 ? "shfl-scan compaction" : "ballot compaction",
           best * 1e3, n * 4 / (best * 1e-3) / 1e12);
  }
  return 0;
}
