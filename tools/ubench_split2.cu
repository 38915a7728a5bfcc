// Where the split fold's f-warp time goes: variants of its chunk loop alone.
#include <cstdio>
#include <cuda_runtime.h>

#include "sl_device.cuh"
using namespace sl;

template <int V>
__global__ void kf(const double* src, int n, double* out, long long* cyc) {
  __shared__ __align__(16) double xb[2][32], fb[2][32];
  const int lane = threadIdx.x & 31;
  long long t0 = clock64();
  double f = 0.0;
  int k = 0;
  double x = frcp_(src[lane]);
  double raw = src[32 + lane];
  for (int c0 = 0; c0 < n; c0 += 32, ++k) {
    const int s = k & 1;
    const double xn = (V & 4) ? raw : frcp_(raw);
    const int jnn = c0 + 64 + lane;
    raw = jnn < n ? src[jnn] : 1.0;
    xb[s][lane] = x;
    __syncwarp();
    double v[32], b[32];
    double mine = 0.0;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const double2 p = reinterpret_cast<const double2*>(xb[s])[t];
      v[2 * t] = p.x;
      v[2 * t + 1] = p.y;
    }
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      b[t] = f;
      if (V & 8) mine = lane == t ? f : mine;
      if (V & 16) { if (lane == 0) fb[s][t] = f; }
      f = fadd_(f, v[t]);
    }
    if (V & 1) {
      if (lane == 0) {
#pragma unroll
        for (int t = 0; t < 16; ++t)
          reinterpret_cast<double2*>(fb[s])[t] = make_double2(b[2 * t], b[2 * t + 1]);
      }
    }
    if (V & 8) fb[s][lane] = mine;
    __syncwarp();
    if (V & 2) asm volatile("bar.arrive 5, 64;");
    if (V & 2) asm volatile("bar.sync 6, 64;");
    x = xn;
  }
  if (lane == 0) {
    out[V] = f + fb[0][3];
    cyc[V] = clock64() - t0;
  }
}

template <int V>
__global__ void kpartner(int n) {  // balances kf's barriers (V & 2)
  for (int c0 = 0; c0 < n; c0 += 32) {
    asm volatile("bar.sync 5, 64;");
    asm volatile("bar.arrive 6, 64;");
  }
}

template <int V>
__global__ void kboth(const double* src, int n, double* out, long long* cyc) {
  if (threadIdx.x < 32) {
    kf<V>(src, n, out, cyc);
  }
}

int main() {
  const int n = 32768;
  static double h[n];
  for (int i = 0; i < n; ++i) h[i] = 0.03 + 1e-7 * (i % 101);
  double *src, *out;
  long long* cyc;
  cudaMalloc(&src, sizeof h);
  cudaMalloc(&out, 64 * 8);
  cudaMallocManaged(&cyc, 64 * 8);
  cudaMemset(cyc, 0, 64 * 8);
  cudaMemcpy(src, h, sizeof h, cudaMemcpyHostToDevice);
  for (int r = 0; r < 2; ++r) {
    kf<0><<<1, 32>>>(src, n, out, cyc);
    kf<1><<<1, 32>>>(src, n, out, cyc);
    kf<4><<<1, 32>>>(src, n, out, cyc);
    kf<5><<<1, 32>>>(src, n, out, cyc);
    kf<8><<<1, 32>>>(src, n, out, cyc);
    kf<16><<<1, 32>>>(src, n, out, cyc);
  }
  cudaDeviceSynchronize();
  printf("chain only (frcp)      %.1f cyc/elem\n", cyc[0] / (double)n);
  printf("+ fb stores            %.1f\n", cyc[1] / (double)n);
  printf("chain only (no frcp)   %.1f\n", cyc[4] / (double)n);
  printf("+ fb stores (no frcp)  %.1f\n", cyc[5] / (double)n);
  printf("select + 1 STS (frcp)  %.1f\n", cyc[8] / (double)n);
  printf("lane-0 STS.64 per elem %.1f\n", cyc[16] / (double)n);
  return 0;
}
