// CPython-sum (Neumaier) fold throughput on one warp: cycles per element for
//  (a) ps_add_nz unrolled over shuffled operands (the current fold),
//  (b) split fold: the f chain alone, then lane-parallel exact errors, then the
//      c chain over the errors (same result bit for bit),
// alone on the SM (1 warp) and with 3 other busy warps on the same SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -Ipaper_2505_23022_b200/csrc -Iinclude -o build/ubench_fold tools/ubench_fold.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "sl_device.cuh"

using namespace sl;

__device__ __forceinline__ void fold_split(PySum& s, double x) {
  // operands of this chunk, warp-uniform registers
  double v[32];
#pragma unroll
  for (int t = 0; t < 32; ++t) v[t] = __shfl_sync(0xffffffffu, x, t);
  const int lane = threadIdx.x & 31;
  double fprev = 0.0;  // f before this lane's element
  double f = s.f;
#pragma unroll
  for (int t = 0; t < 32; ++t) {
    fprev = lane == t ? f : fprev;
    f = fadd_(f, v[t]);
  }
  const double fnew = __shfl_sync(0xffffffffu, f, 0);
  (void)fnew;
  // exact error of fprev + x == t (FastTwoSum on the larger magnitude)
  const double t = fadd_(fprev, x);
  const bool big = fabs(fprev) >= fabs(x);
  const double hi = big ? fprev : x, lo = big ? x : fprev;
  const double err = fadd_(fsub_(hi, t), lo);
  double e[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) e[k] = __shfl_sync(0xffffffffu, err, k);
  double c = s.c;
#pragma unroll
  for (int k = 0; k < 32; ++k) c = fadd_(c, e[k]);
  s.c = c;
  s.f = f;
}

__device__ __forceinline__ void add_twosum(PySum& s, double x) {
  const double t = fadd_(s.f, x);
  const double bp = fsub_(t, s.f);
  const double ap = fsub_(t, bp);
  s.c = fadd_(s.c, fadd_(fsub_(s.f, ap), fsub_(x, bp)));
  s.f = t;
}

// operands through a per-warp shared-memory buffer, read back as 16 x LDS.128
template <int KIND>
__device__ __forceinline__ void fold_smem(PySum& s, double x, double* buf) {
  const int lane = threadIdx.x & 31;
  buf[lane] = x;
  __syncwarp();
  double v[32];
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const double2 p = reinterpret_cast<const double2*>(buf)[t];
    v[2 * t] = p.x;
    v[2 * t + 1] = p.y;
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < 32; ++t) {
    if (KIND == 0) ps_add_nz(s, v[t]);
    else if (KIND == 1) add_twosum(s, v[t]);
    else s.f = fadd_(s.f, v[t]);
  }
}

template <int MODE>
__global__ void k(const double* in, double* out, long long* cyc, int n, int busy) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp > 0) {  // other warps: busy fp64 work (contention), warps 4, 8, 12 share SMSP 0
    if (!busy) return;
    double a = in[lane], b = 1.0000001;
    for (int i = 0; i < n * 4; ++i) a = fadd_(fmul_(a, b), 1e-9);
    out[64 + threadIdx.x] = a;
    return;
  }
  __shared__ __align__(16) double buf[32];
  PySum s;
  ps_init(s);
  ps_add(s, 1.0);
  long long t0 = clock64();
  double x = in[lane];
  for (int c0 = 0; c0 < n; c0 += 32) {
    const double xn = in[(c0 + 32 + lane) & 1023];
    if (MODE == 0)
      ps_add_warp_long(s, x, 32);
    else if (MODE == 1)
      fold_split(s, x);
    else
      fold_smem<MODE - 2>(s, x, buf);
    x = xn;
  }
  long long t1 = clock64();
  if (lane == 0) {
    cyc[MODE * 2 + busy] = t1 - t0;
    out[MODE] = ps_result(s);
  }
}

int main() {
  const int n = 32768;
  double h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = 1.0 / (0.03 + 0.001 * (i % 97));
  double *in, *out;
  long long* cyc;
  cudaMalloc(&in, sizeof h);
  cudaMalloc(&out, 4096 * 8);
  cudaMallocManaged(&cyc, 16 * 8);
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep)
    for (int busy = 0; busy < 2; ++busy) {
      k<0><<<1, 512>>>(in, out, cyc, n, busy);
      k<1><<<1, 512>>>(in, out, cyc, n, busy);
      k<2><<<1, 512>>>(in, out, cyc, n, busy);
      k<3><<<1, 512>>>(in, out, cyc, n, busy);
      k<4><<<1, 512>>>(in, out, cyc, n, busy);
      cudaDeviceSynchronize();
    }
  double r[5];
  cudaMemcpy(r, out, 40, cudaMemcpyDeviceToHost);
  printf("results: %.17g %.17g %.17g %.17g (f only %.17g)\n", r[0], r[1], r[2], r[3], r[4]);
  printf("ps_add_nz fold : alone %.1f  busy %.1f cycles/elem\n", cyc[0] / (double)n, cyc[1] / (double)n);
  printf("split fold     : alone %.1f  busy %.1f cycles/elem\n", cyc[2] / (double)n, cyc[3] / (double)n);
  printf("smem+nz        : alone %.1f  busy %.1f cycles/elem\n", cyc[4] / (double)n, cyc[5] / (double)n);
  printf("smem+twosum    : alone %.1f  busy %.1f cycles/elem\n", cyc[6] / (double)n, cyc[7] / (double)n);
  printf("smem f-chain   : alone %.1f  busy %.1f cycles/elem\n", cyc[8] / (double)n, cyc[9] / (double)n);
  return 0;
}
