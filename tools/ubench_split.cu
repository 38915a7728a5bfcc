// Two-warp split fold (plan_large.cuh split_fold_f / split_fold_c) alone on an
// SM: cycles per element, against ps_add over the same operands.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -Ipaper_2505_23022_b200/csrc -Iinclude -o build/ubench_split tools/ubench_split.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "sl_device.cuh"
using namespace sl;
#include "plan_large.cuh"

__global__ void ksplit(const double* src, int n, double* out, long long* cyc) {
  __shared__ __align__(16) SplitRing ring;
  __shared__ __align__(16) double ebuf[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long t0 = clock64();
  if (warp == 1) {
    const double f = split_fold_f(n, src, [](double t) { return frcp_(t); }, ring, 5, lane);
    if (lane == 0) { out[0] = f; cyc[0] = clock64() - t0; }
  } else if (warp == 2) {
    const double c = split_fold_c(n, ring, 5, ebuf, lane);
    if (lane == 0) { out[1] = c; cyc[1] = clock64() - t0; }
  }
}

__global__ void kref(const double* src, int n, double* out) {
  PySum ps;
  ps_init(ps);
  for (int j = 0; j < n; ++j) ps_add(ps, frcp_(src[j]));
  out[2] = ps.f;
  out[3] = ps.c;
}

int main() {
  const int n = 32768;
  static double h[n];
  for (int i = 0; i < n; ++i) h[i] = (i % 3 == 0) ? 0.03 : (i % 3 == 1 ? 0.05 : 0.1 + 1e-7 * (i % 101));
  double *src, *out;
  long long* cyc;
  cudaMalloc(&src, sizeof h);
  cudaMalloc(&out, 64);
  cudaMallocManaged(&cyc, 64);
  cudaMemcpy(src, h, sizeof h, cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) ksplit<<<1, 128>>>(src, n, out, cyc);
  kref<<<1, 1>>>(src, n, out);
  cudaDeviceSynchronize();
  double o[4];
  cudaMemcpy(o, out, 32, cudaMemcpyDeviceToHost);
  printf("split f %.17g c %.17g | ps_add f %.17g c %.17g | equal %d\n", o[0], o[1], o[2], o[3],
         o[0] == o[2] && o[1] == o[3]);
  printf("cycles/elem: f-warp %.1f c-warp %.1f\n", cyc[0] / (double)n, cyc[1] / (double)n);
  return 0;
}
