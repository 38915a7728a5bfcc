// Dependent-chain latencies on this GPU (cycles per op): DADD, DMUL, DRCP_RN,
// DDIV_RN, 64-bit shfl, shared-memory load, L1-hit global load.  Used to size the
// serial fp64 chains of the config-2 plan kernels.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_lat tools/ubench_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, const double* g, int n) {
  __shared__ double sm[256];
  const int lane = threadIdx.x;
  for (int i = lane; i < 256; i += 32) sm[i] = (double)((i * 7 + 1) & 255);
  __syncwarp();
  double x = out[0], y = 1.0000001;
  long long t0, t1;
  // DADD
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DMUL
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, y);
  t1 = clock64();
  cyc[1] = t1 - t0;
  // DRCP
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x);
  t1 = clock64();
  cyc[2] = t1 - t0;
  // DDIV
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __ddiv_rn(y, x);
  t1 = clock64();
  cyc[3] = t1 - t0;
  // shfl 64-bit chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
  t1 = clock64();
  cyc[4] = t1 - t0;
  // smem dependent load
  int p = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) p = (int)sm[p & 255];
  t1 = clock64();
  cyc[5] = t1 - t0;
  // global dependent load (L1 hit after the first touch)
  int q = lane & 7;
  for (int i = 0; i < 64; ++i) q = (int)g[q & 255];
  t0 = clock64();
  for (int i = 0; i < n; ++i) q = (int)g[q & 255];
  t1 = clock64();
  cyc[6] = t1 - t0;
  // Neumaier step chain (CPython sum): t = s + v; c += ...; s = t
  double s = x, c = 0.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double v = sm[i & 255] * 1e-3;
    const double t = __dadd_rn(s, v);
    const double a = fabs(s) >= fabs(v) ? __dadd_rn(__dsub_rn(s, t), v) : __dadd_rn(__dsub_rn(v, t), s);
    c = __dadd_rn(c, a);
    s = t;
  }
  t1 = clock64();
  cyc[7] = t1 - t0;
  out[1 + lane] = x + p + q + s + c;
}

int main() {
  double *out, *g;
  long long* cyc;
  cudaMalloc(&out, 64 * 8);
  cudaMalloc(&g, 256 * 8);
  cudaMallocManaged(&cyc, 8 * 8);
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = (double)((i * 13 + 5) & 255);
  cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
  cudaMemset(out, 0, 64 * 8);
  const int n = 4096;
  k<<<1, 32>>>(out, cyc, g, n);
  cudaDeviceSynchronize();
  k<<<1, 32>>>(out, cyc, g, n);
  cudaDeviceSynchronize();
  const char* names[] = {"dadd", "dmul", "drcp_rn", "ddiv_rn", "shfl64", "lds_dep", "ldg_l1_dep",
                         "neumaier_step"};
  for (int i = 0; i < 8; ++i) printf("%-14s %6.1f cycles/op\n", names[i], (double)cyc[i] / n);
  return 0;
}
