// Launch cost of an empty kernel by cluster size, block size and dynamic shared
// memory (CUDA events; back-to-back mean of 200, and single launches behind a
// spin kernel after an L2-sized memset, as bench.py times the plan kernels).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubcl tools/ubench_cluster_launch.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_k(int* p) {
  extern __shared__ int sm[];
  if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = sm[0];
}
__global__ void spin_k(long long cyc) {
  long long t0 = clock64();
  while (clock64() - t0 < cyc) {}
}

static float run(int cl, int threads, int smem, bool single, char* flush, size_t fl) {
  cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(empty_k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t c = {};
  c.gridDim = dim3(cl);
  c.blockDim = dim3(threads);
  c.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  c.attrs = at;
  c.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int* nul = nullptr;
  float tot = 0.f;
  const int reps = single ? 20 : 1;
  for (int r = 0; r < reps + 2; ++r) {
    if (single) {
      cudaMemset(flush, r, fl);
      cudaDeviceSynchronize();
      spin_k<<<1, 1>>>(200000);
    }
    cudaEventRecord(e0);
    const int n = single ? 1 : 200;
    for (int i = 0; i < n; ++i) cudaLaunchKernelEx(&c, empty_k, nul);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 2) tot += ms * 1000.f / n;
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return tot / reps;
}

int main() {
  char* flush;
  const size_t fl = 256u << 20;
  cudaMalloc(&flush, fl);
  const int cls[] = {1, 2, 4, 8, 16};
  const int sms[] = {0, 64 << 10, 128 << 10, 200 << 10};
  for (int threads : {256, 1024})
    for (int smem : sms)
      for (int cl : cls) {
        float b2b = run(cl, threads, smem, false, flush, fl);
        float one = run(cl, threads, smem, true, flush, fl);
        printf("threads %4d smem %6d cluster %2d: back-to-back %.2f us, single after flush %.2f us\n",
               threads, smem, cl, b2b, one);
      }
  return 0;
}
