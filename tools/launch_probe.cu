// Launch overhead of an empty persistent-style kernel (148 CTAs x 608
// threads) at several dynamic shared-memory sizes, back to back and after an
// L2-flushing memset.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/launch_probe.cu -o tools/launch_probe
#include <cuda_runtime.h>
#include <cstdio>
__global__ void empty_k(int *p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}
int main() {
  cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  void *flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int kb : {0, 64, 128, 200}) {
    for (int burst : {1, 20}) {
      float best = 1e9;
      for (int rep = 0; rep < 10; ++rep) {
        cudaMemsetAsync(flush, rep, 256 << 20);
        cudaEventRecord(e0);
        for (int i = 0; i < burst; ++i) empty_k<<<148, 608, kb * 1024>>>(nullptr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      printf("smem %3d KB burst %2d: %.2f us per launch\n", kb, burst, best * 1e3 / burst);
    }
  }
  return 0;
}
