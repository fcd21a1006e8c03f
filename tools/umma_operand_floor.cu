// tcgen05.mma SS-mode cost vs N and smem layout (SWIZZLE_NONE vs 128B swizzle).
#include <cstdio>
#include <cstdint>
#include "../paper_1903_07525_b200/csrc/vxb_ptx.cuh"
using namespace vxb;

// layout: 0 = SWIZZLE_NONE (our core-matrix layout), 2 = SWIZZLE_128B K-major
template <int N, int LAYOUT, int ND>
__global__ void bench(int iters, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x3f803f80u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(&tslot, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tm = tslot;
  if (warp == 0 && lane == 0) {
    uint32_t a = smem_u32(smem), b = smem_u32(smem + 48 * 1024);
    const uint32_t idesc = idesc_bf16(128, N);
    uint32_t a_lo, a_hi, b_lo, b_hi;
    if (LAYOUT == 0) {
      a_lo = desc_lo(a, 128); a_hi = desc_hi(256);
      b_lo = desc_lo(b, 128); b_hi = desc_hi(256);
    } else {
      // K-major SW128: rows of 128 B, 8-row atoms 1024 B apart; LBO unused
      a_lo = desc_lo(a, 16); a_hi = desc_hi(1024) | (2u << 29);
      b_lo = desc_lo(b, 16); b_hi = desc_hi(1024) | (2u << 29);
    }
    long long t0 = clock64();
    for (int i = 0; i < iters; i += ND) {
#pragma unroll
      for (int d = 0; d < ND; ++d)
        umma_bf16_lohi(tm + d * 128, a_lo + ((i + d) & 3) * 2, a_hi, b_lo + ((i + d) & 3) * 2, b_hi, idesc, i > 0);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

template <int N, int LAYOUT>
void run() {
  unsigned long long *d, h;
  cudaMalloc(&d, 8 * 148);
  auto k = bench<N, LAYOUT, 4>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  int iters = 8192;
  k<<<148, 128, 100 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("layout %s N=%3d: %.1f cyc/MMA  (%s)\n", LAYOUT ? "SW128" : "NONE ", N, (double)h / iters,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<16, 0>(); run<16, 2>();
  run<32, 0>(); run<32, 2>();
  run<48, 0>(); run<48, 2>();
  run<64, 0>(); run<64, 2>();
  run<96, 0>(); run<96, 2>();
  run<128, 0>(); run<128, 2>();
  run<256, 0>(); run<256, 2>();
  return 0;
}
