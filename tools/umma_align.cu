// tcgen05.mma SS-mode cost vs the A operand's smem alignment (SWIZZLE_NONE).
// The conv's A operand is a shifted view of a halo tile: core matrices (8
// rows x 16 B) start at any 16-byte offset and 8-row groups are SBO = hz*16
// bytes apart.  This measures cycles per M=128, K=16 MMA for a few
// (start step, SBO) pairs.   nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include "../paper_1903_07525_b200/csrc/vxb_ptx.cuh"
using namespace vxb;

template <int N>
__global__ void bench(int iters, uint32_t a_step, uint32_t a_sbo, uint32_t a_lbo,
                      unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 150 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(smem)[i] = 0x3f803f80u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&tslot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tm = tslot;
  if (warp == 0 && lane == 0) {
    uint32_t a = smem_u32(smem), b = smem_u32(smem + 120 * 1024);
    const uint32_t idesc = idesc_bf16(128, N);
    uint32_t a_lo = desc_lo(a, a_lbo), a_hi = desc_hi(a_sbo);
    uint32_t b_lo = desc_lo(b, 128), b_hi = desc_hi(256);
    const uint32_t st = a_step >> 4;
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int d = 0; d < 4; ++d)
        umma_bf16_lohi(tm + d * (N > 128 ? 0 : 128), a_lo + ((i + d) & 7) * st, a_hi, b_lo, b_hi, idesc, i > 0);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm, 512);
  }
}

template <int N>
void run(uint32_t step, uint32_t sbo, uint32_t lbo) {
  unsigned long long *d, h;
  cudaMalloc(&d, 8 * 148);
  auto k = bench<N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  int iters = 8192;
  k<<<148, 128, 160 * 1024>>>(iters, step, sbo, lbo, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("N=%3d a_step=%4u sbo=%4u lbo=%5u: %.1f cyc/MMA (%s)\n", N, step, sbo, lbo,
         (double)h / iters, cudaGetErrorString(e));
  cudaFree(d);
}

template <int N>
void sweep() {
  run<N>(128, 128, 16384);   // core matrices 128-B aligned, dense
  run<N>(256, 256, 16384);   // aligned, gaps
  run<N>(16, 128, 16384);    // start off by 16 B multiples
  run<N>(16, 160, 16384);    // conv 3x3x3 halo (hz = 10)
  run<N>(160, 160, 16384);   // dy step of the same
  run<N>(16, 256, 16384);    // hz = 16 pitch, dz step
  run<N>(256, 384, 16384);   // 128-aligned pitch, aligned step
  run<N>(16, 160, 23056);    // two-chunk K pair, odd LBO
}


// cta_group::2: the leader issues M = 256 MMAs (128 rows per SM), B split
// between the two CTAs; cycles per instruction as seen by the leader
template <int N>
__global__ void __cluster_dims__(2, 1, 1) bench_pair(int iters, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  for (int i = threadIdx.x; i < 150 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(smem)[i] = 0x3f803f80u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc_pair(&tslot, 512);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  uint32_t tm = tslot;
  if (rank == 0 && warp == 0 && lane == 0) {
    uint32_t a = smem_u32(smem), b = smem_u32(smem + 120 * 1024);
    const uint32_t idesc = idesc_bf16(256, N);
    uint32_t a_lo = desc_lo(a, 16384), a_hi = desc_hi(160);
    uint32_t b_lo = desc_lo(b, 128), b_hi = desc_hi(256);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int d = 0; d < 4; ++d)
        umma_bf16_pair_lohi(tm + d * 96, a_lo + ((i + d) & 7), a_hi, b_lo, b_hi, idesc, i > 0);
    }
    umma_commit_pair(&bar, 0x3);
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  if (rank == 1 && warp == 0) {
    if (lane == 0) mbar_wait(&bar, 0);
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tm, 512);
  }
}

template <int N>
void run_pair() {
  unsigned long long *d, h;
  cudaMalloc(&d, 8 * 148);
  auto k = bench_pair<N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  int iters = 8192;
  k<<<148, 128, 160 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("PAIR M=256 N=%3d: %.1f cyc/instr (%s)\n", N, (double)h / iters, cudaGetErrorString(e));
  cudaFree(d);
}


// commit cadence: an M=128 N=128 MMA stream (4 independent accumulators)
// with a tcgen05.commit to a (never waited) mbarrier every K MMAs, or a
// commit every K MMAs plus a wait on an already-completed barrier phase
template <int MODE>
__global__ void bench_commit(int iters, int every, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  __shared__ uint64_t bar, bar2, done;
  __shared__ uint32_t tslot;
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 150 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(smem)[i] = 0x3f803f80u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&tslot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tm = tslot;
  if (warp == 0 && lane == 0) {
    mbar_arrive(&bar2);   // phase 0 of bar2 complete: waits on it return at once
    uint32_t a = smem_u32(smem), b = smem_u32(smem + 120 * 1024);
    const uint32_t idesc = idesc_bf16(128, 128);
    uint32_t a_lo = desc_lo(a, 16384), a_hi = desc_hi(160);
    uint32_t b_lo = desc_lo(b, 128), b_hi = desc_hi(256);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int d = 0; d < 4; ++d)
        umma_bf16_lohi(tm + d * 128, a_lo + ((i + d) & 7), a_hi, b_lo, b_hi, idesc, i > 0);
      if (((i + 4) % every) == 0) {
        if (MODE >= 1) umma_commit(&bar);
        if (MODE == 2) {
          mbar_wait(&bar2, 0);
          tc_fence_after();
        }
      }
    }
    umma_commit(&done);
    mbar_wait(&done, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm, 512);
  }
}

template <int MODE>
void run_commit(int every) {
  unsigned long long *d, h;
  cudaMalloc(&d, 8 * 148);
  auto k = bench_commit<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  int iters = 8192;
  k<<<148, 128, 160 * 1024>>>(iters, every, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("commit mode %d every %3d MMAs: %.1f cyc/MMA (%s)\n", MODE, every, (double)h / iters,
         cudaGetErrorString(e));
  cudaFree(d);
}


// issue/execute overlap: 2 MMAs (N = 128, independent accumulators) then X
// dependent integer adds on the issuing thread, repeated
template <int X, int K = 2>
__global__ void bench_gap(int iters, unsigned long long *out, int *sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  __shared__ uint64_t done;
  __shared__ uint32_t tslot;
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 150 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t *>(smem)[i] = 0x3f803f80u;
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(&tslot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tm = tslot;
  if (warp == 0 && lane == 0) {
    uint32_t a = smem_u32(smem), b = smem_u32(smem + 120 * 1024);
    const uint32_t idesc = idesc_bf16(128, 128);
    uint32_t a_lo = desc_lo(a, 16384), a_hi = desc_hi(160);
    uint32_t b_lo = desc_lo(b, 128), b_hi = desc_hi(256);
    int acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; i += K) {
#pragma unroll
      for (int q = 0; q < K; ++q)
        umma_bf16_lohi(tm + (q & 3) * 128, a_lo + q, a_hi, b_lo, b_hi, idesc, i > 0);
#pragma unroll
      for (int x = 0; x < X; ++x) asm volatile("add.u32 %0, %0, %1;" : "+r"(acc) : "r"(i));
    }
    umma_commit(&done);
    mbar_wait(&done, 0);
    out[blockIdx.x] = clock64() - t0;
    sink[blockIdx.x] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm, 512);
  }
}

template <int X, int K = 2>
void run_gap() {
  unsigned long long *d, h;
  int *sk;
  cudaMalloc(&d, 8 * 148);
  cudaMalloc(&sk, 4 * 148);
  auto k = bench_gap<X, K>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  int iters = 8192;
  k<<<148, 128, 160 * 1024>>>(iters, d, sk);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%d MMAs + %3d dependent adds: %.1f cyc/MMA (%s)\n", K, X, (double)h / iters,
         cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sk);
}

int main() {
  run_gap<0, 8>();
  run_gap<64, 8>();
  run_gap<128, 8>();
  run_gap<192, 8>();
  run_gap<256, 8>();
  run_gap<0, 16>();
  run_gap<256, 16>();
  run_gap<512, 16>();
  run_gap<0>();
  run_gap<8>();
  run_gap<16>();
  run_gap<32>();
  run_gap<64>();
  run_gap<128>();

  for (int every : {4, 8, 16, 32, 64, 1 << 20}) {
    run_commit<1>(every);
    run_commit<2>(every);
  }

  run_pair<16>();
  run_pair<32>();
  run_pair<48>();
  run_pair<64>();
  run_pair<96>();
  run_pair<128>();
  run_pair<192>();
  run_pair<256>();
  sweep<16>();
  sweep<48>();
  sweep<96>();
  sweep<128>();
  run<192>(16, 160, 16384);
  return 0;
}
