// TMA throughput of two A-tile box shapes over a blocked bf16 volume
// (chunk, x, y, z, 8 lanes): the conv's current 4-D box (8*hz, hy, hx, 1)
// with 16-byte rows flattened into dim 0, and a 5-D box (8, hz, hy, 1, 1)
// whose innermost dimension is a single 16-byte row (z-row tiles).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/tma_probe.cu -o tools/tma_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sptr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int DIMS>
__global__ void probe(const __grid_constant__ CUtensorMap m, int loads, int bytes, int nx, int ny,
                      int nz, int hx, int hy, int hz) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[2];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sptr(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t ph[2] = {0, 0};
  for (int i = 0; i < loads; ++i) {
    const int s = i & 1;
    if (i >= 2) {   // wait for the load two back into this slot
      asm volatile(
          "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra W_%=;\n}" ::"r"(sptr(&bar[s])), "r"(ph[s]));
      ph[s] ^= 1;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(&bar[s])),
                 "r"(bytes));
    const int t = blockIdx.x + i * gridDim.x;
    const int c = t & 3, r = t >> 2;
    const int x = (r % (nx / hx)) * hx, y = ((r / (nx / hx)) % (ny / 16)) * 16,
              z = ((r / (nx / hx) / (ny / 16)) % (nz / 128)) * 128;
    void *dst = smem + s * 65536;
    if (DIMS == 4)
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sptr(dst)),
          "l"(&m), "r"(z * 8), "r"(y), "r"(x), "r"(c), "r"(sptr(&bar[s]))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sptr(dst)),
          "l"(&m), "r"(0), "r"(z - 1), "r"(y), "r"(x), "r"(c), "r"(sptr(&bar[s]))
          : "memory");
  }
  for (int s = 0; s < 2; ++s)
    asm volatile(
        "{\n\t.reg .pred p;\nV_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra V_%=;\n}" ::"r"(sptr(&bar[s])), "r"(ph[s]));
}

typedef CUresult (*Enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                        const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                        CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                        CUtensorMapFloatOOBfill);

int main() {
  const int C = 4, NX = 216, NY = 192, NZ = 192;   // 509 MB of bf16: larger than L2
  const size_t elems = size_t(C) * NX * NY * NZ * 8;
  void *buf;
  cudaMalloc(&buf, elems * 2);
  cudaMemset(buf, 0, elems * 2);
  void *fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Enc enc = reinterpret_cast<Enc>(fn);
  const cuuint64_t sz = 16, sy = sz * NZ, sx = sy * NY, sc = sx * NX;
  cudaFuncSetAttribute(probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(probe<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  const int grid = 148, loads = 400;
  for (int mode = 0; mode < 3; ++mode) {
    CUtensorMap m;
    CUresult r;
    int bytes;
    if (mode == 0) {   // current 3x3x3 A box: 8 x-slices x 18 y x 10 z
      cuuint64_t dims[4] = {cuuint64_t(8) * NZ, NY, NX, C};
      cuuint64_t str[3] = {sy, sx, sc};
      cuuint32_t box[4] = {80, 18, 8, 1}, es[4] = {1, 1, 1, 1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, str, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      bytes = 80 * 18 * 8 * 2;
    } else {           // z-row box: 130 z x 10 y (x one plane); mode 2: 34 z x 10 y x 4 x
      cuuint64_t dims[5] = {8, NZ, NY, NX, C};
      cuuint64_t str[4] = {sz, sy, sx, sc};
      cuuint32_t box[5] = {8, mode == 1 ? 130u : 34u, 10, mode == 1 ? 1u : 4u, 1},
                 es[5] = {1, 1, 1, 1, 1};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, buf, dims, str, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      bytes = 8 * box[1] * box[2] * box[3] * 2;
    }
    if (r != CUDA_SUCCESS) {
      printf("mode %d encode failed %d\n", mode, int(r));
      continue;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0)
        probe<4><<<grid, 32, 131072>>>(m, loads, bytes, NX, NY, NZ, 8, 16, 8);
      else
        probe<5><<<grid, 32, 131072>>>(m, loads, bytes, NX, NY, NZ, 1, 16, 128);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("mode %d box bytes %d: %.3f ms, %.0f GB/s (err %s)\n", mode, bytes, ms,
             double(bytes) * loads * grid / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
