// ops.cu — bandwidth kernels and the CUDA-core convolution paths.
//
//   direct conv      generic strides / kernel sizes (reference a1 semantics,
//                    _kernels.pyx:44-179) on CUDA cores; also the subimage
//                    debug primitive (_kernels.pyx:182-271)
//   gather deconv    transposed conv for k != stride (kernels_py.py:162-196)
//   pool             ops.pool (ops.py:63-86)
//   eltwise          ops.eltwise (ops.py:50-60)
//   affine_act       ops.linear_transform + ops.activation (ops.py:89-102)
//   mergecrop        ops.mergecrop (ops.py:113-136)
//   pad_copy         ops.pad_copy (ops.py:105-110)
//   copy             to_blocked / from_blocked (blocked.py:209-231)
//
// All element-wise kernels work on one 8-fmap chunk per thread: for the
// blocked bf16 layout that is one 16-byte load/store, z fastest across the
// warp so a warp touches 512 contiguous bytes.
#include <algorithm>
#include <cuda_bf16.h>
#include "vxb_internal.h"

namespace vxb {



__device__ __forceinline__ long long voff(const DView &v, int b, int c, int x, int y, int z) {
  return b * v.s[0] + (v.blocked ? (c >> 3) * v.s[1] + (c & 7) : c * v.s[1]) + x * v.s[2] +
         y * v.s[3] + z * v.s[4];
}
// element access; split bf16 (VXB_BF16X2, blocked) holds hi at i and lo at
// i + s[1]/2, the value is their (exact) fp32 sum
__device__ __forceinline__ float vld(const DView &v, long long i) {
  if (v.dtype == VXB_BF16X2) {
    const __nv_bfloat16 *p = static_cast<const __nv_bfloat16 *>(v.data);
    return __bfloat162float(p[i]) + __bfloat162float(p[i + (v.s[1] >> 1)]);
  }
  return v.dtype == VXB_BF16 ? __bfloat162float(static_cast<const __nv_bfloat16 *>(v.data)[i])
                             : static_cast<const float *>(v.data)[i];
}
__device__ __forceinline__ void vst(const DView &v, long long i, float f) {
  if (v.dtype == VXB_BF16X2) {
    __nv_bfloat16 *p = static_cast<__nv_bfloat16 *>(v.data);
    const __nv_bfloat16 hi = __float2bfloat16_rn(f);
    p[i] = hi;
    p[i + (v.s[1] >> 1)] = __float2bfloat16_rn(f - __bfloat162float(hi));
  } else if (v.dtype == VXB_BF16) {
    static_cast<__nv_bfloat16 *>(v.data)[i] = __float2bfloat16_rn(f);
  } else {
    static_cast<float *>(v.data)[i] = f;
  }
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4 &u, float (&r)[8]) {
  const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    r[2 * i] = f.x;
    r[2 * i + 1] = f.y;
  }
}
// hi = bf16(r), lo = bf16(r - hi), 8 lanes each
__device__ __forceinline__ void f32_to_split8(const float (&r)[8], uint4 &hi, uint4 &lo) {
  __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&hi);
  __nv_bfloat162 *l = reinterpret_cast<__nv_bfloat162 *>(&lo);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    h[i] = __floats2bfloat162_rn(r[2 * i], r[2 * i + 1]);
    const float2 f = __bfloat1622float2(h[i]);
    l[i] = __floats2bfloat162_rn(r[2 * i] - f.x, r[2 * i + 1] - f.y);
  }
}

// chunk-granular access: lanes [0, 8) of chunk `ch` at voxel (b,x,y,z)
__device__ __forceinline__ void ld_chunk(const DView &v, int b, int ch, int x, int y, int z,
                                         float (&r)[8]) {
  if (v.blocked) {
    long long o = b * v.s[0] + ch * v.s[1] + x * v.s[2] + y * v.s[3] + z * v.s[4];
    if (v.dtype == VXB_BF16X2) {
      const __nv_bfloat16 *p = static_cast<const __nv_bfloat16 *>(v.data) + o;
      float lo[8];
      bf16x8_to_f32(*reinterpret_cast<const uint4 *>(p), r);
      bf16x8_to_f32(*reinterpret_cast<const uint4 *>(p + (v.s[1] >> 1)), lo);
#pragma unroll
      for (int i = 0; i < 8; ++i) r[i] += lo[i];
    } else if (v.dtype == VXB_BF16) {
      uint4 u = *reinterpret_cast<const uint4 *>(static_cast<const __nv_bfloat16 *>(v.data) + o);
      const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float2 f = __bfloat1622float2(h[i]);
        r[2 * i] = f.x;
        r[2 * i + 1] = f.y;
      }
    } else {
      const float *p = static_cast<const float *>(v.data) + o;
      float4 a = *reinterpret_cast<const float4 *>(p), c = *reinterpret_cast<const float4 *>(p + 4);
      r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
      r[4] = c.x; r[5] = c.y; r[6] = c.z; r[7] = c.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int c = ch * 8 + i;
      r[i] = c < v.c ? vld(v, voff(v, b, c, x, y, z)) : 0.f;
    }
  }
}
// writes all 8 lanes for blocked views (caller zeroes lanes >= c), valid
// channels only for standard views
__device__ __forceinline__ void st_chunk(const DView &v, int b, int ch, int x, int y, int z,
                                         const float (&r)[8]) {
  if (v.blocked) {
    long long o = b * v.s[0] + ch * v.s[1] + x * v.s[2] + y * v.s[3] + z * v.s[4];
    if (v.dtype == VXB_BF16X2) {
      uint4 hi, lo;
      f32_to_split8(r, hi, lo);
      __nv_bfloat16 *p = static_cast<__nv_bfloat16 *>(v.data) + o;
      *reinterpret_cast<uint4 *>(p) = hi;
      *reinterpret_cast<uint4 *>(p + (v.s[1] >> 1)) = lo;
    } else if (v.dtype == VXB_BF16) {
      uint4 u;
      __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(r[2 * i], r[2 * i + 1]);
      *reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(v.data) + o) = u;
    } else {
      float *p = static_cast<float *>(v.data) + o;
      *reinterpret_cast<float4 *>(p) = make_float4(r[0], r[1], r[2], r[3]);
      *reinterpret_cast<float4 *>(p + 4) = make_float4(r[4], r[5], r[6], r[7]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int c = ch * 8 + i;
      if (c < v.c) vst(v, voff(v, b, c, x, y, z), r[i]);
    }
  }
}

__device__ __forceinline__ float act_fn(float v, int act, float alpha) {
  if (act == VXB_ACT_RELU) return v > 0.f ? v : 0.f;
  if (act == VXB_ACT_ELU) return v > 0.f ? v : alpha * expm1f(v);
  if (act == VXB_ACT_SIGMOID) return 1.f / (1.f + expf(-v));
  return v;
}

// 3-D launch grid: x covers y*z (z fastest, coalesced), y = x, z = batch*chunk
struct ChunkIdx {
  int b, ch, x, y, z;
};

__device__ __forceinline__ bool chunk_index3(int nch, int Y, int Z, ChunkIdx &o) {
  const int yz = blockIdx.x * blockDim.x + threadIdx.x;
  if (yz >= Y * Z) return false;
  o.y = yz / Z;
  o.z = yz - o.y * Z;
  o.x = blockIdx.y;
  o.b = blockIdx.z / nch;
  o.ch = blockIdx.z - o.b * nch;
  return true;
}

__device__ __forceinline__ void zero_tail_lanes(float (&r)[8], int ch, int c) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (ch * 8 + i >= c) r[i] = 0.f;
}

// ------------------------------------------------------------------ copy
__global__ void copy_kernel(DView src, DView dst) {
  pdl_begin();
  ChunkIdx k;
  int nch = (dst.c + 7) >> 3;
  if (chunk_index3(nch, dst.y, dst.z, k)) {
    float r[8];
    ld_chunk(src, k.b, k.ch, k.x, k.y, k.z, r);
    zero_tail_lanes(r, k.ch, dst.c);
    st_chunk(dst, k.b, k.ch, k.x, k.y, k.z, r);
  }
}

__global__ void zero_kernel(DView dst) {
  pdl_begin();
  ChunkIdx k;
  int nch = (dst.c + 7) >> 3;
  if (chunk_index3(nch, dst.y, dst.z, k)) {
    float r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (dst.blocked) {
      st_chunk(dst, k.b, k.ch, k.x, k.y, k.z, r);
    } else {
      for (int l = 0; l < 8; ++l)
        if (k.ch * 8 + l < dst.c) vst(dst, voff(dst, k.b, k.ch * 8 + l, k.x, k.y, k.z), 0.f);
    }
  }
}

// ------------------------------------------------------------------ pool
// max: seed with the first window element, then max in (dx,dy,dz) order with
// np.maximum NaN propagation; avg: fp32 sum in the same order, / kvol.
__global__ void pool_kernel(DView in, DView out, int kx, int ky, int kz, int sx, int sy, int sz,
                            int mode) {
  pdl_begin();
  ChunkIdx k;
  int nch = (out.c + 7) >> 3;
  if (chunk_index3(nch, out.y, out.z, k)) {
    float r[8], t[8];
    bool first = true;
    for (int dx = 0; dx < kx; ++dx)
      for (int dy = 0; dy < ky; ++dy)
        for (int dz = 0; dz < kz; ++dz) {
          ld_chunk(in, k.b, k.ch, k.x * sx + dx, k.y * sy + dy, k.z * sz + dz, t);
          if (first) {
#pragma unroll
            for (int l = 0; l < 8; ++l) r[l] = t[l];
            first = false;
          } else if (mode == VXB_POOL_MAX) {
#pragma unroll
            for (int l = 0; l < 8; ++l) r[l] = (t[l] > r[l] || t[l] != t[l]) ? t[l] : r[l];
          } else {
#pragma unroll
            for (int l = 0; l < 8; ++l) r[l] += t[l];
          }
        }
    if (mode == VXB_POOL_AVG) {
      float kv = static_cast<float>(kx * ky * kz);
#pragma unroll
      for (int l = 0; l < 8; ++l) r[l] = r[l] / kv;
    }
    zero_tail_lanes(r, k.ch, out.c);
    st_chunk(out, k.b, k.ch, k.x, k.y, k.z, r);
  }
}

// Max pool fast path: bf16 blocked in/out, window (KX, 2, 2) = stride (the
// U-net pools: 2x2x2 in config 4, 1x2x2 in config 5).  All 4*KX 16-byte
// window loads are issued before the reduction (the generic kernel's runtime
// window loop exposes each load's latency), then the same seeded
// (dx, dy, dz)-order comparison as pool_kernel / ops.pool (NaN-propagating).
template <int KX>
__global__ void pool_max_bf16_kernel(DView in, DView out) {
  pdl_begin();
  ChunkIdx k;
  const int nch = (out.c + 7) >> 3;
  if (!chunk_index3(nch, out.y, out.z, k)) return;
  const __nv_bfloat16 *base = static_cast<const __nv_bfloat16 *>(in.data) + k.b * in.s[0] +
                              k.ch * in.s[1] + (k.x * KX) * in.s[2] + (2 * k.y) * in.s[3] +
                              (2 * k.z) * in.s[4];
  uint4 v[KX * 4];
#pragma unroll
  for (int dx = 0; dx < KX; ++dx)
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
      for (int dz = 0; dz < 2; ++dz)
        v[(dx * 2 + dy) * 2 + dz] = __ldg(reinterpret_cast<const uint4 *>(
            base + dx * in.s[2] + dy * in.s[3] + dz * in.s[4]));
  float r[8];
  {
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v[0]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      r[2 * i] = f.x;
      r[2 * i + 1] = f.y;
    }
  }
#pragma unroll
  for (int w = 1; w < KX * 4; ++w) {
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v[w]);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      r[2 * i] = (f.x > r[2 * i] || f.x != f.x) ? f.x : r[2 * i];
      r[2 * i + 1] = (f.y > r[2 * i + 1] || f.y != f.y) ? f.y : r[2 * i + 1];
    }
  }
  zero_tail_lanes(r, k.ch, out.c);
  st_chunk(out, k.b, k.ch, k.x, k.y, k.z, r);
}

// ------------------------------------------------------------------ eltwise
__global__ void eltwise_kernel(DView a, DView b, DView out, int op) {
  pdl_begin();
  ChunkIdx k;
  int nch = (out.c + 7) >> 3;
  if (chunk_index3(nch, out.y, out.z, k)) {
    float ra[8], rb[8], r[8];
    ld_chunk(a, k.b, k.ch, k.x, k.y, k.z, ra);
    ld_chunk(b, k.b, k.ch, k.x, k.y, k.z, rb);
#pragma unroll
    for (int l = 0; l < 8; ++l)
      r[l] = op == VXB_ELT_ADD ? ra[l] + rb[l] : (op == VXB_ELT_MUL ? ra[l] * rb[l] : ra[l] / rb[l]);
    zero_tail_lanes(r, k.ch, out.c);
    st_chunk(out, k.b, k.ch, k.x, k.y, k.z, r);
  }
}

// ------------------------------------------------------------------ affine + act
__global__ void affine_act_kernel(DView in, DView out, const float *mult, const float *add, int act,
                                  float alpha) {
  pdl_begin();
  ChunkIdx k;
  int nch = (out.c + 7) >> 3;
  if (chunk_index3(nch, out.y, out.z, k)) {
    float r[8];
    ld_chunk(in, k.b, k.ch, k.x, k.y, k.z, r);
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      int c = k.ch * 8 + l;
      if (c < out.c) {
        float v = r[l];
        if (mult) v = v * mult[c];
        if (add) v = v + add[c];
        r[l] = act_fn(v, act, alpha);
      }
    }
    zero_tail_lanes(r, k.ch, out.c);
    st_chunk(out, k.b, k.ch, k.x, k.y, k.z, r);
  }
}

// ------------------------------------------------------------------ mergecrop
__global__ void mergecrop_kernel(DView a, DView b, DView out, int oax, int oay, int oaz, int obx,
                                 int oby, int obz) {
  pdl_begin();
  ChunkIdx k;
  int nch = (out.c + 7) >> 3;
  if (chunk_index3(nch, out.y, out.z, k)) {
    float r[8];
    if ((a.c & 7) == 0 && a.blocked && b.blocked) {
      int ach = a.c >> 3;
      if (k.ch < ach)
        ld_chunk(a, k.b, k.ch, k.x + oax, k.y + oay, k.z + oaz, r);
      else
        ld_chunk(b, k.b, k.ch - ach, k.x + obx, k.y + oby, k.z + obz, r);
    } else {
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        int c = k.ch * 8 + l;
        if (c < a.c)
          r[l] = vld(a, voff(a, k.b, c, k.x + oax, k.y + oay, k.z + oaz));
        else if (c < a.c + b.c)
          r[l] = vld(b, voff(b, k.b, c - a.c, k.x + obx, k.y + oby, k.z + obz));
        else
          r[l] = 0.f;
      }
    }
    zero_tail_lanes(r, k.ch, out.c);
    st_chunk(out, k.b, k.ch, k.x, k.y, k.z, r);
  }
}

// ------------------------------------------------------------------ pad copy
__global__ void pad_copy_kernel(DView in, DView out, int px, int py, int pz) {
  pdl_begin();
  ChunkIdx k;
  int nch = (out.c + 7) >> 3;
  if (chunk_index3(nch, out.y, out.z, k)) {
    float r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int x = k.x - px, y = k.y - py, z = k.z - pz;
    if (x >= 0 && y >= 0 && z >= 0 && x < in.x && y < in.y && z < in.z)
      ld_chunk(in, k.b, k.ch, x, y, z, r);
    zero_tail_lanes(r, k.ch, out.c);
    st_chunk(out, k.b, k.ch, k.x, k.y, k.z, r);
  }
}

// ------------------------------------------------------------------ direct conv
// One CTA = 128 output voxels (2 x 8 x 8) x 16 output fmaps.  Input chunks
// are staged through shared memory (fp32), weights too.  Packed weight
// layout: [cout_group(16)][in_chunk][tap][8 in][16 out] fp32.


constexpr int DT_X = 2, DT_Y = 8, DT_Z = 8, DCO = 16;

__global__ void __launch_bounds__(128) conv_direct_kernel(DirectParams p) {
  pdl_begin();
  extern __shared__ float dsm[];
  const int taps = p.kx * p.ky * p.kz;
  float *patch = dsm;                                   // [hx][hy][hz][8]
  float *wsm = dsm + p.hx * p.hy * p.hz * 8;            // [tap][8][16]
  int t = blockIdx.x;
  int tz = t % p.tiles_z;
  t /= p.tiles_z;
  int ty = t % p.tiles_y;
  int tx = t / p.tiles_y;
  const int cg = blockIdx.y, b = blockIdx.z;
  const int lx = threadIdx.x / (DT_Y * DT_Z), ly = (threadIdx.x / DT_Z) % DT_Y,
            lz = threadIdx.x % DT_Z;
  const int x0 = tx * DT_X, y0 = ty * DT_Y, z0 = tz * DT_Z;
  const int ox = x0 + lx, oy = y0 + ly, oz = z0 + lz;
  float acc[DCO];
#pragma unroll
  for (int i = 0; i < DCO; ++i) acc[i] = 0.f;
  const int in_chunks = (p.cin + 7) >> 3;
  const int npatch = p.hx * p.hy * p.hz;
  for (int ch = 0; ch < in_chunks; ++ch) {
    const int lanes = min(8, p.cin - ch * 8);
    __syncthreads();
    for (int i = threadIdx.x; i < npatch; i += blockDim.x) {
      int iz = i % p.hz, iy = (i / p.hz) % p.hy, ix = i / (p.hz * p.hy);
      int gx = x0 * p.sx - p.px + ix, gy = y0 * p.sy - p.py + iy, gz = z0 * p.sz - p.pz + iz;
      float r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (gx >= 0 && gy >= 0 && gz >= 0 && gx < p.in.x && gy < p.in.y && gz < p.in.z)
        ld_chunk(p.in, b, ch, gx, gy, gz, r);
#pragma unroll
      for (int l = 0; l < 8; ++l) patch[i * 8 + l] = r[l];
    }
    const float *wsrc = p.w + (static_cast<long long>(cg) * in_chunks + ch) * taps * 8 * DCO;
    for (int i = threadIdx.x; i < taps * 8 * DCO; i += blockDim.x) wsm[i] = wsrc[i];
    __syncthreads();
    for (int dx = 0; dx < p.kx; ++dx)
      for (int dy = 0; dy < p.ky; ++dy)
        for (int dz = 0; dz < p.kz; ++dz) {
          const int tap = (dx * p.ky + dy) * p.kz + dz;
          const float *src =
              patch + (((lx * p.sx + dx) * p.hy + ly * p.sy + dy) * p.hz + lz * p.sz + dz) * 8;
          const float *wt = wsm + tap * 8 * DCO;
          for (int l = 0; l < lanes; ++l) {
            const float v = src[l];
#pragma unroll
            for (int o = 0; o < DCO; ++o) acc[o] = fmaf(v, wt[l * DCO + o], acc[o]);
          }
        }
  }
  if (ox >= p.out.x || oy >= p.out.y || oz >= p.out.z) return;
#pragma unroll
  for (int h = 0; h < DCO / 8; ++h) {
    const int ch = cg * (DCO / 8) + h;
    if (ch * 8 >= p.cout) continue;
    float r[8], bv[8];
    if (p.has_base) ld_chunk(p.base, b, ch, ox, oy, oz, bv);
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      int c = ch * 8 + l;
      if (c < p.cout) {
        float init = p.bias[c];
        if (p.has_base) init += (p.scale ? p.scale[c] : 1.f) * bv[l];
        r[l] = act_fn(init + acc[h * 8 + l], p.act, p.alpha);
      } else {
        r[l] = 0.f;
      }
    }
    st_chunk(p.out, b, ch, ox, oy, oz, r);
  }
}

// ------------------------------------------------------------------ subimage
// one input chunk -> one output patch, through memory (test primitive)


__global__ void subimage_kernel(SubParams p) {
  pdl_begin();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int nb = p.out.n;
  int total = nb * p.ex * p.ey * p.ez * 8;
  if (i >= total) return;
  int o = i % 8;
  int v = i / 8;
  int zz = v % p.ez;
  v /= p.ez;
  int yy = v % p.ey;
  v /= p.ey;
  int xx = v % p.ex;
  int b = v / p.ex;
  int x = p.x0 + xx, y = p.y0 + yy, z = p.z0 + zz;
  int co = p.ob * 8 + o;
  long long oo = b * p.out.s[0] + p.ob * p.out.s[1] + o + x * p.out.s[2] + y * p.out.s[3] +
                 z * p.out.s[4];
  float acc;
  if (p.first) {
    acc = co < p.cout ? p.bias[co] : 0.f;
    if (p.has_base && co < p.cout)
      acc += (p.scale ? p.scale[co] : 1.f) *
             vld(p.base, b * p.base.s[0] + p.ob * p.base.s[1] + o + x * p.base.s[2] +
                             y * p.base.s[3] + z * p.base.s[4]);
  } else {
    acc = vld(p.out, oo);
  }
  for (int dx = 0; dx < p.kx; ++dx)
    for (int dy = 0; dy < p.ky; ++dy)
      for (int dz = 0; dz < p.kz; ++dz)
        for (int l = 0; l < 8; ++l) {
          int ci = p.ib * 8 + l;
          if (ci >= p.cin || co >= p.cout) continue;
          float xv = vld(p.in, b * p.in.s[0] + p.ib * p.in.s[1] + l +
                                   (x * p.sx + dx) * p.in.s[2] + (y * p.sy + dy) * p.in.s[3] +
                                   (z * p.sz + dz) * p.in.s[4]);
          float wv = p.w[(((static_cast<long long>(co) * p.cin + ci) * p.kx + dx) * p.ky + dy) *
                             p.kz + dz];
          acc = fmaf(xv, wv, acc);
        }
  if (p.last) acc = co < p.cout ? act_fn(acc, p.act, p.alpha) : 0.f;
  vst(p.out, oo, acc);
}

// ------------------------------------------------------------------ gather deconv
// out[o] = act(bias + [base] + sum_{ci,d: (o-d)%s==0} in[(o-d)/s] W[co][ci][d])


__global__ void deconv_gather_kernel(GatherDeconvParams p) {
  pdl_begin();
  ChunkIdx k;
  int nch = (p.out.c + 7) >> 3;
  if (chunk_index3(nch, p.out.y, p.out.z, k)) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int dx = 0; dx < p.kx; ++dx) {
      int ix = k.x - dx;
      if (ix < 0 || ix % p.sx) continue;
      ix /= p.sx;
      if (ix >= p.in.x) continue;
      for (int dy = 0; dy < p.ky; ++dy) {
        int iy = k.y - dy;
        if (iy < 0 || iy % p.sy) continue;
        iy /= p.sy;
        if (iy >= p.in.y) continue;
        for (int dz = 0; dz < p.kz; ++dz) {
          int iz = k.z - dz;
          if (iz < 0 || iz % p.sz) continue;
          iz /= p.sz;
          if (iz >= p.in.z) continue;
          for (int ci = 0; ci < p.cin; ++ci) {
            float xv = vld(p.in, voff(p.in, k.b, ci, ix, iy, iz));
#pragma unroll
            for (int l = 0; l < 8; ++l) {
              int co = k.ch * 8 + l;
              if (co < p.cout)
                acc[l] = fmaf(xv,
                              p.w[(((static_cast<long long>(co) * p.cin + ci) * p.kx + dx) * p.ky +
                                   dy) * p.kz + dz],
                              acc[l]);
            }
          }
        }
      }
    }
    float r[8], bv[8];
    if (p.has_base) ld_chunk(p.base, k.b, k.ch, k.x, k.y, k.z, bv);
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      int co = k.ch * 8 + l;
      if (co < p.cout) {
        float init = p.bias[co];
        if (p.has_base) init += (p.scale ? p.scale[co] : 1.f) * bv[l];
        r[l] = act_fn(init + acc[l], p.act, p.alpha);
      } else {
        r[l] = 0.f;
      }
    }
    st_chunk(p.out, k.b, k.ch, k.x, k.y, k.z, r);
  }
}

// ------------------------------------------------------------------ launchers

static dim3 grid3(const DView &v, int threads) {
  return dim3((v.y * v.z + threads - 1) / threads, v.x, v.n * ((v.c + 7) / 8));
}

// Network-boundary pack: fp32 NCDHW (z contiguous) -> bf16 blocked (or split
// bf16: hi and lo chunks).  Each thread converts 4 consecutive z of one
// 8-fmap chunk: 8 float4 loads (one per fmap plane, 512 B per warp
// instruction) and 4 16-byte stores (8 when split).
// One pack item: 4 consecutive z of one 8-fmap chunk at (b, ch, x, y).
__device__ __forceinline__ void pack_item(const DView &src, const DView &dst, int b, int ch, int x,
                                          int y, int z) {
  float v[8][4];
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    const int c = ch * 8 + l;
    if (c < src.c) {
      const float4 f = *reinterpret_cast<const float4 *>(
          static_cast<const float *>(src.data) + b * src.s[0] + c * src.s[1] + x * src.s[2] +
          y * src.s[3] + z);
      v[l][0] = f.x; v[l][1] = f.y; v[l][2] = f.z; v[l][3] = f.w;
    } else {
      v[l][0] = v[l][1] = v[l][2] = v[l][3] = 0.f;
    }
  }
  __nv_bfloat16 *o = static_cast<__nv_bfloat16 *>(dst.data) + b * dst.s[0] + ch * dst.s[1] +
                     x * dst.s[2] + y * dst.s[3] + z * dst.s[4];
  if (dst.dtype == VXB_BF16X2) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float r[8];
#pragma unroll
      for (int l = 0; l < 8; ++l) r[l] = v[l][q];
      uint4 hi, lo;
      f32_to_split8(r, hi, lo);
      *reinterpret_cast<uint4 *>(o + q * dst.s[4]) = hi;
      *reinterpret_cast<uint4 *>(o + q * dst.s[4] + (dst.s[1] >> 1)) = lo;
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[2 * k][q], v[2 * k + 1][q]);
    *reinterpret_cast<uint4 *>(o + q * dst.s[4]) = u;
  }
}

__global__ void pack_std_f32_kernel(DView src, DView dst) {
  pdl_begin();
  const int zq = dst.z >> 2;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dst.y * zq) return;
  const int y = i / zq, z = (i - y * zq) * 4, x = blockIdx.y;
  const int nch = (dst.c + 7) >> 3;
  const int b = blockIdx.z / nch, ch = blockIdx.z - b * nch;
  pack_item(src, dst, b, ch, x, y, z);
}

// Independent variant (VXB_COPY_INDEPENDENT): reads only a network input and
// writes a buffer no kernel before it in the stream touches, so it skips
// griddepcontrol.wait and may run beside its predecessor (the previous
// network's persistent conv, whose one CTA per SM leaves room for one pack
// CTA).  Its dependents launch only when it completes.  (A grid-stride
// variant with 4 CTAs per SM measured slower: 1.05 vs 0.89 ms per config-2
// step — fewer loads in flight, and no full-occupancy tail once the conv
// ends.)
__global__ void pack_std_f32_indep_kernel(DView src, DView dst, int trigger) {
  if (trigger) pdl_trigger();
  const int zq = dst.z >> 2;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dst.y * zq) return;
  const int y = i / zq, z = (i - y * zq) * 4, x = blockIdx.y;
  const int nch = (dst.c + 7) >> 3;
  const int b = blockIdx.z / nch, ch = blockIdx.z - b * nch;
  pack_item(src, dst, b, ch, x, y, z);
}

// z-window pack of a single-channel network input for a conv with kz z-taps
// (pad pz): lane l of output voxel (x, y, z) holds in(x, y, z + l - pz), lanes
// >= kz and out-of-range taps zero.  The conv then runs as a (kx, ky, 1)
// kernel over kz "channels" (w'(co, l, dx, dy, 0) = w(co, 0, dx, dy, l)):
// half the K steps of the 1-channel conv, whose 8-lane chunks were 7/8
// padding.  Each thread writes 4 consecutive z (4 x 16-byte chunks).
template <bool INDEP, bool WIN = false>
__global__ void pack_zwin_kernel(DView src, DView dst, int kz, int pz, int trigger,
                                 const __grid_constant__ ZwinWindows win) {
  if (!INDEP) pdl_begin();
  else if (trigger) pdl_trigger();
  const int zq = (dst.z + 3) >> 2;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dst.y * zq) return;
  const int y = i / zq, z0 = (i - y * zq) * 4, x = blockIdx.y, b = blockIdx.z;
  // WIN: batch entry b reads its own window of one source volume (the
  // patches of a tiled run, gathered while packing)
  const float *row = static_cast<const float *>(src.data) + (WIN ? win.off[b] : b * src.s[0]) +
                     x * src.s[2] + y * src.s[3];
  float v[4 + 8 - 1];
#pragma unroll
  for (int j = 0; j < 11; ++j) {
    const int zz = z0 + j - pz;
    v[j] = (j < 3 + kz && zz >= 0 && zz < src.z) ? row[zz * src.s[4]] : 0.f;
  }
  __nv_bfloat16 *o = static_cast<__nv_bfloat16 *>(dst.data) + b * dst.s[0] + x * dst.s[2] +
                     y * dst.s[3];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (z0 + q >= dst.z) break;
    float r[8];
#pragma unroll
    for (int l = 0; l < 8; ++l) r[l] = l < kz ? v[q + l] : 0.f;
    if (dst.dtype == VXB_BF16X2) {
      uint4 hi, lo;
      f32_to_split8(r, hi, lo);
      *reinterpret_cast<uint4 *>(o + (z0 + q) * dst.s[4]) = hi;
      *reinterpret_cast<uint4 *>(o + (z0 + q) * dst.s[4] + (dst.s[1] >> 1)) = lo;
      continue;
    }
    uint4 u;
    __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(r[2 * k], r[2 * k + 1]);
    *reinterpret_cast<uint4 *>(o + (z0 + q) * dst.s[4]) = u;
  }
}

// The reverse at the output boundary: bf16 blocked -> fp32 NCDHW.
__global__ void unpack_std_f32_kernel(DView src, DView dst) {
  pdl_begin();
  const int zq = src.z >> 2;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= src.y * zq) return;
  const int y = i / zq, z = (i - y * zq) * 4, x = blockIdx.y;
  const int nch = (src.c + 7) >> 3;
  const int b = blockIdx.z / nch, ch = blockIdx.z - b * nch;
  const __nv_bfloat16 *p = static_cast<const __nv_bfloat16 *>(src.data) + b * src.s[0] +
                           ch * src.s[1] + x * src.s[2] + y * src.s[3] + z * src.s[4];
  float v[4][8];
  const bool split = src.dtype == VXB_BF16X2;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    bf16x8_to_f32(*reinterpret_cast<const uint4 *>(p + q * src.s[4]), v[q]);
    if (split) {
      float lo[8];
      bf16x8_to_f32(*reinterpret_cast<const uint4 *>(p + q * src.s[4] + (src.s[1] >> 1)), lo);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[q][k] += lo[k];
    }
  }
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    const int c = ch * 8 + l;
    if (c < dst.c)
      *reinterpret_cast<float4 *>(static_cast<float *>(dst.data) + b * dst.s[0] + c * dst.s[1] +
                                  x * dst.s[2] + y * dst.s[3] + z) =
          make_float4(v[0][l], v[1][l], v[2][l], v[3][l]);
  }
}

static bool std_f32_vec4(const DView &t) {
  return !t.blocked && t.dtype == VXB_F32 && t.s[4] == 1 && (t.z & 3) == 0 &&
         (reinterpret_cast<uintptr_t>(t.data) & 15) == 0 && (t.s[0] & 3) == 0 &&
         (t.s[1] & 3) == 0 && (t.s[2] & 3) == 0 && (t.s[3] & 3) == 0;
}
static bool blocked_bf16(const DView &t) { return t.blocked && t.dtype == VXB_BF16; }
// bf16 or split bf16 blocked (the boundary pack / unpack kernels handle both)
static bool blocked_bf16ish(const DView &t) {
  return t.blocked && (t.dtype == VXB_BF16 || t.dtype == VXB_BF16X2);
}

static int pack_trigger() {
  const char *v = getenv("VXB_PACK_TRIGGER");
  return v && atoi(v) ? 1 : 0;
}

int launch_copy(const DView &src, const DView &dst, cudaStream_t s, bool independent) {
  if (std_f32_vec4(src) && blocked_bf16ish(dst)) {
    dim3 g((dst.y * (dst.z >> 2) + 127) / 128, dst.x, dst.n * ((dst.c + 7) / 8));
    if (independent)
      return check_cuda(launch_pdl_prio(pack_std_f32_indep_kernel, g, dim3(128), 0, s, true, src,
                                        dst, pack_trigger()),
                        "pack_std_f32_indep_kernel");
    return check_cuda(launch_pdl(pack_std_f32_kernel, g, dim3(128), 0, s, src, dst),
                      "pack_std_f32_kernel");
  }
  if (blocked_bf16ish(src) && std_f32_vec4(dst)) {
    dim3 g((src.y * (src.z >> 2) + 127) / 128, src.x, src.n * ((src.c + 7) / 8));
    return check_cuda(launch_pdl(unpack_std_f32_kernel, g, dim3(128), 0, s, src, dst),
                      "unpack_std_f32_kernel");
  }
  return check_cuda(launch_pdl(copy_kernel, grid3(dst, 256), dim3(256), 0, s, src, dst),
                    "copy_kernel");
}
// One block row per (window, 256-element span of its z rows): consecutive
// threads move consecutive z elements (float4 when the window allows), so a
// warp reads and writes contiguous 512-byte runs of both volumes.
__global__ void __launch_bounds__(256) copy_windows_kernel(const __grid_constant__ WinBatch b) {
  pdl_begin();
  const WinCopy &w = b.w[blockIdx.y];
  const int zq = w.vec4 ? w.ext[4] >> 2 : w.ext[4];      // z elements (or float4s) per row
  const long long rows = static_cast<long long>(w.ext[0]) * w.ext[1] * w.ext[2] * w.ext[3];
  const long long total = rows * zq;
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long r = e / zq;
    const int zz = static_cast<int>(e - r * zq);
    const int y = static_cast<int>(r % w.ext[3]);
    r /= w.ext[3];
    const int x = static_cast<int>(r % w.ext[2]);
    r /= w.ext[2];
    const int c = static_cast<int>(r % w.ext[1]);
    const int n = static_cast<int>(r / w.ext[1]);
    const long long so = n * w.ss[0] + c * w.ss[1] + x * w.ss[2] + y * w.ss[3];
    const long long d = n * w.ds[0] + c * w.ds[1] + x * w.ds[2] + y * w.ds[3];
    if (w.vec4)
      reinterpret_cast<float4 *>(w.dst + d)[zz] =
          __ldg(reinterpret_cast<const float4 *>(w.src + so) + zz);
    else
      w.dst[d + zz] = __ldg(w.src + so + zz);
  }
}

int launch_copy_windows(const WinBatch &b, cudaStream_t s) {
  if (b.count <= 0) return VXB_OK;
  long long most = 1;
  for (int i = 0; i < b.count; ++i) {
    const WinCopy &w = b.w[i];
    const long long e = static_cast<long long>(w.ext[0]) * w.ext[1] * w.ext[2] * w.ext[3] *
                        (w.vec4 ? w.ext[4] >> 2 : w.ext[4]);
    most = std::max(most, e);
  }
  // enough blocks per window to cover the SMs a few times over
  const int bx = static_cast<int>(std::min<long long>((most + 255) / 256, 4096));
  return check_cuda(launch_pdl(copy_windows_kernel, dim3(bx, b.count), dim3(256), 0, s, b),
                    "copy_windows_kernel");
}

int launch_pack_zwin(const DView &src, const DView &dst, int kz, int pz, cudaStream_t s,
                     bool independent) {
  dim3 g((dst.y * ((dst.z + 3) >> 2) + 127) / 128, dst.x, dst.n);
  ZwinWindows none;
  none.off[0] = 0;
  if (independent)
    return check_cuda(launch_pdl_prio(pack_zwin_kernel<true>, g, dim3(128), 0, s, true, src, dst,
                                      kz, pz, pack_trigger(), none),
                      "pack_zwin_kernel");
  return check_cuda(
      launch_pdl(pack_zwin_kernel<false>, g, dim3(128), 0, s, src, dst, kz, pz, 0, none),
      "pack_zwin_kernel");
}
int launch_pack_zwin_windows(const DView &src, const ZwinWindows &w, const DView &dst, int kz,
                             int pz, cudaStream_t s) {
  dim3 g((dst.y * ((dst.z + 3) >> 2) + 127) / 128, dst.x, dst.n);
  return check_cuda(
      launch_pdl(pack_zwin_kernel<false, true>, g, dim3(128), 0, s, src, dst, kz, pz, 0, w),
      "pack_zwin_kernel");
}
int launch_zero(const DView &dst, cudaStream_t s) {
  return check_cuda(launch_pdl(zero_kernel, grid3(dst, 256), dim3(256), 0, s, dst), "zero_kernel");
}
int launch_pool(const DView &in, const DView &out, const int *w, const int *st, int mode,
                cudaStream_t s) {
  const bool fast = mode == VXB_POOL_MAX && blocked_bf16(in) && blocked_bf16(out) &&
                    (w[0] == 1 || w[0] == 2) && w[1] == 2 && w[2] == 2 && st[0] == w[0] &&
                    st[1] == 2 && st[2] == 2 && in.s[4] == 8 && out.s[4] == 8;
  if (fast)
    return check_cuda(w[0] == 2 ? launch_pdl(pool_max_bf16_kernel<2>, grid3(out, 256), dim3(256),
                                             0, s, in, out)
                                : launch_pdl(pool_max_bf16_kernel<1>, grid3(out, 256), dim3(256),
                                             0, s, in, out),
                      "pool_max_bf16_kernel");
  return check_cuda(launch_pdl(pool_kernel, grid3(out, 256), dim3(256), 0, s, in, out, w[0], w[1],
                               w[2], st[0], st[1], st[2], mode),
                    "pool_kernel");
}
int launch_eltwise(const DView &a, const DView &b, const DView &out, int op, cudaStream_t s) {
  return check_cuda(launch_pdl(eltwise_kernel, grid3(out, 256), dim3(256), 0, s, a, b, out, op),
                    "eltwise_kernel");
}
int launch_affine_act(const DView &in, const DView &out, const float *m, const float *a, int act,
                      float alpha, cudaStream_t s) {
  return check_cuda(launch_pdl(affine_act_kernel, grid3(out, 256), dim3(256), 0, s, in, out, m, a,
                               act, alpha),
                    "affine_act_kernel");
}
int launch_mergecrop(const DView &a, const DView &b, const DView &out, const int *oa,
                     const int *ob, cudaStream_t s) {
  return check_cuda(launch_pdl(mergecrop_kernel, grid3(out, 256), dim3(256), 0, s, a, b, out,
                               oa[0], oa[1], oa[2], ob[0], ob[1], ob[2]),
                    "mergecrop_kernel");
}
int launch_pad_copy(const DView &in, const DView &out, const int *pads, cudaStream_t s) {
  return check_cuda(launch_pdl(pad_copy_kernel, grid3(out, 256), dim3(256), 0, s, in, out,
                               pads[0], pads[1], pads[2]),
                    "pad_copy_kernel");
}

int launch_conv_direct(DirectParams p, cudaStream_t s) {
  p.tiles_x = (p.out.x + DT_X - 1) / DT_X;
  p.tiles_y = (p.out.y + DT_Y - 1) / DT_Y;
  p.tiles_z = (p.out.z + DT_Z - 1) / DT_Z;
  p.hx = (DT_X - 1) * p.sx + p.kx;
  p.hy = (DT_Y - 1) * p.sy + p.ky;
  p.hz = (DT_Z - 1) * p.sz + p.kz;
  size_t smem = (static_cast<size_t>(p.hx) * p.hy * p.hz * 8 +
                 static_cast<size_t>(p.kx) * p.ky * p.kz * 8 * DCO) *
                sizeof(float);
  if (smem > 227 * 1024)
    return set_error(VXB_EUNSUPPORTED, "direct conv: staged patch of %zu bytes exceeds smem", smem);
  if (int rc = ensure_smem_attr(conv_direct_kernel, 227 * 1024,
                                "cudaFuncSetAttribute(conv_direct)"))
    return rc;
  dim3 grid(p.tiles_x * p.tiles_y * p.tiles_z, (p.cout + DCO - 1) / DCO, p.out.n);
  return check_cuda(launch_pdl(conv_direct_kernel, grid, dim3(128), smem, s, p),
                    "conv_direct_kernel");
}

int launch_subimage(const SubParams &p, cudaStream_t s) {
  int total = p.out.n * p.ex * p.ey * p.ez * 8;
  return check_cuda(launch_pdl(subimage_kernel, dim3((total + 127) / 128), dim3(128), 0, s, p),
                    "subimage_kernel");
}

int launch_deconv_gather(const GatherDeconvParams &p, cudaStream_t s) {
  return check_cuda(launch_pdl(deconv_gather_kernel, grid3(p.out, 128), dim3(128), 0, s, p),
                    "deconv_gather_kernel");
}

}  // namespace vxb
