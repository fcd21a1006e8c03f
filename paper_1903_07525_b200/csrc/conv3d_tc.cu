// conv3d_tc.cu — direct 3D convolution as a tcgen05/TMEM implicit GEMM.
//
// Replaces the reference hot loop _kernels.conv3d (_kernels.pyx:44-179) with
// its vec8 FMA micro-kernels (convcore.h:19-52).  Semantics follow the
// reference contract (kernels_py.py:7-10, _kernels.pyx:112-175):
//     out = act(bias' + [base_scale .] base + sum_{ib,dx,dy,dz,i} in * K')
// cross-correlation (no flip), stride 1, zero padding virtual.
//
// Mapping:
//   M  = output voxels.  A CTA tile is bx slices x 16 x 8 (z); every
//        slice is one 128-row UMMA (rows = y*8 + z for x-slices) with its own
//        TMEM accumulator of nt fp32 columns.
//   N  = output fmaps (nt per tile, padded to 16).
//   K  = input fmaps x taps, consumed in "steps" of 16 bf16: either two
//        8-fmap chunks at one tap, or (odd last chunk) one chunk at two
//        adjacent z taps.
//   A operand: for each group of <=2 input chunks, one TMA box per chunk
//        brings the halo tile (bx+kx-1, 16+ky-1, 8+kz-1 voxels, 16 B each)
//        into shared memory as a dense [x][y][z] array of 16-byte rows.
//        That is exactly the SWIZZLE_NONE K-major core-matrix layout, so the
//        operand for tap (dx,dy,dz) is just the descriptor start address
//        moved by ((dx*hy + dy)*hz + dz)*16 bytes: no im2col, the halo is
//        read from HBM/L2 once per tile and every tap reuses it from smem.
//        Out-of-range coordinates are zero-filled by TMA = 'same' padding.
//   B operand: weights pre-packed on the host into per-step slabs in the
//        core-matrix layout; streamed with cp.async.bulk (or loaded once and
//        kept resident when the whole filter bank fits).
//   Low/mid fmap counts (3*nt <= 256) fold the 3 taps along the slice axis
//        into N (mma_group_fold): slices along x for 3x3x3, along y for
//        1x3x3 (rows are then 16 x by 8 z).
// Warp roles: w0 = A (halo) TMA producer, w1 = MMA issuer (+TMEM owner),
// w2 = B (weights) producer, w3..w14 = epilogue (TMEM -> regs -> bias/base/
// act -> global).  Persistent CTAs walk the tile list; TMEM accumulators are
// double buffered when they fit so the epilogue of tile i overlaps the MMAs
// of tile i+1.  CTA pairs (cta_group::2, M = 256) split the weight stream of
// unfolded convs.  Experimental (VXB_TC_STREAM): the streamed fold walks whole
// x columns with the output slices' accumulators in a TMEM ring
// (mma_group_stream).
#include <cuda_bf16.h>
#include <type_traits>
#include "vxb_internal.h"
#include "vxb_ptx.cuh"

namespace vxb {

struct GroupInfo {
  int seg, chunk0, nch, steps;
};

__device__ __forceinline__ GroupInfo group_info(const TcParams &p, int g) {
  int g0 = (p.seg_chunks[0] + 1) >> 1;
  int seg = g < g0 ? 0 : 1;
  int j = seg ? g - g0 : g;
  int c = p.seg_chunks[seg];
  int nch = min(2, c - 2 * j);
  int steps = nch == 2 ? p.kx * p.ky * p.kz : p.kx * p.ky * ((p.kz + 1) >> 1);
  if (p.fold) steps /= 3;   // the slice-axis taps ride in N
  GroupInfo gi{seg, 2 * j, nch, steps};
  return gi;
}

struct TileCoord {
  int rep, nt, b, x0, y0, z0;
  bool dummy;   // padding tile of a CTA pair: loads as tile 0, stores nothing
};

__device__ __forceinline__ int fdiv(int t, unsigned long long m) {
  return static_cast<int>((static_cast<unsigned long long>(static_cast<unsigned>(t)) * m) >> 40);
}

__device__ __forceinline__ TileCoord decode_tile(const TcParams &p, int t) {
  TileCoord c;
  const int rn = fdiv(t, p.dm[0]);
  int sp = t - rn * p.spatial_pad;
  c.dummy = sp >= p.spatial_real;
  if (c.dummy) sp = 0;
  t = sp + rn * p.spatial_real;
  int q = fdiv(t, p.dm[1]);
  const int tz = t - q * p.tiles_z;
  t = q;
  q = fdiv(t, p.dm[2]);
  const int ty = t - q * p.tiles_y;
  t = q;
  q = fdiv(t, p.dm[3]);
  const int tx = t - q * p.tiles_x;
  t = q;
  q = fdiv(t, p.dm[4]);
  c.b = t - q * p.nb;
  t = q;
  q = fdiv(t, p.dm[5]);
  c.nt = t - q * p.n_tiles;
  c.rep = q;
  c.x0 = tx * p.ex;
  c.y0 = ty * p.ey;
  c.z0 = tz * TILE_Z;
  return c;
}

// Fast ELU for the tensor-core epilogue: alpha*(2^(v*log2 e) - 1), selected
// branch-free (a data-dependent branch per value tripled the epilogue time).
// Absolute error ~1e-7 near 0, far below the bf16 operand rounding.
// 2^x in one MUFU.EX2 (ftz: inputs below -126 give 0, i.e. e^v - 1 = -1 for
// v < -87, exact to fp32); __expf adds range-scaling FMULs around the MUFU
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_elu(float v, float alpha) {
  const float m = fmaf(alpha, ex2_ftz(v * 1.4426950408889634f), -alpha);
  return v > 0.f ? v : m;
}
__device__ __forceinline__ float fast_sigmoid(float v) {
  return rcp_ftz(1.f + ex2_ftz(v * -1.4426950408889634f));
}
__device__ __forceinline__ float apply_act(float v, int act, float alpha) {
  if (act == VXB_ACT_RELU) return v > 0.f ? v : 0.f;
  if (act == VXB_ACT_ELU) return v > 0.f ? v : alpha * expm1f(v);
  if (act == VXB_ACT_SIGMOID) return 1.f / (1.f + expf(-v));
  return v;
}

// split bf16 (VXB_BF16X2): 8 lanes = a hi and a lo bf16 chunk, s[1]/2 apart
__device__ __forceinline__ void unpack_bf16x8(const uint4 &u, float (&x)[8]) {
  const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    x[2 * i] = f.x;
    x[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void split8(const float (&x)[8], uint4 &hi, uint4 &lo) {
  __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&hi);
  __nv_bfloat162 *l = reinterpret_cast<__nv_bfloat162 *>(&lo);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    h[i] = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
    const float2 f = __bfloat1622float2(h[i]);
    l[i] = __floats2bfloat162_rn(x[2 * i] - f.x, x[2 * i + 1] - f.y);
  }
}
__device__ __forceinline__ void store8_split(const EpiView &v, long long off, const float (&x)[8]) {
  uint4 hi, lo;
  split8(x, hi, lo);
  __nv_bfloat16 *p = static_cast<__nv_bfloat16 *>(v.data) + off;
  *reinterpret_cast<uint4 *>(p) = hi;
  *reinterpret_cast<uint4 *>(p + (v.s[1] >> 1)) = lo;
}

__device__ __forceinline__ void load8(const EpiView &v, long long off, bool blocked_lane_stride1,
                                      float (&x)[8]) {
  if (v.dtype == VXB_BF16X2) {   // blocked only
    const __nv_bfloat16 *p = static_cast<const __nv_bfloat16 *>(v.data) + off;
    float lo[8];
    unpack_bf16x8(*reinterpret_cast<const uint4 *>(p), x);
    unpack_bf16x8(*reinterpret_cast<const uint4 *>(p + (v.s[1] >> 1)), lo);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] += lo[i];
    return;
  }
  if (v.dtype == VXB_BF16) {
    const __nv_bfloat16 *p = static_cast<const __nv_bfloat16 *>(v.data) + off;
    if (blocked_lane_stride1) {
      uint4 u = *reinterpret_cast<const uint4 *>(p);
      const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float2 f = __bfloat1622float2(h[i]);
        x[2 * i] = f.x;
        x[2 * i + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = __bfloat162float(p[i * v.s[1]]);
    }
  } else {
    const float *p = static_cast<const float *>(v.data) + off;
    if (blocked_lane_stride1) {
      float4 a = *reinterpret_cast<const float4 *>(p);
      float4 b = *reinterpret_cast<const float4 *>(p + 4);
      x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
      x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = p[i * v.s[1]];
    }
  }
}

// store lanes [0, nvalid) of one 8-fmap chunk; blocked layouts get all 8
// lanes (tail lanes are written as zero, ops.py:18-23 zero_tail semantics)
__device__ __forceinline__ void store8(const EpiView &v, long long off, bool blocked,
                                       int nvalid, const float (&x)[8]) {
  if (v.dtype == VXB_BF16X2) {   // blocked only
    store8_split(v, off, x);
    return;
  }
  if (v.dtype == VXB_BF16) {
    __nv_bfloat16 *p = static_cast<__nv_bfloat16 *>(v.data) + off;
    if (blocked) {
      uint4 u;
      __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
      *reinterpret_cast<uint4 *>(p) = u;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < nvalid) p[i * v.s[1]] = __float2bfloat16_rn(x[i]);
    }
  } else {
    float *p = static_cast<float *>(v.data) + off;
    if (blocked) {
      *reinterpret_cast<float4 *>(p) = make_float4(x[0], x[1], x[2], x[3]);
      *reinterpret_cast<float4 *>(p + 4) = make_float4(x[4], x[5], x[6], x[7]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < nvalid) p[i * v.s[1]] = x[i];
    }
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void dbg_mark(const TcParams &p, int it, int slot) {
  if (p.dbg && it < 64) p.dbg[(static_cast<size_t>(blockIdx.x) * 64 + it) * 8 + slot] = gtimer();
}
// SM clock counter next to a timestamp (effective clock = dclock / dns)
__device__ __forceinline__ void dbg_clock(const TcParams &p, int it, int slot) {
  if (p.dbg && it > 0 && it < 64)
    p.dbg[(static_cast<size_t>(blockIdx.x) * 64 + it) * 8 + slot] = clock64();
}

// Epilogue warps (a multiple of 4: EPI/4 per TMEM lane quarter).  16 when
// the 104-register budget allows (608 threads = 63.2 K registers); the
// fp32-input variant adds 4 converter warps and keeps 12.
#ifndef VXB_EPI_WARPS
#define VXB_EPI_WARPS 16
#endif
__host__ __device__ constexpr int epi_warps(bool f32in) { return f32in ? 12 : VXB_EPI_WARPS; }
// registers per thread: warps are spread over the 4 SM sub-partitions
// (16 K registers each), so 19-20 warps need <= 96 per thread; 15-16 warps
// (12 epilogue warps + roles + converters) fit 104
#if VXB_EPI_WARPS > 12
#define VXB_TC_MAXNREG 96
#else
#define VXB_TC_MAXNREG 104
#endif
constexpr int CVT_WARPS = 4;                      // fp32-input converters (F32IN)
__host__ __device__ constexpr int tc_threads(bool f32in) {
  return 96 + 32 * epi_warps(f32in) + (f32in ? 32 * CVT_WARPS : 0);
}

// Lean epilogue (bf16 blocked output, optional bf16 blocked residual): per
// 16-column item of a tile, the element offsets of its two 8-fmap halves
// relative to the thread's row in slice 0 of the tile (output and residual)
// and its first channel within the N tile, built once per CTA.
struct LeanEnt {
  long long o0, o1, b0, b1;
  int ch, pad;
};
constexpr int LEAN_TAB = 16;   // nt <= 256: <= 16 column items

// Lean epilogue: per-tile origin computed once by the A producer (which
// decodes the tile anyway) instead of by all 16 epilogue warps: element
// offsets of the tile's (row 0, slice 0) in the output and residual views,
// the tile's row / z / slice origins and its N-tile column.  A ring of
// TINFO slots, each published with an mbarrier arrive; the producer runs at
// most na + acc_stages tiles ahead of the epilogue.
struct TileInfo {
  long long o_off, b_off, p_off;   // output, residual, fused-pool view offsets
  int rc0, z0, sc0, nt0, dummy;
  int ns, slot0;   // streamed fold: slices to finish and the ring slot of the first
  int pad[3];
};
constexpr int TINFO = 16;
static_assert(6 + MAX_ACC < TINFO, "TileInfo ring: the producer runs <= na + acc stages ahead");

// Byte offsets inside the dynamic smem block (all derivable from p).
struct SmemMap {
  uint32_t a, b, stg, bias, scale, head, hpart, ltab, stab, bars;
};
// streamed fold: one 32-word operand table per (ring phase, slab), built
// once per CTA (StreamTab layout: d[8] b[8] id[8] wa[2] wb[2] wid[2])
constexpr int STAB_WORDS = 32;
__host__ __device__ inline SmemMap smem_map(const TcParams &p) {
  SmemMap m;
  m.a = 0;
  m.b = p.na * p.a_stage_bytes;
  m.stg = m.b + p.nb_stages * p.b_stage_bytes;
  m.bias = m.stg + p.n_stg * p.stg_bytes;
  const uint32_t cpad = p.n_tiles * p.nt;
  m.scale = m.bias + cpad * 4;
  m.head = m.scale + cpad * 4;                 // fused head weights [head_cout][cpad]
  // fused head: per-row partial dot products of every column item [item][row]
  m.hpart = (m.head + (p.head_cout > 0 ? 4 * cpad * 4 : 0) + 15) & ~15u;
  m.ltab = m.hpart + (p.head_cout > 0 ? p.bx * (p.nt >> 4) * 128 * 16 : 0);
  m.stab = m.ltab + (p.lean ? LEAN_TAB * sizeof(LeanEnt) + TINFO * sizeof(TileInfo) : 0);
  m.bars = m.stab + (p.stream ? p.st_nphase * p.st_nslab * STAB_WORDS * 4 : 0);
  return m;
}

// Epilogue variants are compile-time so every instantiation carries only its
// own code (a kernel with all variants inlined thrashes the instruction cache).
//   ACT: VXB_ACT_* or -1 (runtime); FASTOUT: blocked bf16 output with fast
//   activations; BASE: fused residual operand.
__device__ __forceinline__ void store8_bf16_blocked(const EpiView &v, long long off,
                                                    const float (&x)[8]) {
  uint4 u;
  __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
  *reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(v.data) + off) = u;
}


// ---------------------------------------------------------------- MMA issue
// One group (<= 2 input chunks x all taps) of MMAs.  Everything is passed by
// value and kept in scalar locals so that, executed by a convergent warp,
// ptxas holds the descriptors in uniform registers.
struct MmaCtx {
  uint64_t *b_full, *b_empty;
  int nb_stages, bsteps, resident, first_tile_iter, cluster;
};

template <int BX, bool PAIRM>
__device__ __forceinline__ void mma_group(
    const uint32_t a_lo0, const uint32_t a_hi, const uint32_t b_base0, const uint32_t b_stage_bytes,
    const uint32_t b_hi, const uint32_t b_inc, const uint32_t slice_inc, const uint32_t d_base,
    const uint32_t nt, const uint32_t idesc, const int steps, const int tz_n, const uint32_t dz_step,
    const uint32_t dy_wrap, const uint32_t dx_wrap, const int ky, const MmaCtx &cx, int &b_st,
    int &b_ph, uint32_t &acc) {
  int tz = 0, ty = 0;
  uint32_t off = 0;
  for (int s0 = 0; s0 < steps; s0 += cx.bsteps) {
    const int n = min(cx.bsteps, steps - s0);
    if (cx.resident) {
      if (cx.first_tile_iter) mbar_wait(&cx.b_full[b_st], 0);
    } else {
      mbar_wait(&cx.b_full[b_st], b_ph);
    }
    tc_fence_after();
    uint32_t b_lo = desc_lo(b_base0 + b_st * b_stage_bytes, 128u);
    for (int i = 0; i < n; ++i) {
      umma_step_elect<BX, PAIRM>(d_base, a_lo0 + off, a_hi, b_lo, b_hi, idesc, acc, nt, slice_inc);
      acc = 1;
      b_lo += b_inc;
      off += dz_step;
      if (++tz == tz_n) {
        tz = 0;
        off += dy_wrap;
        if (++ty == ky) {
          ty = 0;
          off += dx_wrap;
        }
      }
    }
    if (!cx.resident) {
      if (PAIRM)
        umma_commit_pair_elect(&cx.b_empty[b_st], 0x3);
      else if (cx.cluster == 2)
        umma_commit_mc_elect(&cx.b_empty[b_st], 0x3);   // frees the slot in both CTAs
      else
        umma_commit_elect(&cx.b_empty[b_st]);
    }
    if (++b_st == cx.nb_stages) {
      b_st = 0;
      b_ph ^= 1;
    }
  }
}

// Folded variant: K steps run over the taps across the slice axis's
// neighbours (dy or dx) and z only; the 3 slice-axis taps are stacked in the
// B slab as N blocks [w(d=2); w(d=1); w(d=0)].  Input slice j feeds output
// slices j-2..j, so one MMA of N = (#valid d) x nt writes the contiguous
// accumulator columns of those slices: BX+2 MMAs per step instead of 3*BX.
// The first step of a tile initialises every slice with its d=0 term
// (accumulate = 0) before the overlapping MMAs accumulate on top.
template <int BX>
__device__ __forceinline__ void mma_group_fold(
    const uint32_t a_lo0, const uint32_t a_hi, const uint32_t b_base0, const uint32_t b_stage_bytes,
    const uint32_t b_hi, const uint32_t slab_inc, const uint32_t blk_inc, const uint32_t slice_inc,
    const uint32_t d_base, const uint32_t nt, const uint32_t id1, const uint32_t id2,
    const uint32_t id3, const int steps, const int tz_n, const uint32_t dz_step,
    const uint32_t a_wrap, const MmaCtx &cx, int &b_st, int &b_ph, uint32_t &first) {
  int tz = 0;
  uint32_t off = 0;
  for (int s0 = 0; s0 < steps; s0 += cx.bsteps) {
    const int n = min(cx.bsteps, steps - s0);
    if (cx.resident) {
      if (cx.first_tile_iter) mbar_wait(&cx.b_full[b_st], 0);
    } else {
      mbar_wait(&cx.b_full[b_st], b_ph);
    }
    tc_fence_after();
    uint32_t b_lo = desc_lo(b_base0 + b_st * b_stage_bytes, 128u);
    auto advance = [&]() {
      b_lo += slab_inc;
      off += dz_step;
      if (++tz == tz_n) {
        tz = 0;
        off += a_wrap;
      }
    };
    int i = 0;
    if (first) {
      // the tile's first K step (peeled so the steady loop has no branch)
      const uint32_t a_lo = a_lo0 + off;
      if constexpr (BX >= 2) {
        umma_fold_first<BX>(d_base, a_lo, a_hi, b_lo, b_hi, id1, id2, id3, nt, slice_inc, blk_inc);
      } else {
        umma_bf16_lohi_elect(d_base, a_lo, a_hi, b_lo + 2 * blk_inc, b_hi, id1, 0u);
#pragma unroll
        for (int j = 1; j < BX + 2; ++j) {
          const int dlo = j - BX + 1 > 1 ? j - BX + 1 : 1, dhi = j < 2 ? j : 2;
          const uint32_t idn = dhi - dlo == 0 ? id1 : id2;
          umma_bf16_lohi_elect(d_base + (j - dhi) * nt, a_lo + j * slice_inc, a_hi,
                               b_lo + (2 - dhi) * blk_inc, b_hi, idn, 1u);
        }
      }
      first = 0;
      advance();
      i = 1;
    }
    for (; i < n; ++i) {
      const uint32_t a_lo = a_lo0 + off;
      if constexpr (BX >= 2) {
        // one asm block per step: interior slices (shared B, N = 3nt), then
        // the tail and head slices
        umma_fold_step<BX>(d_base, a_lo, a_hi, b_lo, b_hi, id1, id2, id3, nt, slice_inc, blk_inc);
      } else {
        // BX = 1: input slices 0..2 each feed the single output slice
#pragma unroll
        for (int j = 0; j < 3; ++j)
          umma_bf16_lohi_elect(d_base, a_lo + j * slice_inc, a_hi, b_lo + (2 - j) * blk_inc, b_hi,
                               id1, 1u);
      }
      advance();
    }
    if (!cx.resident) umma_commit_elect(&cx.b_empty[b_st]);
    if (++b_st == cx.nb_stages) {
      b_st = 0;
      b_ph ^= 1;
    }
  }
}

// Folded CTA-pair variant (cta_group::2, M = 256: each MMA covers the same
// slice of both CTAs' tiles, B split by rows between the pair).  Every MMA
// runs at N = 3nt from the start of the slab, so the split is the same for
// all of them: input slice j writes slices j-2..j (D = d_base + j*nt, where
// d_base is the column of slice -2) and the edge slices' extra terms land in
// the scratch columns around the tile.  At N <= 96 an M = 256 instruction
// costs what an M = 128 one does (~45-50 cycles, tools/umma_align.cu), so the
// pair halves the MMA time per tile of the low-fmap convs.  The first step of
// a tile writes input slices j = 0, 3, 6, .. with accumulate off (their
// 3-slice ranges tile the accumulator without overlap), then j = 1 mod 3 and
// j = 2 mod 3 accumulate on top.
template <int BX>
__device__ __forceinline__ void mma_group_fold_pair(
    const uint32_t a_lo0, const uint32_t a_hi, const uint32_t b_base0, const uint32_t b_stage_bytes,
    const uint32_t b_hi, const uint32_t slab_inc, const uint32_t slice_inc, const uint32_t d_base,
    const uint32_t nt, const uint32_t id3, const int steps, const int tz_n, const uint32_t dz_step,
    const uint32_t a_wrap, const MmaCtx &cx, int &b_st, int &b_ph, uint32_t &first) {
  constexpr int C = BX + 2;
  int tz = 0;
  uint32_t off = 0;
  for (int s0 = 0; s0 < steps; s0 += cx.bsteps) {
    const int n = min(cx.bsteps, steps - s0);
    if (cx.resident) {
      if (cx.first_tile_iter) mbar_wait(&cx.b_full[b_st], 0);
    } else {
      mbar_wait(&cx.b_full[b_st], b_ph);
    }
    tc_fence_after();
    uint32_t b_lo = desc_lo(b_base0 + b_st * b_stage_bytes, 128u);
    auto advance = [&]() {
      b_lo += slab_inc;
      off += dz_step;
      if (++tz == tz_n) {
        tz = 0;
        off += a_wrap;
      }
    };
    int i = 0;
    if (first) {
      const uint32_t a_lo = a_lo0 + off;
      umma_pair_run<(C + 2) / 3>(d_base, a_lo, a_hi, b_lo, b_hi, id3, 0u, 3 * nt, 3 * slice_inc);
      umma_pair_run<(C + 1) / 3>(d_base + nt, a_lo + slice_inc, a_hi, b_lo, b_hi, id3, 1u, 3 * nt,
                                 3 * slice_inc);
      umma_pair_run<C / 3>(d_base + 2 * nt, a_lo + 2 * slice_inc, a_hi, b_lo, b_hi, id3, 1u,
                           3 * nt, 3 * slice_inc);
      first = 0;
      advance();
      i = 1;
    }
    for (; i < n; ++i) {
      // j = 0, 3, .. then 1, 4, .. then 2, 5, ..: consecutive MMAs never
      // touch the same accumulator slices (no read-after-write stalls)
      const uint32_t a_lo = a_lo0 + off;
      umma_pair_run<(C + 2) / 3>(d_base, a_lo, a_hi, b_lo, b_hi, id3, 1u, 3 * nt, 3 * slice_inc);
      umma_pair_run<(C + 1) / 3>(d_base + nt, a_lo + slice_inc, a_hi, b_lo, b_hi, id3, 1u, 3 * nt,
                                 3 * slice_inc);
      umma_pair_run<C / 3>(d_base + 2 * nt, a_lo + 2 * slice_inc, a_hi, b_lo, b_hi, id3, 1u,
                           3 * nt, 3 * slice_inc);
      advance();
    }
    if (!cx.resident) umma_commit_pair_elect(&cx.b_empty[b_st], 0x3);
    if (++b_st == cx.nb_stages) {
      b_st = 0;
      b_ph ^= 1;
    }
  }
}

// Streamed fold (TcParams::stream): one slab of `cnt` <= 8 input slices jmin
// .. jmin + cnt - 1 (halo coordinates) of a column.  Input slice j carries the
// taps d in [dlo, dhi] = [max(0, j - S + 1), min(2, j)] to the output slices
// j - d; their accumulators are consecutive slots of a ring of `slots` TMEM
// slices starting at (rb + j - dhi) mod slots, so one MMA of N = (dhi - dlo
// + 1) nt serves them (two where the range wraps around the ring).  Every MMA
// accumulates: the epilogue leaves each slot zeroed after reading it.  The
// per-slice operands are worked out once per slab (StreamTab, registers);
// within a K step the input slices go in stride-3 order so that consecutive
// MMAs never touch the same slots (no accumulator read-after-write stalls).
struct StreamCtx {
  int jmin, cnt, S, rb, slots;
};
constexpr int STREAM_BX = 8;
struct StreamTab {
  uint32_t d[STREAM_BX], b[STREAM_BX], id[STREAM_BX];   // main MMA: D column, B block offset, idesc
  // at most two input slices of a slab wrap around the ring: their second
  // MMA (D column 0): A slice offset, B block offset, idesc (0 = none)
  uint32_t wa[2], wb[2], wid[2];
};
// Entry i (0..7: input slice i of the slab; 8: the wrapped parts) of the
// operand table of slab t at ring phase ph, written to shared memory by one
// thread in the kernel prologue.
__device__ __forceinline__ void stream_table_entry(const TcParams &p, uint32_t *tab, int ph, int t,
                                                   int i, const uint32_t blk_inc,
                                                   const uint32_t slice_inc) {
  const int mask = p.st_slots - 1;
  const int rb = (ph * p.ox) & mask;
  const int jmin = p.st_j0 + t * p.bx;
  const int cnt = min(p.bx, p.st_nin - t * p.bx);
  const uint32_t id1 = idesc_bf16(128, p.nt), id2 = idesc_bf16(128, 2 * p.nt),
                 id3 = idesc_bf16(128, 3 * p.nt);
  auto entry = [&](int k, int &r, int &nn, int &n1, int &dhi) {
    const int j = jmin + k;
    dhi = min(2, j);
    const int dlo = max(0, j - p.ox + 1);
    nn = dhi - dlo + 1;
    r = (rb + j - dhi) & mask;
    n1 = min(nn, p.st_slots - r);
  };
  if (i < STREAM_BX) {
    int r, nn, n1, dhi;
    entry(i, r, nn, n1, dhi);
    tab[i] = r * p.nt;
    tab[8 + i] = (2 - dhi) * blk_inc;
    tab[16 + i] = n1 == 1 ? id1 : (n1 == 2 ? id2 : id3);
  } else {
    uint32_t w[6] = {0u, 0u, 0u, 0u, 0u, 0u};
    int nw = 0;
    for (int k = 0; k < cnt; ++k) {
      int r, nn, n1, dhi;
      entry(k, r, nn, n1, dhi);
      if (n1 < nn && nw < 2) {
        w[nw] = k * slice_inc;
        w[2 + nw] = (2 - dhi + n1) * blk_inc;
        w[4 + nw] = nn - n1 == 1 ? id1 : id2;
        ++nw;
      }
    }
    for (int k = 0; k < 6; ++k) tab[24 + k] = w[k];
    tab[30] = tab[31] = 0u;
  }
}
// the MMA warp's copy of a table: lane l reads word l, every word is then
// broadcast so that ptxas keeps the operands in uniform registers
__device__ __forceinline__ void stream_table_load(const uint32_t *tab, const uint32_t d0,
                                                  StreamTab &tb) {
  const uint32_t v = tab[threadIdx.x & 31];
#pragma unroll
  for (int i = 0; i < STREAM_BX; ++i) {
    tb.d[i] = d0 + __shfl_sync(0xffffffffu, v, i);
    tb.b[i] = __shfl_sync(0xffffffffu, v, 8 + i);
    tb.id[i] = __shfl_sync(0xffffffffu, v, 16 + i);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    tb.wa[k] = __shfl_sync(0xffffffffu, v, 24 + k);
    tb.wb[k] = __shfl_sync(0xffffffffu, v, 26 + k);
    tb.wid[k] = __shfl_sync(0xffffffffu, v, 28 + k);
  }
}
template <int CNT>
__device__ __forceinline__ void mma_group_stream(
    const uint32_t a_lo0, const uint32_t a_hi, const uint32_t b_base0, const uint32_t b_stage_bytes,
    const uint32_t b_hi, const uint32_t slab_inc, const uint32_t slice_inc, const uint32_t d0,
    const int steps, const int tz_n, const uint32_t dz_step, const uint32_t a_wrap,
    const MmaCtx &cx, const StreamTab &tb, int &b_st) {
  int tz = 0;
  uint32_t off = 0;
  for (int s0 = 0; s0 < steps; s0 += cx.bsteps) {
    const int n = min(cx.bsteps, steps - s0);
    if (cx.first_tile_iter) mbar_wait(&cx.b_full[b_st], 0);   // resident weights
    tc_fence_after();
    uint32_t b_lo = desc_lo(b_base0 + b_st * b_stage_bytes, 128u);
    for (int i0 = 0; i0 < n; ++i0) {
      const uint32_t a_lo = a_lo0 + off;
      umma_stream_step<CNT>(a_lo, a_hi, b_lo, b_hi, slice_inc, tb.d, tb.b, tb.id);
      if (tb.wid[0]) {
        umma_bf16_lohi_elect(d0, a_lo + tb.wa[0], a_hi, b_lo + tb.wb[0], b_hi, tb.wid[0], 1u);
        if (tb.wid[1])
          umma_bf16_lohi_elect(d0, a_lo + tb.wa[1], a_hi, b_lo + tb.wb[1], b_hi, tb.wid[1], 1u);
      }
      b_lo += slab_inc;
      off += dz_step;
      if (++tz == tz_n) {
        tz = 0;
        off += a_wrap;
      }
    }
    ++b_st;
  }
}

template <int ACT, bool FASTOUT, bool BASE, bool PAIR, bool F32IN, bool POOL = false,
          bool HEAD = false, bool LEAN = false, bool STREAM = false>
__global__ void __maxnreg__(VXB_TC_MAXNREG)
    conv3d_tc_kernel(const __grid_constant__ TcParams p, const __grid_constant__ TcMaps maps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int EPI_WARPS = epi_warps(F32IN);
  // warp index broadcast from lane 0 so ptxas treats each role's code as
  // warp-uniform (as CUTLASS's canonical_warp_idx_sync does)
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const SmemMap sm = smem_map(p);
  pdl_trigger();
  if (threadIdx.x == 0) dbg_mark(p, 0, 5);

  uint8_t *a_buf = smem + sm.a;
  uint8_t *b_buf = smem + sm.b;
  float *s_bias = reinterpret_cast<float *>(smem + sm.bias);
  float *s_scale = reinterpret_cast<float *>(smem + sm.scale);
  float *s_head = reinterpret_cast<float *>(smem + sm.head);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + sm.bars);
  uint64_t *a_full = bars;
  uint64_t *a_empty = a_full + p.na;
  uint64_t *b_full = a_empty + p.na;
  uint64_t *b_empty = b_full + p.nb_stages;
  uint64_t *t_full = b_empty + p.nb_stages;
  uint64_t *t_empty = t_full + MAX_ACC;
  uint64_t *stg_full = t_empty + MAX_ACC;           // F32IN staging ring
  uint64_t *stg_empty = stg_full + p.n_stg;
  uint64_t *info_full = stg_empty + p.n_stg;          // lean: TileInfo ring slots
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(stg_empty + p.n_stg + (p.lean ? TINFO : 0));
  uint8_t *stg_buf = smem + sm.stg;

  // CTA pairs (cluster 2) walk pairs of tiles in lockstep so they can share
  // one B (weight) stream through TMA multicast
  // (broadcast so ptxas knows it is warp-uniform: an opaque asm result would
  // make everything under `crank == 0` look divergent, and the MMA issue loop
  // then routes every descriptor through R2UR / VOTEU / BRA.DIV sequences)
  const int crank =
      p.cluster == 2 ? __shfl_sync(0xffffffffu, static_cast<int>(cluster_rank()), 0) : 0;
  const int first_tile = (blockIdx.x / p.cluster) * p.cluster + crank;
  const int tile_step = gridDim.x;
  const uint16_t pair_mask = 0x3;
  const int acc_stride = p.acc_stride;
  const uint32_t tmem_cols = static_cast<uint32_t>(p.tmem_cols);

  // one-time setup by all threads: guard bytes behind every chunk array
  // (read with zero weight by odd-chunk z-pair steps) and the per-fmap
  // epilogue vectors
  for (int s = 0; s < p.na; ++s)
    for (int c = 0; c < p.chunk_slots; ++c) {
      uint8_t *g = a_buf + s * p.a_stage_bytes + c * p.chunk_stride + p.chunk_bytes;
      for (int i = threadIdx.x; i < 32; i += blockDim.x) reinterpret_cast<uint32_t *>(g)[i] = 0u;
    }
  const int cpad = p.n_tiles * p.nt;
  LeanEnt *ltab = reinterpret_cast<LeanEnt *>(smem + sm.ltab);
  TileInfo *tinfo = reinterpret_cast<TileInfo *>(smem + sm.ltab + LEAN_TAB * sizeof(LeanEnt));
  if (LEAN)
    for (int ci = threadIdx.x; ci < (p.nt >> 4); ci += blockDim.x) {
      const int cc = ci << 4;
      int rep = 0, ch = cc;
      if (p.zpair) {
        const int rp = cc / (2 * p.rep_n), rem = cc - rp * 2 * p.rep_n;
        rep = 2 * rp;
        ch = (rem >> 4) << 3;
      } else if (p.rep_n) {
        rep = cc / p.rep_n;
        ch = cc - rep * p.rep_n;
      }
      const long long oc = static_cast<long long>(ch >> 3) * p.out.s[1];
      const long long bc = static_cast<long long>(ch >> 3) * p.base.s[1];
      LeanEnt e;
      e.o0 = (p.rep_n ? p.out_rep_off[rep] : 0) + oc;
      e.o1 = p.zpair ? p.out_rep_off[rep + 1] + oc : e.o0 + p.out.s[1];
      e.b0 = (p.rep_n ? p.base_rep_off[rep] : 0) + bc;
      e.b1 = p.zpair ? p.base_rep_off[rep + 1] + bc : e.b0 + p.base.s[1];
      e.ch = ch;
      e.pad = 0;
      ltab[ci] = e;
    }
  if constexpr (STREAM) {
    uint32_t *stab_s = reinterpret_cast<uint32_t *>(smem + sm.stab);
    const uint32_t blk_w = (p.nt * SLAB_ROW_BYTES) >> 4, sl_w = p.a_slice_inc >> 4;
    for (int e = threadIdx.x; e < p.st_nphase * p.st_nslab * 9; e += blockDim.x) {
      const int tb_i = e / 9, i = e - tb_i * 9;
      stream_table_entry(p, stab_s + tb_i * STAB_WORDS, tb_i / p.st_nslab, tb_i % p.st_nslab, i,
                         blk_w, sl_w);
    }
  }
  fence_proxy_async_smem();

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&maps.m[0]);
    if (p.seg_chunks[1] > 0) prefetch_tmap(&maps.m[1]);
    for (int i = 0; i < p.na; ++i) {
      // F32IN: the stage is full once every converter warp (of both CTAs of a
      // pair) has written its rows; otherwise the TMA bytes complete it
      mbar_init(&a_full[i], F32IN ? CVT_WARPS * (PAIR ? 2 : 1) : 1);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < p.n_stg; ++i) {
      mbar_init(&stg_full[i], 1);
      mbar_init(&stg_empty[i], CVT_WARPS);
    }
    for (int i = 0; i < p.nb_stages; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], PAIR ? 1 : p.cluster);
    }
    for (int i = 0; i < MAX_ACC; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], PAIR ? 2 * EPI_WARPS : EPI_WARPS);
    }
    if (LEAN)
      for (int i = 0; i < TINFO; ++i) mbar_init(&info_full[i], 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    if (PAIR) {
      tmem_alloc_pair(tmem_slot, tmem_cols);
      tmem_relinquish_pair();
    } else {
      tmem_alloc(tmem_slot, tmem_cols);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (p.cluster == 2) cluster_sync_all();   // peer barriers initialised before multicast
  tc_fence_after();
  // broadcast (not a plain smem load) so the compiler knows it is warp-uniform
  // and keeps everything derived from it in uniform registers
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  pdl_wait();   // activations (inputs, residual, output buffer) belong to the predecessor until here

  if (warp == 0) {
    // ===================== A producer: halo tiles (TMA 4-D boxes) ==========
    if (STREAM && lane == 0) {
      // streamed fold: whole columns, slab by slab along x (no x halo)
      int a_st = 0, a_ph = 0, pit = 0, rb = 0;
      const int smask = p.st_slots - 1;
      for (int col = blockIdx.x; col < p.st_ncols; col += gridDim.x) {
        const int tz = col % p.tiles_z, q1 = col / p.tiles_z;
        const int ty = q1 % p.tiles_y, b = q1 / p.tiles_y;
        const int y0 = ty * TILE_Y, z0 = tz * TILE_Z;
        int dprev = -1;   // last output slice handed to the epilogue so far
        for (int t = 0; t < p.st_nslab; ++t, ++pit) {
          const int jmin = p.st_j0 + t * p.bx;
          const int cnt = min(p.bx, p.st_nin - t * p.bx);
          // output slices complete after this slab: all whose last input
          // slice (s + 2) lies in it, the rest of the column after the last
          const int dhi = t == p.st_nslab - 1 ? p.ox - 1 : min(p.ox - 1, jmin + cnt - 3);
          const int dlo = dprev + 1;
          TileInfo ti;
          ti.rc0 = y0;
          ti.z0 = z0;
          ti.sc0 = dlo;
          ti.nt0 = 0;
          ti.dummy = 0;
          ti.ns = max(0, dhi - dlo + 1);
          ti.slot0 = (rb + dlo) & smask;
          dprev = max(dprev, dhi);
          ti.o_off = b * p.out.s[0] + static_cast<long long>(y0) * p.out.s[3] +
                     static_cast<long long>(z0) * p.out.s[4] +
                     static_cast<long long>(dlo) * p.out.s[2] + p.out_rep_off[0];
          ti.b_off = b * p.base.s[0] + static_cast<long long>(y0) * p.base.s[3] +
                     static_cast<long long>(z0) * p.base.s[4] +
                     static_cast<long long>(dlo) * p.base.s[2] + p.base_rep_off[0];
          ti.p_off = 0;
          if (p.pool)
            ti.p_off = b * p.pool_out.s[0] + static_cast<long long>(dlo) * p.pool_out.s[2] +
                       static_cast<long long>(y0 >> 1) * p.pool_out.s[3] +
                       static_cast<long long>(z0 >> 1) * p.pool_out.s[4];
          for (int i = 0; i < 3; ++i) ti.pad[i] = 0;
          tinfo[pit & (TINFO - 1)] = ti;
          mbar_arrive(&info_full[pit & (TINFO - 1)]);
          for (int g = 0; g < p.n_groups; ++g) {
            GroupInfo gi = group_info(p, g);
            mbar_wait_sleep(&a_empty[a_st], a_ph ^ 1);
            if (g == 0) dbg_mark(p, pit, 0);
            mbar_expect_tx(&a_full[a_st], gi.nch * p.chunk_bytes);
            const int *off = p.seg_off[gi.seg];
            const int cx = jmin - p.pad[0] + off[0];
            const int cy = y0 - p.pad[1] + off[1];
            const int cz = (z0 - p.pad[2] + off[2]) * LANES;
            for (int ci = 0; ci < gi.nch; ++ci)
              tma_load_4d(a_buf + a_st * p.a_stage_bytes + ci * p.chunk_stride, &maps.m[gi.seg],
                          &a_full[a_st], cz, cy, cx, b * p.seg_bstride[gi.seg] + gi.chunk0 + ci);
            if (++a_st == p.na) {
              a_st = 0;
              a_ph ^= 1;
            }
          }
        }
        rb = (rb + p.ox) & smask;
      }
    } else if (lane == 0) {
      int a_st = 0, a_ph = 0, s_st = 0, s_ph = 0;
      int pit = 0;
      for (int tile = first_tile; tile < p.total_tiles; tile += tile_step, ++pit) {
        TileCoord tc = decode_tile(p, tile);
        if constexpr (LEAN) {
          TileInfo ti;
          const int ra_dim = p.slice_y ? 2 : 3, sl_dim = p.slice_y ? 3 : 2;
          ti.rc0 = p.slice_y ? tc.x0 : tc.y0;
          ti.z0 = tc.z0;
          ti.sc0 = p.slice_y ? tc.y0 : tc.x0;
          ti.nt0 = tc.nt * p.nt;
          ti.dummy = tc.dummy;
          ti.o_off = tc.b * p.out.s[0] + static_cast<long long>(ti.rc0) * p.out.s[ra_dim] +
                     static_cast<long long>(ti.z0) * p.out.s[4] +
                     static_cast<long long>(ti.sc0) * p.out.s[sl_dim] +
                     (p.rep_n ? 0 : p.out_rep_off[tc.rep]) + (ti.nt0 >> 3) * p.out.s[1];
          ti.b_off = tc.b * p.base.s[0] + static_cast<long long>(ti.rc0) * p.base.s[ra_dim] +
                     static_cast<long long>(ti.z0) * p.base.s[4] +
                     static_cast<long long>(ti.sc0) * p.base.s[sl_dim] +
                     (p.rep_n ? 0 : p.base_rep_off[tc.rep]) + (ti.nt0 >> 3) * p.base.s[1];
          ti.p_off = 0;
          if (p.pool)   // the pooled tile origin (tiles start at even y, z)
            ti.p_off = tc.b * p.pool_out.s[0] + static_cast<long long>(ti.sc0) * p.pool_out.s[2] +
                       static_cast<long long>(ti.rc0 >> 1) * p.pool_out.s[3] +
                       static_cast<long long>(ti.z0 >> 1) * p.pool_out.s[4] +
                       (ti.nt0 >> 3) * p.pool_out.s[1];
          ti.ns = ti.slot0 = 0;
          for (int i = 0; i < 3; ++i) ti.pad[i] = 0;
          tinfo[pit & (TINFO - 1)] = ti;
          mbar_arrive(&info_full[pit & (TINFO - 1)]);   // release: the epilogue acquires
        }
        for (int g = 0; g < p.n_groups; ++g) {
          GroupInfo gi = group_info(p, g);
          mbar_wait_sleep(&a_empty[a_st], a_ph ^ 1);
          if (g == 0) dbg_mark(p, pit, 0);
          // pair mode: the leader's barrier counts both CTAs' bytes
          if (p.dbg_mode & 2) {
            if (!PAIR || crank == 0) mbar_arrive(&a_full[a_st]);
            if (++a_st == p.na) {
              a_st = 0;
              a_ph ^= 1;
            }
            continue;
          }
          if (F32IN) {
            // fp32 NCDHW input: one (hzb, hy, 1, 8) box per chunk and halo
            // x-slice into the staging ring; the converter warps fill the stage
            const int *off = p.seg_off[0];
            const int cx = tc.x0 - p.pad[0] + off[0];
            const int cy = tc.y0 - p.pad[1] + off[1];
            const int cz = tc.z0 - p.pad[2] + off[2] - p.f32in_zshift;   // 16-byte aligned
            for (int ci = 0; ci < gi.nch; ++ci)
              for (int xs = 0; xs < p.hx; xs += p.f32in_xb) {
                mbar_wait_sleep(&stg_empty[s_st], s_ph ^ 1);
                if (p.dbg_mode & 128) {
                  mbar_arrive(&stg_full[s_st]);
                } else {
                  mbar_expect_tx(&stg_full[s_st], p.stg_bytes);
                  // (batch folded into the channel coordinate: c + b * C)
                  tma_load_4d(stg_buf + s_st * p.stg_bytes, &maps.m[0], &stg_full[s_st], cz, cy,
                              cx + xs, (gi.chunk0 + ci) * LANES + tc.b * p.f32in_cstride);
                }
                if (++s_st == p.n_stg) {
                  s_st = 0;
                  s_ph ^= 1;
                }
              }
            if (++a_st == p.na) {
              a_st = 0;
              a_ph ^= 1;
            }
            continue;
          }
          if (!PAIR || crank == 0)
            mbar_expect_tx(&a_full[a_st], gi.nch * p.chunk_bytes * (PAIR ? 2 : 1));
          const int *off = p.seg_off[gi.seg];
          const int cx = tc.x0 - p.pad[0] + off[0];
          const int cy = tc.y0 - p.pad[1] + off[1];
          const int cz = (tc.z0 - p.pad[2] + off[2]) * LANES;
          for (int ci = 0; ci < gi.nch; ++ci) {
            const int chunk = tc.b * p.seg_bstride[gi.seg] + gi.chunk0 + ci;
            if (PAIR)
              tma_load_4d_pair(a_buf + a_st * p.a_stage_bytes + ci * p.chunk_stride,
                               &maps.m[gi.seg], &a_full[a_st], cz, cy, cx, chunk);
            else
              tma_load_4d(a_buf + a_st * p.a_stage_bytes + ci * p.chunk_stride, &maps.m[gi.seg],
                          &a_full[a_st], cz, cy, cx, chunk);
          }
          if (++a_st == p.na) {
            a_st = 0;
            a_ph ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ===================== B producer: weight slabs (bulk copies) ==========
    // independent of the A producer so halo loads are never queued behind
    // the weight stream of the current group
    if (lane == 0) {
      int b_st = 0, b_ph = 0;
      const uint32_t slab = static_cast<uint32_t>(p.slab_bytes);
      for (int tile = first_tile; tile < p.total_tiles; tile += tile_step) {
        if (p.resident && tile != first_tile) break;   // resident bank: loaded once
        TileCoord tc = decode_tile(p, STREAM ? 0 : tile);
        const uint8_t *wbase = p.w + tc.rep * p.w_rep_stride + tc.nt * p.w_ntile_stride;
        long long step_base = 0;
        for (int g = 0; g < p.n_groups; ++g) {
          GroupInfo gi = group_info(p, g);
          for (int s0 = 0; s0 < gi.steps; s0 += p.bsteps) {
            const int n = min(p.bsteps, gi.steps - s0);
            const uint32_t bytes = n * slab;
            mbar_wait_sleep(&b_empty[b_st], b_ph ^ 1);
            if (p.dbg_mode & 4) {
              if (!PAIR || crank == 0) mbar_arrive(&b_full[b_st]);
            } else if (PAIR) {
              // this CTA's half (rows [crank*nt/2, ..)) of bsteps slabs; the
              // box always spans bsteps steps (extra steps are never read)
              if (crank == 0) mbar_expect_tx(&b_full[b_st], 2 * p.b_stage_bytes);
              const int step0 = static_cast<int>((static_cast<long long>(tc.rep) * p.n_tiles +
                                                  tc.nt) * p.w_steps + step_base + s0);
              tma_load_4d_pair(b_buf + b_st * p.b_stage_bytes, &maps.w, &b_full[b_st], 0, 0,
                               crank, step0);
            } else if (p.cluster == 2) {
              mbar_expect_tx(&b_full[b_st], bytes);
              // each CTA of the pair fetches one half and multicasts it to both
              const uint32_t hb = bytes >> 1;
              bulk_load_mc(b_buf + b_st * p.b_stage_bytes + crank * hb,
                           wbase + (step_base + s0) * slab + crank * hb, hb, &b_full[b_st],
                           pair_mask);
            } else {
              mbar_expect_tx(&b_full[b_st], bytes);
              bulk_load(b_buf + b_st * p.b_stage_bytes, wbase + (step_base + s0) * slab, bytes,
                        &b_full[b_st]);
            }
            if (++b_st == p.nb_stages) {
              b_st = 0;
              b_ph ^= 1;
            }
          }
          step_base += gi.steps;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    // The issue loop paces N >= 128 convs (one tcgen05.mma per ~64 cycles).
    // The whole warp walks the schedule in convergent, warp-uniform control
    // flow so ptxas keeps descriptors in uniform registers; the MMA asm
    // elects one lane.  Descriptors are split in a loop-invariant high word
    // and a low word advanced by constants; the x-slice loop is unrolled.
    if (!PAIR || crank == 0) {
      const uint32_t idesc = idesc_bf16(PAIR ? 256 : 128, p.nt);
      const uint32_t a_base0 = smem_u32(a_buf);
      const uint32_t b_base0 = smem_u32(b_buf);
      const uint32_t slice_inc = p.a_slice_inc >> 4;
      const uint32_t b_inc = (p.slab_bytes / (PAIR ? 2 : 1)) >> 4;
      const uint32_t a_hi = desc_hi(p.a_sbo);
      const uint32_t blk_inc = (p.nt * SLAB_ROW_BYTES) >> 4;
      // (debug mode 16: every folded MMA at N = nt, to time the issue loop)
      const uint32_t idp = idesc_bf16(256, p.fold ? 3 * p.nt : p.nt);   // folded pairs
      const uint32_t id1 = idesc_bf16(128, p.nt),
                     id2 = (p.dbg_mode & 16) ? id1 : idesc_bf16(128, 2 * p.nt),
                     id3 = (p.dbg_mode & 16) ? id1 : idesc_bf16(128, p.fold ? 3 * p.nt : p.nt);
      // folded walk: z taps inside, the other non-slice axis outside
      const uint32_t fold_stride = (p.slice_y ? p.hy * p.hz : p.hz);
      const uint32_t b_hi = desc_hi(256u);
      MmaCtx cx;
      cx.b_full = b_full;
      cx.b_empty = b_empty;
      cx.nb_stages = p.nb_stages;
      cx.bsteps = p.bsteps;
      cx.resident = p.resident;
      cx.cluster = p.cluster;
      int a_st = 0, a_ph = 0, b_st = 0, b_ph = 0;
      // Count this CTA's tiles up front: a loop bound compared against a
      // tile index derived from blockIdx makes ptxas treat the whole loop as
      // divergent, and every MMA operand then goes through R2UR.BROADCAST
      // (~5 extra instructions per MMA, which bounded the N = 128 convs).
      const int my_tiles =
          STREAM ? (static_cast<int>(blockIdx.x) < p.st_ncols
                        ? (p.st_ncols - static_cast<int>(blockIdx.x) + tile_step - 1) / tile_step *
                              p.st_nslab
                        : 0)
                 : (first_tile < p.total_tiles
                        ? (p.total_tiles - first_tile + tile_step - 1) / tile_step
                        : 0);
      const bool no_mma = (p.dbg_mode & 8) && p.resident;   // debug: epilogue-only timing
      // The tile loop is instantiated per (walk, tile width): the dispatch
      // happens once per kernel, not once per K group (per-group work in the
      // issue loop costs MMA throughput).
      auto tiles = [&](auto bx_c, auto kind_c) {
        constexpr int BXV = decltype(bx_c)::value;
        constexpr int KIND = decltype(kind_c)::value;   // 0 plain, 1 folded, 2 folded pair
        // accumulator stage of tile `it`: it % acc_stages, phase (it / acc_stages) & 1
        int acc = -1, acc_ph = 1;
        StreamCtx sc;   // streamed fold: slab within the column, ring base
        sc.S = p.ox;
        sc.rb = 0;
        sc.slots = p.st_slots;
        int st_t = 0, st_ph = 0;
        StreamTab stab;
        if constexpr (KIND == 3) {
          // the epilogue warps zeroed the accumulator ring (t_full[MAX_ACC - 1])
          if (my_tiles > 0) mbar_wait(&t_full[MAX_ACC - 1], 0);
          tc_fence_after();
        }
        for (int it = 0; it < my_tiles; ++it) {
          if constexpr (KIND == 3) {
            // (the slab's operand table was worked out while the previous
            // slab's MMAs drained: see the end of the loop body)
            if (it == 0) {
              sc.jmin = p.st_j0;
              sc.cnt = min(p.bx, p.st_nin);
              stream_table_load(reinterpret_cast<const uint32_t *>(smem + sm.stab), tmem_base,
                                stab);
            }
          }
          if (++acc == p.acc_stages) acc = 0;
          if (acc == 0) acc_ph ^= 1;
          mbar_wait(&t_empty[acc], acc_ph ^ 1);
          tc_fence_after();
          const uint32_t d_base = tmem_base + acc * acc_stride;
          uint32_t accumulate = 0, first = 1;
          if (p.resident) b_st = 0;
          cx.first_tile_iter = it == 0;
          for (int g = 0; g < p.n_groups; ++g) {
            GroupInfo gi = group_info(p, g);
            mbar_wait(&a_full[a_st], a_ph);
            tc_fence_after();
            if (g == 0 && lane == 0) {
              dbg_mark(p, it, 1);
              dbg_clock(p, it, 5);
            }
            const bool pair = gi.nch == 2;
            const int tz_n = pair ? p.kz : (p.kz + 1) >> 1;
            const uint32_t dz_step = pair ? 1u : 2u;
            const uint32_t a_lo0 =
                desc_lo(a_base0 + a_st * p.a_stage_bytes, pair ? p.chunk_stride : 16u);
            if (!no_mma) {
              if constexpr (KIND == 3) {
                auto run = [&](auto cnt_c) {
                  mma_group_stream<decltype(cnt_c)::value>(
                      a_lo0, a_hi, b_base0, p.b_stage_bytes, b_hi, b_inc, slice_inc, tmem_base,
                      gi.steps, tz_n, dz_step, fold_stride - tz_n * dz_step, cx, stab, b_st);
                };
                switch (sc.cnt) {
                  case 1: run(std::integral_constant<int, 1>{}); break;
                  case 2: run(std::integral_constant<int, 2>{}); break;
                  case 3: run(std::integral_constant<int, 3>{}); break;
                  case 4: run(std::integral_constant<int, 4>{}); break;
                  case 5: run(std::integral_constant<int, 5>{}); break;
                  case 6: run(std::integral_constant<int, 6>{}); break;
                  case 7: run(std::integral_constant<int, 7>{}); break;
                  default: run(std::integral_constant<int, 8>{}); break;
                }
              } else if constexpr (KIND == 2) {
                mma_group_fold_pair<BXV>(a_lo0, a_hi, b_base0, p.b_stage_bytes, b_hi, b_inc,
                                         slice_inc, d_base, p.nt, idp, gi.steps, tz_n, dz_step,
                                         fold_stride - tz_n * dz_step, cx, b_st, b_ph, first);
              } else if constexpr (KIND == 1) {
                mma_group_fold<BXV>(a_lo0, a_hi, b_base0, p.b_stage_bytes, b_hi, b_inc, blk_inc,
                                    slice_inc, d_base, p.nt, id1, id2, id3, gi.steps, tz_n,
                                    dz_step, fold_stride - tz_n * dz_step, cx, b_st, b_ph, first);
              } else {
                mma_group<BXV, PAIR>(a_lo0, a_hi, b_base0, p.b_stage_bytes, b_hi, b_inc,
                                     slice_inc, d_base, p.nt, idesc, gi.steps, tz_n, dz_step,
                                     p.hz - tz_n * dz_step, (p.hy - p.ky) * p.hz, p.ky, cx,
                                     b_st, b_ph, accumulate);
              }
            }
            if (PAIR)
              umma_commit_pair_elect(&a_empty[a_st], pair_mask);
            else
              umma_commit_elect(&a_empty[a_st]);
            if (++a_st == p.na) {
              a_st = 0;
              a_ph ^= 1;
            }
          }
          if (PAIR)
            umma_commit_pair_elect(&t_full[acc], pair_mask);
          else
            umma_commit_elect(&t_full[acc]);
          if (lane == 0) {
            dbg_mark(p, it, 2);
            dbg_clock(p, it, 6);
          }
          if constexpr (KIND == 3) {
            if (++st_t == p.st_nslab) {
              st_t = 0;
              if (++st_ph == p.st_nphase) st_ph = 0;
            }
            sc.jmin = p.st_j0 + st_t * p.bx;
            sc.cnt = min(p.bx, p.st_nin - st_t * p.bx);
            // the next slab's operand table (while this slab's MMAs drain)
            if (!(p.dbg_mode & 4096))   // (debug: keep the first slab's table)
              stream_table_load(reinterpret_cast<const uint32_t *>(smem + sm.stab) +
                                    (st_ph * p.st_nslab + st_t) * STAB_WORDS,
                                tmem_base, stab);
          }
        }
      };
      using I1 = std::integral_constant<int, 1>;
      using I2 = std::integral_constant<int, 2>;
      using I3 = std::integral_constant<int, 3>;
      using I4 = std::integral_constant<int, 4>;
      using I6 = std::integral_constant<int, 6>;
      using I8 = std::integral_constant<int, 8>;
      using K0 = std::integral_constant<int, 0>;
      using K1 = std::integral_constant<int, 1>;
      using K2 = std::integral_constant<int, 2>;
      using K3 = std::integral_constant<int, 3>;
      if constexpr (STREAM) {
        tiles(I1{}, K3{});
      } else if (p.fold) {
        auto folded = [&](auto kind_c) {
          switch (p.bx) {
            case 1: tiles(I1{}, kind_c); break;
            case 2: tiles(I2{}, kind_c); break;
            case 3: tiles(I3{}, kind_c); break;
            case 4: tiles(I4{}, kind_c); break;
            case 6: tiles(I6{}, kind_c); break;
            default: tiles(I8{}, kind_c); break;
          }
        };
        if constexpr (PAIR) folded(K2{});
        else folded(K1{});
      } else {
        switch (p.bx) {
          case 1: tiles(I1{}, K0{}); break;
          case 2: tiles(I2{}, K0{}); break;
          case 3: tiles(I3{}, K0{}); break;
          case 4: tiles(I4{}, K0{}); break;
          case 6: tiles(I6{}, K0{}); break;
          default: tiles(I8{}, K0{}); break;
        }
      }
    }
    __syncwarp();
  } else if (F32IN && warp >= 3 + EPI_WARPS) {
    // ===================== fp32 -> bf16 chunk converters (F32IN) ============
    // Staging slot = (8 c, xb, hy, hzb) fp32 of xb halo x-slices.  A work item
    // is one z-pair of a staging row: 8 float2 loads (one per channel plane)
    // give two voxels' 8 channels, written as two 16-byte bf16x8 rows of the
    // A stage's chunk array.  Pairs start at even staging positions (8-byte
    // loads), so with an odd z shift the first / last pair of a row holds one
    // voxel outside the halo, which is not stored.
    const int ct = threadIdx.x - 32 * (3 + EPI_WARPS);   // 0 .. 32*CVT_WARPS-1
    constexpr int NT = 32 * CVT_WARPS;
    const int rows = p.hy * p.hz;
    const int zs = p.f32in_zshift;
    const int p0 = zs >> 1;                              // first pair (staging position 2*p0)
    const int np = ((zs + p.hz + 1) >> 1) - p0;          // pairs per row
    const int per_x = p.hy * np;
    const int cstride = p.f32in_xb * p.hy * p.hzb;       // fp32 elements per channel plane
    // this thread's first item and the stride, split into (x, y, pair)
    const int s_x = NT / per_x, s_y = (NT % per_x) / np, s_p = NT % np;
    int a_st = 0, s_st = 0, s_ph = 0;
    for (int tile = first_tile; tile < p.total_tiles; tile += tile_step) {
      for (int g = 0; g < p.n_groups; ++g) {
        GroupInfo gi = group_info(p, g);
        uint8_t *abase = a_buf + a_st * p.a_stage_bytes;
        for (int ci = 0; ci < gi.nch; ++ci)
          for (int xs0 = 0; xs0 < p.hx; xs0 += p.f32in_xb) {
            mbar_wait(&stg_full[s_st], s_ph);
            const float *src0 = reinterpret_cast<const float *>(stg_buf + s_st * p.stg_bytes);
            const int nxs = min(p.f32in_xb, p.hx - xs0);
            uint4 *dst0 = reinterpret_cast<uint4 *>(abase + ci * p.chunk_stride) + xs0 * rows;
            int xi = ct / per_x, y = (ct % per_x) / np, pp = ct % np;
            if (p.dbg_mode & 64) xi = nxs;
            while (xi < nxs) {
              const int zp = 2 * (pp + p0);                // staging position of the pair
              const float *q = src0 + (xi * p.hy + y) * p.hzb + zp;
              float2 v[8];
#pragma unroll
              for (int c = 0; c < 8; ++c) v[c] = *reinterpret_cast<const float2 *>(q + c * cstride);
              uint4 lo, hi;
              __nv_bfloat162 *hl = reinterpret_cast<__nv_bfloat162 *>(&lo);
              __nv_bfloat162 *hh = reinterpret_cast<__nv_bfloat162 *>(&hi);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                hl[i] = __floats2bfloat162_rn(v[2 * i].x, v[2 * i + 1].x);
                hh[i] = __floats2bfloat162_rn(v[2 * i].y, v[2 * i + 1].y);
              }
              const int z = zp - zs;                       // halo z of the pair's first voxel
              uint4 *d = dst0 + xi * rows + y * p.hz + z;
              if (z >= 0) d[0] = lo;
              if (z + 1 < p.hz) d[1] = hi;
              // advance by NT items: (x, y, pair) with carries
              pp += s_p;
              y += s_y;
              xi += s_x;
              if (pp >= np) {
                pp -= np;
                ++y;
              }
              if (y >= p.hy) {
                y -= p.hy;
                ++xi;
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&stg_empty[s_st]);
            if (++s_st == p.n_stg) {
              s_st = 0;
              s_ph ^= 1;
            }
          }
        // the tensor core reads the stage through the async proxy
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (PAIR)
            mbar_arrive_cta_release(&a_full[a_st], 0);
          else
            mbar_arrive(&a_full[a_st]);
        }
        if (++a_st == p.na) a_st = 0;
      }
    }
  } else {
    // ===================== epilogue (EPI_WARPS warps, EPI_WARPS/4 per quarter) ==
    // Work item = (slice, 16 accumulator columns).  The TMEM load of item k+1
    // and the residual loads of items k+1, k+2 are in flight while item k is
    // finished (software pipeline).
    // per-fmap epilogue vectors (bias, residual scale, head weights) are
    // staged by the epilogue warps only, after the CTA-wide setup, so their
    // global-memory latency overlaps the first tile's loads and MMAs
    {
      const int et = threadIdx.x - 96;
      for (int c = et; c < cpad; c += 32 * EPI_WARPS) {
        // taps in N: column -> channel of its tap (z-pair order: see TcParams::zpair)
        int cr = c;
        if (p.rep_n) {
          const int rem = p.zpair ? c % (2 * p.rep_n) : c % p.rep_n;
          cr = p.zpair ? ((rem >> 4) << 3) + (rem & 7) : rem;
        }
        s_bias[c] = cr < p.cout ? p.bias[cr] : 0.f;
        s_scale[c] = (cr < p.cout && p.scale) ? p.scale[cr] : 1.f;
      }
      if (HEAD)
        for (int i = et; i < 4 * cpad; i += 32 * EPI_WARPS) {
          const int j = i / cpad, c = i - j * cpad;
          s_head[i] = (j < p.head_cout && c < p.cout) ? p.head_w[j * p.cout + c] : 0.f;
        }
      if constexpr (STREAM) {
        // streamed fold: every MMA accumulates, so the ring starts zeroed
        // (and the epilogue zeroes each slot again after reading it)
        const uint32_t tq = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        for (int u = (warp - 3) >> 2; u < (p.st_slots * p.nt) >> 4; u += EPI_WARPS / 4)
          tmem_st16_zero(tq + u * 16);
        tmem_wait_st();
        tc_fence_before();
      }
      named_bar_sync(2, 32 * EPI_WARPS);
      if (STREAM && warp == 3 && lane == 0) mbar_arrive(&t_full[MAX_ACC - 1]);
    }
    const int q = warp & 3;                   // TMEM lane quarter this warp may access
    const int sub = (warp - 3) >> 2;          // which share of the work items
    constexpr int NSUB = EPI_WARPS / 4;
    const int row = q * 32 + lane;            // MMA row == TMEM lane
    const int ra = row >> 3, zz = row & 7;    // row-axis offset (y, or x with slice_y), z
    const int col_items = p.nt >> 4;
    // item -> (slice, column offset) without a division: items < 2^16, so
    // a multiply-high by ceil(2^32 / col_items) is exact
    const uint32_t cmagic = col_items > 1 ? 0xffffffffu / col_items + 1u : 0u;
    auto split_item = [&](int item, int &s, int &cc) {
      s = col_items > 1 ? static_cast<int>(__umulhi(static_cast<uint32_t>(item), cmagic)) : item;
      cc = (item - s * col_items) << 4;
    };
    const EpiView &ov = p.out;
    const EpiView &bvw = p.base;
    const int act = ACT >= 0 ? ACT : p.act;
    const bool braw = BASE && bvw.dtype == VXB_BF16 && bvw.blocked;
    int it = 0;
    int acc = -1, acc_ph = 1;   // accumulator stage it % acc_stages and its phase
    const int ra_dim = p.slice_y ? 2 : 3, sl_dim = p.slice_y ? 3 : 2;
    // lean: this thread's row offset inside a tile (per kernel)
    const long long ra_oo = LEAN ? ra * ov.s[ra_dim] + zz * ov.s[4] : 0;
    const long long ra_bo = LEAN && BASE ? ra * bvw.s[ra_dim] + zz * bvw.s[4] : 0;
    // lean + fused pool: lanes with (y, z) both even store the 2x2 max
    const long long ra_po = LEAN ? (ra >> 1) * p.pool_out.s[3] + (zz >> 1) * p.pool_out.s[4] : 0;
    // (streamed fold: the CTA's columns x slabs, in the producer's order)
    const int n_items =
        STREAM ? (static_cast<int>(blockIdx.x) < p.st_ncols
                      ? (p.st_ncols - static_cast<int>(blockIdx.x) + tile_step - 1) / tile_step *
                            p.st_nslab
                      : 0)
               : (first_tile < p.total_tiles
                      ? (p.total_tiles - first_tile + tile_step - 1) / tile_step
                      : 0);
    for (; it < n_items; ++it) {
      const int tile = first_tile + it * tile_step;
      TileCoord tc;
      int rc, z, sc0;
      int st_ns = 0, st_slot0 = 0;
      bool yz_ok;
      long long lo_off = 0, lb_off = 0, lp_off = 0;
      int nt0;
      if constexpr (LEAN) {
        // the producer published this tile's origin (TileInfo ring)
        const int slot = it & (TINFO - 1);
        mbar_wait_sleep(&info_full[slot], static_cast<uint32_t>((it / TINFO) & 1));
        const TileInfo &ti = tinfo[slot];
        rc = ti.rc0 + ra;
        z = ti.z0 + zz;
        sc0 = ti.sc0;
        nt0 = ti.nt0;
        yz_ok = rc < (p.slice_y ? p.ox : p.oy) && z < p.oz && !ti.dummy;
        lo_off = ti.o_off + ra_oo;
        lb_off = ti.b_off + ra_bo;
        lp_off = ti.p_off + ra_po;
        st_ns = ti.ns;
        st_slot0 = ti.slot0;
        tc.rep = 0;
        tc.nt = 0;
        tc.b = 0;
        tc.x0 = tc.y0 = tc.z0 = 0;
        tc.dummy = ti.dummy;
      } else {
        tc = decode_tile(p, tile);
        rc = (p.slice_y ? tc.x0 : tc.y0) + ra;
        z = tc.z0 + zz;
        sc0 = p.slice_y ? tc.y0 : tc.x0;
        yz_ok = rc < (p.slice_y ? p.ox : p.oy) && z < p.oz && !tc.dummy;
        nt0 = tc.nt * p.nt;
      }
      if (++acc == p.acc_stages) acc = 0;
      if (acc == 0) acc_ph ^= 1;
      const int slim = p.slice_y ? p.oy : p.ox;
      // only the tile's slices inside the output are finished (a last tile
      // along the slice axis may hold fewer than bx; 18 = 8 + 8 + 2)
      const int nsv = STREAM ? st_ns : (tc.dummy ? 0 : min(p.bx, slim - sc0));
      const int items = nsv * col_items;
      // (replica offsets are added per item: with taps in N (rep_n) every
      // 16-column item belongs to one tap)
      const long long orow = LEAN ? 0 : tc.b * ov.s[0] + rc * ov.s[ra_dim] + z * ov.s[4];
      const long long brow = LEAN ? 0 : tc.b * bvw.s[0] + rc * bvw.s[ra_dim] + z * bvw.s[4];
      // item column -> (replica, first channel of the item)
      // (z-pair order: rep is the item's dz = 0 tap, its second half is rep + 1
      // at the same channels)
      auto item_rep = [&](int cc, int &rep, int &ch) {
        if (p.zpair) {
          const int rp = cc / (2 * p.rep_n), rem = cc - rp * 2 * p.rep_n;
          rep = 2 * rp;
          ch = (rem >> 4) << 3;
        } else if (p.rep_n) {
          rep = cc / p.rep_n;
          ch = cc - rep * p.rep_n;
        } else {
          rep = tc.rep;
          ch = tc.nt * p.nt + cc;
        }
      };
      const uint32_t tbase =
          tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * acc_stride + p.slice0_col;
      // lean epilogue: this thread's row in slice 0 of the tile (N tile and
      // tile replica included); items add the slice and their LeanEnt offsets
      __nv_bfloat16 *lo_row = nullptr;
      const __nv_bfloat16 *lb_row = nullptr;
      if constexpr (LEAN) {
        lo_row = static_cast<__nv_bfloat16 *>(ov.data) + lo_off;
        if (BASE) lb_row = static_cast<const __nv_bfloat16 *>(bvw.data) + lb_off;
      }

      auto taddr_of = [&](int item) {
        int s, cc;
        split_item(item, s, cc);
        if constexpr (STREAM)   // slice s of this slab: slot (slot0 + s) of the TMEM ring
          return tbase + ((st_slot0 + s) & (p.st_slots - 1)) * p.nt + cc;
        return tbase + s * p.nt + cc;
      };
      // residual operand: bf16 blocked bases are prefetched raw two items
      // ahead (the first ones before the accumulator is even ready); other
      // layouts are read at use
      auto base_issue = [&](int item, uint4 (&d)[2]) {
        if constexpr (LEAN) {
          int s, cc;
          split_item(item, s, cc);
          const LeanEnt &e = ltab[cc >> 4];
          const int c0 = nt0 + e.ch, c1 = p.zpair ? c0 : c0 + 8;
          d[0] = d[1] = make_uint4(0u, 0u, 0u, 0u);
          if (yz_ok && sc0 + s < slim) {
            const __nv_bfloat16 *q = lb_row + s * bvw.s[sl_dim];
            if (p.zpair_v8) {
              if (c0 < p.cout) ld_nc_v8(q + e.b0, d[0], d[1]);
            } else {
              if (c0 < p.cout) d[0] = __ldg(reinterpret_cast<const uint4 *>(q + e.b0));
              if (c1 < p.cout) d[1] = __ldg(reinterpret_cast<const uint4 *>(q + e.b1));
            }
          }
          return;
        }
        int s, cc, rep, ch;
        split_item(item, s, cc);
        item_rep(cc, rep, ch);
        const int x = sc0 + s;
        const bool ok = yz_ok && x < slim;
        const __nv_bfloat16 *bp = static_cast<const __nv_bfloat16 *>(bvw.data) + brow +
                                  p.base_rep_off[rep] + x * bvw.s[sl_dim];
        if (p.zpair) {
          // both halves: the same chunk at dz = 0 and dz = 1 (adjacent rows)
          d[0] = d[1] = make_uint4(0u, 0u, 0u, 0u);
          if (ok && ch < p.cout) {
            const __nv_bfloat16 *q = bp + (ch >> 3) * bvw.s[1];
            if (p.zpair_v8) {
              ld_nc_v8(q, d[0], d[1]);
            } else {
              d[0] = __ldg(reinterpret_cast<const uint4 *>(q));
              d[1] = __ldg(reinterpret_cast<const uint4 *>(q + p.base_rep_off[rep + 1] -
                                                              p.base_rep_off[rep]));
            }
          }
          return;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c0 = ch + h * 8;
          d[h] = make_uint4(0u, 0u, 0u, 0u);
          if (ok && c0 < p.cout) d[h] = __ldg(reinterpret_cast<const uint4 *>(bp + (c0 >> 3) * bvw.s[1]));
        }
      };
      auto base_get = [&](int item, const uint4 (&d)[2], float (&bv)[16]) {
        if (braw) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const __nv_bfloat162 *hv = reinterpret_cast<const __nv_bfloat162 *>(&d[h]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 f = __bfloat1622float2(hv[i]);
              bv[h * 8 + 2 * i] = f.x;
              bv[h * 8 + 2 * i + 1] = f.y;
            }
          }
          return;
        }
        int s, cc, rep, ch;
        split_item(item, s, cc);
        item_rep(cc, rep, ch);
        const int x = sc0 + s;
        const bool ok = yz_ok && x < slim;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float t8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          const int c0 = p.zpair ? ch : ch + h * 8;
          const int rp = p.zpair ? rep + h : rep;
          if (ok && c0 < p.cout)
            load8(bvw, brow + p.base_rep_off[rp] + x * bvw.s[sl_dim] +
                           (bvw.blocked ? (c0 >> 3) * bvw.s[1] : c0 * bvw.s[1]),
                  bvw.blocked, t8);
#pragma unroll
          for (int i = 0; i < 8; ++i) bv[h * 8 + i] = t8[i];
        }
      };
      auto finish = [&](int item, const uint32_t (&rv)[16], const float (&bv)[16]) {
        if constexpr (LEAN) {
          // bias (+ scale . residual), activation, bf16 pack, two 16-byte
          // stores (or one 32-byte store for z-paired deconv taps)
          int s, cc;
          split_item(item, s, cc);
          const LeanEnt &e = ltab[cc >> 4];
          const int c0 = nt0 + e.ch, c1 = p.zpair ? c0 : c0 + 8;
          const int col = nt0 + cc;
          // (packed pairs: FADD2 / FFMA2 / FMUL2 for the bias, the residual and
          // the exponent's scaling -- bit-identical to the scalar forms)
          uint32_t w[8];
          // the per-fmap vectors are read as 16-byte words (all lanes read
          // the same address): every LDS is a shared-memory wavefront that
          // competes with the MMAs' operand reads (C28 1x3x3, 18x768x768:
          // 338 us with eight 8-byte bias reads per item, 297 us with none)
          float4 bq[4], sq[4];
#pragma unroll
          for (int i4 = 0; i4 < 4; ++i4) {
            bq[i4] = (p.dbg_mode & 2048) ? make_float4(p.alpha, p.alpha, p.alpha, p.alpha)
                                         : *reinterpret_cast<const float4 *>(s_bias + col + 4 * i4);
            if (BASE) sq[i4] = *reinterpret_cast<const float4 *>(s_scale + col + 4 * i4);
          }
#pragma unroll
          for (int i2 = 0; i2 < 8; ++i2) {
            const float2 b2 = (i2 & 1) ? make_float2(bq[i2 >> 1].z, bq[i2 >> 1].w)
                                       : make_float2(bq[i2 >> 1].x, bq[i2 >> 1].y);
            float2 r = fadd2(make_float2(__uint_as_float(rv[2 * i2]), __uint_as_float(rv[2 * i2 + 1])),
                             b2);
            if (BASE) {
              const float2 c2 = (i2 & 1) ? make_float2(sq[i2 >> 1].z, sq[i2 >> 1].w)
                                         : make_float2(sq[i2 >> 1].x, sq[i2 >> 1].y);
              r = ffma2(c2, make_float2(bv[2 * i2], bv[2 * i2 + 1]), r);
            }
            if (ACT == VXB_ACT_RELU) {
              r.x = fmaxf(r.x, 0.f);
              r.y = fmaxf(r.y, 0.f);
            } else if (ACT == VXB_ACT_ELU) {
              const float2 t = fmul2(r, make_float2(1.4426950408889634f, 1.4426950408889634f));
              const float ex = ex2_ftz(t.x), ey = ex2_ftz(t.y);
              r.x = r.x > 0.f ? r.x : fmaf(p.alpha, ex, -p.alpha);
              r.y = r.y > 0.f ? r.y : fmaf(p.alpha, ey, -p.alpha);
            }
            __nv_bfloat162 h = __floats2bfloat162_rn(r.x, r.y);
            w[i2] = *reinterpret_cast<uint32_t *>(&h);
          }
          if (p.pool) {
            // MaxPool 1x2x2 / 1x2x2 of the stored values (ops.py:63-86):
            // rows (y, z) (y, z+1) (y+1, z) (y+1, z+1) are lanes l, l+1,
            // l+8, l+9; packed-bf16 max, NaN-propagating like np.maximum
            uint32_t m[8];
#pragma unroll
            // (two steps: z neighbour, then the y neighbour of that maximum:
            // 16 shuffles per item instead of 24; shuffles share the
            // shared-memory crossbar with the MMAs' operand reads)
            for (int i = 0; i < 8; ++i) {
              const uint32_t t1 = __shfl_down_sync(0xffffffffu, w[i], 1);
              __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162 *>(&w[i]);
              a = __hmax2_nan(a, *reinterpret_cast<const __nv_bfloat162 *>(&t1));
              const uint32_t t2 =
                  __shfl_down_sync(0xffffffffu, *reinterpret_cast<uint32_t *>(&a), 8);
              a = __hmax2_nan(a, *reinterpret_cast<const __nv_bfloat162 *>(&t2));
              m[i] = *reinterpret_cast<uint32_t *>(&a);
            }
            if ((lane & 9) == 0 && sc0 + s < slim && !tc.dummy && (rc >> 1) < p.pool_oy &&
                (z >> 1) < p.pool_oz) {
              __nv_bfloat16 *pp = static_cast<__nv_bfloat16 *>(p.pool_out.data) + lp_off +
                                  s * p.pool_out.s[2] + (e.ch >> 3) * p.pool_out.s[1];
              if (c0 < p.cout) *reinterpret_cast<uint4 *>(pp) = make_uint4(m[0], m[1], m[2], m[3]);
              if (c0 + 8 < p.cout)
                *reinterpret_cast<uint4 *>(pp + p.pool_out.s[1]) = make_uint4(m[4], m[5], m[6], m[7]);
            }
          }
          if (yz_ok && sc0 + s < slim) {
            __nv_bfloat16 *o = lo_row + s * ov.s[sl_dim];
            if (p.zpair_v8) {
              if (c0 < p.cout) st_v8(o + e.o0, w);
            } else {
              if (c0 < p.cout)
                *reinterpret_cast<uint4 *>(o + e.o0) = make_uint4(w[0], w[1], w[2], w[3]);
              if (c1 < p.cout)
                *reinterpret_cast<uint4 *>(o + e.o1) = make_uint4(w[4], w[5], w[6], w[7]);
            }
          }
          return;
        }
        int s, cc, rep, ch;
        split_item(item, s, cc);
        item_rep(cc, rep, ch);
        const int x = sc0 + s;
        const bool valid = yz_ok && x < slim;   // stores only; all lanes run the math
        const long long obase0 = orow + p.out_rep_off[rep] + x * ov.s[sl_dim];
        uint32_t zp_w[8];                       // z-pair: both halves, one 32-byte store
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c0 = p.zpair ? ch : ch + h * 8;        // output channel
          const int col = tc.nt * p.nt + cc + h * 8;       // bias / scale column
          const long long obase =
              p.zpair && h ? orow + p.out_rep_off[rep + 1] + x * ov.s[sl_dim] : obase0;
          if (c0 >= p.cout) break;
          const int nvalid = min(8, p.cout - c0);
          const float4 b0 = *reinterpret_cast<const float4 *>(s_bias + col);
          const float4 b1 = *reinterpret_cast<const float4 *>(s_bias + col + 4);
          const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
          float r[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) r[i] = __uint_as_float(rv[h * 8 + i]) + bb[i];
          if (BASE) {
            const float4 s0 = *reinterpret_cast<const float4 *>(s_scale + col);
            const float4 s1 = *reinterpret_cast<const float4 *>(s_scale + col + 4);
            const float sc[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i] = fmaf(sc[i], bv[h * 8 + i], r[i]);
          }
          if (FASTOUT) {
            if (act == VXB_ACT_RELU) {
#pragma unroll
              for (int i = 0; i < 8; ++i) r[i] = fmaxf(r[i], 0.f);
            } else if (act == VXB_ACT_ELU) {
#pragma unroll
              for (int i = 0; i < 8; ++i) r[i] = fast_elu(r[i], p.alpha);
            } else if (act == VXB_ACT_SIGMOID) {
#pragma unroll
              for (int i = 0; i < 8; ++i) r[i] = fast_sigmoid(r[i]);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i] = apply_act(r[i], act, p.alpha);
          }
          // tail lanes (ops.py:18-23 zero_tail): with zero-padded weights,
          // bias 0 and zero base lanes they already hold act(0) = 0 for
          // none / relu / elu; only sigmoid (and the runtime-act variant)
          // must clear them
          if ((ACT < 0 || ACT == VXB_ACT_SIGMOID || !FASTOUT) && nvalid < 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (i >= nvalid) r[i] = 0.f;
          }
          if (POOL) {
            // bf16 blocked output with a fused MaxPool 1x2x2 / 1x2x2
            // (ops.py:63-86) of the stored values: rows (y, z) (y, z+1)
            // (y+1, z) (y+1, z+1) sit in lanes l, l+1, l+8, l+9; the max runs
            // on the packed bf16 pairs (NaN-propagating, like np.maximum)
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              __nv_bfloat162 h2 = __floats2bfloat162_rn(r[2 * i], r[2 * i + 1]);
              w[i] = *reinterpret_cast<uint32_t *>(&h2);
            }
            if (valid)
              *reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(ov.data) + obase +
                                         (c0 >> 3) * ov.s[1]) = make_uint4(w[0], w[1], w[2], w[3]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const uint32_t t1 = __shfl_down_sync(0xffffffffu, w[i], 1);
              const uint32_t t2 = __shfl_down_sync(0xffffffffu, w[i], 8);
              const uint32_t t3 = __shfl_down_sync(0xffffffffu, w[i], 9);
              __nv_bfloat162 m = *reinterpret_cast<const __nv_bfloat162 *>(&w[i]);
              m = __hmax2_nan(m, *reinterpret_cast<const __nv_bfloat162 *>(&t1));
              m = __hmax2_nan(m, *reinterpret_cast<const __nv_bfloat162 *>(&t2));
              m = __hmax2_nan(m, *reinterpret_cast<const __nv_bfloat162 *>(&t3));
              w[i] = *reinterpret_cast<uint32_t *>(&m);
            }
            const int py = rc >> 1, pz = z >> 1;
            if ((lane & 9) == 0 && x < slim && !tc.dummy && py < p.pool_oy && pz < p.pool_oz) {
              const EpiView &pv = p.pool_out;
              *reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(pv.data) + tc.b * pv.s[0] +
                                         x * pv.s[2] + py * pv.s[3] + pz * pv.s[4] +
                                         (c0 >> 3) * pv.s[1]) = make_uint4(w[0], w[1], w[2], w[3]);
            }
          } else if (FASTOUT) {
            if (p.zpair_v8) {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                __nv_bfloat162 h2 = __floats2bfloat162_rn(r[2 * i], r[2 * i + 1]);
                zp_w[4 * h + i] = *reinterpret_cast<uint32_t *>(&h2);
              }
              if (h == 1 && valid)
                st_v8(static_cast<__nv_bfloat16 *>(ov.data) + obase0 + (c0 >> 3) * ov.s[1], zp_w);
            } else if (ov.blocked) {
              if (valid && !(p.dbg_mode & 512)) {
                if (ov.dtype == VXB_BF16X2)
                  store8_split(ov, obase + (c0 >> 3) * ov.s[1], r);
                else
                  store8_bf16_blocked(ov, obase + (c0 >> 3) * ov.s[1], r);
              }
            } else if (valid) {
              // fused unpack: fp32 NCDHW network output written directly
              // (one pointer walked across the channel planes)
              float *op = static_cast<float *>(ov.data) + obase + c0 * ov.s[1];
              const long long cs = ov.s[1];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                if (i < nvalid) *op = r[i];
                op += cs;
              }
            }
          } else if (valid) {
            store8(ov, obase + (ov.blocked ? (c0 >> 3) * ov.s[1] : c0 * ov.s[1]), ov.blocked,
                   nvalid, r);
          }
        }
      };

      if constexpr (HEAD) {
        // Fused 1x1x1 head.  (1) Column items run balanced over the epilogue
        // warps through the plain epilogue's pipeline (TMEM load of the next
        // item and residual loads two items ahead in flight); each item's
        // activated values feed head_cout partial dot products over its 16
        // fmaps (even / odd fmap pairs, FFMA2), written to smem as one float4
        // per row.  (2) After a barrier of the epilogue warps, the warps owning
        // a slice fold its items' partials in column order, add the head bias,
        // activate and store the fp32 network output; a second barrier frees
        // the partials for the next tile.  The activated values are never
        // stored.
        const EpiView &hv = p.head_out;
        float4 *hpart = reinterpret_cast<float4 *>(smem + sm.hpart);   // [slice][item][row]
        auto head_item = [&](int item, const uint32_t (&rv)[16], const float (&bq)[16]) {
          int s_, cc;
          split_item(item, s_, cc);
          const int col = tc.nt * p.nt + cc;
          float2 hs2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                           make_float2(0.f, 0.f)};
#pragma unroll
          for (int i4 = 0; i4 < 4; ++i4) {
            const float4 b4 = *reinterpret_cast<const float4 *>(s_bias + col + 4 * i4);
            float2 r[2] = {fadd2(make_float2(__uint_as_float(rv[4 * i4]), __uint_as_float(rv[4 * i4 + 1])),
                                 make_float2(b4.x, b4.y)),
                           fadd2(make_float2(__uint_as_float(rv[4 * i4 + 2]),
                                             __uint_as_float(rv[4 * i4 + 3])),
                                 make_float2(b4.z, b4.w))};
            if (BASE) {
              const float4 c4 = *reinterpret_cast<const float4 *>(s_scale + col + 4 * i4);
              r[0] = ffma2(make_float2(c4.x, c4.y), make_float2(bq[4 * i4], bq[4 * i4 + 1]), r[0]);
              r[1] = ffma2(make_float2(c4.z, c4.w), make_float2(bq[4 * i4 + 2], bq[4 * i4 + 3]), r[1]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (act == VXB_ACT_RELU) {
                r[h].x = fmaxf(r[h].x, 0.f);
                r[h].y = fmaxf(r[h].y, 0.f);
              } else if (act == VXB_ACT_ELU) {
                const float2 t = fmul2(r[h], make_float2(1.4426950408889634f, 1.4426950408889634f));
                const float ex = ex2_ftz(t.x), ey = ex2_ftz(t.y);
                r[h].x = r[h].x > 0.f ? r[h].x : fmaf(p.alpha, ex, -p.alpha);
                r[h].y = r[h].y > 0.f ? r[h].y : fmaf(p.alpha, ey, -p.alpha);
              } else if (act == VXB_ACT_SIGMOID) {
                r[h].x = fast_sigmoid(r[h].x);
                r[h].y = fast_sigmoid(r[h].y);
              }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 hw = *reinterpret_cast<const float4 *>(s_head + j * cpad + col + 4 * i4);
              hs2[j] = ffma2(r[0], make_float2(hw.x, hw.y), hs2[j]);
              hs2[j] = ffma2(r[1], make_float2(hw.z, hw.w), hs2[j]);
            }
          }
          hpart[item * 128 + row] = make_float4(hs2[0].x + hs2[0].y, hs2[1].x + hs2[1].y,
                                                hs2[2].x + hs2[2].y, hs2[3].x + hs2[3].y);
        };
        // (computing only head_cout <= 3 rows, selected per item, measured
        // slower: 1.64-1.67 vs 1.58 ms per 36 patches)
        uint32_t ra[16], rb[16];
        uint4 qa[2], qb[2];
        float bq[16];
        int item = sub;
        if (braw) {
          if (item < items) base_issue(item, qa);
          if (item + NSUB < items) base_issue(item + NSUB, qb);
        }
        mbar_wait_sleep(&t_full[acc], static_cast<uint32_t>(acc_ph));
        tc_fence_after();
        if (item < items) tmem_ld16_issue(taddr_of(item), ra);
        while (item < items) {
          const int nxt = item + NSUB;
          tmem_wait_ld16(ra);
          if (nxt < items) tmem_ld16_issue(taddr_of(nxt), rb);
          if (BASE) base_get(item, qa, bq);
          head_item(item, ra, bq);
          if (braw && item + 2 * NSUB < items) base_issue(item + 2 * NSUB, qa);
          if (nxt >= items) break;
          const int nn = nxt + NSUB;
          tmem_wait_ld16(rb);
          if (nn < items) tmem_ld16_issue(taddr_of(nn), ra);
          if (BASE) base_get(nxt, qb, bq);
          head_item(nxt, rb, bq);
          if (braw && nxt + 2 * NSUB < items) base_issue(nxt + 2 * NSUB, qb);
          item = nn;
        }
        // the accumulator stage is free for the next tile's MMAs
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_empty[acc]);
        named_bar_sync(1, EPI_WARPS * 32);
        for (int s_ = sub; s_ < nsv; s_ += NSUB) {
          float hsum[4] = {0.f, 0.f, 0.f, 0.f};
          for (int c_ = 0; c_ < col_items; ++c_) {
            const float4 v = hpart[(s_ * col_items + c_) * 128 + row];
            hsum[0] += v.x;
            hsum[1] += v.y;
            hsum[2] += v.z;
            hsum[3] += v.w;
          }
          const int x = sc0 + s_;
          if (yz_ok && x < slim) {
            float *op = static_cast<float *>(hv.data) + tc.b * hv.s[0] + rc * hv.s[ra_dim] +
                        z * hv.s[4] + x * hv.s[sl_dim];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < p.head_cout)
                op[j * hv.s[1]] = p.head_act == VXB_ACT_SIGMOID
                                      ? fast_sigmoid(hsum[j] + p.head_b[j])   // ~1e-7 absolute
                                      : apply_act(hsum[j] + p.head_b[j], p.head_act, p.head_alpha);
          }
        }
        named_bar_sync(1, EPI_WARPS * 32);   // partials free for the next tile
        continue;
      }
      uint32_t ra[16], rb[16];
      uint4 qa[2], qb[2];
      float bv[16];
      int item = (p.dbg_mode & 1) ? items : sub;
      if (braw) {
        if (item < items) base_issue(item, qa);
        if (item + NSUB < items) base_issue(item + NSUB, qb);
      }
      mbar_wait_sleep(&t_full[acc], static_cast<uint32_t>(acc_ph));
      if (warp == 3 && lane == 0) dbg_mark(p, it, 3);
      tc_fence_after();
      if (item < items) tmem_ld16_issue(taddr_of(item), ra);
      while (item < items) {
        const int nxt = item + NSUB;
        tmem_wait_ld16(ra);
        if constexpr (STREAM) tmem_st16_zero(taddr_of(item));
        if (warp == 3 && lane == 0 && item == sub) dbg_mark(p, it, 7);
        if (nxt < items) tmem_ld16_issue(taddr_of(nxt), rb);
        if (BASE) base_get(item, qa, bv);
        if (!(p.dbg_mode & 256)) finish(item, ra, bv);
        if (braw && item + 2 * NSUB < items) base_issue(item + 2 * NSUB, qa);
        if (nxt >= items) break;
        const int nn = nxt + NSUB;
        tmem_wait_ld16(rb);
        if constexpr (STREAM) tmem_st16_zero(taddr_of(nxt));
        if (nn < items) tmem_ld16_issue(taddr_of(nn), ra);
        if (BASE) base_get(nxt, qb, bv);
        if (!(p.dbg_mode & 256)) finish(nxt, rb, bv);
        if (braw && nxt + 2 * NSUB < items) base_issue(nxt + 2 * NSUB, qb);
        item = nn;
      }
      if constexpr (STREAM) tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR)
          mbar_arrive_cta(&t_empty[acc], 0);   // the leader's MMA waits for both CTAs
        else
          mbar_arrive(&t_empty[acc]);
      }
      if (warp == 3 && lane == 0) dbg_mark(p, it, 4);
    }
  }

  __syncthreads();
  if (threadIdx.x == 0) dbg_mark(p, 0, 6);
  if (p.cluster == 2) cluster_sync_all();   // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    if (PAIR)
      tmem_dealloc_pair(tmem_base, tmem_cols);
    else
      tmem_dealloc(tmem_base, tmem_cols);
  }
}

// ---------------------------------------------------------------- host side

size_t tc_smem_bytes(const TcParams &p) {
  return smem_map(p).bars +
         (2 * p.na + 2 * p.nb_stages + 2 * MAX_ACC + 2 * p.n_stg + (p.lean ? TINFO : 0)) *
             sizeof(uint64_t) +
         16;
}

template <int ACT, bool FASTOUT, bool BASE, bool PAIR, bool F32IN = false, bool POOL = false,
          bool HEAD = false, bool LEAN = false, bool STREAM = false>
static int launch_variant(const TcParams &p, const TcMaps &maps, int grid, cudaStream_t stream,
                          size_t smem) {
  auto kern = conv3d_tc_kernel<ACT, FASTOUT, BASE, PAIR, F32IN, POOL, HEAD, LEAN, STREAM>;
  if (int rc = ensure_smem_attr(kern, 232448, "cudaFuncSetAttribute(conv3d_tc)")) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tc_threads(F32IN));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[3];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  attr[na].id = cudaLaunchAttributePriority;
  attr[na].val.priority = launch_priority(false);
  ++na;
  if (p.cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = p.cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return check_cuda(cudaLaunchKernelEx(&cfg, kern, p, maps), "conv3d_tc_kernel launch");
}

template <bool PAIR>
static int launch_f32in(const TcParams &p, const TcMaps &maps, int grid, cudaStream_t s,
                        size_t smem) {
  switch (p.act) {
    case VXB_ACT_RELU:
      return launch_variant<VXB_ACT_RELU, true, false, PAIR, true>(p, maps, grid, s, smem);
    case VXB_ACT_ELU:
      return launch_variant<VXB_ACT_ELU, true, false, PAIR, true>(p, maps, grid, s, smem);
    case VXB_ACT_SIGMOID:
      return launch_variant<VXB_ACT_SIGMOID, true, false, PAIR, true>(p, maps, grid, s, smem);
    default: return launch_variant<VXB_ACT_NONE, true, false, PAIR, true>(p, maps, grid, s, smem);
  }
}

template <bool BASE, bool PAIR>
static int launch_act(const TcParams &p, const TcMaps &maps, int grid, cudaStream_t s,
                      size_t smem) {
  const bool fast = ((p.out.dtype == VXB_BF16 || p.out.dtype == VXB_BF16X2) && p.out.blocked) ||
                    (p.out.dtype == VXB_F32 && !p.out.blocked);
  if (p.head_cout > 0) {
    if (PAIR || p.f32in || p.pool || p.rep_n || p.reps != 1 || p.n_tiles != 1)
      return set_error(VXB_EUNSUPPORTED,
                       "fused head: single-CTA tiles, one N tile, no fp32 input / pooling");
    // (the activation of the producing conv is compile-time for ELU / ReLU:
    // a runtime selection sits inside the head's innermost loops)
    switch (p.act) {
      case VXB_ACT_ELU:
        return launch_variant<VXB_ACT_ELU, true, BASE, false, false, false, true>(p, maps, grid, s,
                                                                                  smem);
      case VXB_ACT_RELU:
        return launch_variant<VXB_ACT_RELU, true, BASE, false, false, false, true>(p, maps, grid, s,
                                                                                   smem);
      default:
        return launch_variant<-1, true, BASE, false, false, false, true>(p, maps, grid, s, smem);
    }
  }
  if (p.pool && !p.lean) {
    if (PAIR || p.f32in || p.out.dtype != VXB_BF16 || !p.out.blocked ||
        p.pool_out.dtype != VXB_BF16 || !p.pool_out.blocked)
      return set_error(VXB_EUNSUPPORTED,
                       "fused pooling: bf16 blocked output and pool view, single-CTA tiles");
    // activation at run time: two instances (with / without residual) only
    return launch_variant<-1, true, BASE, false, false, true>(p, maps, grid, s, smem);
  }
  if (p.f32in) {
    if (BASE || !fast)
      return set_error(VXB_EUNSUPPORTED,
                       "fp32-input conv: no residual operand, output bf16 blocked or fp32 NCDHW");
    return launch_f32in<PAIR>(p, maps, grid, s, smem);
  }
  if (!fast) {
    if (PAIR) return set_error(VXB_EUNSUPPORTED, "pair mode needs a blocked bf16 output");
    return launch_variant<-1, false, BASE, false>(p, maps, grid, s, smem);
  }
  if (p.lean && p.stream) {
    if (PAIR) return set_error(VXB_EUNSUPPORTED, "streamed fold: single-CTA tiles");
    switch (p.act) {
      case VXB_ACT_RELU:
        return launch_variant<VXB_ACT_RELU, true, BASE, false, false, false, false, true, true>(
            p, maps, grid, s, smem);
      case VXB_ACT_ELU:
        return launch_variant<VXB_ACT_ELU, true, BASE, false, false, false, false, true, true>(
            p, maps, grid, s, smem);
      default:
        return launch_variant<VXB_ACT_NONE, true, BASE, false, false, false, false, true, true>(
            p, maps, grid, s, smem);
    }
  }
  if (p.lean) {
    // bf16 blocked output (and residual): the lean epilogue (tc_lean_ok)
    switch (p.act) {
      case VXB_ACT_RELU:
        return launch_variant<VXB_ACT_RELU, true, BASE, PAIR, false, false, false, true>(p, maps,
                                                                                          grid, s,
                                                                                          smem);
      case VXB_ACT_ELU:
        return launch_variant<VXB_ACT_ELU, true, BASE, PAIR, false, false, false, true>(p, maps,
                                                                                         grid, s,
                                                                                         smem);
      default:
        return launch_variant<VXB_ACT_NONE, true, BASE, PAIR, false, false, false, true>(p, maps,
                                                                                          grid, s,
                                                                                          smem);
    }
  }
  switch (p.act) {
    case VXB_ACT_RELU:
      return launch_variant<VXB_ACT_RELU, true, BASE, PAIR>(p, maps, grid, s, smem);
    case VXB_ACT_ELU: return launch_variant<VXB_ACT_ELU, true, BASE, PAIR>(p, maps, grid, s, smem);
    case VXB_ACT_SIGMOID:
      return launch_variant<VXB_ACT_SIGMOID, true, BASE, PAIR>(p, maps, grid, s, smem);
    default: return launch_variant<VXB_ACT_NONE, true, BASE, PAIR>(p, maps, grid, s, smem);
  }
}

int launch_conv3d_tc(const TcParams &p, const TcMaps &maps, int grid, cudaStream_t stream) {
  const size_t smem = tc_smem_bytes(p);
  if (p.pair)
    return p.has_base ? launch_act<true, true>(p, maps, grid, stream, smem)
                      : launch_act<false, true>(p, maps, grid, stream, smem);
  return p.has_base ? launch_act<true, false>(p, maps, grid, stream, smem)
                    : launch_act<false, false>(p, maps, grid, stream, smem);
}

}  // namespace vxb
