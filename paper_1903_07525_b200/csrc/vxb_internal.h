// vxb_internal.h — host/device shared parameter blocks and helpers.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../include/vxb.h"

namespace vxb {

constexpr int LANES = 8;          // fmaps per chunk (blocked.py DEFAULT_SIMD_WIDTH)
constexpr int TILE_Y = 16;        // output tile rows along y per 128-row MMA
constexpr int TILE_Z = 8;         // output tile along z (one 8-row core-matrix group)
constexpr int SLAB_ROW_BYTES = 32;  // one B row: 16 bf16 of K
constexpr int MAX_REPS = 8;
// TMEM accumulator stages: tiles whose MMAs may run ahead of the epilogue
// (as many as fit in the 512 TMEM columns, see tc_configure)
constexpr int MAX_ACC = 6;

// Epilogue view of an output / base tensor, element strides.
struct EpiView {
  void *data;
  long long s[5];   // batch, chunk (or channel when !blocked), x, y, z
  int dtype;        // VXB_BF16 / VXB_F32
  int blocked;
};

// Parameters of the tcgen05 implicit-GEMM convolution kernel.
struct TcParams {
  int nb;                      // batch
  int ox, oy, oz;              // output extents
  int tiles_x, tiles_y, tiles_z;
  int n_tiles, reps, total_tiles;
  // fast division of tile indices: q = (t * m) >> 40 with m = ceil(2^40 / d)
  // for d = spatial_pad, tiles_z, tiles_y, tiles_x, nb, n_tiles (exact while
  // t * d < 2^40, checked on the host); replaces six runtime integer
  // divisions per tile in every epilogue warp
  unsigned long long dm[6];
  int spatial_real, spatial_pad;  // tiles per (rep, ntile); padded to the cluster size
  int cluster;                    // 1, or 2 = CTA pair sharing B via TMA multicast
  int pair;                       // cta_group::2 MMA (M = 256), each CTA holds half of B
  int bx;                      // slices per CTA tile (each slice = 128 MMA rows)
  int nt;                      // N per tile (multiple of 16)
  // Slice axis: slices run along x (rows = 16 y x 8 z) or, with slice_y,
  // along y (rows = 16 x x 8 z).  fold: the 3 taps along the slice axis are
  // folded into N (one MMA per input slice covers up to 3 output slices).
  int slice_y, fold;
  int ex, ey;                  // tile extents along x and y
  int slab_bytes;              // B bytes per K step (nt rows, or 3*nt when folded)
  int a_slice_inc, a_sbo;      // smem bytes between slices / between 8-row groups
  // fp32 NCDHW input converted in the kernel (no separate pack): TMA boxes of
  // (hzb z, hy y, 1 x, 8 c) fp32 land in a staging ring, converter warps write
  // the bf16 chunk rows of the A stage
  int f32in, stg_bytes, n_stg, hzb;
  int f32in_cstride;           // channel-coordinate distance between batches
  int f32in_zshift;            // box z start is rounded down to 16 B: rows start this far in
  int f32in_xb;                // halo x-slices per staging box
  int acc_stages;              // TMEM accumulator stages
  // TMEM columns between accumulator stages, and from a stage's base to its
  // slice 0.  Folded CTA-pair tiles (fold && pair) issue every MMA at N = 3nt,
  // so input slices 0 and bx+1 also write the two slices before / after the
  // tile: stage s spans slices -2..bx+1 and neighbouring stages share their
  // 2nt-column scratch band (stride (bx+2)nt, slice 0 at +2nt).
  int acc_stride, slice0_col, tmem_cols;
  // Streamed fold (folded x taps, single CTA, resident weights, lean
  // epilogue): a CTA walks whole columns (all x of one 16 y x 8 z block) slab
  // by slab; the accumulators of the column's output slices live in a ring
  // of st_slots TMEM slices, input slice j writes output slices j-2..j
  // wherever they fall in the ring, so there are no per-tile fold edges and
  // no x halo re-reads.  Input slices st_j0 .. st_j0 + st_nin - 1 (halo
  // coordinates) can be non-zero; slab t holds bx of them.
  int stream, st_j0, st_nin, st_nslab, st_slots, st_ncols;
  int st_nphase;   // ring phases: column k starts at slot (k * ox) mod st_slots, period st_nphase
  int kx, ky, kz;
  int hx, hy, hz;              // halo tile extents
  int pad[3];
  // input segments (fused concat): chunk counts, crop offsets, batch chunk stride
  int seg_chunks[2];
  int seg_off[2][3];
  int seg_bstride[2];          // chunk-index stride between batches in the TMA map
  int n_groups;
  int chunk_bytes;             // bytes of one TMA'd chunk array (hx*hy*hz*16)
  int chunk_stride;            // smem distance between the two chunk arrays of a stage
  int chunk_slots;             // chunk arrays per A stage (1 or 2)
  int a_stage_bytes, b_stage_bytes;
  int na, nb_stages;           // ring depths
  int bsteps;                  // K steps per B stage
  int resident;                // weights loaded once, kept in smem
  const uint8_t *w;
  long long w_ntile_stride, w_rep_stride;   // bytes
  int w_steps;                 // K steps per (rep, ntile)
  const float *bias, *scale;
  EpiView out, base;
  long long out_rep_off[MAX_REPS], base_rep_off[MAX_REPS];
  int rep_n;                   // deconv taps in N: columns per tap (0 = taps are tile replicas)
  int zpair;                   // taps in N with z-stride 2: the dz = 0 / 1 taps of each 8-fmap
                               // chunk are adjacent 8-column halves of one 16-column item
                               // (their output rows are adjacent: one 32-byte store)
  int zpair_v8;                // zpair outputs (and residuals) moved as 32-byte accesses
  int lean;                    // lean epilogue: bf16 blocked output, bf16 blocked residual if
                               // any, act none / relu / elu, no pooling / head / fp32 input
  int cout, act;
  float alpha;
  int has_base;
  // fused 1x2x2 max pool of the stored output (VXB_POOL_FUSED_MAX122)
  int pool, pool_oy, pool_oz;
  EpiView pool_out;
  // fused 1x1x1 head (vxb_conv_desc.head_*): head_out = act(head_b + head_w . y)
  const float *head_w, *head_b;
  int head_cout, head_act;
  float head_alpha;
  EpiView head_out;
  unsigned long long *dbg;     // optional per-tile phase timestamps (VXB_TC_DEBUG)
  int dbg_mode;                // VXB_TC_DBGMODE (timing experiments, wrong results): 1 no
                               // epilogue, 2 no A loads, 4 no B loads, 8 no MMAs (resident B),
                               // 16 folded MMAs at N = nt, 64 no fp32 conversion, 128 no fp32
                               // TMA, 256 epilogue TMEM loads only, 512 no bf16 output stores,
                               // 2048 lean epilogue without its bias smem reads, 4096 streamed
                               // fold keeps the first slab's operand table
};

struct TcMaps {
  CUtensorMap m[2];
  CUtensorMap w;   // packed weights (pair mode): (128 B, nt/8, half, step)
};


// ---- CUDA-core kernels (ops.cu)
struct DView {
  void *data;
  long long s[5];
  int dtype, blocked;
  int n, c, x, y, z;
};

struct DirectParams {
  DView in, out, base;
  const float *w, *bias, *scale;
  int cin, cout, kx, ky, kz, sx, sy, sz, px, py, pz;
  int act, has_base;
  float alpha;
  int tiles_x, tiles_y, tiles_z;
  int hx, hy, hz;  // staged input patch extents
};

struct SubParams {
  DView in, out, base;
  const float *w, *bias, *scale;  // w: standard (cout, cin, kx, ky, kz)
  int cin, cout, kx, ky, kz, sx, sy, sz;
  int ib, ob, x0, y0, z0, ex, ey, ez, first, last, act, has_base;
  float alpha;
};

struct GatherDeconvParams {
  DView in, out, base;
  const float *w, *bias, *scale;  // standard (cout, cin, kx, ky, kz)
  int cin, cout, kx, ky, kz, sx, sy, sz, act, has_base;
  float alpha;
};

int launch_copy(const DView &src, const DView &dst, cudaStream_t s, bool independent = false);
// batched window copies (fp32, z contiguous): up to WIN_MAX (src, dst) pairs
// of equal extents in one launch (DeviceTiler's patch gather / scatter)
constexpr int WIN_MAX = 16;
struct WinCopy {
  const float *src;
  float *dst;
  long long ss[4], ds[4];   // n, c, x, y strides (elements); z stride is 1
  int ext[5];               // n, c, x, y, z
  int vec4;                 // z extent, pointers and strides allow float4 moves
};
struct WinBatch {
  WinCopy w[WIN_MAX];
  int count;
};
int launch_copy_windows(const WinBatch &b, cudaStream_t s);
// z-window pack reading one window per batch entry (element offsets into a
// source volume that shares the view's strides)
constexpr int ZWIN_MAX = 64;
struct ZwinWindows {
  long long off[ZWIN_MAX];
};
int launch_pack_zwin_windows(const DView &src, const ZwinWindows &w, const DView &dst, int kz,
                             int pz, cudaStream_t s);
int launch_pack_zwin(const DView &src, const DView &dst, int kz, int pz, cudaStream_t s,
                     bool independent);
int launch_zero(const DView &dst, cudaStream_t s);
int launch_pool(const DView &in, const DView &out, const int *w, const int *st, int mode,
                cudaStream_t s);
int launch_eltwise(const DView &a, const DView &b, const DView &out, int op, cudaStream_t s);
int launch_affine_act(const DView &in, const DView &out, const float *m, const float *a, int act,
                      float alpha, cudaStream_t s);
int launch_mergecrop(const DView &a, const DView &b, const DView &out, const int *oa,
                     const int *ob, cudaStream_t s);
int launch_pad_copy(const DView &in, const DView &out, const int *pads, cudaStream_t s);
int launch_conv_direct(DirectParams p, cudaStream_t s);
int launch_subimage(const SubParams &p, cudaStream_t s);
int launch_deconv_gather(const GatherDeconvParams &p, cudaStream_t s);

// ---- tensor-core conv (conv3d_tc.cu)
size_t tc_smem_bytes(const TcParams &p);
int launch_conv3d_tc(const TcParams &p, const TcMaps &maps, int grid, cudaStream_t stream);
constexpr int DCO_DIRECT = 16;  // output fmaps per direct-conv CTA

// status helpers (vxb_abi.cu)
int set_error(int code, const char *fmt, ...);
int check_cuda(cudaError_t e, const char *what);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-device setting:
// done once per (kernel, device), thread-safe (run_tiled drives several GPUs
// from one thread each).  Keyed by the kernel's address: every instantiation
// of a template kernel is its own function.
bool smem_attr_done(const void *kern, int dev);   // vxb_abi.cu
void smem_attr_mark(const void *kern, int dev);
template <typename... KArgs>
int ensure_smem_attr(void (*kern)(KArgs...), int bytes, const char *what) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return check_cuda(e, what);
  const void *k = reinterpret_cast<const void *>(kern);
  if (smem_attr_done(k, dev)) return 0;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return check_cuda(e, what);
  smem_attr_mark(k, dev);
  return 0;
}

// ---- programmatic dependent launch (PDL)
// Every vxb kernel is launched with programmatic stream serialization: it
// may start while its predecessor drains, signals its own dependents at
// entry, and waits for the predecessor's completion (griddepcontrol.wait)
// before touching activations.  The conv kernel does its setup (barriers,
// TMEM, bias/scale staging) before the wait, overlapping the previous
// kernel's tail.  VXB_PDL=0 launches plainly (the wait is then a no-op).
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_begin() {
  pdl_trigger();
  pdl_wait();
}
#endif
bool pdl_enabled();

// Launch priority: every kernel runs at the device's highest priority except
// background work (independent network-input packs, PlanBatch), which runs at
// the lowest, so its CTAs only take SM slots the convolutions leave free.
int launch_priority(bool background);

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_prio(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t stream, bool background, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  attr[na].id = cudaLaunchAttributePriority;
  attr[na].val.priority = launch_priority(background);
  ++na;
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<Args &&>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args &&...args) {
  return launch_pdl_prio(kern, grid, block, smem, stream, false, static_cast<Args &&>(args)...);
}

}  // namespace vxb
