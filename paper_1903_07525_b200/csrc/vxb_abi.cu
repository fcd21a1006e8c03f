// vxb_abi.cu — the extern "C" boundary (include/vxb.h): validation, path
// selection, host-side weight packing, TMA descriptor encoding, launches.
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>
#include "vxb_internal.h"

namespace vxb {

static thread_local std::string g_last_error;

int set_error(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_cuda(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return VXB_OK;
  return set_error(VXB_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

static inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
static inline int round_up(int a, int b) { return ceil_div(a, b) * b; }

static int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

// programmatic dependent launch: VXB_PDL (default on), overridden per host
// thread by vxb_set_pdl (a runner captures its graph with its own setting)
static thread_local int t_pdl_override = -1;
bool pdl_enabled() {
  if (t_pdl_override >= 0) return t_pdl_override != 0;
  return env_int("VXB_PDL", 1) != 0;
}
int set_pdl_override(int mode) {
  const int prev = t_pdl_override;
  t_pdl_override = mode < 0 ? -1 : (mode ? 1 : 0);
  return prev;
}

static std::mutex g_attr_mu;
static std::set<std::pair<const void *, int>> g_attr_done;
bool smem_attr_done(const void *kern, int dev) {
  std::lock_guard<std::mutex> g(g_attr_mu);
  return g_attr_done.count({kern, dev}) != 0;
}
void smem_attr_mark(const void *kern, int dev) {
  std::lock_guard<std::mutex> g(g_attr_mu);
  g_attr_done.insert({kern, dev});
}
int launch_priority(bool background) {
  static int lo = 0, hi = 0, init = 0;
  if (!init) {
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) lo = hi = 0;
    if (!env_int("VXB_PRIORITIES", 1)) lo = hi = 0;
    init = 1;
  }
  return background ? lo : hi;
}

static DView to_dview(const vxb_tensor &t) {
  DView v;
  v.data = t.data;
  for (int i = 0; i < 5; ++i) v.s[i] = t.s[i];
  v.dtype = t.dtype;
  v.blocked = t.blocked;
  v.n = t.n;
  v.c = t.c;
  v.x = t.x;
  v.y = t.y;
  v.z = t.z;
  return v;
}

static EpiView to_epi(const vxb_tensor &t) {
  EpiView v;
  v.data = t.data;
  for (int i = 0; i < 5; ++i) v.s[i] = t.s[i];
  v.dtype = t.dtype;
  v.blocked = t.blocked;
  return v;
}

static int check_view(const vxb_tensor *t, const char *what) {
  if (!t || !t->data) return set_error(VXB_EINVAL, "%s: null tensor", what);
  if (t->dtype != VXB_BF16 && t->dtype != VXB_F32 && t->dtype != VXB_BF16X2)
    return set_error(VXB_EINVAL, "%s: bad dtype %d", what, t->dtype);
  if (t->dtype == VXB_BF16X2 && (!t->blocked || t->s[1] % 16 != 0))
    return set_error(VXB_EINVAL,
                     "%s: split bf16 views are blocked with the lo plane at s[1]/2 (s[1] %% 16 == 0)",
                     what);
  if (t->n < 1 || t->c < 1 || t->x < 1 || t->y < 1 || t->z < 1)
    return set_error(VXB_EINVAL, "%s: non-positive extent (%d,%d,%d,%d,%d)", what, t->n, t->c,
                     t->x, t->y, t->z);
  if (t->blocked) {
    size_t esz = t->dtype == VXB_F32 ? 4 : 2;
    uintptr_t a = reinterpret_cast<uintptr_t>(t->data);
    if (a % (8 * esz) != 0)
      return set_error(VXB_EINVAL, "%s: blocked view base must be %zu-byte aligned", what, 8 * esz);
    for (int i = 0; i < 5; ++i)
      if (t->s[i] % 8 != 0)
        return set_error(VXB_EINVAL, "%s: blocked view strides must be multiples of 8", what);
  }
  return VXB_OK;
}

static cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// A split (VXB_BF16X2) input as the two bf16 K segments the tensor-core conv
// reads: `both` = every chunk's hi and lo planes as 2*CB chunks of 8 lanes
// (hi_0, lo_0, hi_1, lo_1, ...), `hi` = the CB hi planes alone.  Weights
// packed with VXB_PREC_X3 multiply them by bf16(W) and bf16(W - bf16(W)).
static void split_segments(const vxb_tensor &t, vxb_tensor &both, vxb_tensor &hi) {
  const int cb = (t.c + 7) / 8;
  both = t;
  both.dtype = VXB_BF16;
  both.c = 16 * cb;
  both.s[1] = t.s[1] / 2;
  hi = t;
  hi.dtype = VXB_BF16;
  hi.c = 8 * cb;
}

// ------------------------------------------------------------------ TC geometry

struct TcGroup {
  int seg, chunk0, nch, steps;
};

struct TcLayout {
  int npad, n_tiles, nt;
  int fold;         // 0, 1 = x taps folded into N (slices along x), 2 = y taps (slices along y)
  int slab;         // B bytes per device K step
  int seg_chunks[2];
  std::vector<TcGroup> groups;
  long long steps;  // device K steps per (rep, ntile)
};

// Tap folding (conv3d_tc.cu mma_group_fold): with 3 taps along the slice axis
// and 3*nt <= 256, one MMA per input slice serves up to 3 output slices.
// 3x3x3 folds x (slices along x); 1x3x3 folds y (slices along y).
static int tc_fold_axis(int nt, const int k[3]) {
  if (env_int("VXB_TC_FOLD", 1) == 0 || 3 * nt > 256) return 0;
  if (k[0] == 3) return 1;
  if (k[0] == 1 && k[1] == 3) return 2;
  return 0;
}

static bool is_tc(int path) {
  return path == VXB_PATH_TC || path == VXB_PATH_TC_UNFOLDED ||
         (path >= VXB_PATH_TC_N128 && path <= VXB_PATH_TC_N16);
}
static bool path_folds(int path) { return path != VXB_PATH_TC_UNFOLDED; }
static int path_nt_cap(int path) {
  switch (path) {
    case VXB_PATH_TC_N128: return 128;
    case VXB_PATH_TC_N64: return 64;
    case VXB_PATH_TC_N32: return 32;
    case VXB_PATH_TC_N16: return 16;
    default: return 256;
  }
}

static TcLayout tc_layout(int cin0, int cin1, int cout, const int k[3], bool allow_fold = true,
                          int nt_cap = 256) {
  TcLayout L;
  L.npad = round_up(cout, 16);
  L.n_tiles = ceil_div(L.npad, nt_cap);
  L.nt = round_up(ceil_div(L.npad, L.n_tiles), 16);
  L.fold = allow_fold ? tc_fold_axis(L.nt, k) : 0;
  L.slab = (L.fold ? 3 : 1) * L.nt * SLAB_ROW_BYTES;
  L.seg_chunks[0] = ceil_div(cin0, 8);
  L.seg_chunks[1] = cin1 > 0 ? ceil_div(cin1, 8) : 0;
  L.steps = 0;
  for (int seg = 0; seg < 2; ++seg) {
    int c = L.seg_chunks[seg];
    for (int j = 0; 2 * j < c; ++j) {
      TcGroup g;
      g.seg = seg;
      g.chunk0 = 2 * j;
      g.nch = std::min(2, c - 2 * j);
      g.steps = g.nch == 2 ? k[0] * k[1] * k[2] : k[0] * k[1] * ceil_div(k[2], 2);
      if (L.fold) g.steps /= 3;
      L.groups.push_back(g);
      L.steps += g.steps;
    }
  }
  return L;
}

static size_t tc_bytes_per_rep(const TcLayout &L) {
  return static_cast<size_t>(L.n_tiles) * L.steps * L.slab;
}

static inline uint16_t f32_to_bf16_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) {  // inf / nan
    uint16_t h = static_cast<uint16_t>(u >> 16);
    if (u & 0x007fffffu) h |= 0x40;
    return h;
  }
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return static_cast<uint16_t>(u >> 16);
}

// Pack w (cout, cin, kx, ky, kz) fp32 into per-step UMMA B slabs, bf16.
// wtap(co, ci, dx, dy, dz) gives the weight; deconv reuses this with k=1.
template <class WFn>
static void tc_pack(const TcLayout &L, int cin0, int cin1, int cout, const int k[3], WFn wtap,
                    uint8_t *dst) {
  const int slab = L.slab;
  const int kzh = ceil_div(k[2], 2);
  for (int nti = 0; nti < L.n_tiles; ++nti) {
    long long step_base = static_cast<long long>(nti) * L.steps;
    for (const TcGroup &g : L.groups) {
      const int cin_seg = g.seg == 0 ? cin0 : cin1;
      const int cbase = g.seg == 0 ? 0 : cin0;
      const int taps = g.steps * (L.fold ? 3 : 1);
      for (int t = 0; t < taps; ++t) {
        int dx, dy, dz;
        if (g.nch == 2) {
          dz = t % k[2];
          dy = (t / k[2]) % k[1];
          dx = t / (k[2] * k[1]);
        } else {
          dz = 2 * (t % kzh);
          dy = (t / kzh) % k[1];
          dx = t / (kzh * k[1]);
        }
        // device step and N block of this tap (unfolded: the tap order itself)
        const int tzn = g.nch == 2 ? k[2] : kzh, tzi = g.nch == 2 ? dz : dz / 2;
        int step = t, blk = 0;
        if (L.fold == 1) {
          step = dy * tzn + tzi;
          blk = 2 - dx;
        } else if (L.fold == 2) {
          step = dx * tzn + tzi;
          blk = 2 - dy;
        }
        uint16_t *s = reinterpret_cast<uint16_t *>(dst + (step_base + step) * slab) +
                      blk * L.nt * SLAB_ROW_BYTES / 2;
        for (int n = 0; n < L.nt; ++n) {
          const int co = nti * L.nt + n;
          for (int kk = 0; kk < 16; ++kk) {
            const int h = kk >> 3, l = kk & 7;
            int chunk = g.chunk0, tz = dz;
            if (g.nch == 2)
              chunk += h;
            else
              tz += h;
            const int cl = chunk * 8 + l;
            float v = 0.f;
            if (co < cout && cl < cin_seg && tz < k[2]) v = wtap(co, cbase + cl, dx, dy, tz);
            const size_t byte = static_cast<size_t>(n >> 3) * 256 + h * 128 + (n & 7) * 16 + l * 2;
            s[byte / 2] = f32_to_bf16_bits(v);
          }
        }
      }
      step_base += g.steps;
    }
  }
}

struct TcConfig {
  int bx, acc, na, nb, bsteps, resident, chunk_bytes, chunk_stride, chunk_slots, a_stage,
      b_stage;
  int pair;   // cta_group::2 tiles (each CTA holds half of every B stage)
  size_t smem;
};

// other_tiles: tiles over the non-slice axes x batch x N tiles x reps.
static const int kTileOverhead = 3;

// TMEM columns of the accumulator stages (see TcParams::acc_stride)
static int tc_tmem_cols(int bx, int nt, int acc, bool fold_pair) {
  return fold_pair ? acc * (bx + 2) * nt + 2 * nt : acc * bx * nt;
}

// can_pair: the conv may run as CTA pairs (pair_mode 1: always, 2: only with
// streamed weights); fold_pair: it is a folded conv that pairs (TMEM layout)
static int tc_configure(const TcLayout &L, const int k[3], int slice_extent, long long other_tiles,
                        int sms, int reps, int reserved, bool f32in, bool can_pair,
                        int pair_mode, bool fold_pair, TcConfig &c, int reserved_per_slice = 0,
                        int stream_bx = 0) {
  // room for bias/scale/barriers, plus the fp32-input staging ring if any
  // (and per-slice epilogue scratch: the fused head's partials)
  const int budget0 = 227 * 1024 - 6144 - reserved;
  c.acc = env_int("VXB_TC_ACC", 2);
  if (c.acc != 1 && c.acc != 2) c.acc = 2;
  int bx_cap = env_int("VXB_TC_BX", 8);
  // Slices per tile: minimise (waves of persistent CTAs) x (per-tile cost):
  // MMAs per K step (bx + 2 folded, bx unfolded) plus a fixed per-tile
  // overhead (decode, barrier round trips, epilogue drain) worth ~3 slices.
  // Large layers thus take the slice count with the least padding along the
  // axis (6 for the 18-deep axis of config 5, 8 for 32 or 128); layers with
  // fewer tiles than SMs shrink their tiles until every SM has work.  Ties go
  // to the larger tile.
  c.bx = 1;
  long long best = -1;
  for (int cand : {8, 6, 4, 3, 2, 1}) {
    if (cand > bx_cap || tc_tmem_cols(cand, L.nt, c.acc, fold_pair) > 512) continue;
    // (unfolded tiles of 3 / 6 slices: VXB_TC_UNF36=0 restores 1, 2, 4, 8)
    if (!L.fold && (cand & (cand - 1)) && !env_int("VXB_TC_UNF36", 1)) continue;
    long long tiles = static_cast<long long>(ceil_div(slice_extent, cand)) * other_tiles;
    if (fold_pair) tiles = (tiles + 1) / 2 * 2;
    const long long waves = (tiles + sms - 1) / sms;
    // a folded pair issues bx + 2 MMAs per step for two tiles (one per SM)
    const long long cost = fold_pair ? waves * ((cand + 2) + 2 * kTileOverhead)
                                     : waves * 2 * ((L.fold ? cand + 2 : cand) + kTileOverhead);
    if (best < 0 || cost < best) {
      best = cost;
      c.bx = cand;
    }
  }
  // streamed fold (run_tc): the slab width is given, the accumulators are a
  // TMEM ring, the A box has no halo along the slice axis and the weights
  // must stay resident
  if (stream_bx) c.bx = stream_bx;
  if (!stream_bx && tc_tmem_cols(c.bx, L.nt, c.acc, fold_pair) > 512)
    return set_error(VXB_EUNSUPPORTED, "TMEM overflow");
  bool any_pair = false;
  int max_steps = 1;
  for (const TcGroup &g : L.groups) {
    any_pair |= g.nch == 2;
    max_steps = std::max(max_steps, g.steps);
  }
  const int slab = L.slab;
  // fp32-input convs buffer their input in the staging ring: two A stages
  int na_cap = f32in ? std::max(2, std::min(4, env_int("VXB_TC_F32IN_NA", 2)))
                        : std::max(2, std::min(6, env_int("VXB_TC_NA", 3)));
  for (;;) {
    const int budget = budget0 - c.bx * reserved_per_slice;
    const int sx = L.fold == 2 ? TILE_Y : c.bx, sy = L.fold == 2 ? c.bx : TILE_Y;
    const int hx = sx + (stream_bx ? 0 : k[0] - 1), hy = sy + k[1] - 1, hz = TILE_Z + k[2] - 1;
    c.chunk_bytes = hx * hy * hz * 16;
    c.chunk_stride = round_up(c.chunk_bytes + 128, 128);
    c.chunk_slots = any_pair ? 2 : 1;
    c.a_stage = c.chunk_slots * c.chunk_stride;
    c.na = na_cap;
    // resident weights: whole filter bank of the (single) N tile in smem
    long long total_w = L.steps * slab;
    c.resident = 0;
    if (reps * L.n_tiles == 1 && c.na * c.a_stage + total_w <= budget) {
      c.bsteps = max_steps;
      int nbs = 0;
      for (const TcGroup &g : L.groups) nbs += ceil_div(g.steps, c.bsteps);
      c.b_stage = c.bsteps * slab;
      if (c.na * c.a_stage + static_cast<long long>(nbs) * c.b_stage <= budget) {
        c.resident = 1;
        c.nb = nbs;
      }
    }
    c.pair = can_pair && (pair_mode == 1 || !c.resident);
    if (c.resident) c.b_stage = c.b_stage / (c.pair ? 2 : 1);
    if (!c.resident) {
      // Streamed weights: as few B stages per K group as fit (ring >= 2).
      // Every stage boundary costs the MMA warp a b_full wait + commit round
      // trip (~300 cycles measured: C128 1x3x3 stages of 8+1 steps 147 us,
      // one 9-step stage 127 us; C64 3x3x3 one 9-step stage 88.6 us, 5+4
      // steps 92.4 us; deeper rings of smaller stages measured no better).
      const int half = c.pair ? 2 : 1;
      const int env_bs = env_int("VXB_TC_BSTEPS", 0);
      const int avail = budget - c.na * c.a_stage;
      const int min_ring = env_int("VXB_TC_BRING", 2);
      c.bsteps = 0;
      for (int parts = 1; parts <= max_steps && !env_bs; ++parts) {
        const int bs = ceil_div(max_steps, parts);
        const int stage = bs * slab / half;
        if (stage <= 64 * 1024 && avail / stage >= min_ring) {
          c.bsteps = bs;
          break;
        }
      }
      if (!c.bsteps) c.bsteps = std::max(1, std::min(max_steps, env_bs ? env_bs : 32768 / slab));
      c.b_stage = c.bsteps * slab / half;
      c.nb = std::min(c.pair ? 6 : 4, avail / c.b_stage);
      while (c.nb < 2 && c.bsteps > 1) {
        c.bsteps = (c.bsteps + 1) / 2;
        c.b_stage = c.bsteps * slab / half;
        c.nb = std::min(c.pair ? 6 : 4, avail / c.b_stage);
      }
    }
    if (stream_bx && c.resident) break;
    if (stream_bx && na_cap <= 2) return VXB_EUNSUPPORTED;   // caller falls back (no error text)
    if (!stream_bx && c.nb >= 1 && (c.resident || c.nb >= 2)) break;
    if (na_cap > 2) {
      --na_cap;
      continue;
    }
    if (c.bx == 1) return set_error(VXB_EUNSUPPORTED, "conv tile does not fit in shared memory");
    c.bx /= 2;
  }
  // Accumulator stages: with two, the MMAs of tile i + 2 wait for the whole
  // epilogue of tile i, and when MMA and epilogue times are close the pair of
  // chains runs at (MMA + epilogue + hand-off latencies) / 2 per tile instead
  // of max(MMA, epilogue) (C28 1x3x3 on 18x768x768: MMAs alone 249 us,
  // epilogue alone 226 us, together 338 us).  Small tiles leave TMEM columns
  // free: use them for more stages (VXB_TC_ACC_MAX, default 4).
  if (stream_bx) c.acc = 2;
  if (c.acc == 2 && !stream_bx) {
    const int acc_max = std::min(MAX_ACC, env_int("VXB_TC_ACC_MAX", 4));
    while (c.acc < acc_max && tc_tmem_cols(c.bx, L.nt, c.acc + 1, fold_pair) <= 512) ++c.acc;
  }
  c.smem = static_cast<size_t>(c.na) * c.a_stage + static_cast<size_t>(c.nb) * c.b_stage +
           (2 * c.na + 2 * c.nb + 2 * MAX_ACC) * sizeof(uint64_t) + 16;
  return VXB_OK;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 4-D map over a blocked bf16 view: (lane*z, y, x, batch*chunk)
static int make_input_map(const vxb_tensor &t, int hx, int hy, int hz, CUtensorMap *m,
                          int *bstride) {
  if (t.dtype != VXB_BF16 || !t.blocked)
    return set_error(VXB_EINVAL, "tensor-core conv input must be a blocked bf16 view");
  if (t.s[4] != 8)
    return set_error(VXB_EINVAL, "tensor-core conv input: z stride must be 8 (got %lld)",
                     static_cast<long long>(t.s[4]));
  const int nch = ceil_div(t.c, 8);
  long long total = nch;
  *bstride = 0;
  if (t.n > 1) {
    if (t.s[0] % t.s[1] != 0)
      return set_error(VXB_EINVAL, "tensor-core conv input: batch stride not a chunk multiple");
    *bstride = static_cast<int>(t.s[0] / t.s[1]);
    total = static_cast<long long>(t.n - 1) * *bstride + nch;
  }
  EncodeTiledFn enc = get_encode();
  if (!enc) return set_error(VXB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(8) * t.z, static_cast<cuuint64_t>(t.y),
                        static_cast<cuuint64_t>(t.x), static_cast<cuuint64_t>(total)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(t.s[3]) * 2,
                           static_cast<cuuint64_t>(t.s[2]) * 2,
                           static_cast<cuuint64_t>(t.s[1]) * 2};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(8 * hz), static_cast<cuuint32_t>(hy),
                       static_cast<cuuint32_t>(hx), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, t.data, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(VXB_ECUDA, "cuTensorMapEncodeTiled failed (%d): dims %llu %llu %llu %llu",
                     static_cast<int>(r), (unsigned long long)dims[0],
                     (unsigned long long)dims[1], (unsigned long long)dims[2],
                     (unsigned long long)dims[3]);
  return VXB_OK;
}

static void *g_dbg = nullptr;
static const size_t kDbgBytes = 1024 * 64 * 8 * sizeof(unsigned long long);

// SM count of the calling thread's current device (cached per device: the
// threads of a multi-GPU run_tiled each drive their own device)
static int device_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (dev >= 0 && dev < 64) {
    const int c = __atomic_load_n(&cache[dev], __ATOMIC_RELAXED);
    if (c > 0) return c;
  }
  int sms = -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  if (dev >= 0 && dev < 64) __atomic_store_n(&cache[dev], sms, __ATOMIC_RELAXED);
  return sms;
}

struct TcLaunch {
  const vxb_tensor *in[2];
  int off[2][3];
  int cin0, cin1, cout;
  int k[3], pad[3];
  int ox, oy, oz, nb;
  int reps;
  int rep_n;        // > 0: the reps ride in N (rep_n columns each), one tile computes all
  int zpair;        // rep_n layout with the dz = 0 / 1 taps interleaved per 8-fmap chunk
  long long out_rep_off[MAX_REPS], base_rep_off[MAX_REPS];
  EpiView out, base;
  int has_base;
  const void *w;
  const float *bias, *scale;
  int act;
  float alpha;
  bool allow_fold;
  int nt_cap;
  int pool;
  EpiView pool_out;
  // fused 1x1x1 head
  const float *head_w, *head_b;
  int head_cout, head_act;
  float head_alpha;
  EpiView head_out;
};

// (set while a conv whose streamed configuration did not fit is configured
// again as tiles)
static thread_local bool g_no_stream = false;

static int run_tc(const TcLaunch &a_in, cudaStream_t stream) {
  TcLaunch a = a_in;
  const int n_cols = a.rep_n ? a.reps * a.rep_n : a.cout;   // GEMM N over all taps in N
  const int rep_offsets = a.reps;
  if (a.rep_n) a.reps = 1;                                   // one tile covers every tap
  TcLayout L = tc_layout(a.cin0, a.cin1, n_cols, a.k, a.allow_fold, a.nt_cap > 0 ? a.nt_cap : 256);
  TcConfig c;
  const int slice_y = L.fold == 2;
  int sms = device_sms();
  if (sms <= 0) return set_error(VXB_ECUDA, "no CUDA device");
  // The tile shape (and with it the MMA order, hence the fp32 summation
  // order) is chosen from ONE batch entry's tile count, so a batch of
  // volumes (rebatched plans: several patches per launch) computes every
  // entry bit-identically to a batch-1 run.
  const long long other_tiles = static_cast<long long>(ceil_div(slice_y ? a.ox : a.oy, TILE_Y)) *
                                ceil_div(a.oz, TILE_Z) * L.n_tiles * a.reps;
  // fp32 NCDHW input (the network's own input tensor): converted in-kernel
  const vxb_tensor &x0 = *a.in[0];
  const bool f32in = x0.dtype == VXB_F32 && !x0.blocked;
  // staging ring: ~80 KB of fp32 boxes in flight covers the TMA latency at
  // the input rate of the low-fmap convs (each box <= 16 KB: xb x-slices)
  const int kStgBudget = env_int("VXB_TC_STG_KB", 80) * 1024;
  int stg_bytes = 0, hzb = 0, zshift = 0;
  if (f32in) {
    if (a.in[1] || a.has_base)
      return set_error(VXB_EUNSUPPORTED,
                       "fp32-input conv supports one input segment and no residual operand");
    if (x0.s[4] != 1 || (reinterpret_cast<uintptr_t>(x0.data) & 15) || (x0.s[3] * 4) % 16 ||
        (x0.s[2] * 4) % 16 || (x0.s[1] * 4) % 16 || (x0.n > 1 && (x0.s[0] * 4) % 16))
      return set_error(VXB_EINVAL,
                       "fp32-input conv needs a z-contiguous view with 16-byte aligned rows");
    // TMA needs the box's innermost (z) start 16-byte aligned: boxes start at
    // the halo origin rounded down to 4 floats (tile origins are multiples of
    // 8, so the shift is a per-layer constant) and rows are 16-byte multiples
    zshift = (((a.off[0][2] - a.pad[2]) % 4) + 4) % 4;
    hzb = round_up(zshift + TILE_Z + a.k[2] - 1, 4);
    stg_bytes = kStgBudget;
  }
  // folded low-fmap convs run as CTA pairs when N = 3nt <= 96: an M = 256
  // MMA then costs what an M = 128 one does (tools/umma_align.cu)
  const int pair_env = env_int("VXB_TC_PAIR", 1);
  const bool out_ok = ((a.out.dtype == VXB_BF16 || a.out.dtype == VXB_BF16X2) && a.out.blocked) ||
                      (a.out.dtype == VXB_F32 && !a.out.blocked);
  // Measured (config-2 shapes, 128x256x256): 3x3x3 at nt = 16 gains 14 %;
  // 1x3x3 and nt = 32 lose (their tiles are bound by the A-halo stream, and
  // the pair couples two CTAs' loads), so only that case pairs by default.
  const int fp_env = env_int("VXB_TC_FOLDPAIR", 1);
  const bool fold_pair = L.fold && L.nt <= 32 && pair_env == 1 && fp_env &&
                         (fp_env == 2 || (L.fold == 1 && L.nt == 16)) && !a.pool && !f32in &&
                         out_ok;
  // weight-streaming convs run as CTA pairs sharing one B stream
  // (cta_group::2: M = 256 per MMA, each CTA ingests and reads only half of
  // every weight slab, halving the smem traffic that bounds high-fmap
  // convs); resident-weight unfolded convs pair too (one M = 256 instruction
  // serves two SMs at the per-instruction floor).  A pair needs >= 2 tiles:
  // checked at the widest tile, so any tile width chosen below has them.
  const long long spatial_min =
      static_cast<long long>(ceil_div(slice_y ? a.oy : a.ox, 8)) *
      ceil_div(slice_y ? a.ox : a.oy, TILE_Y) * ceil_div(a.oz, TILE_Z);
  const bool can_pair = (!L.fold || fold_pair) && !a.pool && !a.head_cout && spatial_min >= 2 &&
                        L.nt % 16 == 0 && L.nt / 8 <= 256 && out_ok &&
                        (pair_env == 1 || pair_env == 2);
  // a fused head keeps its weights in smem (4 rows x the padded fmaps) and
  // one float4 partial per row and column item of a tile (<= 8 slices)
  const int head_smem = a.head_cout ? 4 * L.n_tiles * L.nt * 4 + 16 : 0;
  const int head_slice = a.head_cout ? (L.nt / 16) * 128 * 16 : 0;
  // Streamed fold (TcParams::stream): x-folded convs with a lean epilogue
  // whose columns fill the SMs (one batch entry's columns decide, so batched
  // launches stay bit-identical to single ones).  VXB_TC_STREAM: 0 off, 1
  // (default) = nt == 32 convs without fused pooling, 2 = every eligible
  // conv.  Measured (C28 3x3x3, 16 patches of 18x192x192): 483 vs 505 us
  // tiled (571 vs 578 with a residual operand; 368 vs 434 at x = 14); with
  // fused pooling the streamed epilogue is slower (1.53 vs 1.45 ms per 36
  // patches), so those stay tiled.
  const bool lean_ok = env_int("VXB_TC_LEAN", 1) && !f32in && !a.head_cout &&
                       (!a.pool || (a.pool_out.dtype == VXB_BF16 && a.pool_out.blocked)) &&
                       a.out.dtype == VXB_BF16 && a.out.blocked &&
                       (!a.has_base || (a.base.dtype == VXB_BF16 && a.base.blocked)) &&
                       (a.act == VXB_ACT_NONE || a.act == VXB_ACT_RELU || a.act == VXB_ACT_ELU);
  const int st_env = g_no_stream ? 0 : env_int("VXB_TC_STREAM", 1);
  int st_bx = 0, st_j0 = 0, st_nin = 0, st_nslab = 0, st_slots = 0;
  if (st_env && L.fold == 1 && lean_ok && a.reps == 1 && !a.rep_n && L.n_tiles == 1 && a.k[0] == 3) {
    st_slots = 1;
    while (st_slots * 2 * L.nt <= 512) st_slots *= 2;
    // input slices (halo coordinates j: x_in = j - pad + off) that can be non-zero
    int j0 = 0, j1 = a.ox + 1;
    bool same = true;
    for (int sg = 0; sg < 2; ++sg) {
      if (!a.in[sg]) continue;
      const int lo = std::max(0, a.pad[0] - a.off[sg][0]);
      const int hi = std::min(a.ox + 1, a.in[sg]->x - 1 + a.pad[0] - a.off[sg][0]);
      if (sg == 0) {
        j0 = lo;
        j1 = hi;
      } else if (lo != j0 || hi != j1) {
        same = false;
      }
    }
    const int bx_max = std::min(8, (st_slots - 2) / 2);
    const long long cols_one = static_cast<long long>(ceil_div(a.oy, TILE_Y)) * ceil_div(a.oz, TILE_Z);
    if (same && j0 <= 2 && j1 >= a.ox - 1 && j1 >= j0 && bx_max >= 1 &&
        (st_env == 2 ||
         // (columns are the unit of work: one entry's columns must fill whole
         // waves of CTAs -- config 4's 153 columns over 148 SMs would take
         // two waves for 1.03 waves of work)
         (L.nt == 32 && !a.pool && cols_one >= sms &&
          cols_one * 10 >= ceil_div(cols_one, sms) * sms * 9))) {
      st_j0 = j0;
      st_nin = j1 - j0 + 1;
      st_nslab = ceil_div(st_nin, bx_max);
      st_bx = ceil_div(st_nin, st_nslab);
    }
  }
  int rc = VXB_EUNSUPPORTED;
  if (st_bx) {
    rc = tc_configure(L, a.k, a.ox, other_tiles, sms, a.reps, stg_bytes + head_smem, f32in, false,
                      pair_env, false, c, head_slice, st_bx);
    if (rc) st_bx = 0;   // weights do not stay resident beside the A ring: tiled walk
  }
  if (!st_bx)
    rc = tc_configure(L, a.k, slice_y ? a.oy : a.ox, other_tiles, sms, a.reps,
                      stg_bytes + head_smem, f32in, can_pair && !(fold_pair && a.head_cout),
                      pair_env, fold_pair && !a.head_cout, c, head_slice);
  if (rc) return rc;
  TcParams p;
  memset(&p, 0, sizeof(p));
  p.nb = a.nb;
  p.ox = a.ox;
  p.oy = a.oy;
  p.oz = a.oz;
  p.bx = c.bx;
  p.nt = L.nt;
  p.acc_stages = c.acc;
  p.slice_y = slice_y;
  p.fold = L.fold != 0;
  p.ex = slice_y ? TILE_Y : c.bx;
  p.ey = slice_y ? c.bx : TILE_Y;
  p.slab_bytes = L.slab;
  p.tiles_x = ceil_div(a.ox, p.ex);
  p.tiles_y = ceil_div(a.oy, p.ey);
  p.tiles_z = ceil_div(a.oz, TILE_Z);
  p.n_tiles = L.n_tiles;
  p.reps = a.reps;
  const long long spatial = static_cast<long long>(p.tiles_x) * p.tiles_y * p.tiles_z * p.nb;
  p.pair = c.pair;
  p.cluster = p.pair || (!c.resident && env_int("VXB_TC_CLUSTER", 1) == 2 && spatial >= 2) ? 2 : 1;
  const long long spatial_pad = (spatial + p.cluster - 1) / p.cluster * p.cluster;
  long long total = spatial_pad * p.n_tiles * p.reps;
  if (total > 0x7fffffffLL) return set_error(VXB_EUNSUPPORTED, "too many tiles");
  p.spatial_real = static_cast<int>(spatial);
  p.spatial_pad = static_cast<int>(spatial_pad);
  p.total_tiles = static_cast<int>(total);
  {
    const int ds[6] = {p.spatial_pad, p.tiles_z, p.tiles_y, p.tiles_x, p.nb, p.n_tiles};
    for (int i = 0; i < 6; ++i) {
      const unsigned long long d = static_cast<unsigned long long>(std::max(1, ds[i]));
      if (static_cast<unsigned long long>(total) * d >= (1ull << 40))
        return set_error(VXB_EUNSUPPORTED, "tile grid too large for the fast tile decode");
      p.dm[i] = ((1ull << 40) + d - 1) / d;
    }
  }
  p.kx = a.k[0];
  p.ky = a.k[1];
  p.kz = a.k[2];
  p.hx = p.ex + (st_bx ? 0 : a.k[0] - 1);
  p.hy = p.ey + a.k[1] - 1;
  p.hz = TILE_Z + a.k[2] - 1;
  p.a_slice_inc = (slice_y ? p.hz : p.hy * p.hz) * 16;
  p.a_sbo = (slice_y ? p.hy * p.hz : p.hz) * 16;
  for (int i = 0; i < 3; ++i) p.pad[i] = a.pad[i];
  TcMaps maps;
  memset(&maps, 0, sizeof(maps));
  for (int s = 0; s < 2; ++s) {
    p.seg_chunks[s] = L.seg_chunks[s];
    if (!p.seg_chunks[s]) continue;
    for (int i = 0; i < 3; ++i) p.seg_off[s][i] = a.off[s][i];
    if (f32in) continue;
    rc = make_input_map(*a.in[s], p.hx, p.hy, p.hz, &maps.m[s], &p.seg_bstride[s]);
    if (rc) return rc;
  }
  if (f32in) {
    p.f32in = 1;
    p.hzb = hzb;
    const int slice_bytes = LANES * p.hy * hzb * 4;
    p.f32in_xb = std::max(1, std::min(p.hx, 16384 / slice_bytes));
    p.stg_bytes = p.f32in_xb * slice_bytes;
    p.n_stg = std::max(2, std::min(8, kStgBudget / p.stg_bytes));
    p.f32in_zshift = zshift;
    EncodeTiledFn enc = get_encode();
    if (!enc) return set_error(VXB_ECUDA, "cuTensorMapEncodeTiled unavailable");
    // 4-D (z, y, x, batch*channel): lanes past C must read as zero, so a
    // batch > 1 needs whole chunks (C % 8 == 0) and a channel-stride batch
    if (x0.n > 1 && (x0.c % LANES || x0.s[0] != x0.s[1] * x0.c))
      return set_error(VXB_EUNSUPPORTED,
                       "fp32-input conv with batch > 1 needs C %% 8 == 0 and packed batches");
    p.f32in_cstride = x0.c;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(x0.z), static_cast<cuuint64_t>(x0.y),
                          static_cast<cuuint64_t>(x0.x),
                          static_cast<cuuint64_t>(x0.c) * x0.n};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(x0.s[3]) * 4,
                             static_cast<cuuint64_t>(x0.s[2]) * 4,
                             static_cast<cuuint64_t>(x0.s[1]) * 4};
    cuuint32_t box[4] = {static_cast<cuuint32_t>(hzb), static_cast<cuuint32_t>(p.hy),
                         static_cast<cuuint32_t>(p.f32in_xb), static_cast<cuuint32_t>(LANES)};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(&maps.m[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x0.data, dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
      return set_error(VXB_ECUDA, "fp32 input tensor map failed (%d)", static_cast<int>(r));
    if (env_int("VXB_PRINT", 0))
      fprintf(stderr, "f32in map dims %llu %llu %llu %llu str %llu %llu %llu box %u %u %u %u "
              "hx %d hy %d hz %d bx %d stg %d smem-a %d nb %d bst %d na %d\n",
              (unsigned long long)dims[0], (unsigned long long)dims[1], (unsigned long long)dims[2],
              (unsigned long long)dims[3], (unsigned long long)strides[0],
              (unsigned long long)strides[1], (unsigned long long)strides[2], box[0], box[1],
              box[2], box[3], p.hx, p.hy, p.hz, c.bx, p.stg_bytes, c.a_stage, c.nb, c.b_stage,
              c.na);
  }
  p.n_groups = static_cast<int>(L.groups.size());
  p.chunk_bytes = c.chunk_bytes;
  p.chunk_stride = c.chunk_stride;
  p.chunk_slots = c.chunk_slots;
  p.a_stage_bytes = c.a_stage;
  p.b_stage_bytes = c.b_stage;
  p.na = c.na;
  p.nb_stages = c.nb;
  p.bsteps = c.bsteps;
  p.resident = c.resident;
  p.w = static_cast<const uint8_t *>(a.w);
  p.w_steps = static_cast<int>(L.steps);
  if (p.pair) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return set_error(VXB_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t slab = static_cast<cuuint64_t>(L.slab);
    // a slab is R rows (nt, or 3nt folded) x 32 B; each CTA takes R/2 rows =
    // R/8 units of 128 B
    const cuuint64_t units = static_cast<cuuint64_t>(L.slab) / SLAB_ROW_BYTES / 8;
    cuuint64_t dims[4] = {128, units, 2, static_cast<cuuint64_t>(a.reps) * L.n_tiles * L.steps};
    cuuint64_t strides[3] = {128, slab / 2, slab};
    cuuint32_t box[4] = {128, static_cast<cuuint32_t>(units), 1,
                         static_cast<cuuint32_t>(c.bsteps)};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(&maps.w, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void *>(a.w), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(VXB_ECUDA, "weight tensor map failed (%d)", (int)r);
  }
  p.w_ntile_stride = L.steps * L.slab;
  p.w_rep_stride = static_cast<long long>(tc_bytes_per_rep(L));
  p.bias = a.bias;
  p.scale = a.scale;
  p.out = a.out;
  p.base = a.base;
  p.has_base = a.has_base;
  if (a.pool) {
    // the epilogue pools over (y, z) row pairs of one 128-row slice
    if (slice_y) return set_error(VXB_EUNSUPPORTED, "fused pooling needs x-sliced tiles");
    p.pool = 1;
    p.pool_out = a.pool_out;
    p.pool_oy = a.oy / 2;
    p.pool_oz = a.oz / 2;
  }
  for (int r = 0; r < MAX_REPS; ++r) {
    p.out_rep_off[r] = a.out_rep_off[r];
    p.base_rep_off[r] = a.base_rep_off[r];
  }
  p.rep_n = a.rep_n;
  p.zpair = a.zpair;
  if (a.zpair) {
    // 32-byte stores / residual loads need the dz = 0 row 32-byte aligned:
    // every offset of a dz = 0 row is a multiple of 16 elements
    auto al32 = [&](const EpiView &v, const long long *roff) {
      if (!v.data) return true;
      if (v.dtype != VXB_BF16 || !v.blocked || (reinterpret_cast<uintptr_t>(v.data) & 31)) return false;
      for (int i = 0; i < 5; ++i)
        if (i != 4 && v.s[i] % 16) return false;
      if (v.s[4] != 16) return false;
      for (int r = 0; r < a.reps; r += 2)
        if (roff[r] % 16 || roff[r + 1] != roff[r] + 8) return false;
      return true;
    };
    p.zpair_v8 = al32(a.out, a.out_rep_off) && (!a.has_base || al32(a.base, a.base_rep_off));
  }
  (void)rep_offsets;
  p.head_w = a.head_w;
  p.head_b = a.head_b;
  p.head_cout = a.head_cout;
  p.head_act = a.head_act;
  p.head_alpha = a.head_alpha;
  p.head_out = a.head_out;
  p.cout = a.cout;
  p.act = a.act;
  p.alpha = a.alpha;
  // lean epilogue (conv3d_tc.cu LeanEnt): the common bf16 blocked case
  p.lean = env_int("VXB_TC_LEAN", 1) && !f32in && !a.head_cout &&
           (!p.pool || (!p.pair && a.pool_out.dtype == VXB_BF16 && a.pool_out.blocked)) &&
           a.out.dtype == VXB_BF16 && a.out.blocked &&
           (!a.has_base || (a.base.dtype == VXB_BF16 && a.base.blocked)) &&
           (a.act == VXB_ACT_NONE || a.act == VXB_ACT_RELU || a.act == VXB_ACT_ELU) &&
           L.nt <= 256;
  p.dbg_mode = env_int("VXB_TC_DBGMODE", 0);
  if (env_int("VXB_TC_DEBUG", 0)) {
    if (!g_dbg) {
      cudaError_t e = cudaMalloc(&g_dbg, kDbgBytes);
      if (e != cudaSuccess) return check_cuda(e, "debug buffer");
    }
    cudaMemsetAsync(g_dbg, 0, kDbgBytes, stream);
    p.dbg = static_cast<unsigned long long *>(g_dbg);
  }
  const bool fp = p.pair && p.fold;
  p.acc_stride = (fp ? p.bx + 2 : p.bx) * p.nt;
  p.slice0_col = fp ? 2 * p.nt : 0;
  int cols = tc_tmem_cols(p.bx, p.nt, p.acc_stages, fp);
  if (st_bx) {
    p.stream = 1;
    p.st_j0 = st_j0;
    p.st_nin = st_nin;
    p.st_nslab = st_nslab;
    p.st_slots = st_slots;
    p.st_ncols = p.tiles_y * p.tiles_z * p.nb;
    {
      int a_ = a.ox % st_slots, b_ = st_slots;   // period of (k * ox) mod slots
      while (a_) {
        const int t_ = b_ % a_;
        b_ = a_;
        a_ = t_;
      }
      p.st_nphase = st_slots / b_;
    }
    p.acc_stride = 0;
    cols = st_slots * p.nt;
    total = static_cast<long long>(p.st_ncols) * st_nslab;
    p.total_tiles = static_cast<int>(total);
  }
  p.tmem_cols = 32;
  while (p.tmem_cols < cols) p.tmem_cols <<= 1;
  if (p.tmem_cols > 512) return set_error(VXB_EUNSUPPORTED, "TMEM overflow (%d columns)", cols);
  c.smem = tc_smem_bytes(p);
  if (c.smem > 227 * 1024 && p.stream) {
    // the ring's operand tables and the lean tables did not fit beside the
    // resident weights: the tiled walk instead
    g_no_stream = true;
    const int rc2 = run_tc(a_in, stream);
    g_no_stream = false;
    return rc2;
  }
  if (c.smem > 227 * 1024) return set_error(VXB_EUNSUPPORTED, "conv needs %zu B smem", c.smem);
  // persistent: one CTA per SM (480 threads x ~100 registers leaves no room
  // for a second one, and the smem ring is sized for the whole SM)
  int grid = static_cast<int>(std::min<long long>(p.stream ? p.st_ncols : total,
                                                 static_cast<long long>(sms)));
  grid = std::max(p.cluster, grid / p.cluster * p.cluster);
  if (env_int("VXB_PRINT", 0))
    fprintf(stderr,
            "conv3d_tc cin %d+%d cout %d k %d%d%d out %dx%dx%d: nt %d ntiles %d fold %d pair %d "
            "bx %d acc %d na %d nb %d bsteps %d resident %d tiles %d grid %d smem %zu tmem %d "
            "stream %d (j0 %d nin %d slabs %d slots %d)\n",
            a.cin0, a.cin1, a.cout, a.k[0], a.k[1], a.k[2], a.ox, a.oy, a.oz, p.nt, p.n_tiles,
            L.fold, p.pair, p.bx, p.acc_stages, p.na, p.nb_stages, p.bsteps, p.resident,
            p.total_tiles, grid, c.smem, p.tmem_cols, p.stream, p.st_j0, p.st_nin, p.st_nslab,
            p.st_slots);
  return launch_conv3d_tc(p, maps, grid, stream);
}

// x3 precision: the conv's K segments over a split input of cin fmaps
static inline int x3_cin0(int cin) { return 16 * ceil_div(cin, 8); }
static inline int x3_cin1(int cin) { return 8 * ceil_div(cin, 8); }

static inline float bf16_bits_to_f32(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static inline float bf16_round_host(float v) { return bf16_bits_to_f32(f32_to_bf16_bits(v)); }

// Weight of K column ci of the x3 segments (split_segments): ci < 16 CB is
// lane ci % 8 of plane (ci / 8) % 2 of chunk ci / 16 -> bf16(W); ci >= 16 CB
// is the hi plane again -> bf16(W - bf16(W)).  Lanes past cin are zero.
template <class WFn>
static float x3_weight(WFn wstd, int cin, int co, int ci, int dx, int dy, int dz) {
  const int c0 = x3_cin0(cin);
  const bool lo_term = ci >= c0;
  const int c = lo_term ? ci - c0 : (ci / 16) * 8 + (ci % 8);
  if (c >= cin) return 0.f;
  const float v = wstd(co, c, dx, dy, dz);
  const float hi = bf16_round_host(v);
  return lo_term ? v - hi : hi;
}

}  // namespace vxb

using namespace vxb;

extern "C" {

int vxb_abi_version(void) { return VXB_ABI_VERSION; }

int vxb_set_pdl(int mode) { return vxb::set_pdl_override(mode); }
const char *vxb_last_error(void) { return g_last_error.c_str(); }
int vxb_device_sms(void) { return device_sms(); }

size_t vxb_debug_read(unsigned long long *host, size_t count) {
  if (!g_dbg || !host) return 0;
  size_t n = std::min(count, kDbgBytes / sizeof(unsigned long long));
  if (cudaMemcpy(host, g_dbg, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  return n;
}

int vxb_conv_select(int cin, int cout, const int k[3], const int stride[3]) {
  (void)cin;
  (void)cout;
  if (stride[0] == 1 && stride[1] == 1 && stride[2] == 1 && TILE_Z + k[2] - 1 <= 32 &&
      TILE_Y + k[1] - 1 <= 256 && k[0] <= 64 && k[0] >= 1 && k[1] >= 1 && k[2] >= 1)
    return VXB_PATH_TC;
  return VXB_PATH_DIRECT;
}

static int device_sms_or(int fallback) {
  const int n = device_sms();
  return n > 0 ? n : fallback;
}

int vxb_conv_select_shape(int cin, int cout, const int k[3], const int stride[3],
                          const int out_xyz[3]) {
  return vxb_conv_select_shape_b(cin, cout, k, stride, out_xyz, 1);
}

int vxb_conv_select_shape_b(int cin, int cout, const int k[3], const int stride[3],
                            const int out_xyz[3], int batch) {
  int path = vxb_conv_select(cin, cout, k, stride);
  if (path != VXB_PATH_TC || !out_xyz) return path;
  const TcLayout L = tc_layout(cin, 0, cout, k);
  if (L.fold == 2 && out_xyz[0] > 0 && ceil_div(out_xyz[0], TILE_Y) * TILE_Y * 4 > out_xyz[0] * 5)
    return VXB_PATH_TC_UNFOLDED;   // > 25% of the 16-row x tiles would be padding
  // Too few output tiles for the SMs even at one slice per tile (deep U-net
  // levels: 9^3 .. 24^3 voxels, or 18x12x12 in config 5)?  Narrower N tiles
  // multiply the tile count and shorten each tile's MMAs; every N tile
  // re-reads the (small, L2-resident) input.  Take the widest N tile that
  // gives one tile per SM.
  const int sms = std::max(1, device_sms_or(148));
  // (all batch entries count: a rebatched plan runs several patches per
  // launch.  The N split never changes a result -- every output column
  // accumulates the same K steps in the same order -- so batch-1 and
  // batch-B runs stay bit-identical; config 5 at 12 patches per launch:
  // 80 -> 80 3x3x3 unsplit 24 us vs 45 us in N tiles of 32, tools/conv_sweep.py)
  const long long sp = static_cast<long long>(out_xyz[0]) * ceil_div(out_xyz[1], TILE_Y) *
                       ceil_div(out_xyz[2], TILE_Z) * std::max(1, batch);
  if (sp * L.n_tiles >= sms) return path;
  if (L.npad > 128) {
    // wide layers (CTA-pair MMAs when unsplit): the widest split that fills
    // the SMs, else 64-wide tiles
    const TcLayout L128 = tc_layout(cin, 0, cout, k, true, 128);
    if (sp * L128.n_tiles >= sms) return VXB_PATH_TC_N128;
    return VXB_PATH_TC_N64;
  }
  if (L.npad > 96) return path;   // 96-128 fmaps: one CTA-pair N tile beats two halves (measured)
  // narrow (folded, single-CTA) layers: waves x per-MMA cycles of the N tile
  // (SS-mode floor max(45.5, 32 + N/4), N = 3 nt when folded); the K work of
  // a tile does not depend on the split
  static const int kCaps[4] = {256, 64, 32, 16};
  static const int kPaths[4] = {VXB_PATH_TC, VXB_PATH_TC_N64, VXB_PATH_TC_N32, VXB_PATH_TC_N16};
  int best = path;
  double best_cost = 1e30;
  for (int i = 0; i < 4; ++i) {
    const TcLayout Li = tc_layout(cin, 0, cout, k, true, kCaps[i]);
    const long long waves = (sp * Li.n_tiles + sms - 1) / sms;
    const int n = Li.fold ? 3 * Li.nt : Li.nt;
    const double cost = static_cast<double>(waves) * std::max(45.5, 32.0 + n / 4.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = kPaths[i];
    }
  }
  return best;
}

static size_t direct_bytes(int cin, int cout, const int k[3]) {
  return static_cast<size_t>(ceil_div(cout, DCO_DIRECT)) * ceil_div(cin, 8) * k[0] * k[1] * k[2] *
         8 * DCO_DIRECT * sizeof(float);
}

size_t vxb_conv_weights_bytes3(int cin0, int cin1, int cout, const int k[3], const int stride[3],
                               int path, int prec) {
  if (prec == VXB_PREC_X3) {
    if (cin1 != 0) return 0;
    if (path == 0) path = vxb_conv_select(cin0, cout, k, stride);
    if (is_tc(path))
      return tc_bytes_per_rep(tc_layout(x3_cin0(cin0), x3_cin1(cin0), cout, k, path_folds(path),
                                        path_nt_cap(path)));
    return direct_bytes(cin0, cout, k);   // CUDA cores read split inputs as fp32 sums
  }
  if (path == 0) path = vxb_conv_select(cin0 + cin1, cout, k, stride);
  if (is_tc(path))
    return tc_bytes_per_rep(tc_layout(cin0, cin1, cout, k, path_folds(path), path_nt_cap(path)));
  return direct_bytes(cin0 + cin1, cout, k);
}

size_t vxb_conv_weights_bytes2(int cin0, int cin1, int cout, const int k[3], const int stride[3],
                               int path) {
  return vxb_conv_weights_bytes3(cin0, cin1, cout, k, stride, path, VXB_PREC_BF16);
}

size_t vxb_conv_weights_bytes(int cin, int cout, const int k[3], const int stride[3], int path) {
  return vxb_conv_weights_bytes2(cin, 0, cout, k, stride, path);
}

int vxb_conv_pack_weights3(const float *w, int cin0, int cin1, int cout, const int k[3],
                           const int stride[3], int path, int prec, void *dst, size_t dst_bytes) {
  const int cin = cin0 + cin1;
  if (!w || !dst) return set_error(VXB_EINVAL, "pack: null pointer");
  if (prec != VXB_PREC_BF16 && prec != VXB_PREC_X3)
    return set_error(VXB_EINVAL, "pack: bad precision %d", prec);
  if (prec == VXB_PREC_X3 && cin1 != 0)
    return set_error(VXB_EUNSUPPORTED, "pack: x3 precision takes a single input segment");
  if (path == 0) path = vxb_conv_select(cin, cout, k, stride);
  size_t need = vxb_conv_weights_bytes3(cin0, cin1, cout, k, stride, path, prec);
  if (dst_bytes < need) return set_error(VXB_EINVAL, "pack: need %zu bytes, got %zu", need, dst_bytes);
  auto wtap = [&](int co, int ci, int dx, int dy, int dz) {
    return w[((((static_cast<size_t>(co) * cin) + ci) * k[0] + dx) * k[1] + dy) * k[2] + dz];
  };
  if (is_tc(path)) {
    if (prec == VXB_PREC_X3) {
      const int a = x3_cin0(cin), b = x3_cin1(cin);
      TcLayout L = tc_layout(a, b, cout, k, path_folds(path), path_nt_cap(path));
      auto wx3 = [&](int co, int ci, int dx, int dy, int dz) {
        return x3_weight(wtap, cin, co, ci, dx, dy, dz);
      };
      tc_pack(L, a, b, cout, k, wx3, static_cast<uint8_t *>(dst));
      return VXB_OK;
    }
    TcLayout L = tc_layout(cin0, cin1, cout, k, path_folds(path), path_nt_cap(path));
    tc_pack(L, cin0, cin1, cout, k, wtap, static_cast<uint8_t *>(dst));
    return VXB_OK;
  }
  // direct: [cout_group][in_chunk][tap][8 in][16 out] fp32
  float *o = static_cast<float *>(dst);
  const int taps = k[0] * k[1] * k[2], ich = ceil_div(cin, 8), ncg = ceil_div(cout, DCO_DIRECT);
  size_t idx = 0;
  for (int cg = 0; cg < ncg; ++cg)
    for (int ch = 0; ch < ich; ++ch)
      for (int t = 0; t < taps; ++t) {
        const int dz = t % k[2], dy = (t / k[2]) % k[1], dx = t / (k[2] * k[1]);
        for (int l = 0; l < 8; ++l)
          for (int oo = 0; oo < DCO_DIRECT; ++oo, ++idx) {
            const int ci = ch * 8 + l, co = cg * DCO_DIRECT + oo;
            o[idx] = (ci < cin && co < cout) ? wtap(co, ci, dx, dy, dz) : 0.f;
          }
      }
  return VXB_OK;
}

int vxb_conv_pack_weights2(const float *w, int cin0, int cin1, int cout, const int k[3],
                           const int stride[3], int path, void *dst, size_t dst_bytes) {
  return vxb_conv_pack_weights3(w, cin0, cin1, cout, k, stride, path, VXB_PREC_BF16, dst,
                                dst_bytes);
}

int vxb_conv_pack_weights(const float *w, int cin, int cout, const int k[3], const int stride[3],
                          int path, void *dst, size_t dst_bytes) {
  return vxb_conv_pack_weights2(w, cin, 0, cout, k, stride, path, dst, dst_bytes);
}

int vxb_conv3d(const vxb_conv_desc *d, void *stream) {
  if (!d) return set_error(VXB_EINVAL, "conv3d: null descriptor");
  int rc;
  if ((rc = check_view(&d->in0, "conv3d.in0"))) return rc;
  if ((rc = check_view(&d->out, "conv3d.out"))) return rc;
  const bool two = d->in1.data != nullptr;
  if (two && (rc = check_view(&d->in1, "conv3d.in1"))) return rc;
  const bool additive = d->base.data != nullptr;
  if (additive && (rc = check_view(&d->base, "conv3d.base"))) return rc;
  if (!d->w_packed || !d->bias) return set_error(VXB_EINVAL, "conv3d: null weights/bias");
  const int cin0 = d->in0.c, cin1 = two ? d->in1.c : 0;
  if (cin0 + cin1 != d->cin)
    return set_error(VXB_EINVAL, "conv3d: cin %d != input fmaps %d", d->cin, cin0 + cin1);
  if (d->out.c != d->cout)
    return set_error(VXB_EINVAL, "conv3d: out view has %d fmaps, cout %d", d->out.c, d->cout);
  for (int i = 0; i < 3; ++i)
    if (d->k[i] < 1 || d->stride[i] < 1 || d->pad[i] < 0)
      return set_error(VXB_EINVAL, "conv3d: bad kernel/stride/pad");
  if (d->act < 0 || d->act > 3) return set_error(VXB_EINVAL, "conv3d: bad act %d", d->act);
  // extents: every output voxel's window (after the segment's crop offset)
  // lies inside the input plus its virtual zero padding; batches agree; a
  // residual operand has the output's shape (the epilogue reads it at
  // output coordinates)
  {
    const int oe[3] = {d->out.x, d->out.y, d->out.z};
    for (int sg = 0; sg < (two ? 2 : 1); ++sg) {
      const vxb_tensor &t = sg ? d->in1 : d->in0;
      const int *off = sg ? d->off1 : d->off0;
      const int ie[3] = {t.x, t.y, t.z};
      if (t.n != d->out.n)
        return set_error(VXB_EINVAL, "conv3d: in%d batch %d != out batch %d", sg, t.n, d->out.n);
      for (int i = 0; i < 3; ++i)
        if (off[i] < 0 || (oe[i] - 1) * d->stride[i] + d->k[i] > ie[i] - off[i] + 2 * d->pad[i])
          return set_error(VXB_EINVAL,
                           "conv3d: output extent %d on axis %d needs more than in%d extent %d "
                           "(offset %d, pad %d, k %d, stride %d)",
                           oe[i], i, sg, ie[i], off[i], d->pad[i], d->k[i], d->stride[i]);
    }
    if (additive && (d->base.n != d->out.n || d->base.c != d->out.c || d->base.x != d->out.x ||
                     d->base.y != d->out.y || d->base.z != d->out.z))
      return set_error(VXB_EINVAL, "conv3d: base view must have the output's shape");
  }
  const bool split_in = d->in0.dtype == VXB_BF16X2;
  if (d->prec != VXB_PREC_BF16 && d->prec != VXB_PREC_X3)
    return set_error(VXB_EINVAL, "conv3d: bad prec %d", d->prec);
  if (split_in != (d->prec == VXB_PREC_X3))
    return set_error(VXB_EINVAL,
                     "conv3d: a split (VXB_BF16X2) input needs VXB_PREC_X3 weights and vice versa");
  if (split_in && two)
    return set_error(VXB_EUNSUPPORTED, "conv3d: split inputs take a single input segment");
  const int path = d->path ? d->path : vxb_conv_select(d->cin, d->cout, d->k, d->stride);
  cudaStream_t s = as_stream(stream);
  if (is_tc(path)) {
    if (d->stride[0] != 1 || d->stride[1] != 1 || d->stride[2] != 1)
      return set_error(VXB_EUNSUPPORTED, "tensor-core conv requires stride 1");
    TcLaunch a;
    memset(&a, 0, sizeof(a));
    a.allow_fold = path_folds(path);
    a.nt_cap = path_nt_cap(path);
    vxb_tensor both, hi;
    if (split_in) {
      split_segments(d->in0, both, hi);
      a.in[0] = &both;
      a.in[1] = &hi;
    } else {
      a.in[0] = &d->in0;
      a.in[1] = two ? &d->in1 : nullptr;
    }
    for (int i = 0; i < 3; ++i) {
      a.off[0][i] = d->off0[i];
      a.off[1][i] = split_in ? d->off0[i] : d->off1[i];
      a.k[i] = d->k[i];
      a.pad[i] = d->pad[i];
    }
    a.cin0 = split_in ? x3_cin0(cin0) : cin0;
    a.cin1 = split_in ? x3_cin1(cin0) : cin1;
    a.cout = d->cout;
    a.ox = d->out.x;
    a.oy = d->out.y;
    a.oz = d->out.z;
    a.nb = d->out.n;
    a.reps = 1;
    a.out = to_epi(d->out);
    a.has_base = additive;
    if (additive) a.base = to_epi(d->base);
    a.w = d->w_packed;
    a.bias = d->bias;
    a.scale = additive ? d->base_scale : nullptr;
    a.act = d->act;
    a.alpha = d->alpha;
    if (d->pool_mode == VXB_POOL_FUSED_MAX122) {
      if (split_in || d->out.dtype == VXB_BF16X2)
        return set_error(VXB_EUNSUPPORTED, "fused pooling: bf16 storage only");
      if ((rc = check_view(&d->pool_out, "conv3d.pool_out"))) return rc;
      const vxb_tensor &pv = d->pool_out;
      if (pv.n != d->out.n || pv.c != d->cout || pv.x != d->out.x || pv.y != d->out.y / 2 ||
          pv.z != d->out.z / 2)
        return set_error(VXB_EINVAL, "conv3d.pool_out must be (n, cout, x, y/2, z/2)");
      a.pool = 1;
      a.pool_out = to_epi(pv);
    } else if (d->pool_mode != VXB_POOL_FUSED_NONE) {
      return set_error(VXB_EINVAL, "conv3d: bad pool_mode %d", d->pool_mode);
    }
    if (d->head_cout) {
      const vxb_tensor &h = d->head_out;
      if ((rc = check_view(&h, "conv3d.head_out"))) return rc;
      if (d->head_cout < 0 || d->head_cout > 4 || !d->head_w || !d->head_b)
        return set_error(VXB_EINVAL, "conv3d: fused head needs 1..4 fmaps, weights and bias");
      if (h.dtype != VXB_F32 || h.blocked || h.n != d->out.n || h.c != d->head_cout ||
          h.x != d->out.x || h.y != d->out.y || h.z != d->out.z)
        return set_error(VXB_EINVAL,
                         "conv3d.head_out must be an fp32 standard view (n, head_cout, ox, oy, oz)");
      if (d->head_act < 0 || d->head_act > 3 || d->pool_mode != VXB_POOL_FUSED_NONE)
        return set_error(VXB_EINVAL, "conv3d: bad head activation / head with pooling");
      a.head_w = d->head_w;
      a.head_b = d->head_b;
      a.head_cout = d->head_cout;
      a.head_act = d->head_act;
      a.head_alpha = d->head_alpha;
      a.head_out = to_epi(h);
    }
    return run_tc(a, s);
  }
  if (d->pool_mode != VXB_POOL_FUSED_NONE)
    return set_error(VXB_EUNSUPPORTED, "fused pooling needs the tensor-core conv path");
  if (d->head_cout)
    return set_error(VXB_EUNSUPPORTED, "a fused head needs the tensor-core conv path");
  if (two) return set_error(VXB_EUNSUPPORTED, "direct conv path takes a single input");
  DirectParams p;
  memset(&p, 0, sizeof(p));
  p.in = to_dview(d->in0);
  p.out = to_dview(d->out);
  if (additive) p.base = to_dview(d->base);
  p.w = static_cast<const float *>(d->w_packed);
  p.bias = d->bias;
  p.scale = additive ? d->base_scale : nullptr;
  p.cin = d->cin;
  p.cout = d->cout;
  p.kx = d->k[0];
  p.ky = d->k[1];
  p.kz = d->k[2];
  p.sx = d->stride[0];
  p.sy = d->stride[1];
  p.sz = d->stride[2];
  // crop offsets fold into a negative pad
  p.px = d->pad[0] - d->off0[0];
  p.py = d->pad[1] - d->off0[1];
  p.pz = d->pad[2] - d->off0[2];
  p.act = d->act;
  p.alpha = d->alpha;
  p.has_base = additive;
  return launch_conv_direct(p, s);
}

int vxb_conv3d_subimage(const vxb_conv_desc *d, const float *w_std, int in_chunk, int out_chunk,
                        const int origin[3], const int extent[3], int first, int last,
                        void *stream) {
  int rc;
  if (!d || !w_std) return set_error(VXB_EINVAL, "subimage: null argument");
  if ((rc = check_view(&d->in0, "subimage.in"))) return rc;
  if ((rc = check_view(&d->out, "subimage.out"))) return rc;
  if (!d->in0.blocked || !d->out.blocked)
    return set_error(VXB_EINVAL, "subimage: blocked views required");
  SubParams p;
  memset(&p, 0, sizeof(p));
  p.in = to_dview(d->in0);
  p.out = to_dview(d->out);
  p.has_base = d->base.data != nullptr;
  if (p.has_base) p.base = to_dview(d->base);
  p.w = w_std;
  p.bias = d->bias;
  p.scale = d->base_scale;
  p.cin = d->cin;
  p.cout = d->cout;
  p.kx = d->k[0];
  p.ky = d->k[1];
  p.kz = d->k[2];
  p.sx = d->stride[0];
  p.sy = d->stride[1];
  p.sz = d->stride[2];
  p.ib = in_chunk;
  p.ob = out_chunk;
  p.x0 = origin[0];
  p.y0 = origin[1];
  p.z0 = origin[2];
  p.ex = extent[0];
  p.ey = extent[1];
  p.ez = extent[2];
  p.first = first;
  p.last = last;
  p.act = d->act;
  p.alpha = d->alpha;
  return launch_subimage(p, as_stream(stream));
}

// ------------------------------------------------------------------ deconv

static bool deconv_tc_ok(const int k[3], const int stride[3]) {
  return k[0] == stride[0] && k[1] == stride[1] && k[2] == stride[2] &&
         k[0] * k[1] * k[2] <= MAX_REPS;
}
static bool deconv_tc(const int k[3], const int stride[3], int path) {
  return path != VXB_PATH_DIRECT && deconv_tc_ok(k, stride);
}

// Taps in N: with k == stride every output voxel takes exactly one tap, so a
// k-tap deconv is one 1x1x1 GEMM with N = taps x round_up(cout, 16): the
// input tile is read once for all taps and the epilogue sends each 16-column
// item to its tap's (strided) output voxels.  Used when N fits one MMA
// (config 5's 1x2x2 deconvs: 4 x 32..64); otherwise every tap is a tile
// replica (config 4's 2x2x2 deconvs at 128-512 fmaps).
static int deconv_rep_n(int cout, const int k[3], const int stride[3], int path) {
  if (!deconv_tc(k, stride, path)) return 0;
  const int reps = k[0] * k[1] * k[2];
  const int ntr = round_up(cout, 16);
  if (reps < 2 || reps * ntr > 256 || !env_int("VXB_DECONV_REPN", 1)) return 0;
  return ntr;
}

// z-pair column order for taps in N with a z stride of 2 (config 5's 1x2x2
// deconvs): column n of tap r, fmap co is
//   (r / 2) * 2 rn + (co / 8) * 16 + (r % 2) * 8 + co % 8,
// so a 16-column epilogue item holds one 8-fmap chunk at dz = 0 and dz = 1,
// whose outputs are adjacent 16-byte rows (one 32-byte store instead of two
// half-sector writes 32 bytes apart)
static bool deconv_zpair(int rep_n, const int k[3], const int stride[3]) {
  return rep_n > 0 && k[2] == 2 && stride[2] == 2 && env_int("VXB_DECONV_ZPAIR", 1);
}

// K segments of a tensor-core deconv's 1x1x1 GEMM: the input fmaps, or the
// two x3 segments over a split input
static void deconv_segments(int cin, int prec, int &c0, int &c1) {
  c0 = prec == VXB_PREC_X3 ? x3_cin0(cin) : cin;
  c1 = prec == VXB_PREC_X3 ? x3_cin1(cin) : 0;
}

size_t vxb_deconv_weights_bytes3(int cin, int cout, const int k[3], const int stride[3], int path,
                                 int prec) {
  int one[3] = {1, 1, 1}, c0, c1;
  deconv_segments(cin, prec, c0, c1);
  if (const int rn = deconv_rep_n(cout, k, stride, path))
    return tc_bytes_per_rep(tc_layout(c0, c1, k[0] * k[1] * k[2] * rn, one));
  if (deconv_tc(k, stride, path))
    return static_cast<size_t>(k[0] * k[1] * k[2]) * tc_bytes_per_rep(tc_layout(c0, c1, cout, one));
  return static_cast<size_t>(cout) * cin * k[0] * k[1] * k[2] * sizeof(float);
}

size_t vxb_deconv_weights_bytes(int cin, int cout, const int k[3], const int stride[3],
                                int path) {
  return vxb_deconv_weights_bytes3(cin, cout, k, stride, path, VXB_PREC_BF16);
}

int vxb_deconv_pack_weights3(const float *w, int cin, int cout, const int k[3],
                             const int stride[3], int path, int prec, void *dst,
                             size_t dst_bytes) {
  if (!w || !dst) return set_error(VXB_EINVAL, "deconv pack: null pointer");
  if (prec != VXB_PREC_BF16 && prec != VXB_PREC_X3)
    return set_error(VXB_EINVAL, "deconv pack: bad precision %d", prec);
  if (path == VXB_PATH_TC && !deconv_tc_ok(k, stride))
    return set_error(VXB_EUNSUPPORTED, "tensor-core deconv needs k == stride, <= 8 taps");
  size_t need = vxb_deconv_weights_bytes3(cin, cout, k, stride, path, prec);
  if (dst_bytes < need) return set_error(VXB_EINVAL, "deconv pack: need %zu bytes", need);
  if (!deconv_tc(k, stride, path)) {
    memcpy(dst, w, need);
    return VXB_OK;
  }
  int one[3] = {1, 1, 1}, c0, c1;
  deconv_segments(cin, prec, c0, c1);
  // weight of GEMM K column ci for output column co at tap (dx, dy, dz)
  auto wk = [&](int co, int ci, int dx, int dy, int dz) -> float {
    auto wstd = [&](int o, int i, int a, int b, int c) {
      return w[((((static_cast<size_t>(o) * cin) + i) * k[0] + a) * k[1] + b) * k[2] + c];
    };
    if (prec == VXB_PREC_X3) return x3_weight(wstd, cin, co, ci, dx, dy, dz);
    return wstd(co, ci, dx, dy, dz);
  };
  if (const int rn = deconv_rep_n(cout, k, stride, path)) {
    // column co' = tap * rn + co, taps in (dx, dy, dz) order
    const int reps = k[0] * k[1] * k[2];
    TcLayout L = tc_layout(c0, c1, reps * rn, one);
    const bool zp = deconv_zpair(rn, k, stride);
    auto wtap = [&](int cop, int ci, int, int, int) {
      int r = cop / rn, co = cop - r * rn;
      if (zp) {
        const int rp = cop / (2 * rn), rem = cop - rp * 2 * rn;
        r = 2 * rp + ((rem >> 3) & 1);
        co = ((rem >> 4) << 3) + (rem & 7);
      }
      if (co >= cout) return 0.f;
      const int dz = r % k[2], dy = (r / k[2]) % k[1], dx = r / (k[2] * k[1]);
      return wk(co, ci, dx, dy, dz);
    };
    tc_pack(L, c0, c1, reps * rn, one, wtap, static_cast<uint8_t *>(dst));
    return VXB_OK;
  }
  TcLayout L = tc_layout(c0, c1, cout, one);
  size_t per = tc_bytes_per_rep(L);
  int r = 0;
  for (int dx = 0; dx < k[0]; ++dx)
    for (int dy = 0; dy < k[1]; ++dy)
      for (int dz = 0; dz < k[2]; ++dz, ++r) {
        auto wtap = [&](int co, int ci, int, int, int) { return wk(co, ci, dx, dy, dz); };
        tc_pack(L, c0, c1, cout, one, wtap, static_cast<uint8_t *>(dst) + r * per);
      }
  return VXB_OK;
}

int vxb_deconv_pack_weights(const float *w, int cin, int cout, const int k[3], const int stride[3],
                            int path, void *dst, size_t dst_bytes) {
  return vxb_deconv_pack_weights3(w, cin, cout, k, stride, path, VXB_PREC_BF16, dst, dst_bytes);
}

int vxb_deconv3d(const vxb_deconv_desc *d, void *stream) {
  if (!d) return set_error(VXB_EINVAL, "deconv3d: null descriptor");
  int rc;
  if ((rc = check_view(&d->in, "deconv3d.in"))) return rc;
  if ((rc = check_view(&d->out, "deconv3d.out"))) return rc;
  const bool additive = d->base.data != nullptr;
  if (additive && (rc = check_view(&d->base, "deconv3d.base"))) return rc;
  if (d->in.c != d->cin || d->out.c != d->cout)
    return set_error(VXB_EINVAL, "deconv3d: fmap counts do not match the views");
  for (int i = 0; i < 3; ++i) {
    int ext = i == 0 ? d->in.x : (i == 1 ? d->in.y : d->in.z);
    int oext = i == 0 ? d->out.x : (i == 1 ? d->out.y : d->out.z);
    if ((ext - 1) * d->stride[i] + d->k[i] != oext)
      return set_error(VXB_EINVAL, "deconv3d: output extent mismatch on axis %d", i);
  }
  cudaStream_t s = as_stream(stream);
  if (d->path == VXB_PATH_TC && !deconv_tc_ok(d->k, d->stride))
    return set_error(VXB_EUNSUPPORTED, "tensor-core deconv needs k == stride, <= 8 taps");
  const bool split_in = d->in.dtype == VXB_BF16X2;
  if (d->prec != VXB_PREC_BF16 && d->prec != VXB_PREC_X3)
    return set_error(VXB_EINVAL, "deconv3d: bad prec %d", d->prec);
  if (split_in != (d->prec == VXB_PREC_X3))
    return set_error(VXB_EINVAL,
                     "deconv3d: a split (VXB_BF16X2) input needs VXB_PREC_X3 weights and vice versa");
  if (deconv_tc(d->k, d->stride, d->path)) {
    TcLaunch a;
    memset(&a, 0, sizeof(a));
    vxb_tensor both, hi;
    if (split_in) {
      split_segments(d->in, both, hi);
      a.in[0] = &both;
      a.in[1] = &hi;
    } else {
      a.in[0] = &d->in;
      a.in[1] = nullptr;
    }
    for (int i = 0; i < 3; ++i) a.k[i] = 1;
    deconv_segments(d->cin, d->prec, a.cin0, a.cin1);
    a.cout = d->cout;
    a.ox = d->in.x;
    a.oy = d->in.y;
    a.oz = d->in.z;
    a.nb = d->in.n;
    a.reps = d->k[0] * d->k[1] * d->k[2];
    a.rep_n = deconv_rep_n(d->cout, d->k, d->stride, d->path);
    a.zpair = deconv_zpair(a.rep_n, d->k, d->stride);
    a.out = to_epi(d->out);
    for (int i = 0; i < 3; ++i) a.out.s[2 + i] = d->out.s[2 + i] * d->stride[i];
    a.has_base = additive;
    if (additive) {
      a.base = to_epi(d->base);
      for (int i = 0; i < 3; ++i) a.base.s[2 + i] = d->base.s[2 + i] * d->stride[i];
    }
    int r = 0;
    for (int dx = 0; dx < d->k[0]; ++dx)
      for (int dy = 0; dy < d->k[1]; ++dy)
        for (int dz = 0; dz < d->k[2]; ++dz, ++r) {
          a.out_rep_off[r] = dx * d->out.s[2] + dy * d->out.s[3] + dz * d->out.s[4];
          if (additive)
            a.base_rep_off[r] = dx * d->base.s[2] + dy * d->base.s[3] + dz * d->base.s[4];
        }
    a.w = d->w_packed;
    a.bias = d->bias;
    a.scale = additive ? d->base_scale : nullptr;
    a.act = d->act;
    a.alpha = d->alpha;
    return run_tc(a, s);
  }
  GatherDeconvParams p;
  memset(&p, 0, sizeof(p));
  p.in = to_dview(d->in);
  p.out = to_dview(d->out);
  p.has_base = additive;
  if (additive) p.base = to_dview(d->base);
  p.w = static_cast<const float *>(d->w_packed);
  p.bias = d->bias;
  p.scale = additive ? d->base_scale : nullptr;
  p.cin = d->cin;
  p.cout = d->cout;
  p.kx = d->k[0];
  p.ky = d->k[1];
  p.kz = d->k[2];
  p.sx = d->stride[0];
  p.sy = d->stride[1];
  p.sz = d->stride[2];
  p.act = d->act;
  p.alpha = d->alpha;
  return launch_deconv_gather(p, s);
}

// ------------------------------------------------------------------ ops

static int same_shape(const vxb_tensor *a, const vxb_tensor *b, const char *what) {
  if (a->n != b->n || a->c != b->c || a->x != b->x || a->y != b->y || a->z != b->z)
    return set_error(VXB_EINVAL, "%s: shape mismatch", what);
  return VXB_OK;
}

int vxb_pool3d(const vxb_tensor *in, const vxb_tensor *out, const int window[3],
               const int stride[3], int mode, void *stream) {
  int rc;
  if ((rc = check_view(in, "pool.in")) || (rc = check_view(out, "pool.out"))) return rc;
  if (mode != VXB_POOL_MAX && mode != VXB_POOL_AVG) return set_error(VXB_EINVAL, "pool: mode");
  const int ie[3] = {in->x, in->y, in->z}, oe[3] = {out->x, out->y, out->z};
  for (int i = 0; i < 3; ++i) {
    if (window[i] < 1 || stride[i] < 1 || window[i] > ie[i])
      return set_error(VXB_EINVAL, "pool: bad window/stride on axis %d", i);
    if ((ie[i] - window[i]) / stride[i] + 1 != oe[i])
      return set_error(VXB_EINVAL, "pool: output extent mismatch on axis %d", i);
  }
  if (in->n != out->n || in->c != out->c) return set_error(VXB_EINVAL, "pool: n/c mismatch");
  return launch_pool(to_dview(*in), to_dview(*out), window, stride, mode, as_stream(stream));
}

int vxb_eltwise(const vxb_tensor *a, const vxb_tensor *b, const vxb_tensor *out, int op,
                void *stream) {
  int rc;
  if ((rc = check_view(a, "eltwise.a")) || (rc = check_view(b, "eltwise.b")) ||
      (rc = check_view(out, "eltwise.out")))
    return rc;
  if ((rc = same_shape(a, b, "eltwise")) || (rc = same_shape(a, out, "eltwise"))) return rc;
  if (op < 0 || op > 2) return set_error(VXB_EINVAL, "eltwise: op %d", op);
  return launch_eltwise(to_dview(*a), to_dview(*b), to_dview(*out), op, as_stream(stream));
}

int vxb_affine_act(const vxb_tensor *in, const vxb_tensor *out, const float *mult,
                   const float *add, int act, float alpha, void *stream) {
  int rc;
  if ((rc = check_view(in, "affine.in")) || (rc = check_view(out, "affine.out"))) return rc;
  if ((rc = same_shape(in, out, "affine_act"))) return rc;
  if (act < 0 || act > 3) return set_error(VXB_EINVAL, "affine_act: act %d", act);
  return launch_affine_act(to_dview(*in), to_dview(*out), mult, add, act, alpha,
                           as_stream(stream));
}

int vxb_mergecrop(const vxb_tensor *a, const vxb_tensor *b, const vxb_tensor *out, void *stream) {
  int rc;
  if ((rc = check_view(a, "mergecrop.a")) || (rc = check_view(b, "mergecrop.b")) ||
      (rc = check_view(out, "mergecrop.out")))
    return rc;
  const int ea[3] = {a->x, a->y, a->z}, eb[3] = {b->x, b->y, b->z};
  const int eo[3] = {out->x, out->y, out->z};
  int oa[3], ob[3];
  for (int i = 0; i < 3; ++i) {
    int common = std::min(ea[i], eb[i]);
    if (eo[i] != common) return set_error(VXB_EINVAL, "mergecrop: output extent mismatch");
    oa[i] = (ea[i] - common) / 2;  // shapes.crop_offsets: floor
    ob[i] = (eb[i] - common) / 2;
  }
  if (out->c != a->c + b->c || a->n != b->n || out->n != a->n)
    return set_error(VXB_EINVAL, "mergecrop: fmap/batch mismatch");
  return launch_mergecrop(to_dview(*a), to_dview(*b), to_dview(*out), oa, ob, as_stream(stream));
}

int vxb_pad_copy(const vxb_tensor *in, const vxb_tensor *out, const int pads[3], void *stream) {
  int rc;
  if ((rc = check_view(in, "pad.in")) || (rc = check_view(out, "pad.out"))) return rc;
  if (out->x != in->x + 2 * pads[0] || out->y != in->y + 2 * pads[1] ||
      out->z != in->z + 2 * pads[2] || in->c != out->c || in->n != out->n)
    return set_error(VXB_EINVAL, "pad_copy: shape mismatch");
  return launch_pad_copy(to_dview(*in), to_dview(*out), pads, as_stream(stream));
}

int vxb_copy(const vxb_tensor *src, const vxb_tensor *dst, void *stream) {
  int rc;
  if ((rc = check_view(src, "copy.src")) || (rc = check_view(dst, "copy.dst"))) return rc;
  if ((rc = same_shape(src, dst, "copy"))) return rc;
  return launch_copy(to_dview(*src), to_dview(*dst), as_stream(stream));
}

int vxb_copy_ex(const vxb_tensor *src, const vxb_tensor *dst, int flags, void *stream) {
  int rc;
  if ((rc = check_view(src, "copy.src")) || (rc = check_view(dst, "copy.dst"))) return rc;
  if ((rc = same_shape(src, dst, "copy"))) return rc;
  if (flags & ~VXB_COPY_INDEPENDENT) return set_error(VXB_EINVAL, "copy: unknown flags %d", flags);
  return launch_copy(to_dview(*src), to_dview(*dst), as_stream(stream),
                     (flags & VXB_COPY_INDEPENDENT) != 0);
}

int vxb_copy_windows(const vxb_tensor *src, const vxb_tensor *dst, int count, void *stream) {
  if (count < 0 || (count > 0 && (!src || !dst)))
    return set_error(VXB_EINVAL, "copy_windows: bad arguments");
  for (int base = 0; base < count; base += WIN_MAX) {
    WinBatch b;
    memset(&b, 0, sizeof(b));
    b.count = std::min(WIN_MAX, count - base);
    for (int i = 0; i < b.count; ++i) {
      const vxb_tensor &a = src[base + i], &d = dst[base + i];
      int rc;
      if ((rc = check_view(&a, "copy_windows.src")) || (rc = check_view(&d, "copy_windows.dst")))
        return rc;
      if (a.dtype != VXB_F32 || d.dtype != VXB_F32 || a.blocked || d.blocked || a.s[4] != 1 ||
          d.s[4] != 1)
        return set_error(VXB_EINVAL, "copy_windows: fp32 standard views with contiguous z");
      if ((rc = same_shape(&a, &d, "copy_windows"))) return rc;
      WinCopy &w = b.w[i];
      w.src = static_cast<const float *>(a.data);
      w.dst = static_cast<float *>(d.data);
      for (int k = 0; k < 4; ++k) {
        w.ss[k] = a.s[k];
        w.ds[k] = d.s[k];
      }
      w.ext[0] = a.n; w.ext[1] = a.c; w.ext[2] = a.x; w.ext[3] = a.y; w.ext[4] = a.z;
      bool v4 = a.z % 4 == 0 && !(reinterpret_cast<uintptr_t>(a.data) & 15) &&
                !(reinterpret_cast<uintptr_t>(d.data) & 15);
      for (int k = 0; k < 4; ++k) v4 = v4 && a.s[k] % 4 == 0 && d.s[k] % 4 == 0;
      w.vec4 = v4;
    }
    if (int rc = launch_copy_windows(b, as_stream(stream))) return rc;
  }
  return VXB_OK;
}

int vxb_pack_zwin(const vxb_tensor *src, const vxb_tensor *dst, int kz, int pz, int flags,
                  void *stream) {
  int rc;
  if ((rc = check_view(src, "pack_zwin.src")) || (rc = check_view(dst, "pack_zwin.dst")))
    return rc;
  if (src->blocked || src->dtype != VXB_F32 || src->c != 1)
    return set_error(VXB_EINVAL, "pack_zwin: source must be a 1-channel fp32 standard view");
  if (!dst->blocked || (dst->dtype != VXB_BF16 && dst->dtype != VXB_BF16X2) || dst->c != kz ||
      kz < 1 || kz > 8)
    return set_error(VXB_EINVAL,
                     "pack_zwin: destination must be (split) bf16 blocked with c == kz <= 8");
  if (pz < 0 || dst->n != src->n || dst->x != src->x || dst->y != src->y ||
      dst->z != src->z + 2 * pz - kz + 1)
    return set_error(VXB_EINVAL, "pack_zwin: shape mismatch (dst z = src z + 2 pz - kz + 1)");
  if (flags & ~VXB_COPY_INDEPENDENT) return set_error(VXB_EINVAL, "pack_zwin: unknown flags");
  return launch_pack_zwin(to_dview(*src), to_dview(*dst), kz, pz, as_stream(stream),
                          (flags & VXB_COPY_INDEPENDENT) != 0);
}

int vxb_pack_zwin_windows(const vxb_tensor *src, int count, const vxb_tensor *dst, int kz, int pz,
                          void *stream) {
  int rc;
  if (!src || !dst || count < 1 || count > ZWIN_MAX || count != dst->n)
    return set_error(VXB_EINVAL, "pack_zwin_windows: need 1..%d windows, one per dst entry",
                     ZWIN_MAX);
  if ((rc = check_view(dst, "pack_zwin_windows.dst"))) return rc;
  ZwinWindows w;
  memset(&w, 0, sizeof(w));
  for (int b = 0; b < count; ++b) {
    const vxb_tensor &a = src[b];
    if ((rc = check_view(&a, "pack_zwin_windows.src"))) return rc;
    if (a.blocked || a.dtype != VXB_F32 || a.c != 1 || a.n != 1 || a.x != src[0].x ||
        a.y != src[0].y || a.z != src[0].z)
      return set_error(VXB_EINVAL, "pack_zwin_windows: 1-channel fp32 windows of one shape");
    for (int i = 2; i < 5; ++i)
      if (a.s[i] != src[0].s[i])
        return set_error(VXB_EINVAL, "pack_zwin_windows: windows of one volume (same strides)");
    w.off[b] = (static_cast<const char *>(a.data) - static_cast<const char *>(src[0].data)) /
               static_cast<long long>(sizeof(float));
  }
  if (!dst->blocked || (dst->dtype != VXB_BF16 && dst->dtype != VXB_BF16X2) || dst->c != kz ||
      kz < 1 || kz > 8 || pz < 0 || dst->x != src[0].x || dst->y != src[0].y ||
      dst->z != src[0].z + 2 * pz - kz + 1)
    return set_error(VXB_EINVAL, "pack_zwin_windows: destination shape");
  return launch_pack_zwin_windows(to_dview(src[0]), w, to_dview(*dst), kz, pz, as_stream(stream));
}

int vxb_zero(const vxb_tensor *t, void *stream) {
  int rc;
  if ((rc = check_view(t, "zero"))) return rc;
  return launch_zero(to_dview(*t), as_stream(stream));
}

}  // extern "C"
