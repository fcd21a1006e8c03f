/*
 * vxb.h — C ABI of the B200 (sm_100a) volumetric-convolution engine.
 *
 * This is the drop-in boundary for the hot path of the reference engine
 * (voxplan, a Python + Cython restatement of PZnet, arXiv 1903.07525).
 * Every entry point replaces one callable the reference's runtime invokes
 * per plan step; the reference interface each one replaces is cited next
 * to it (paths relative to the reference's pkg/src/voxplan/).
 *
 * Conventions
 *  - All device memory is owned by the caller; entry points never allocate
 *    device memory (cf. _kernels.pyx:81-83, which only mallocs a scratch
 *    accumulator).  Host-side packing functions write caller buffers.
 *  - Every launch is asynchronous on the caller's stream (cudaStream_t
 *    passed as void*).  Nothing synchronises.
 *  - Return value: 0 on success, nonzero VXB_E* on failure; the message is
 *    available from vxb_last_error() (thread-local).  The Python layer maps
 *    a nonzero status onto voxplan's ExecutionError (errors.py:55-56).
 *  - Activations live in the channel-blocked layout of the reference
 *    (blocked.py:1-9): (batch, ceil(C/8), X, Y, Z, 8), lane = fmap % 8,
 *    with lanes past the logical fmap count held at zero.  Element type is
 *    bf16 (VXB_BF16) on the production path, split bf16 (VXB_BF16X2) on the
 *    fp32-accurate path, fp32 (VXB_F32) at network boundaries.  A view carries element strides so the interior of a halo
 *    allocation, a crop window or a channel slice of a concat buffer are
 *    all addressable without copies (blocked.py:57-110).
 */
#ifndef VXB_H
#define VXB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VXB_ABI_VERSION 5

/* element types */
#define VXB_BF16 0
#define VXB_F32 1
/* split bf16 ("x3" precision): every element is held as two bf16 values,
 * hi = bf16(v) and lo = bf16(v - hi), so hi + lo keeps ~16 significant bits
 * (fp32 storage bytes, values exact in fp32).  Blocked views only: the lo
 * plane of every chunk lies s[1]/2 elements after its hi plane, i.e. the
 * storage of a dense tensor is (batch, ceil(C/8), 2, X, Y, Z, 8) bf16.  A
 * tensor-core conv reads a split input as two bf16 K segments,
 * [hi, lo] x bf16(W) and [hi] x bf16(W - bf16(W)) (weights packed with
 * VXB_PREC_X3), which reproduces fp32 arithmetic to ~1e-5 relative. */
#define VXB_BF16X2 2

/* weight-packing precisions (vxb_conv_pack_weights3 / vxb_deconv_pack_weights3) */
#define VXB_PREC_BF16 0   /* bf16(W): inputs bf16 */
#define VXB_PREC_X3 1     /* split inputs: [bf16(W); bf16(W); bf16(W - bf16(W))] */

/* activation codes: identical to kernels_cy.py:19 (_ACT_CODE) */
#define VXB_ACT_NONE 0
#define VXB_ACT_RELU 1
#define VXB_ACT_ELU 2
#define VXB_ACT_SIGMOID 3

/* status codes */
#define VXB_OK 0
#define VXB_EINVAL 1
#define VXB_EUNSUPPORTED 2
#define VXB_ECUDA 3

/* conv paths chosen by vxb_conv_select */
#define VXB_PATH_TC 1     /* tcgen05/TMEM implicit GEMM, TMA-fed */
#define VXB_PATH_DIRECT 2 /* CUDA-core direct convolution (Cin<8, strides, big k) */
#define VXB_PATH_TC_UNFOLDED 3 /* tensor-core path without slice-axis tap folding */
#define VXB_PATH_TC_N128 4     /* tensor-core path, output fmaps in N tiles of <= 128 */
#define VXB_PATH_TC_N64 5      /* tensor-core path, output fmaps in N tiles of <= 64 */
#define VXB_PATH_TC_N32 6      /* tensor-core path, output fmaps in N tiles of <= 32 */
#define VXB_PATH_TC_N16 7      /* tensor-core path, output fmaps in N tiles of 16 */

/* pooling modes: ops.py:63-86 */
#define VXB_POOL_MAX 0
#define VXB_POOL_AVG 1
/* pooling fused into a conv epilogue (vxb_conv_desc.pool_mode): max over
 * 1x2x2 windows with stride 1x2x2 of the stored (rounded) conv output, the
 * following MaxPool step of the reference (ops.py:63-86) */
#define VXB_POOL_FUSED_NONE 0
#define VXB_POOL_FUSED_MAX122 1

/* eltwise ops: ops.py:50-60 */
#define VXB_ELT_ADD 0
#define VXB_ELT_MUL 1
#define VXB_ELT_DIV 2

/*
 * A view of one activation tensor.  Logical shape (n, c, x, y, z).
 *  blocked == 1: element (b, f, i, j, k) lives at
 *      data + b*s[0] + (f/8)*s[1] + i*s[2] + j*s[3] + k*s[4] + (f%8)
 *  blocked == 0 (standard NCDHW, used at the network boundary):
 *      data + b*s[0] + f*s[1] + i*s[2] + j*s[3] + k*s[4]
 * Strides are in elements.
 */
typedef struct vxb_tensor {
  void *data;
  int32_t dtype;
  int32_t blocked;
  int32_t n, c, x, y, z;
  int32_t pad_;
  int64_t s[5];
} vxb_tensor;

/*
 * One fused convolution step: y = act(bias' + [scale.]base + sum x*K').
 * Replaces _kernels.conv3d (_kernels.pyx:44-179) as driven by
 * kernels_cy.conv3d (kernels_cy.py:49-57) over a ConvInvocation
 * (kernels_py.py:24-44).  Zero padding is virtual: input coordinates
 * outside [0, extent) read as zero (TMA out-of-bounds fill), which replaces
 * the reference's Pad step / halo buffers (ops.py:105-110, ir.py:343-383).
 * Two input segments may be given: the conv then reads channels of in0
 * followed by channels of in1, i.e. a fused MergeCrop (ops.py:113-136);
 * off0/off1 are the per-segment crop offsets in voxels.
 */
typedef struct vxb_conv_desc {
  vxb_tensor in0;
  vxb_tensor in1;          /* in1.data == NULL: single input */
  int32_t off0[3], off1[3];
  vxb_tensor out;          /* out view; logical (n, cout, ox, oy, oz) */
  vxb_tensor base;         /* base.data == NULL: not additive */
  const void *w_packed;    /* from vxb_conv_pack_weights */
  const float *bias;       /* [cout] fp32 */
  const float *base_scale; /* [cout] fp32 or NULL */
  int32_t cin, cout;
  int32_t k[3];
  int32_t stride[3];
  int32_t pad[3];
  int32_t act;
  float alpha;
  int32_t path;            /* 0 = auto (vxb_conv_select) */
  int32_t pool_mode;       /* VXB_POOL_FUSED_*: also write the pooled output (ops.pool fused) */
  int32_t prec;            /* VXB_PREC_* the weights were packed with (X3 <=> split input) */
  int32_t reserved[5];
  vxb_tensor pool_out;     /* pooled view, logical (n, cout, ox, oy/2, oz/2) */
  /* Fused 1x1x1 head: the network's next step when it is a 1x1x1 conv that
   * alone reads this conv's output (the U-nets' output layer, SURVEY §8f
   * rank 3).  head_out = head_act(head_b + head_w . y), y = this conv's
   * activated output per voxel, which is then never stored (out gives only
   * the shape).  head_w: (head_cout, cout) fp32; head_out: fp32 standard
   * (NCDHW) view (n, head_cout, ox, oy, oz).  head_cout 0 = no head. */
  const float *head_w;
  const float *head_b;
  int32_t head_cout;       /* 0 .. 4 */
  int32_t head_act;        /* VXB_ACT_* */
  float head_alpha;
  int32_t head_reserved_;
  vxb_tensor head_out;
} vxb_conv_desc;

/* Transposed convolution (kernels_py.deconv3d, kernels_py.py:162-196):
 * out = act(bias + [base] + scatter_taps(in @ W_tap)).  k == stride takes the
 * tensor-core path (one 1x1x1 GEMM per tap, written to a strided output
 * view); other geometries take a gather kernel on CUDA cores. */
typedef struct vxb_deconv_desc {
  vxb_tensor in;
  vxb_tensor out;
  vxb_tensor base;         /* optional fused skip-add operand (same shape as out) */
  const void *w_packed;    /* from vxb_deconv_pack_weights */
  const float *bias;
  const float *base_scale;
  int32_t cin, cout;
  int32_t k[3];
  int32_t stride[3];
  int32_t act;
  float alpha;
  int32_t path;            /* 0 = auto, VXB_PATH_TC (k == stride), VXB_PATH_DIRECT (gather) */
  int32_t prec;            /* VXB_PREC_* the weights were packed with (X3 <=> split input) */
  int32_t reserved[6];
} vxb_deconv_desc;

/* ---- library ---- */
int vxb_abi_version(void);
const char *vxb_last_error(void);
/* number of SMs of the current device, or -1 */
int vxb_device_sms(void);
/* debug: with VXB_TC_DEBUG=1 the tensor-core conv records per-tile phase
 * timestamps (ns, [cta][tile<64][8]) of its last launch; copies up to count */
size_t vxb_debug_read(unsigned long long *host, size_t count);

/* launches from the calling host thread use programmatic dependent launch
 * (mode 1), plain stream order (0), or the VXB_PDL environment default (-1,
 * on); returns the previous mode.  Graph captures record the mode in force. */
int vxb_set_pdl(int mode);

/* ---- convolution (kernels_cy.conv3d / _kernels.conv3d) ---- */
int vxb_conv_select(int cin, int cout, const int k[3], const int stride[3]);
/* as vxb_conv_select, knowing the output extent: a 1x3x3 conv whose x extent
 * pads badly to the 16-row tiles of y-sliced folding (e.g. x = 18) gets
 * VXB_PATH_TC_UNFOLDED; a layer with too few output tiles to fill the SMs
 * (deep U-net levels) splits its output fmaps into narrower N tiles
 * (VXB_PATH_TC_N128 / _N64).  Replaces the same per-layer choice the
 * reference makes once per bind (kernels_cy.py:22-27 lane-kernel cache). */
int vxb_conv_select_shape(int cin, int cout, const int k[3], const int stride[3],
                          const int out_xyz[3]);
/* as vxb_conv_select_shape for a launch over `batch` volumes of that extent
 * (the N-tile split counts the tiles of every batch entry) */
int vxb_conv_select_shape_b(int cin, int cout, const int k[3], const int stride[3],
                            const int out_xyz[3], int batch);
/* bytes of the packed weight image for a conv of this geometry */
size_t vxb_conv_weights_bytes(int cin, int cout, const int k[3], const int stride[3],
                              int path);
/* host-side packing of a standard (cout, cin, kx, ky, kz) fp32 kernel bank
 * (the reference's weight order, shapes.py:104-110) into dst (host memory);
 * replaces blocked.kernel_to_blocked + kernels_cy._lane_kernel
 * (blocked.py:260-278, kernels_cy.py:22-27). */
int vxb_conv_pack_weights(const float *w, int cin, int cout, const int k[3],
                          const int stride[3], int path, void *dst, size_t dst_bytes);
/* two-segment variants for a conv fused with MergeCrop: the first cin0
 * input fmaps come from in0, the next cin1 from in1 (ops.py:113-136) */
size_t vxb_conv_weights_bytes2(int cin0, int cin1, int cout, const int k[3],
                               const int stride[3], int path);
int vxb_conv_pack_weights2(const float *w, int cin0, int cin1, int cout, const int k[3],
                           const int stride[3], int path, void *dst, size_t dst_bytes);
/* precision-aware variants: prec VXB_PREC_BF16 is the plain packing above;
 * VXB_PREC_X3 packs the weights of a conv whose input is split bf16
 * (VXB_BF16X2, single input segment: cin1 must be 0) */
size_t vxb_conv_weights_bytes3(int cin0, int cin1, int cout, const int k[3],
                               const int stride[3], int path, int prec);
int vxb_conv_pack_weights3(const float *w, int cin0, int cin1, int cout, const int k[3],
                           const int stride[3], int path, int prec, void *dst,
                           size_t dst_bytes);
int vxb_conv3d(const vxb_conv_desc *d, void *stream);

/* Sub-image primitive (kernels_py.subimage / _kernels.subimage,
 * _kernels.pyx:182-271): one input chunk's contribution to one output patch,
 * through memory.  first: init from bias (+[scale.]base); last: apply act.
 * Debug/test entry, CUDA cores, fp32 weights (cout, cin, k) standard order. */
int vxb_conv3d_subimage(const vxb_conv_desc *d, const float *w_std, int in_chunk,
                        int out_chunk, const int origin[3], const int extent[3],
                        int first, int last, void *stream);

/* ---- deconvolution ---- */
size_t vxb_deconv_weights_bytes(int cin, int cout, const int k[3], const int stride[3],
                                int path);
int vxb_deconv_pack_weights(const float *w, int cin, int cout, const int k[3],
                            const int stride[3], int path, void *dst, size_t dst_bytes);
size_t vxb_deconv_weights_bytes3(int cin, int cout, const int k[3], const int stride[3],
                                 int path, int prec);
int vxb_deconv_pack_weights3(const float *w, int cin, int cout, const int k[3],
                             const int stride[3], int path, int prec, void *dst,
                             size_t dst_bytes);
int vxb_deconv3d(const vxb_deconv_desc *d, void *stream);

/* ---- bandwidth kernels (ops.py) ---- */
/* ops.pool, ops.py:63-86 (window/stride per axis, no border handling) */
int vxb_pool3d(const vxb_tensor *in, const vxb_tensor *out, const int window[3],
               const int stride[3], int mode, void *stream);
/* ops.eltwise, ops.py:50-60 */
int vxb_eltwise(const vxb_tensor *a, const vxb_tensor *b, const vxb_tensor *out, int op,
                void *stream);
/* ops.linear_transform + ops.activation (ops.py:89-102), fused:
 * out = act(x*mult + add); mult/add NULL = identity; act VXB_ACT_* */
int vxb_affine_act(const vxb_tensor *in, const vxb_tensor *out, const float *mult,
                   const float *add, int act, float alpha, void *stream);
/* ops.mergecrop, ops.py:113-136 + shapes.crop_offsets (shapes.py:35-37) */
int vxb_mergecrop(const vxb_tensor *a, const vxb_tensor *b, const vxb_tensor *out,
                  void *stream);
/* ops.pad_copy, ops.py:105-110 (out is the dense inflated tensor) */
int vxb_pad_copy(const vxb_tensor *in, const vxb_tensor *out, const int pads[3],
                 void *stream);
/* layout transforms to_blocked / from_blocked (blocked.py:209-231):
 * generic strided copy between any two views of the same logical shape,
 * converting dtype; tail lanes of a blocked destination are zeroed. */
int vxb_copy(const vxb_tensor *src, const vxb_tensor *dst, void *stream);
/* count (src[i] -> dst[i]) copies of equally shaped fp32 standard views
 * (z contiguous) in one launch per 16: the patch gather / scatter of tiled
 * execution (the reference's per-tile numpy slicing, tiling.py:189-237) */
int vxb_copy_windows(const vxb_tensor *src, const vxb_tensor *dst, int count, void *stream);
/* vxb_pack_zwin over a batch whose entry b is read from window src[b]
 * (1-channel fp32 views into one volume): the patch gather of a tiled run
 * fused into the network's input pack; count == dst->n <= 64 */
int vxb_pack_zwin_windows(const vxb_tensor *src, int count, const vxb_tensor *dst, int kz, int pz,
                          void *stream);
/* vxb_copy with flags.  VXB_COPY_INDEPENDENT: the copy reads nothing the
 * previous kernel in the stream writes and writes nothing it touches (a
 * network-input pack), so it may start beside that kernel instead of after
 * it (programmatic launch without a grid-dependency wait).  Used by
 * PlanBatch to overlap one network's input pack with the previous network's
 * convolution (runner.py). */
#define VXB_COPY_INDEPENDENT 1
int vxb_copy_ex(const vxb_tensor *src, const vxb_tensor *dst, int flags, void *stream);
/* z-window pack of a 1-channel fp32 network input for a conv with kz z-taps
 * and z padding pz (the first layer of both U-nets; blocked.to_blocked,
 * blocked.py:209-231, followed by the conv's own z taps): lane l of dst voxel
 * (x, y, z) = src(x, y, z + l - pz) (zero outside), lanes >= kz zero, so the
 * conv runs as a (kx, ky, 1) kernel over kz lanes with
 * w'(co, l, dx, dy, 0) = w(co, 0, dx, dy, l).  dst: bf16 blocked, c == kz,
 * z == src z + 2 pz - kz + 1.  flags: VXB_COPY_INDEPENDENT as for vxb_copy_ex. */
int vxb_pack_zwin(const vxb_tensor *src, const vxb_tensor *dst, int kz, int pz, int flags,
                  void *stream);
/* fill a whole view (all lanes) with zeros */
int vxb_zero(const vxb_tensor *t, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* VXB_H */
