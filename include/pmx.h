/*
 * pmx.h -- C ABI of libpmx.so, the sm_100a kernels behind the pillarmix-compatible
 * API (package paper_2601_12638_b200).
 *
 * The reference (pillarmix, /root/reference/pkg/src/pillarmix = "pm/") is pure
 * Python + numpy and has no FFI: its seam is the Python functions listed per
 * entry point below.  Each entry point replaces one of them; the Python host
 * layer (paper_2601_12638_b200/*.py) keeps the reference names, argument meaning
 * and exception types, and binds this header through ctypes
 * (paper_2601_12638_b200/_native.py).  INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Every buffer is caller-owned DEVICE memory
 *    unless the parameter name says host; the library never allocates on the hot
 *    path (scratch comes in through `ws`).
 *  - Every call is stream-ordered on `stream` (a cudaStream_t) and asynchronous;
 *    no call synchronises the device, so all of them can be captured into CUDA
 *    graphs.
 *  - Activations are NHWC.  Frames of a batch are independent.
 *  - Status codes: 0 = ok.  On failure pmx_last_error() (thread-local) holds a
 *    message; the Python layer maps PMX_ERR_INVALID to ValueError and the others
 *    to RuntimeError, mirroring the reference's exception types.
 *  - No CPU fallback exists: without a CUDA device every call fails with
 *    PMX_ERR_CUDA.
 */
#ifndef PMX_H_
#define PMX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* pmx_stream_t; /* == cudaStream_t */

typedef enum {
  PMX_OK = 0,
  PMX_ERR_INVALID = 1,     /* bad shape / argument (ValueError in Python) */
  PMX_ERR_CUDA = 2,        /* CUDA runtime failure or no device */
  PMX_ERR_UNSUPPORTED = 3  /* valid request outside what the kernels cover */
} pmx_status;

/* PMX_F32X2: an f32 activation stored as a (hi, lo) pair for the 3xTF32 tensor-core
 * path of FP32 layers -- hi = the value rounded to TF32 (nearest even, low 13
 * mantissa bits zero), lo = value - hi (exact in f32), hi + lo == value bit for bit.
 * A pixel holds 2S f32 elements: hi of channel c at [c], lo at [S + c], so the
 * c_stride of an F32X2 tensor is 2S and the lo plane is c_stride / 2 away. */
typedef enum { PMX_F32 = 0, PMX_F16 = 1, PMX_I8 = 2, PMX_F64 = 3, PMX_F32X2 = 4 } pmx_dtype;

#define PMX_ABI_VERSION 3

const char* pmx_last_error(void);
int32_t pmx_abi_version(void);
/* Name of the conv backend pmx_conv() uses for (in_dtype, kind): "tcgen05" or "simt". */
const char* pmx_conv_backend(int32_t in_dtype, int32_t kind);
/* Stream-ordered zero fill (canvas clearing; cudaMemsetAsync, graph-capturable). */
pmx_status pmx_zero(void* ptr, size_t bytes, pmx_stream_t stream);

/* ------------------------------------------------------------------------
 * K1 quantization math -- replaces pm/quant.py:98-147.
 * Codes are bit-exact with clip(rint(f64(x) / scale), -128, 127): an f32
 * estimate is refined by an IEEE f64 division inside a guard band around
 * every .5 tie.
 * ---------------------------------------------------------------------- */

/* pm/quant.py:98-103 quantize(x, QuantParams(scale)) -> int codes (int32 out, like numpy).
 * x_dtype: PMX_F32 (activations; guard-band kernel) or PMX_F64 (API inputs that
 * are not f32, divided in f64 directly as the reference does). */
pmx_status pmx_quantize(const void* x, int32_t x_dtype, int64_t n, double scale, int32_t* codes,
                        pmx_stream_t stream);
/* pm/quant.py:114-116 fake_quant(t, qp) -> f32(f64(code) * scale). */
pmx_status pmx_fake_quant(const void* x, int32_t x_dtype, int64_t n, double scale, float* out,
                          pmx_stream_t stream);
/* pm/quant.py:136-141 (codes part) and pm/model.py:276-279: per-row (axis 0)
 * weight quantization.  `scales` is a device f64 [rows] array.  Writes int8
 * codes (may be NULL) and the dequantized f32 weight (may be NULL). */
pmx_status pmx_quantize_rows(const float* w, int64_t rows, int64_t cols, const double* scales,
                             int8_t* codes, float* dequant, pmx_stream_t stream);
/* pm/quant.py:144-147 fp16_roundtrip: clip +-65504, RNE to binary16.  Either
 * output may be NULL: f32 round-tripped values and/or raw binary16 bits. */
pmx_status pmx_fp16_roundtrip(const float* x, int64_t n, float* out_f32, uint16_t* out_f16,
                              pmx_stream_t stream);

/* ------------------------------------------------------------------------
 * K2 min/max observers -- replaces pm/quant.py:179-188 and the observe_fn
 * record of pm/calibration.py:116-124.  Observers are device uint32 pairs of
 * order-preserving float keys {min_key, max_key}; widen with atomics, so they
 * are exact and order-independent.  Decode: key>=0x80000000 ? key^0x80000000
 * : ~key gives the float bits.  NaN/Inf widen the pair to a non-finite value,
 * which the host reports like the reference.
 * ---------------------------------------------------------------------- */
pmx_status pmx_minmax_init(uint32_t* keys, int64_t n_pairs, pmx_stream_t stream);
pmx_status pmx_minmax(const void* x, int64_t n, int32_t dtype, uint32_t* keys,
                      pmx_stream_t stream);
/* f64 observer (API inputs in f64, e.g. pm/quant.py:179-188 on float64 arrays):
 * same protocol with uint64 keys {min_key, max_key}. */
pmx_status pmx_minmax_f64_init(uint64_t* keys, pmx_stream_t stream);
pmx_status pmx_minmax_f64(const double* x, int64_t n, uint64_t* keys, pmx_stream_t stream);

/* ------------------------------------------------------------------------
 * K3 pillarize -- replaces pm/scenes.py:155-193 (binning, ascending flat-id
 * pillar order, first-come truncation to max_points), extended with an origin
 * offset and a max-pillars cap (keep the cells whose first point has the
 * smallest scene index; identity when the cap does not bind).
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t grid_h;      /* rows (y) */
  int32_t grid_w;      /* cols (x) */
  int32_t max_points;  /* M, points kept per pillar (1..32) */
  int32_t max_pillars; /* P cap; <= 0 means uncapped (then Pcap must be grid_h*grid_w) */
  float x_min, y_min;  /* origin */
  float cell_w, cell_h;
} pmx_grid;

/* Scratch bytes for pmx_pillarize. */
size_t pmx_pillarize_workspace(const pmx_grid* grid, int32_t batch, int64_t max_points_per_frame);

/* points: [total, 4] f32 (x, y, z|intensity, r) rows, frames concatenated;
 * frame_offsets: device int64 [batch + 1].  Outputs per frame b (Pcap slots):
 * coords [B, Pcap, 2] int32 (row, col); counts [B, Pcap] int32 kept points;
 * pt_idx [B, Pcap, M] int32 frame-local point index in scene order, -1 padding;
 * n_pillars [B] int32.  Slots >= n_pillars are left untouched. */
pmx_status pmx_pillarize(const float* points, const int64_t* frame_offsets, int32_t batch,
                         int64_t max_points_per_frame, const pmx_grid* grid, int32_t pcap,
                         int32_t* coords, int32_t* counts, int32_t* pt_idx, int32_t* n_pillars,
                         void* ws, size_t ws_bytes, pmx_stream_t stream);

/* The cell -> pillar-slot map pmx_pillarize leaves in `ws`: device int32
 * [B, grid_h, grid_w], the kept pillar's slot + 1 in that cell, 0 if empty
 * (every cell is written on every call; valid until `ws` is reused).  Input of
 * pmx_conv_gather.  Returns NULL on bad arguments. */
const int32_t* pmx_pillarize_cell_map(const pmx_grid* grid, int32_t batch, int64_t max_points_per_frame,
                                      const void* ws);

/* Materialise padded per-pillar features [B, Pcap, M, F] f32 (zero padded) and
 * the mask [B, Pcap, M] u8 -- the PillarSample of pm/tensor_ops.py:60-77.
 * n_features = 5: (x, y, i, x-mx, y-my), pm/scenes.py:186-192 (points' third
 * column is the intensity); n_features = 9: (x, y, z, r, x-mx, y-my, z-mz,
 * x-xc, y-yc), SURVEY App. B.2. */
pmx_status pmx_pillar_features(const float* points, const int64_t* frame_offsets, int32_t batch,
                               const pmx_grid* grid, int32_t pcap, int32_t n_features,
                               const int32_t* coords, const int32_t* counts,
                               const int32_t* pt_idx, const int32_t* n_pillars, float* features,
                               uint8_t* mask, pmx_stream_t stream);

/* ------------------------------------------------------------------------
 * Output descriptor shared by the layer kernels: the producer epilogue writes
 * its (post-BN, post-ReLU) f32 value once per consumer format.  Heads use F32.
 * ---------------------------------------------------------------------- */
typedef struct {
  void* ptr;         /* NHWC destination */
  double scale;      /* PMX_I8 only: consumer activation scale (codes = quantize(y, scale)) */
  int32_t dtype;     /* PMX_F32 / PMX_F16 / PMX_I8 / PMX_F32X2 */
  int32_t c_stride;  /* elements per pixel in the destination (PMX_F32X2: 2S, both planes) */
  int32_t c_offset;  /* first destination channel (concat slice) */
  int32_t _reserved;
} pmx_out;

#define PMX_MAX_OUTS 3

/* ------------------------------------------------------------------------
 * K4+K5 fused pillar feature net: (feature augmentation) -> layer-1 precision
 * transform -> linear -> folded BN -> ReLU -> masked max over points -> scatter
 * onto the NHWC canvas in every consumer format.  Replaces pm/model.py:334-355
 * (linear branch of _run_weight_layer :271-307, max_over_points
 * pm/tensor_ops.py:163-173, scatter_pillars :138-160).  The canvas must be
 * zeroed by the caller (cudaMemsetAsync) -- empty cells stay 0 in every format.
 * ---------------------------------------------------------------------- */
enum { PMX_PFN_FROM_POINTS9 = 0, PMX_PFN_FROM_FEATURES = 1 };

typedef struct {
  int32_t source;     /* PMX_PFN_FROM_POINTS9 or PMX_PFN_FROM_FEATURES */
  int32_t in_dtype;   /* layer-1 precision (PMX_F32/F16/I8) */
  int32_t n_features; /* F: 9 for POINTS9, any 1..16 for FROM_FEATURES */
  int32_t channels;   /* C out, 1..64 */
  int32_t max_points; /* M */
  int32_t relu;
  double in_scale;    /* PMX_I8: layer-1 activation scale */
} pmx_pfn_desc;

/* weight: [C, F] in the layer precision (f32 / f16 bits / int8 codes);
 * alpha: PMX_I8 only, f32(s_x * s_w[c]) per channel; bias [C] f32 (BN folded).
 * FROM_FEATURES reads features [B, Pcap, M, F] f32 + mask [B, Pcap, M] u8;
 * POINTS9 recomputes the 9 features from points + pt_idx.
 * in_keys (may be NULL): observer of layer 1's input (features incl. padding);
 * out_keys (may be NULL): observer of the canvas (pooled values, 0 if any cell empty). */
pmx_status pmx_pfn_scatter(const pmx_pfn_desc* desc, const pmx_grid* grid, int32_t batch,
                           int32_t pcap, const float* points, const int64_t* frame_offsets,
                           const float* features, const uint8_t* mask, const int32_t* coords,
                           const int32_t* counts, const int32_t* pt_idx,
                           const int32_t* n_pillars, const void* weight, const float* alpha,
                           const float* bias, const float* bn_post, const pmx_out* outs,
                           int32_t n_outs, uint32_t* in_keys, uint32_t* out_keys,
                           pmx_stream_t stream);

/* Same computation as pmx_pfn_scatter, but the pooled pillar features are written
 * densely per pillar slot -- outs[o] row b * pcap + p, rows >= n_pillars[b]
 * untouched -- instead of onto a canvas (scatter_pillars pm/tensor_ops.py:138-160
 * then happens virtually inside pmx_conv_gather: no canvas memset or write). */
pmx_status pmx_pfn_pillars(const pmx_pfn_desc* desc, const pmx_grid* grid, int32_t batch,
                           int32_t pcap, const float* points, const int64_t* frame_offsets,
                           const float* features, const uint8_t* mask, const int32_t* coords,
                           const int32_t* counts, const int32_t* pt_idx,
                           const int32_t* n_pillars, const void* weight, const float* alpha,
                           const float* bias, const float* bn_post, const pmx_out* outs,
                           int32_t n_outs, uint32_t* in_keys, uint32_t* out_keys,
                           pmx_stream_t stream);

/* ------------------------------------------------------------------------
 * K6-K10 implicit-GEMM layer kernel -- replaces conv2d pm/tensor_ops.py:109-131
 * / linear :80-91 under the precision dispatch of pm/model.py:271-307, plus the
 * KITTI neck deconvolution (kernel == stride).
 *   INT8: int8 codes x int8 codes -> exact int32, y = f32(acc) * alpha[c] + bias[c]
 *   FP16: binary16 x binary16 -> f32, y = acc + bias[c]
 *   FP32: f32 x f32 -> f32,          y = acc + bias[c]
 *   FP32 as PMX_F32X2 (3xTF32 on tcgen05): x = hi + lo, w = w_hi + w_lo, acc =
 *         sum hi*w_hi + lo*w_hi + hi*w_lo (kind::tf32, f32 accumulate),
 *         y = acc + bias[c]; in_c_stride / in_c_offset count f32 elements of the
 *         hi plane's pixel (lo at + in_c_stride / 2); weights are prepacked per tap
 *         as [w_hi | w_hi | w_lo] (K = taps * 3 * Cin, w_hi = tf32 rounding of w).
 * then ReLU, then one store per pmx_out (int8 codes are exact quantize()).
 * Weight layouts: CONV2D [Cout, kh, kw, Cin]; DECONV2D [(dy, dx, co), Cin]
 * (k*k*Cout rows).  alpha/bias are per output channel (Cout).
 * ---------------------------------------------------------------------- */
enum { PMX_CONV2D = 0, PMX_DECONV2D = 1 };

typedef struct {
  int32_t kind;         /* PMX_CONV2D / PMX_DECONV2D */
  int32_t in_dtype;     /* layer precision = input and weight storage type */
  int32_t batch, in_h, in_w, in_c;
  int32_t in_c_stride;  /* channels per input pixel in the source buffer (>= in_c) */
  int32_t in_c_offset;  /* first source channel */
  int32_t out_c;
  int32_t k_h, k_w, stride_h, stride_w, pad_h, pad_w;
  int32_t out_h, out_w; /* output extents (deconv: in * stride) */
  int32_t relu;
} pmx_conv_desc;

size_t pmx_conv_workspace(const pmx_conv_desc* desc);
/* Nonzero if pmx_conv runs desc on the tcgen05 tensor-core kernels (0: the SIMT kernel):
 * bit 0 set; bit 1 = the 2-CTA-cluster (cta_group::2, M = 256) plan; bits 2-3 = the
 * operand mode (0 3x3 per-tap TMA, 1 GEMM, 2 halo tile with resident weights). */
int32_t pmx_conv_tc_supported(const pmx_conv_desc* desc);

/* bn_post (may be NULL): unfolded batch norm applied after the bias as
 * (y - mean[c]) * factor[c] + beta[c] in f32 (pm/model.py:252-258); device
 * [3, Cout] = {mean, factor, beta}.  The same argument exists on pmx_pfn_scatter.
 * out_keys (may be NULL): observer widened with every output value y. */
pmx_status pmx_conv(const pmx_conv_desc* desc, const void* x, const void* w, const float* alpha,
                    const float* bias, const float* bn_post, const pmx_out* outs, int32_t n_outs,
                    uint32_t* out_keys, void* ws, size_t ws_bytes, pmx_stream_t stream);

/* pmx_conv on the pillar canvas without materialising it (the first backbone
 * conv): x[b, y, x, c] = feats[(b * pcap + cell_map[b, y, x] - 1) * in_c_stride +
 * in_c_offset + c], or 0 where cell_map == 0.  desc describes the canvas (in_h /
 * in_w = grid, in_c_stride = channels per pillar row).  Bit-identical to pmx_conv
 * on the scattered canvas.  Only the tcgen05 halo shapes (3x3, stride 1/2, 64 or
 * 128 bytes of channels, int8/f16): PMX_ERR_UNSUPPORTED otherwise -- the caller
 * then scatters a canvas and calls pmx_conv. */
int32_t pmx_conv_gather_supported(const pmx_conv_desc* desc); /* 1 if pmx_conv_gather runs desc */
pmx_status pmx_conv_gather(const pmx_conv_desc* desc, const void* feats, const int32_t* cell_map,
                           int32_t pcap, const void* w, const float* alpha, const float* bias,
                           const float* bn_post, const pmx_out* outs, int32_t n_outs,
                           uint32_t* out_keys, pmx_stream_t stream);

/* Force a backend for testing: 0 = automatic, 1 = SIMT reference kernel only,
 * 2 = tcgen05 without the halo variant.  Thread-local: applies to later calls made
 * by the calling thread only (no process-wide state). */
void pmx_set_conv_backend(int32_t mode);
/* Debug (thread-local, like pmx_set_conv_backend): when non-NULL, tcgen05 conv launches record per-role clock64 stamps of
 * CTA 0 into buf[10][64]: rows 0-7 producer/MMA/epilogue hand-offs per tile, row 8
 * = kernel entry, setup done, resident weights landed, teardown; row 9 = MMA loop top. */
void pmx_debug_trace(unsigned long long* buf);
/* Debug (trace builds, -DPMX_CONV_TRACE): every tcgen05 conv CTA launched after this
 * call appends {launch tag << 32 | cta, t_entry, t_after_griddepcontrol_wait, t_exit}
 * (%globaltimer ns) at buf[1 + 4 * atomicAdd(buf[0], 1)]; tags count launches from 0.
 * NULL turns it off.  A no-op in production builds. */
void pmx_debug_timeline(unsigned long long* buf);

/* ------------------------------------------------------------------------
 * K9+K10 fused: a neck deconvolution (kernel == stride, Cout == 128, INT8 or FP16
 * input) whose output feeds only the concat of the three 1x1 INT8 heads
 * (pm/model.py:329-331 heads on the trunk; pm/model.py:271-307 INT8 head inputs).
 * The deconv's output tile is quantized with the heads' activation scale (the int8
 * codes the concat would hold) and multiplied right away, on the tensor core, by its
 * 128-channel slice of the heads' weight codes; the int32 partial sums of the heads
 * (order-free, exact) accumulate over the three deconvs in `partial`, and the last one
 * applies the heads' epilogue -- so the 384-channel concat is never written or read.
 * Results equal pmx_conv(deconv) -> concat -> pmx_conv(heads) bit for bit.
 * ---------------------------------------------------------------------- */
typedef struct {
  const int8_t* w_codes;    /* [32, 128] int8 head weight codes for this deconv's concat
                               slice (row n = head output channel; rows >= n_heads zero) */
  int32_t n_heads;          /* total head output channels, <= 20 (partial rows hold 20) */
  int32_t stage;            /* 0: write partial; 1: partial += ; 2: partial + this -> heads */
  double in_scale;          /* the heads' activation scale (codes = quantize(y, in_scale)) */
  int32_t* partial;         /* int32 [ps, ps, B, out_h / ps, out_w / ps, 20]: output pixel
                               (b, y, x) at [y % ps, x % ps, b, y / ps, x / ps] */
  float* heads;             /* stage 2: f32 NHWC [B * out_h * out_w, heads_c_stride] */
  int32_t heads_c_stride;
  int32_t part_stride;      /* ps: a power of two dividing out_h and out_w (the largest stride) */
  const float* head_alpha;  /* stage 2: f32(s_in * s_w[n]), [n_heads] */
  const float* head_bias;   /* stage 2: [n_heads] */
} pmx_head_fuse;

/* 1 if pmx_deconv_heads runs desc. */
int32_t pmx_deconv_heads_supported(const pmx_conv_desc* desc);
pmx_status pmx_deconv_heads(const pmx_conv_desc* desc, const void* x, const void* w, const float* alpha,
                            const float* bias, const pmx_head_fuse* heads, pmx_stream_t stream);

/* Stage an f32 [pixels, c] tensor into every consumer format (the precision
 * transform of pm/model.py:273-285 applied to a graph input), optionally
 * widening an observer with its values. */
pmx_status pmx_cast_out(const float* x, int64_t pixels, int32_t c, const pmx_out* outs, int32_t n_outs,
                        uint32_t* keys, pmx_stream_t stream);

/* Nearest 2x upsample of an NHWC tensor (pm/tensor_ops.py:176-178), any dtype. */
pmx_status pmx_upsample2x(const void* x, int32_t dtype, int32_t batch, int32_t h, int32_t w,
                          int32_t c, void* out, pmx_stream_t stream);

/* ------------------------------------------------------------------------
 * K11 anchor decode + top-k (KITTI extension; no reference counterpart --
 * conventions of pm/detector.py:266-307: f64-exact ordering, stable ties).
 * Candidates: flat anchor index a = (y * W + x) * n_anchors + k, ranked by f32
 * cls logit descending, ties to the lower index.  Boxes: SECOND delta coder.
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t n_anchors;   /* A (<= 4); cls has A channels, box 7A, dir 2A */
  int32_t k;           /* top-k (<= 512) */
  float x_min, y_min, stride_x, stride_y;
  float anchor_z, anchor_w, anchor_l, anchor_h;
  float rotations[4];
  float dir_offset;
  float _pad;
} pmx_anchor_desc;

size_t pmx_decode_workspace(const pmx_anchor_desc* desc, int32_t batch, int32_t out_h,
                            int32_t out_w);

/* heads: f32 NHWC [B, H, W, head_c_stride]; cls/box/dir channel offsets.
 * Outputs: topk_idx [B,k] int32, topk_logit [B,k] f32, boxes [B,k,7] f32,
 * dir_label [B,k] int32. */
pmx_status pmx_decode_topk(const pmx_anchor_desc* desc, int32_t batch, int32_t out_h,
                           int32_t out_w, const float* heads, int32_t head_c_stride,
                           int32_t cls_off, int32_t box_off, int32_t dir_off, int32_t* topk_idx,
                           float* topk_logit, float* boxes, int32_t* dir_label, void* ws,
                           size_t ws_bytes, pmx_stream_t stream);

/* ------------------------------------------------------------------------
 * K11b local-peak decode + per-class greedy NMS -- replaces the reference's own
 * decode entry point pm/detector.py:266-307 (decode_and_nms, with _sigmoid
 * :251-252, _local_peaks :255-263, iou_matrix pm/metrics.py:52-66).  f64 scores
 * sigmoid(logit), 3x3 local peaks (ties keep both, NaN never a peak), score >=
 * score_thresh, box = ((j + .5 + dx) * cell_w, (i + .5 + dy) * cell_h,
 * base * exp(clip(dw, +-4)), base * exp(clip(dh, +-4))), stable order by score
 * descending, greedy suppression at IoU >= iou_thresh, classes independent.
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t n_classes, out_h, out_w; /* class map [B, n_classes, out_h, out_w], out_h*out_w <= 16384 */
  int32_t _pad;
  double cell_w, cell_h;           /* field_size / out_w, field_size / out_h */
  double base_size;
  double score_thresh, iou_thresh; /* both in [0, 1] (PMX_ERR_INVALID otherwise, the reference's ValueError) */
} pmx_nms_desc;

/* cls: f32 NCHW [B, n_classes, H, W] logits; reg: f32 NCHW [B, 4, H, W] (dx, dy, dw, dh).
 * dets: f64 [B, n_classes, H*W, 5] -- per (frame, class) the kept detections in the
 * reference's order as (cx, cy, w, h, score); n_dets: int32 [B, n_classes]. */
pmx_status pmx_decode_nms(const pmx_nms_desc* desc, int32_t batch, const float* cls, const float* reg,
                          double* dets, int32_t* n_dets, pmx_stream_t stream);

/* Fixed-size per-frame top-k records for the host / the NCCL gather:
 * records [B, k, 10] f32 = (idx, logit, box[7], dir) with idx and dir as f32
 * (exact below 2^24).  Same layout as paper_2601_12638_b200.distributed.pack_topk;
 * one kernel inside the captured graph instead of four torch ops after it. */
pmx_status pmx_pack_topk_records(int32_t batch, int32_t k, const int32_t* topk_idx,
                                 const float* topk_logit, const float* boxes,
                                 const int32_t* dir_label, float* records, pmx_stream_t stream);

/* ------------------------------------------------------------------------
 * K12 sensitivity-sweep error (BASELINE config 5; SPEC.md:364-372 sweep with the
 * head-output error as the score): out2[0] += sum((a - b)^2), out2[1] += sum(b^2)
 * over n f32 values, accumulated in f64 in a fixed order (deterministic:
 * a fixed number of per-block partials, then one ordered reduction).
 * ws: device scratch of ws_bytes >= pmx_sq_err_workspace() (checked).
 * ---------------------------------------------------------------------- */
size_t pmx_sq_err_workspace(void);
pmx_status pmx_sq_err(const float* a, const float* b, int64_t n, double* out2, double* ws,
                      size_t ws_bytes, pmx_stream_t stream);

/* ------------------------------------------------------------------------
 * QAT (pm/qat.py:79-306) on the GPU: the training forward's pre-activation
 * convolutions and the backward pass over its tape.  f32 throughout; activations
 * NHWC, weights as the model stores them ([Cout, Cin, kh, kw]; a linear layer is a
 * 1x1 conv over rows with batch = rows).  desc: PMX_CONV2D (any kernel / stride /
 * padding) or PMX_DECONV2D (kernel == stride); in_dtype / in_c_stride /
 * in_c_offset / relu are ignored.  Every reduction has a fixed order: a training
 * run is bit-reproducible on one device.
 * ---------------------------------------------------------------------- */
/* out = conv(x, w) + bias, before any ReLU (the tape's pre_act, pm/model.py:286-292) */
pmx_status pmx_train_conv_fwd(const pmx_conv_desc* desc, const float* x, const float* w, const float* bias,
                              float* out, pmx_stream_t stream);
/* dx = the data gradient of dout (pm/qat.py:145-152 col2im; linear :130-131) */
pmx_status pmx_train_conv_dgrad(const pmx_conv_desc* desc, const float* dout, const float* w, float* dx,
                                pmx_stream_t stream);
/* dw = dout^T . im2col(x), db = column sums of dout (pm/qat.py:142-144); either may be NULL */
pmx_status pmx_train_conv_wgrad(const pmx_conv_desc* desc, const float* dout, const float* x, float* dw,
                                float* db, pmx_stream_t stream);
/* np.maximum(x, 0) (NaN propagates) and its adjoint dout * (pre_act > 0) (pm/qat.py:160-161) */
pmx_status pmx_train_relu(const float* x, int64_t n, float* out, pmx_stream_t stream);
pmx_status pmx_train_relu_bwd(const float* dout, const float* pre_act, int64_t n, float* dx, pmx_stream_t stream);
/* clipped STE (pm/qat.py:68-85): out = upstream * (q_min*s <= x <= q_max*s).  Per tensor
 * the bounds are compared as f32 (NumPy 2 promotion of a Python float against an f32
 * array); per row (per-channel weights, scales f64 [rows]) in f64. */
pmx_status pmx_train_ste(const float* x, int64_t n, double scale, int32_t q_min, int32_t q_max,
                         const float* upstream, float* out, pmx_stream_t stream);
pmx_status pmx_train_ste_rows(const float* x, int64_t rows, int64_t cols, const double* scales, int32_t q_min,
                              int32_t q_max, const float* upstream, float* out, pmx_stream_t stream);
/* masked max over points of x [P, M, C] with the np.argmax winner per (pillar, channel)
 * (pm/model.py:338-345); argmax may be NULL.  Adjoint: dx[p, argmax, c] = dout[p, c]. */
pmx_status pmx_train_maxpool(const float* x, const uint8_t* mask, int64_t pillars, int32_t m, int32_t c,
                             float* out, int32_t* argmax, pmx_stream_t stream);
pmx_status pmx_train_maxpool_bwd(const float* dout, const int32_t* argmax, int64_t pillars, int32_t m, int32_t c,
                                 float* dx, pmx_stream_t stream);
/* scatter of pillar rows into a zeroed NHWC canvas (coords int32 [P, 2] = (row, col)) and
 * its adjoint, the gather (pm/tensor_ops.py:138-160, pm/qat.py:184-186) */
pmx_status pmx_train_scatter(const float* feats, const int32_t* coords, int64_t pillars, int32_t c,
                             int32_t grid_w, float* canvas, pmx_stream_t stream);
pmx_status pmx_train_scatter_bwd(const float* dcanvas, const int32_t* coords, int64_t pillars, int32_t c,
                                 int32_t grid_w, float* dfeats, pmx_stream_t stream);
/* adjoint of pmx_upsample2x: each input cell sums its 2x2 block (pm/qat.py:188-190);
 * h, w are the INPUT extents */
pmx_status pmx_train_upsample2x_bwd(const float* dout, int32_t batch, int32_t h, int32_t w, int32_t c,
                                    float* dx, pmx_stream_t stream);
/* out = a + b (f32) -- gradient accumulation, the heads' trunk sum */
pmx_status pmx_train_add(const float* a, const float* b, int64_t n, float* out, pmx_stream_t stream);
/* dst[p, dst_offset + k] = src[p, src_offset + k], k < c: concat and its adjoint */
pmx_status pmx_train_copy_channels(const float* src, int64_t pixels, int32_t c, int32_t src_stride,
                                   int32_t src_offset, float* dst, int32_t dst_stride, int32_t dst_offset,
                                   pmx_stream_t stream);
/* device scratch (bytes) of the f64 reductions below */
size_t pmx_train_reduce_workspace(void);
/* detection_loss (pm/qat.py:92-116) on NHWC maps: cls [hw, n_cls] logits and
 * cls_target (f64), ignore_mask / pos_mask u8 [hw] (ignore may be NULL), reg [hw, n_reg]
 * and reg_target (f64).  d_cls / d_reg get the f32 gradients; sums[0] = sum(w * bce),
 * sums[1] = sum(diff^2), both f64 (the loss is formed on the host). */
pmx_status pmx_train_detection_loss(const float* cls, const double* cls_target, const uint8_t* ignore_mask,
                                    const uint8_t* pos_mask, const float* reg, const double* reg_target,
                                    int64_t hw, int32_t n_cls, int32_t n_reg, double n_pos, double cls_weight,
                                    double reg_weight, double pos_weight, float* d_cls, float* d_reg,
                                    double* sums, double* ws, pmx_stream_t stream);
/* mse_loss (pm/qat.py:119-125): grad = f32(2 (out - target) / n), sum = sum((out - target)^2) */
pmx_status pmx_train_mse_loss(const float* out, const double* target, int64_t n, float* grad, double* sum,
                              double* ws, pmx_stream_t stream);
/* sum of (inv * g)^2 (f32 product and square, f64 sum): the gradient-norm clip */
pmx_status pmx_train_sumsq(const float* g, int64_t n, float inv, double* sum, double* ws, pmx_stream_t stream);
/* SGD step (pm/qat.py:289-301): step = inv * g (momentum: step = mu * v + step, v = step),
 * w -= lr * step, all f32 */
pmx_status pmx_train_sgd(float* w, const float* grad, int64_t n, float inv, float lr, float momentum,
                         float* velocity, pmx_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* PMX_H_ */
