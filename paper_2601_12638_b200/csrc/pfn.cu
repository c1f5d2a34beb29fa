// K4+K5 fused pillar feature net + BEV scatter.
//
// Four threads per pillar, 16 output channels each (64 pillars per 256-thread
// block).  A KITTI pillar holds ~1-3 points, so a lane-per-point warp would idle
// >90% of its lanes; here every thread walks its pillar's points itself: the 9
// features are rebuilt in registers (sequential f32 mean in slot order, matching
// numpy's chunk.mean(axis=0) bit for bit), transformed to layer 1's precision
// (exact int8 codes / binary16 / f32), multiplied against the weights staged once
// per block in shared memory (feature-major, 16-channel float4 rows), max-pooled
// in registers, and the pooled column is written once per consumer format straight
// onto the NHWC canvas (scatter fused; 16-byte vector stores).
// Replaces pm/model.py:334-355 -> _run_weight_layer :271-307 -> linear
// pm/tensor_ops.py:80-91, relu :134, max_over_points :163-173, scatter :138-160.
// INT8: features and weights are integer codes; the 9-term dot product of codes
// (|sum| < 2^18) is exact in f32 FMA, then y = fma(acc, s_x * s_w[c], bias[c]).
#include "pmx_common.cuh"

namespace pmx {

namespace {

constexpr int kMaxF = 16;
constexpr int kMaxC = 64;
constexpr int kTPP = 4;                      // threads per pillar
constexpr int kThreads = 256;
constexpr int kPPB = kThreads / kTPP;        // pillars per block

struct PfnArgs {
  pmx_pfn_desc d;
  pmx_grid g;
  int32_t pcap;
  const float4* points;
  const int64_t* offs;
  const float* features;
  const uint8_t* mask;
  const int32_t* coords;
  const int32_t* counts;
  const int32_t* pt_idx;
  const int32_t* n_pillars;
  const void* weight;
  const float* alpha;
  const float* bias;
  const float* bn_post;
  float in_inv;
  uint32_t* in_keys;
  uint32_t* out_keys;
  int dense;  // pmx_pfn_pillars: rows are pillar slots (b * pcap + p), no canvas
};

template <int DT>
__device__ __forceinline__ float transform_in(float v, const PfnArgs& a) {
  if constexpr (DT == PMX_I8) return (float)quantize_fast(v, a.d.in_scale, a.in_inv);
  else if constexpr (DT == PMX_F16) return __half2float(f16_sat(v));
  else return v;
}

template <int DT, int NF, bool FROM_POINTS>
__global__ void __launch_bounds__(kThreads) pfn_kernel(const PfnArgs a, const Outs outs) {
  __shared__ __align__(16) float ws[kMaxF][kMaxC];  // weights, feature-major
  __shared__ __align__(16) float ps[3][kMaxC];      // alpha (I8), bias, unused
  const int b = blockIdx.y;
  const int F = FROM_POINTS ? 9 : NF;
  const int C = a.d.channels;
  const int M = a.d.max_points;
  for (int e = threadIdx.x; e < kMaxF * kMaxC; e += kThreads) {
    const int j = e / kMaxC, c = e % kMaxC;
    float w = 0.f;
    if (j < F && c < C) {
      if constexpr (DT == PMX_I8) w = (float)reinterpret_cast<const int8_t*>(a.weight)[c * F + j];
      else if constexpr (DT == PMX_F16) w = __half2float(reinterpret_cast<const __half*>(a.weight)[c * F + j]);
      else w = reinterpret_cast<const float*>(a.weight)[c * F + j];
    }
    ws[j][c] = w;
  }
  for (int c = threadIdx.x; c < kMaxC; c += kThreads) {
    ps[0][c] = (DT == PMX_I8 && c < C) ? a.alpha[c] : 1.f;
    ps[1][c] = c < C ? a.bias[c] : 0.f;
  }
  __syncthreads();

  const int P = a.n_pillars[b];
  const int64_t hw = (int64_t)a.g.grid_h * a.g.grid_w;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t zk = f2key(0.0f);
    if (a.out_keys && P < hw) {  // empty cells stay 0 on the canvas
      atomicMin(a.out_keys + 0, zk);
      atomicMax(a.out_keys + 1, zk);
    }
    if (a.in_keys && P == 0) {  // record() of an empty tensor is (0, 0)
      atomicMin(a.in_keys + 0, zk);
      atomicMax(a.in_keys + 1, zk);
    }
  }
  const int p = blockIdx.x * kPPB + threadIdx.x / kTPP;
  const int cq = threadIdx.x % kTPP;
  const int c0 = cq * 16;
  const bool live = p < P && c0 < C;
  const int64_t q = (int64_t)b * a.pcap + (p < P ? p : 0);
  const float INF = __int_as_float(0x7f800000);
  float in_lo = INF, in_hi = -INF;

  float mx[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) mx[j] = -INF;

  if (live) {
    int k;
    float4 ctr = make_float4(0.f, 0.f, 0.f, 0.f);  // cluster mean (x, y, z), pillar centre offsets
    float xc = 0.f, yc = 0.f;
    const float4* fp = nullptr;
    if (FROM_POINTS) {
      k = a.counts[q];
      fp = a.points + a.offs[b];
      float sx = 0.f, sy = 0.f, sz = 0.f;
      for (int s = 0; s < k; ++s) {
        const float4 pt = __ldg(fp + a.pt_idx[q * M + s]);
        sx = __fadd_rn(sx, pt.x);
        sy = __fadd_rn(sy, pt.y);
        sz = __fadd_rn(sz, pt.z);
      }
      const float fk = (float)(k > 0 ? k : 1);
      ctr = make_float4(__fdiv_rn(sx, fk), __fdiv_rn(sy, fk), __fdiv_rn(sz, fk), 0.f);
      const float xoff = (float)((double)a.g.cell_w * 0.5 + (double)a.g.x_min);
      const float yoff = (float)((double)a.g.cell_h * 0.5 + (double)a.g.y_min);
      xc = __fadd_rn(__fmul_rn((float)a.coords[2 * q + 1], a.g.cell_w), xoff);
      yc = __fadd_rn(__fmul_rn((float)a.coords[2 * q + 0], a.g.cell_h), yoff);
      if (k < M) { in_lo = 0.f; in_hi = 0.f; }  // zero padding rows are part of layer 1's input
    } else {
      k = M;
    }
    for (int s = 0; s < k; ++s) {
      float f[kMaxF];
#pragma unroll
      for (int j = 0; j < kMaxF; ++j) f[j] = 0.f;
      if (FROM_POINTS) {
        const float4 pt = __ldg(fp + a.pt_idx[q * M + s]);
        f[0] = pt.x; f[1] = pt.y; f[2] = pt.z; f[3] = pt.w;
        f[4] = __fsub_rn(pt.x, ctr.x); f[5] = __fsub_rn(pt.y, ctr.y); f[6] = __fsub_rn(pt.z, ctr.z);
        f[7] = __fsub_rn(pt.x, xc); f[8] = __fsub_rn(pt.y, yc);
      } else {
        const float* src = a.features + (q * M + s) * F;
#pragma unroll
        for (int j = 0; j < kMaxF; ++j)
          if (j < F) f[j] = src[j];
      }
      if (a.in_keys) {
#pragma unroll
        for (int j = 0; j < kMaxF; ++j)
          if (j < F) { in_lo = nmin(in_lo, f[j]); in_hi = nmax(in_hi, f[j]); }
      }
      if (!FROM_POINTS && a.mask[q * M + s] == 0) continue;  // padding row: no effect on the max
#pragma unroll
      for (int j = 0; j < kMaxF; ++j)
        if (j < F) f[j] = transform_in<DT>(f[j], a);
      float acc[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) acc[c] = 0.f;
#pragma unroll
      for (int j = 0; j < kMaxF; ++j) {
        if (j < F) {
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const float4 w4 = *reinterpret_cast<const float4*>(&ws[j][c0 + 4 * c4]);
            acc[4 * c4 + 0] = __fmaf_rn(f[j], w4.x, acc[4 * c4 + 0]);
            acc[4 * c4 + 1] = __fmaf_rn(f[j], w4.y, acc[4 * c4 + 1]);
            acc[4 * c4 + 2] = __fmaf_rn(f[j], w4.z, acc[4 * c4 + 2]);
            acc[4 * c4 + 3] = __fmaf_rn(f[j], w4.w, acc[4 * c4 + 3]);
          }
        }
      }
      if (a.bn_post == nullptr) {
        // y = fl(acc * alpha + bias) (alpha > 0) and ReLU are monotone, so the max over
        // points commutes with the epilogue: pool the raw sums, finish once below
#pragma unroll
        for (int c = 0; c < 16; ++c) mx[c] = nmax(mx[c], acc[c]);
      } else {
        // unfolded BN may have a negative gamma: finish every point (rare path)
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          float y;
          if constexpr (DT == PMX_I8) y = __fmaf_rn(acc[c], ps[0][c0 + c], ps[1][c0 + c]);
          else y = __fadd_rn(acc[c], ps[1][c0 + c]);
          if (c0 + c < C)
            y = __fadd_rn(__fmul_rn(__fsub_rn(y, a.bn_post[c0 + c]), a.bn_post[C + c0 + c]),
                          a.bn_post[2 * C + c0 + c]);
          if (a.d.relu) y = fmaxf(y, 0.f);
          mx[c] = nmax(mx[c], y);
        }
      }
    }
    if (a.bn_post == nullptr) {
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        float y;
        if constexpr (DT == PMX_I8) y = __fmaf_rn(mx[c], ps[0][c0 + c], ps[1][c0 + c]);
        else y = __fadd_rn(mx[c], ps[1][c0 + c]);
        if (a.d.relu) y = fmaxf(y, 0.f);
        mx[c] = y;
      }
    }
    // scatter the pooled 16-channel run onto the canvas, every consumer format
    const int64_t pix =
        a.dense ? q : ((int64_t)b * a.g.grid_h + a.coords[2 * q]) * a.g.grid_w + a.coords[2 * q + 1];
    const int n_live = C - c0 < 16 ? C - c0 : 16;
#pragma unroll
    for (int o = 0; o < PMX_MAX_OUTS; ++o)
      if (o < outs.n) store16(outs.o[o], pix, c0, mx, n_live);
  }
  if (a.in_keys) block_minmax_commit<kThreads>(in_lo, in_hi, a.in_keys);
  if (a.out_keys) {
    float lo = INF, hi = -INF;
    if (live) {
      const int n_live = C - c0 < 16 ? C - c0 : 16;
      for (int c = 0; c < n_live; ++c) { lo = nmin(lo, mx[c]); hi = nmax(hi, mx[c]); }
    }
    block_minmax_commit<kThreads>(lo, hi, a.out_keys);
  }
}

template <int DT>
pmx_status launch_dt(const PfnArgs& a, const Outs& outs, dim3 grid, cudaStream_t st) {
  if (a.d.source == PMX_PFN_FROM_POINTS9) {
    pfn_kernel<DT, 9, true><<<grid, kThreads, 0, st>>>(a, outs);
  } else {
    switch (a.d.n_features) {
#define PMX_F_CASE(N) \
  case N:             \
    pfn_kernel<DT, N, false><<<grid, kThreads, 0, st>>>(a, outs); break;
      PMX_F_CASE(1) PMX_F_CASE(2) PMX_F_CASE(3) PMX_F_CASE(4) PMX_F_CASE(5) PMX_F_CASE(6)
      PMX_F_CASE(7) PMX_F_CASE(8) PMX_F_CASE(9) PMX_F_CASE(10) PMX_F_CASE(11) PMX_F_CASE(12)
      PMX_F_CASE(13) PMX_F_CASE(14) PMX_F_CASE(15) PMX_F_CASE(16)
#undef PMX_F_CASE
      default:
        return fail(PMX_ERR_INVALID, "n_features must be 1..16");
    }
  }
  return check_launch("pmx_pfn_scatter");
}

}  // namespace
}  // namespace pmx

using namespace pmx;

static pmx_status pfn_impl(int dense, const pmx_pfn_desc* desc, const pmx_grid* grid, int32_t batch, int32_t pcap,
                                      const float* points, const int64_t* frame_offsets, const float* features,
                                      const uint8_t* mask, const int32_t* coords, const int32_t* counts,
                                      const int32_t* pt_idx, const int32_t* n_pillars, const void* weight,
                                      const float* alpha, const float* bias, const float* bn_post,
                                      const pmx_out* outs, int32_t n_outs, uint32_t* in_keys, uint32_t* out_keys,
                                      pmx_stream_t stream) {
  PMX_REQUIRE(desc && grid, "desc/grid is NULL");
  const pmx_pfn_desc d = *desc;
  PMX_REQUIRE(d.channels >= 1 && d.channels <= kMaxC, "PFN channels must be 1..64");
  PMX_REQUIRE(d.max_points >= 1 && d.max_points <= 32 && d.max_points == grid->max_points,
              "PFN max_points must equal the grid's (1..32)");
  PMX_REQUIRE(d.in_dtype >= PMX_F32 && d.in_dtype <= PMX_I8, "bad PFN dtype");
  if (d.source == PMX_PFN_FROM_POINTS9) {
    PMX_REQUIRE(d.n_features == 9 && points && frame_offsets && pt_idx, "POINTS9 needs points, offsets, pt_idx");
  } else if (d.source == PMX_PFN_FROM_FEATURES) {
    PMX_REQUIRE(d.n_features >= 1 && d.n_features <= kMaxF && features && mask, "FROM_FEATURES needs features+mask");
  } else {
    return fail(PMX_ERR_INVALID, "bad PFN source");
  }
  PMX_REQUIRE(d.in_dtype != PMX_I8 || (alpha && d.in_scale > 0.0), "int8 PFN needs alpha and in_scale");
  PMX_REQUIRE(weight && bias && coords && counts && n_pillars, "NULL PFN operand");
  pmx_status st = validate_outs(outs, n_outs, d.channels);
  if (st != PMX_OK) return st;
  if (batch == 0 || pcap == 0) return PMX_OK;
  PfnArgs a;
  a.d = d;
  a.g = *grid;
  a.pcap = pcap;
  a.points = reinterpret_cast<const float4*>(points);
  a.offs = frame_offsets;
  a.features = features;
  a.mask = mask;
  a.coords = coords;
  a.counts = counts;
  a.pt_idx = pt_idx;
  a.n_pillars = n_pillars;
  a.weight = weight;
  a.alpha = alpha;
  a.bias = bias;
  a.bn_post = bn_post;
  a.in_inv = d.in_dtype == PMX_I8 ? (float)(1.0 / d.in_scale) : 1.f;
  a.in_keys = in_keys;
  a.out_keys = out_keys;
  a.dense = dense;
  Outs o = make_outs(outs, n_outs);
  dim3 g((unsigned)ceil_div(pcap, kPPB), (unsigned)batch);
  if (d.in_dtype == PMX_I8) return launch_dt<PMX_I8>(a, o, g, stream);
  if (d.in_dtype == PMX_F16) return launch_dt<PMX_F16>(a, o, g, stream);
  return launch_dt<PMX_F32>(a, o, g, stream);
}

extern "C" pmx_status pmx_pfn_scatter(const pmx_pfn_desc* desc, const pmx_grid* grid, int32_t batch, int32_t pcap,
                                      const float* points, const int64_t* frame_offsets, const float* features,
                                      const uint8_t* mask, const int32_t* coords, const int32_t* counts,
                                      const int32_t* pt_idx, const int32_t* n_pillars, const void* weight,
                                      const float* alpha, const float* bias, const float* bn_post,
                                      const pmx_out* outs, int32_t n_outs, uint32_t* in_keys, uint32_t* out_keys,
                                      pmx_stream_t stream) {
  return pfn_impl(0, desc, grid, batch, pcap, points, frame_offsets, features, mask, coords, counts, pt_idx,
                  n_pillars, weight, alpha, bias, bn_post, outs, n_outs, in_keys, out_keys, stream);
}

extern "C" pmx_status pmx_pfn_pillars(const pmx_pfn_desc* desc, const pmx_grid* grid, int32_t batch, int32_t pcap,
                                      const float* points, const int64_t* frame_offsets, const float* features,
                                      const uint8_t* mask, const int32_t* coords, const int32_t* counts,
                                      const int32_t* pt_idx, const int32_t* n_pillars, const void* weight,
                                      const float* alpha, const float* bias, const float* bn_post,
                                      const pmx_out* outs, int32_t n_outs, uint32_t* in_keys, uint32_t* out_keys,
                                      pmx_stream_t stream) {
  return pfn_impl(1, desc, grid, batch, pcap, points, frame_offsets, features, mask, coords, counts, pt_idx,
                  n_pillars, weight, alpha, bias, bn_post, outs, n_outs, in_keys, out_keys, stream);
}
