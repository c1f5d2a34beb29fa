// K4+K5 fused pillar feature net + BEV scatter.
//
// One warp per pillar, lane = point slot (M <= 32).  The 9 features are built in
// registers (sequential f32 mean via shuffle broadcast, matching numpy's
// chunk.mean(axis=0) bit for bit), transformed to layer 1's precision (exact int8
// codes / binary16 / f32), then every live point is broadcast in turn and each
// lane accumulates its output channels (lane, lane+32).  The running max over
// points stays in registers; the pooled value is written once per consumer
// format straight onto the NHWC canvas (scatter fused, no [P, C] round trip).
// Replaces pm/model.py:334-355 -> _run_weight_layer :271-307 -> linear
// pm/tensor_ops.py:80-91, relu :134, max_over_points :163-173, scatter :138-160.
#include "pmx_common.cuh"

namespace pmx {

namespace {

constexpr int kMaxF = 16;
constexpr int kMaxC = 64;

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
};

template <int DT, int NF, bool FROM_POINTS>
__global__ void __launch_bounds__(256) pfn_kernel(const PfnArgs a, const Outs outs) {
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int p = blockIdx.x * 8 + wid;
  const int P = a.n_pillars[b];
  const int M = a.d.max_points;
  const int F = FROM_POINTS ? 9 : NF;
  const int C = a.d.channels;
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
  if (p >= P) return;
  const int64_t q = (int64_t)b * a.pcap + p;

  // ---- features of this lane's slot
  float f[kMaxF];
#pragma unroll
  for (int j = 0; j < kMaxF; ++j) f[j] = 0.f;
  bool live;
  if (FROM_POINTS) {
    const int k = a.counts[q];
    live = lane < k;
    float4 pt = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) pt = __ldg(a.points + a.offs[b] + a.pt_idx[q * M + lane]);
    float sx = 0.f, sy = 0.f, sz = 0.f;
    for (int s = 0; s < k; ++s) {
      sx = __fadd_rn(sx, __shfl_sync(0xffffffffu, pt.x, s));
      sy = __fadd_rn(sy, __shfl_sync(0xffffffffu, pt.y, s));
      sz = __fadd_rn(sz, __shfl_sync(0xffffffffu, pt.z, s));
    }
    const float fk = (float)(k > 0 ? k : 1);
    const float mx = __fdiv_rn(sx, fk), my = __fdiv_rn(sy, fk), mz = __fdiv_rn(sz, fk);
    const float xoff = (float)((double)a.g.cell_w * 0.5 + (double)a.g.x_min);
    const float yoff = (float)((double)a.g.cell_h * 0.5 + (double)a.g.y_min);
    const float xc = __fadd_rn(__fmul_rn((float)a.coords[2 * q + 1], a.g.cell_w), xoff);
    const float yc = __fadd_rn(__fmul_rn((float)a.coords[2 * q + 0], a.g.cell_h), yoff);
    if (live) {
      f[0] = pt.x; f[1] = pt.y; f[2] = pt.z; f[3] = pt.w;
      f[4] = __fsub_rn(pt.x, mx); f[5] = __fsub_rn(pt.y, my); f[6] = __fsub_rn(pt.z, mz);
      f[7] = __fsub_rn(pt.x, xc); f[8] = __fsub_rn(pt.y, yc);
    }
    if (a.in_keys) {  // layer-1 observer: real rows, plus the zero padding rows if any
      float lo = 0.f, hi = 0.f;
      if (live) {
        lo = f[0]; hi = f[0];
#pragma unroll
        for (int j = 1; j < 9; ++j) { lo = nmin(lo, f[j]); hi = nmax(hi, f[j]); }
      }
      const bool has_pad = k < M;
      if (!live && !has_pad) { lo = __int_as_float(0x7f800000); hi = -lo; }
      if (lane >= M) { lo = __int_as_float(0x7f800000); hi = -lo; }
      block_minmax_commit<256>(lo, hi, a.in_keys);
    }
  } else {
    live = false;
    if (lane < M) {
      live = a.mask[q * M + lane] != 0;
      const float* src = a.features + (q * M + lane) * F;
#pragma unroll
      for (int j = 0; j < kMaxF; ++j)
        if (j < F) f[j] = src[j];
    }
    if (a.in_keys) {
      float lo = __int_as_float(0x7f800000), hi = -lo;
      if (lane < M) {
#pragma unroll
        for (int j = 0; j < kMaxF; ++j)
          if (j < F) { lo = nmin(lo, f[j]); hi = nmax(hi, f[j]); }
      }
      block_minmax_commit<256>(lo, hi, a.in_keys);
    }
  }

  // ---- precision transform of the layer input (pm/model.py:273-285)
  int fq[kMaxF];
  if (DT == PMX_I8) {
#pragma unroll
    for (int j = 0; j < kMaxF; ++j) fq[j] = j < F ? quantize_exact(f[j], a.d.in_scale, a.in_inv) : 0;
  } else if (DT == PMX_F16) {
#pragma unroll
    for (int j = 0; j < kMaxF; ++j) f[j] = __half2float(f16_sat(f[j]));
  }

  // ---- per-lane channels: c0 = lane, c1 = lane + 32
  float w0[kMaxF], w1[kMaxF];
  int iw0[kMaxF], iw1[kMaxF];
  const int c0 = lane, c1 = lane + 32;
  const bool h0 = c0 < C, h1 = c1 < C;
#pragma unroll
  for (int j = 0; j < kMaxF; ++j) {
    w0[j] = w1[j] = 0.f;
    iw0[j] = iw1[j] = 0;
    if (j < F) {
      if (DT == PMX_I8) {
        const int8_t* W = reinterpret_cast<const int8_t*>(a.weight);
        if (h0) iw0[j] = W[c0 * F + j];
        if (h1) iw1[j] = W[c1 * F + j];
      } else if (DT == PMX_F16) {
        const __half* W = reinterpret_cast<const __half*>(a.weight);
        if (h0) w0[j] = __half2float(W[c0 * F + j]);
        if (h1) w1[j] = __half2float(W[c1 * F + j]);
      } else {
        const float* W = reinterpret_cast<const float*>(a.weight);
        if (h0) w0[j] = W[c0 * F + j];
        if (h1) w1[j] = W[c1 * F + j];
      }
    }
  }
  const float al0 = (DT == PMX_I8 && h0) ? a.alpha[c0] : 1.f;
  const float al1 = (DT == PMX_I8 && h1) ? a.alpha[c1] : 1.f;
  const float b0 = h0 ? a.bias[c0] : 0.f, b1 = h1 ? a.bias[c1] : 0.f;
  float bm0 = 0.f, bf0 = 1.f, bb0 = 0.f, bm1 = 0.f, bf1 = 1.f, bb1 = 0.f;
  if (a.bn_post) {
    if (h0) { bm0 = a.bn_post[c0]; bf0 = a.bn_post[C + c0]; bb0 = a.bn_post[2 * C + c0]; }
    if (h1) { bm1 = a.bn_post[c1]; bf1 = a.bn_post[C + c1]; bb1 = a.bn_post[2 * C + c1]; }
  }

  const float NEG_INF = -__int_as_float(0x7f800000);
  float m0 = NEG_INF, m1 = NEG_INF;
  unsigned vm = __ballot_sync(0xffffffffu, live && lane < M);
  while (vm) {
    const int s = __ffs(vm) - 1;
    vm &= vm - 1;
    float y0, y1;
    if (DT == PMX_I8) {
      int acc0 = 0, acc1 = 0;
#pragma unroll
      for (int j = 0; j < kMaxF; ++j) {
        if (j < F) {
          const int v = __shfl_sync(0xffffffffu, fq[j], s);
          acc0 += v * iw0[j];
          acc1 += v * iw1[j];
        }
      }
      y0 = __fadd_rn(__fmul_rn((float)acc0, al0), b0);
      y1 = __fadd_rn(__fmul_rn((float)acc1, al1), b1);
    } else {
      float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
      for (int j = 0; j < kMaxF; ++j) {
        if (j < F) {
          const float v = __shfl_sync(0xffffffffu, f[j], s);
          acc0 = __fmaf_rn(v, w0[j], acc0);
          acc1 = __fmaf_rn(v, w1[j], acc1);
        }
      }
      y0 = __fadd_rn(acc0, b0);
      y1 = __fadd_rn(acc1, b1);
    }
    if (a.bn_post) {
      y0 = __fadd_rn(__fmul_rn(__fsub_rn(y0, bm0), bf0), bb0);
      y1 = __fadd_rn(__fmul_rn(__fsub_rn(y1, bm1), bf1), bb1);
    }
    if (a.d.relu) {
      y0 = fmaxf(y0, 0.f);
      y1 = fmaxf(y1, 0.f);
    }
    m0 = nmax(m0, y0);
    m1 = nmax(m1, y1);
  }

  // ---- scatter the pooled column onto the canvas, every consumer format
  const int64_t pix = ((int64_t)b * a.g.grid_h + a.coords[2 * q]) * a.g.grid_w + a.coords[2 * q + 1];
  if (h0) store_all(outs, pix, c0, m0);
  if (h1) store_all(outs, pix, c1, m1);
  if (a.out_keys) {
    float lo = h0 ? m0 : __int_as_float(0x7f800000), hi = h0 ? m0 : -__int_as_float(0x7f800000);
    if (h1) { lo = nmin(lo, m1); hi = nmax(hi, m1); }
    block_minmax_commit<256>(lo, hi, a.out_keys);
  }
}

template <int DT>
pmx_status launch_dt(const PfnArgs& a, const Outs& outs, dim3 grid, cudaStream_t st) {
  if (a.d.source == PMX_PFN_FROM_POINTS9) {
    pfn_kernel<DT, 9, true><<<grid, 256, 0, st>>>(a, outs);
  } else {
    switch (a.d.n_features) {
#define PMX_F_CASE(N) \
  case N:             \
    pfn_kernel<DT, N, false><<<grid, 256, 0, st>>>(a, outs); break;
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

extern "C" pmx_status pmx_pfn_scatter(const pmx_pfn_desc* desc, const pmx_grid* grid, int32_t batch, int32_t pcap,
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
  Outs o = make_outs(outs, n_outs);
  dim3 g((unsigned)ceil_div(pcap, 8), (unsigned)batch);
  if (d.in_dtype == PMX_I8) return launch_dt<PMX_I8>(a, o, g, stream);
  if (d.in_dtype == PMX_F16) return launch_dt<PMX_F16>(a, o, g, stream);
  return launch_dt<PMX_F32>(a, o, g, stream);
}
