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
#include <type_traits>

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
  int ppw;    // pfn_points_kernel: pillars per warp (32; 16 / 8 when one wave of 32 would leave SMs idle)
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

// POINTS9 path.  A warp takes 32 pillars.
//  Phase A (lane = pillar): counts, coords, the first kSlots points (independent
//   gathers in flight together), the cluster mean as the sequential f32 sum in slot
//   order (numpy's chunk.mean, bit for bit), the 9 features (observer), layer 1's
//   transform -> shared memory.
//  Phase B (lane = output channel pair 2l, 2l+1; weights in registers): for each of the
//   32 pillars, the FMA chain over the features (broadcast shared-memory reads) and the
//   max over points; epilogue once per pillar; 128-byte coalesced row stores.
// Points beyond kSlots (dense clusters, M up to 32) are rebuilt in phase B.
constexpr int kSlots = 4;  // KITTI pillars hold ~1.3 points; more are rebuilt in phase B
// one point record = the 9 transformed features (int8 codes / binary16 values are
// exact in f32) as f32, padded to 48 bytes: phase B reads three broadcast float4 and
// converts nothing
template <int DT>
struct Rec {
  using T = float;
  static constexpr int N = 12;  // elements per record
  static constexpr int BYTES = N * (int)sizeof(T);
};
template <int DT>
constexpr size_t pfn_points_smem() {
  return (size_t)(kThreads / 32) * 32 * kSlots * Rec<DT>::BYTES + (size_t)(kThreads / 32) * 32 * 6 * 4;
}

template <int DT>
#ifndef PMX_PFN_MINB
#define PMX_PFN_MINB 2
#endif
__global__ void __launch_bounds__(kThreads, PMX_PFN_MINB) pfn_points_kernel(const PfnArgs a, const Outs outs) {
  pdl_begin();
#ifdef PMX_PFN_TRACE
  unsigned long long pt0, pt1, pt2;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pt0));
#endif
  using R = Rec<DT>;
  using T = typename R::T;
  extern __shared__ __align__(16) uint8_t pfn_smem[];
  // [warp][pillar][slot] records, then [warp][pillar][6] slow-path metadata
  T (*sf)[32][kSlots][R::N] = reinterpret_cast<T (*)[32][kSlots][R::N]>(pfn_smem);
  float (*smeta)[32][6] =
      reinterpret_cast<float (*)[32][6]>(pfn_smem + (size_t)(kThreads / 32) * 32 * kSlots * R::BYTES);
  const int b = blockIdx.y;
  const int C = a.d.channels;
  const int M = a.d.max_points;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
  const float INF = __int_as_float(0x7f800000);
  const float4* fp = a.points + a.offs[b];
#ifdef PMX_DEBUG_BOUNDS
  const int64_t n_frame = a.offs[b + 1] - a.offs[b];
#define PMX_CHK(cond, what, v)                                                                                \
  do {                                                                                                        \
    if (!(cond)) {                                                                                            \
      printf("pfn check failed: %s value %lld b %d block %d thread %d line %d\n", what, (long long)(v), b,     \
             blockIdx.x, threadIdx.x, __LINE__);                                                              \
      __trap();                                                                                               \
    }                                                                                                         \
  } while (0)
  PMX_CHK(P >= 0 && P <= a.pcap, "n_pillars", P);
#define PMX_PT(i_)                                                                                            \
  ([&](int i__) {                                                                                             \
    if (i__ < 0 || i__ >= n_frame) {                                                                          \
      printf("pfn: point index %d out of [0, %lld) b %d block %d thread %d line %d\n", i__, (long long)n_frame, b, \
             blockIdx.x, threadIdx.x, __LINE__);                                                              \
      __trap();                                                                                               \
    }                                                                                                         \
    return i__;                                                                                               \
  }(i_))
#else
#define PMX_PT(i_) (i_)
#define PMX_CHK(cond, what, v) \
  do {                         \
  } while (0)
#endif
  const float xoff = (float)((double)a.g.cell_w * 0.5 + (double)a.g.x_min);
  const float yoff = (float)((double)a.g.cell_h * 0.5 + (double)a.g.y_min);
  // ---------------- phase A: lane = pillar
  const int p = (blockIdx.x * (kThreads / 32) + warp) * a.ppw + lane;
  const bool live = lane < a.ppw && p < P;
  const int64_t q = (int64_t)b * a.pcap + (live ? p : 0);
  const int k = live ? a.counts[q] : 0;
  const int32_t* idx = a.pt_idx + q * M;
  PMX_CHK(k >= 0 && k <= M, "count", k);
  float in_lo = INF, in_hi = -INF;
  float4 pts[kSlots];
#pragma unroll
  for (int s = 0; s < kSlots; ++s) pts[s] = make_float4(0.f, 0.f, 0.f, 0.f);
  // the first kSlots point indices in one 16-byte load issued next to the count's (not
  // after it): one dependent global round trip less on phase A's gather chain
  static_assert(kSlots == 4, "one int4 of point indices");
  int ids[kSlots];
  if (live && (M & 3) == 0 && (reinterpret_cast<uintptr_t>(a.pt_idx) & 15) == 0) {
    const int4 i4 = __ldg(reinterpret_cast<const int4*>(idx));
    ids[0] = i4.x; ids[1] = i4.y; ids[2] = i4.z; ids[3] = i4.w;
  } else {
#pragma unroll
    for (int s = 0; s < kSlots; ++s) ids[s] = (s < k) ? __ldg(idx + s) : 0;
  }
#pragma unroll
  for (int s = 0; s < kSlots; ++s)
    if (s < k) pts[s] = __ldg(fp + PMX_PT(ids[s]));
  float sx = 0.f, sy = 0.f, sz = 0.f;
#pragma unroll
  for (int s = 0; s < kSlots; ++s)
    if (s < k) {
      sx = __fadd_rn(sx, pts[s].x);
      sy = __fadd_rn(sy, pts[s].y);
      sz = __fadd_rn(sz, pts[s].z);
    }
  for (int s = kSlots; s < k; ++s) {  // dense cluster tail, still in slot order
    const float4 pt = __ldg(fp + PMX_PT(__ldg(idx + s)));
    sx = __fadd_rn(sx, pt.x);
    sy = __fadd_rn(sy, pt.y);
    sz = __fadd_rn(sz, pt.z);
  }
  const float fk = (float)(k > 0 ? k : 1);
  const float mxm = __fdiv_rn(sx, fk), mym = __fdiv_rn(sy, fk), mzm = __fdiv_rn(sz, fk);
  float xc = 0.f, yc = 0.f;
  int64_t mypix = q;  // output row of this lane's pillar (canvas pixel, or the pillar slot)
  if (live) {
    const int2 cc = *reinterpret_cast<const int2*>(a.coords + 2 * q);
    xc = __fadd_rn(__fmul_rn((float)cc.y, a.g.cell_w), xoff);
    yc = __fadd_rn(__fmul_rn((float)cc.x, a.g.cell_h), yoff);
    if (!a.dense) mypix = ((int64_t)b * a.g.grid_h + cc.x) * a.g.grid_w + cc.y;
    PMX_CHK(cc.x >= 0 && cc.x < a.g.grid_h && cc.y >= 0 && cc.y < a.g.grid_w, "coords", cc.x * 100000 + cc.y);
  }
  if (live && k < M) { in_lo = 0.f; in_hi = 0.f; }  // zero padding rows are part of layer 1's input
  auto feats = [&](const float4& pt, float (&f)[9]) {
    f[0] = pt.x; f[1] = pt.y; f[2] = pt.z; f[3] = pt.w;
    f[4] = __fsub_rn(pt.x, mxm); f[5] = __fsub_rn(pt.y, mym); f[6] = __fsub_rn(pt.z, mzm);
    f[7] = __fsub_rn(pt.x, xc); f[8] = __fsub_rn(pt.y, yc);
  };
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    if (s < k) {
      float f[9];
      feats(pts[s], f);
      if (a.in_keys) {
#pragma unroll
        for (int j = 0; j < 9; ++j) { in_lo = nmin(in_lo, f[j]); in_hi = nmax(in_hi, f[j]); }
      }
      float t9[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) t9[j] = transform_in<DT>(f[j], a);  // exact in f32
      float4* dst = reinterpret_cast<float4*>(sf[warp][lane][s]);
      dst[0] = make_float4(t9[0], t9[1], t9[2], t9[3]);
      dst[1] = make_float4(t9[4], t9[5], t9[6], t9[7]);
      dst[2] = make_float4(t9[8], 0.f, 0.f, 0.f);
    }
  }
  if (k > kSlots) {
    smeta[warp][lane][0] = mxm; smeta[warp][lane][1] = mym; smeta[warp][lane][2] = mzm;
    smeta[warp][lane][3] = xc; smeta[warp][lane][4] = yc;
    if (a.in_keys) {
      for (int s = kSlots; s < k; ++s) {
        float f[9];
        feats(__ldg(fp + PMX_PT(__ldg(idx + s))), f);
#pragma unroll
        for (int j = 0; j < 9; ++j) { in_lo = nmin(in_lo, f[j]); in_hi = nmax(in_hi, f[j]); }
      }
    }
  }
  __syncwarp();
#ifdef PMX_PFN_TRACE
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pt1));
#endif
  // ---------------- phase B: two pillars per step; lane = (pillar half, 4 channels)
  const int half = lane >> 4;
  const int c = 4 * (lane & 15);
  float w[4][9];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      const int cc = c + u;
      float v = 0.f;
      if (cc < C) {
        if constexpr (DT == PMX_I8) v = (float)reinterpret_cast<const int8_t*>(a.weight)[cc * 9 + j];
        else if constexpr (DT == PMX_F16) v = __half2float(reinterpret_cast<const __half*>(a.weight)[cc * 9 + j]);
        else v = reinterpret_cast<const float*>(a.weight)[cc * 9 + j];
      }
      w[u][j] = v;
    }
  float al[4], bi[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    al[u] = (DT == PMX_I8 && c + u < C) ? a.alpha[c + u] : 1.f;
    bi[u] = c + u < C ? a.bias[c + u] : 0.f;
  }
  float o_lo = INF, o_hi = -INF;
  // single f16 consumer with 8-byte aligned 4-channel runs (kernel-uniform)
  const bool f16_only = outs.n == 1 && outs.o[0].dtype == PMX_F16 && (outs.o[0].c_stride & 3) == 0 &&
                        (outs.o[0].c_offset & 3) == 0;
  for (int it = 0; it < (a.ppw >> 1); ++it) {
    const int j = 2 * it + half;
    const int kj = __shfl_sync(0xffffffffu, k, j);
    const int kpair = max(kj, __shfl_xor_sync(0xffffffffu, kj, 16));
    if (kpair == 0) continue;  // warp-uniform
    const int64_t qj = __shfl_sync(0xffffffffu, q, j);
    float m[4] = {-INF, -INF, -INF, -INF};
    // live: this half's pillar holds the point (the loop runs to the pair's max count
    // without diverging; a dead slot's products are computed and discarded)
    auto point = [&](const float (&f)[9], bool live) {
      float2 acc01 = make_float2(0.f, 0.f), acc23 = make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        acc01 = __ffma2_rn(make_float2(f[t], f[t]), make_float2(w[0][t], w[1][t]), acc01);
        acc23 = __ffma2_rn(make_float2(f[t], f[t]), make_float2(w[2][t], w[3][t]), acc23);
      }
      const float acc[4] = {acc01.x, acc01.y, acc23.x, acc23.y};
      if (a.bn_post == nullptr) {
        // NaN-propagating max (max.NaN): a NaN product reaches the canvas like numpy's max
#pragma unroll
        for (int u = 0; u < 4; ++u) m[u] = live ? fmax_nan(m[u], acc[u]) : m[u];
      } else if (live) {  // unfolded BN may have a negative gamma: finish every point
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float y;
          if constexpr (DT == PMX_I8) y = __fmaf_rn(acc[u], al[u], bi[u]);
          else y = __fadd_rn(acc[u], bi[u]);
          if (c + u < C)
            y = __fadd_rn(__fmul_rn(__fsub_rn(y, a.bn_post[c + u]), a.bn_post[C + c + u]), a.bn_post[2 * C + c + u]);
          if (a.d.relu) y = fmaxf(y, 0.f);
          m[u] = nmax(m[u], y);
        }
      }
    };
    const int kk = kpair < kSlots ? kpair : kSlots;
    for (int s2 = 0; s2 < kk; ++s2) {  // warp-uniform trip count
      float f[9];
      const float4* src = reinterpret_cast<const float4*>(sf[warp][j][s2]);  // two broadcast addresses
      const float4 f0 = src[0], f1 = src[1], f2 = src[2];
      f[0] = f0.x; f[1] = f0.y; f[2] = f0.z; f[3] = f0.w; f[4] = f1.x; f[5] = f1.y; f[6] = f1.z; f[7] = f1.w;
      f[8] = f2.x;
      point(f, s2 < kj);
    }
    if (kpair > kSlots) {  // dense cluster: rebuild the remaining points (broadcast loads per half)
      const float* mt = smeta[warp][j];
      const int32_t* idj = a.pt_idx + qj * M;
      for (int s2 = kSlots; s2 < kpair; ++s2) {
        if (s2 >= kj) continue;
        const float4 pt = __ldg(fp + PMX_PT(__ldg(idj + s2)));
        float f[9];
        f[0] = pt.x; f[1] = pt.y; f[2] = pt.z; f[3] = pt.w;
        f[4] = __fsub_rn(pt.x, mt[0]); f[5] = __fsub_rn(pt.y, mt[1]); f[6] = __fsub_rn(pt.z, mt[2]);
        f[7] = __fsub_rn(pt.x, mt[3]); f[8] = __fsub_rn(pt.y, mt[4]);
#pragma unroll
        for (int t = 0; t < 9; ++t) f[t] = transform_in<DT>(f[t], a);
        point(f, true);
      }
    }
    // every lane takes part in the shuffle (the halves' pillars may differ in liveness:
    // a shuffle after the divergent `continue` below is undefined and returned garbage)
    const int64_t pix = __shfl_sync(0xffffffffu, mypix, j);
    if (kj == 0 || c >= C) continue;
    float y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      y[u] = m[u];
      if (a.bn_post == nullptr) {
        if constexpr (DT == PMX_I8) y[u] = __fmaf_rn(m[u], al[u], bi[u]);
        else y[u] = __fadd_rn(m[u], bi[u]);
        if (a.d.relu) y[u] = fmaxf(y[u], 0.f);
      }
    }
    const int nl = C - c < 4 ? C - c : 4;
    PMX_CHK(pix >= 0 && pix < (a.dense ? (int64_t)gridDim.y * a.pcap : (int64_t)gridDim.y * hw), "pix", pix);
    if (f16_only && nl == 4) {
      // the common single binary16 consumer (next layer FP16): one 8-byte store
      *reinterpret_cast<uint2*>(reinterpret_cast<__half*>(outs.o[0].ptr) + pix * outs.o[0].c_stride +
                                outs.o[0].c_offset + c) = make_uint2(f16x2_sat(y[0], y[1]), f16x2_sat(y[2], y[3]));
      if (a.out_keys) {
        for (int u = 0; u < nl; ++u) { o_lo = nmin(o_lo, y[u]); o_hi = nmax(o_hi, y[u]); }
      }
      continue;
    }
#pragma unroll
    for (int o = 0; o < PMX_MAX_OUTS; ++o) {
      if (o >= outs.n) break;
      const OutDev& od = outs.o[o];
      const int64_t off = pix * od.c_stride + od.c_offset + c;
      if (nl == 4 && od.dtype == PMX_F16 && (off & 3) == 0) {
        *reinterpret_cast<uint2*>(reinterpret_cast<__half*>(od.ptr) + off) =
            make_uint2(f16x2_sat(y[0], y[1]), f16x2_sat(y[2], y[3]));
      } else if (nl == 4 && od.dtype == PMX_I8 && (off & 3) == 0) {
        uint32_t wd = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) wd |= (uint32_t)(quantize_exact(y[u], od.scale, od.inv) & 0xff) << (8 * u);
        *reinterpret_cast<uint32_t*>(reinterpret_cast<int8_t*>(od.ptr) + off) = wd;
      } else if (nl == 4 && od.dtype == PMX_F32 && (off & 3) == 0) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(od.ptr) + off) = make_float4(y[0], y[1], y[2], y[3]);
      } else {
        for (int u = 0; u < nl; ++u) store_one(od, pix, c + u, y[u]);
      }
    }
    if (a.out_keys) {
      for (int u = 0; u < nl; ++u) { o_lo = nmin(o_lo, y[u]); o_hi = nmax(o_hi, y[u]); }
    }
  }
#ifdef PMX_PFN_TRACE
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pt2));
  if (lane == 0 && (blockIdx.x % 8 == 0) && warp == 0)
    printf("pfn trace blk %d warp %d: start %llu phaseA %llu phaseB %llu keys %d/%d\n", blockIdx.x, warp, pt0 % 1000000,
           pt1 - pt0, pt2 - pt1, a.in_keys != nullptr, a.out_keys != nullptr);
#endif
  if (a.in_keys) block_minmax_commit<kThreads>(in_lo, in_hi, a.in_keys);
  if (a.out_keys) block_minmax_commit<kThreads>(o_lo, o_hi, a.out_keys);
}

template <int DT>
pmx_status launch_dt(const PfnArgs& a, const Outs& outs, dim3 grid, cudaStream_t st) {
  if (a.d.source == PMX_PFN_FROM_POINTS9) {
    // 32 pillars per warp; small batches (one wave of those would leave SMs idle): 16 or
    // 8, a shorter per-warp chain over more warps (batch 1: 63 -> 252 blocks)
    PfnArgs a2 = a;
    a2.ppw = 32;
    {
      static const int fixed = [] {
        const char* e = getenv("PMX_PFN_PPW");  // A/B override: 8, 16 or 32
        return e ? atoi(e) : 0;
      }();
      if (fixed == 8 || fixed == 16 || fixed == 32) {
        a2.ppw = fixed;
      } else {
        while (a2.ppw > 8 && (int64_t)ceil_div(a.pcap, (kThreads / 32) * (a2.ppw / 2)) * grid.y <= 2LL * num_sms())
          a2.ppw /= 2;
      }
    }
    const dim3 g2((unsigned)ceil_div(a.pcap, (kThreads / 32) * a2.ppw), grid.y);
    const size_t sm = pfn_points_smem<DT>();
    PMX_CUDA(cudaFuncSetAttribute(pfn_points_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    PMX_CUDA(launch_pdl(pfn_points_kernel<DT>, g2, dim3(kThreads), sm, st, a2, outs));
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
