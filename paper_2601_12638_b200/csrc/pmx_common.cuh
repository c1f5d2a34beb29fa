// Shared device helpers for libpmx (sm_100a).  Never compile with --use_fast_math:
// the binning divide, the quantize estimate and the fp16 cast must be IEEE.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "pmx.h"

namespace pmx {

// ---------------------------------------------------------------------------
// error plumbing (thread-local message, pmx_last_error)

void set_error(const std::string& msg);
pmx_status fail(pmx_status code, const std::string& msg);
pmx_status check_launch(const char* what);

#define PMX_REQUIRE(cond, msg)                               \
  do {                                                       \
    if (!(cond)) return ::pmx::fail(PMX_ERR_INVALID, (msg)); \
  } while (0)

#define PMX_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return ::pmx::fail(PMX_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

inline int elem_size(int dtype) { return dtype == PMX_F32 ? 4 : (dtype == PMX_F16 ? 2 : 1); }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
constexpr int kNumSMs = 148;

// ---------------------------------------------------------------------------
// exact quantize: clip(rint(f64(x) / scale), -128, 127)   (pm/quant.py:98-103)
//
// q = x * inv (f32) has relative error < 2^-22, i.e. absolute error < 4e-5 for
// |q| < 129, so rint(q) equals rint(x / scale) unless q lies within 1e-3 of a
// half-integer; there the IEEE f64 divide decides (the reference's own op).

struct QScale {
  double s;
  float inv;
};

__host__ inline QScale make_qscale(double s) { return QScale{s, (float)(1.0 / s)}; }

__device__ __forceinline__ int quantize_exact(float x, double s, float inv) {
  float q = __fmul_rn(x, inv);
  float aq = fabsf(q);
  if (!(aq < 129.0f)) {
    if (q != q) return 0;  // NaN: defined as 0 (the reference's cast is undefined)
    return q > 0.0f ? 127 : -128;
  }
  float r = rintf(q);
  float d = fabsf(__fsub_rn(q, r));
  if (fabsf(d - 0.5f) < 1e-3f) {
    double e = __ddiv_rn((double)x, s);
    r = (float)rint(e);
  }
  int c = (int)r;
  return c < -128 ? -128 : (c > 127 ? 127 : c);
}

// Same result as quantize_exact with a short common path: away from ties
// (|frac - .5| >= 1e-3) and inside |q| < 127 the f32 estimate is already exact and
// needs no clamp; everything else (ties, saturation, NaN) takes the exact path.
__device__ __forceinline__ int quantize_fast(float x, double s, float inv) {
  const float q = __fmul_rn(x, inv);
  const float r = rintf(q);
  if (fabsf(__fsub_rn(q, r)) < 0.499f && fabsf(q) < 127.0f) return (int)r;
  return quantize_exact(x, s, inv);
}

// fp16_roundtrip (pm/quant.py:144-147): saturate at +-65504, then RNE.
__device__ __forceinline__ __half f16_sat(float x) {
  if (x != x) return __float2half_rn(x);
  x = fminf(fmaxf(x, -65504.0f), 65504.0f);
  return __float2half_rn(x);
}

// ---------------------------------------------------------------------------
// order-preserving float keys for atomic min/max observers

__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ float key2f(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(b);
}

template <int kThreads>
__device__ __forceinline__ void block_minmax_commit(float lo, float hi, uint32_t* keys) {
  // warp reduce, then one atomic pair per warp (keys are exact, order free)
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0 && lo <= hi) {
    atomicMin(keys + 0, f2key(lo));
    atomicMax(keys + 1, f2key(hi));
  }
}

// NaN-propagating min/max so that a non-finite activation reaches the observer
__device__ __forceinline__ float nmin(float a, float b) { return (b != b || b < a) ? b : a; }
__device__ __forceinline__ float nmax(float a, float b) { return (b != b || b > a) ? b : a; }

// ---------------------------------------------------------------------------
// epilogue stores: one f32 value -> every consumer format

struct OutDev {
  void* ptr;
  double scale;
  float inv;
  int32_t dtype;
  int32_t c_stride;
  int32_t c_offset;
};

struct Outs {
  OutDev o[PMX_MAX_OUTS];
  int32_t n;
};

__host__ inline Outs make_outs(const pmx_out* outs, int n) {
  Outs r{};
  r.n = n;
  for (int i = 0; i < n; ++i) {
    r.o[i].ptr = outs[i].ptr;
    r.o[i].scale = outs[i].scale;
    r.o[i].inv = outs[i].dtype == PMX_I8 ? (float)(1.0 / outs[i].scale) : 1.0f;
    r.o[i].dtype = outs[i].dtype;
    r.o[i].c_stride = outs[i].c_stride;
    r.o[i].c_offset = outs[i].c_offset;
  }
  return r;
}

__device__ __forceinline__ void store_one(const OutDev& o, int64_t pix, int c, float y) {
  int64_t off = pix * o.c_stride + o.c_offset + c;
  if (o.dtype == PMX_F32) {
    reinterpret_cast<float*>(o.ptr)[off] = y;
  } else if (o.dtype == PMX_F16) {
    reinterpret_cast<__half*>(o.ptr)[off] = f16_sat(y);
  } else {
    reinterpret_cast<int8_t*>(o.ptr)[off] = (int8_t)quantize_exact(y, o.scale, o.inv);
  }
}

__device__ __forceinline__ void store_all(const Outs& outs, int64_t pix, int c, float y) {
#pragma unroll
  for (int i = 0; i < PMX_MAX_OUTS; ++i)
    if (i < outs.n) store_one(outs.o[i], pix, c, y);
}

__host__ pmx_status validate_outs(const pmx_out* outs, int n, int c_needed);

}  // namespace pmx
