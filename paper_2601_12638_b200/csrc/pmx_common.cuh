// Shared device helpers for libpmx (sm_100a).  Never compile with --use_fast_math:
// the binning divide, the quantize estimate and the fp16 cast must be IEEE.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>
#include <utility>

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

inline int elem_size(int dtype) { return (dtype == PMX_F32 || dtype == PMX_F32X2) ? 4 : (dtype == PMX_F16 ? 2 : 1); }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
// SM count of the current device (queried once per device, cached): persistent grids
// are sized from it, never from a compile-time constant (other SKUs, MIG slices)
int num_sms();

// ---------------------------------------------------------------------------
// programmatic dependent launch: kernels are launched with programmatic stream
// serialization and start with pdl_begin() -- wait for the predecessor grid (its
// writes visible), then let the successor grid start launching.  The successor's
// launch and block scheduling overlap this kernel; no memory is touched before the
// wait, so the ordering is the plain stream order.  (A no-op without the attribute.)

__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// exact quantize: clip(rint(f64(x) / scale), -128, 127)   (pm/quant.py:98-103)
//
// q = x * inv (f32) has relative error < 2^-22, i.e. absolute error < 4e-5 for
// |q| < 129, so rint(q) equals rint(x / scale) unless q lies within 1e-4 of a
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
  if (fabsf(d - 0.5f) < 1e-4f) {
    double e = __ddiv_rn((double)x, s);
    r = (float)rint(e);
  }
  int c = (int)r;
  return c < -128 ? -128 : (c > 127 ? 127 : c);
}

// |frac(q) - .5| guard band.  q = RN(x * RN(1/s)) is within 2^-23 relative of x / s,
// i.e. within 1.6e-5 absolute for |q| < 128, so outside a 1e-4 band around the .5
// ties RN(q) already equals rint(x / s) and only values inside the band need the
// f64 divide of quantize_exact (pm/quant.py:100).
constexpr float kTieBand = 0.4999f;

// Same result as quantize_exact with a short common path: away from ties and inside
// |q| < 127 the f32 estimate is already exact and needs no clamp; everything else
// (ties, saturation, NaN) takes the exact path.
__device__ __forceinline__ int quantize_fast(float x, double s, float inv) {
  const float q = __fmul_rn(x, inv);
  const float r = rintf(q);
  if (fabsf(__fsub_rn(q, r)) < kTieBand && fabsf(q) < 127.0f) return (int)r;
  return quantize_exact(x, s, inv);
}

// NaN-propagating min / max (PTX max.NaN: FMNMX.NAN; the 3-input form is FMNMX3)
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmax3_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// unsigned division by a runtime constant for numerators < 2^31:
// q = (umulhi(n, m) + n) >> s with s = ceil(log2 d), m = 2^32 (2^s - d) / d + 1
struct FastDiv {
  uint32_t d, m, s;
};

__host__ inline FastDiv make_fastdiv(uint32_t d) {
  uint32_t s = 0;
  while ((1ull << s) < d) ++s;
  const uint64_t m = ((1ull << 32) * ((1ull << s) - d)) / d + 1;
  return FastDiv{d, (uint32_t)m, s};
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) { return (__umulhi(n, f.m) + n) >> f.s; }

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

// TF32 split of an f32 value (PMX_F32X2): hi = round-to-nearest-even to 10 mantissa
// bits, lo = y - hi exactly (|lo| <= 2^-11 |y|); Inf / NaN pass through in hi
__device__ __forceinline__ float tf32_hi(float y) {
  const uint32_t b = __float_as_uint(y);
  if ((b & 0x7f800000u) == 0x7f800000u) return y;
  uint32_t r = (b + 0x0fffu + ((b >> 13) & 1u)) & 0xffffe000u;
  if ((r & 0x7f800000u) == 0x7f800000u) r = b & 0xffffe000u;  // no rounding up into Inf near FLT_MAX
  return __uint_as_float(r);
}
__device__ __forceinline__ float2 tf32_split(float y) {
  const float hi = tf32_hi(y);
  const bool fin = (__float_as_uint(y) & 0x7f800000u) != 0x7f800000u;
  return make_float2(hi, fin ? __fsub_rn(y, hi) : 0.0f);
}

__device__ __forceinline__ void store_one(const OutDev& o, int64_t pix, int c, float y) {
  int64_t off = pix * o.c_stride + o.c_offset + c;
  if (o.dtype == PMX_F32) {
    reinterpret_cast<float*>(o.ptr)[off] = y;
  } else if (o.dtype == PMX_F32X2) {
    const float2 h = tf32_split(y);
    reinterpret_cast<float*>(o.ptr)[off] = h.x;
    reinterpret_cast<float*>(o.ptr)[off + (o.c_stride >> 1)] = h.y;
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

// 16 f32 values -> 16 exact int8 codes (quantize() semantics), packed.  Common
// path: q = y * inv clamped to [lo, 127] with NaN-propagating min/max (exact: clip
// commutes with rint there, and the .5 ties at 127.5 / -128.5 land on the same code
// either way; lo = 0 fuses a preceding ReLU since inv > 0), rounded by the 1.5*2^23
// magic add whose low byte IS the two's-complement code.  One max-reduction of
// |q - rint(q)| flags the rare tie-band value or NaN; then every value is redone on
// the exact f64 path.
__device__ __forceinline__ uint4 quant16(const float (&y)[16], double s, float inv, float lo = -128.0f) {
  // packed f32x2 arithmetic (sm_100): q = y*inv, t = q + M, d = q - (t - M)
  const float2 M2 = make_float2(12582912.0f, 12582912.0f), I2 = make_float2(inv, inv);
  const float2 NEG1 = make_float2(-1.0f, -1.0f);
  uint32_t tb[16];
  float dmax = 0.0f;
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    float2 qv = __fmul2_rn(make_float2(y[j], y[j + 1]), I2);
    qv.x = fmin_nan(fmax_nan(qv.x, lo), 127.0f);
    qv.y = fmin_nan(fmax_nan(qv.y, lo), 127.0f);
    const float2 t = __fadd2_rn(qv, M2);
    const float2 d = __fadd2_rn(qv, __ffma2_rn(t, NEG1, M2));  // q + (M - t), both exact
    dmax = fmax3_nan(dmax, fabsf(d.x), fabsf(d.y));
    tb[j] = __float_as_uint(t.x);
    tb[j + 1] = __float_as_uint(t.y);
  }
  if (!(dmax < kTieBand)) {
    // redo only the flagged values (a tie-band value or NaN); the others keep their
    // magic-add code.  Constant activations (empty canvas regions) make a tie channel
    // hit every pixel, so the per-value patch matters.
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      float2 qv = __fmul2_rn(make_float2(y[j], y[j + 1]), I2);
      qv.x = fmin_nan(fmax_nan(qv.x, lo), 127.0f);
      qv.y = fmin_nan(fmax_nan(qv.y, lo), 127.0f);
      const float2 d = __fadd2_rn(qv, __ffma2_rn(__fadd2_rn(qv, M2), NEG1, M2));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!(fabsf(h ? d.y : d.x) < kTieBand)) {
          const float yj = lo == 0.0f ? fmaxf(y[j + h], 0.0f) : y[j + h];
          tb[j + h] = (uint32_t)quantize_exact(yj, s, inv);
        }
      }
    }
  }
  return make_uint4(__byte_perm(__byte_perm(tb[0], tb[1], 0x0040), __byte_perm(tb[2], tb[3], 0x0040), 0x5410),
                    __byte_perm(__byte_perm(tb[4], tb[5], 0x0040), __byte_perm(tb[6], tb[7], 0x0040), 0x5410),
                    __byte_perm(__byte_perm(tb[8], tb[9], 0x0040), __byte_perm(tb[10], tb[11], 0x0040), 0x5410),
                    __byte_perm(__byte_perm(tb[12], tb[13], 0x0040), __byte_perm(tb[14], tb[15], 0x0040), 0x5410));
}

// fp16_roundtrip semantics for a pair: satfinite == clip(+-65504) then RNE; NaN stays NaN
__device__ __forceinline__ uint32_t f16x2_sat(float lo_v, float hi_v) {
  uint32_t r;
  asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_v), "f"(lo_v));
  return r;
}

// 16 channels of one pixel as (hi, lo) planes: 4 + 4 float4 stores
__device__ __forceinline__ void store16_f32x2(const OutDev& od, int64_t off, const float (&y)[16]) {
  float4* hi = reinterpret_cast<float4*>(reinterpret_cast<float*>(od.ptr) + off);
  float4* lo = reinterpret_cast<float4*>(reinterpret_cast<float*>(od.ptr) + off + (od.c_stride >> 1));
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 a = tf32_split(y[4 * q]), b = tf32_split(y[4 * q + 1]), c = tf32_split(y[4 * q + 2]),
                 d = tf32_split(y[4 * q + 3]);
    hi[q] = make_float4(a.x, b.x, c.x, d.x);
    lo[q] = make_float4(a.y, b.y, c.y, d.y);
  }
}

// 16 consecutive channels of one pixel -> one consumer format (vectorised when the
// run is complete and aligned, element-wise otherwise)
__device__ __forceinline__ void store16(const OutDev& od, int64_t pix, int c0, const float (&y)[16], int n_live) {
  const int64_t off = pix * od.c_stride + od.c_offset + c0;
  if (n_live == 16 && od.dtype == PMX_I8 && (off & 15) == 0) {
    *reinterpret_cast<uint4*>(reinterpret_cast<int8_t*>(od.ptr) + off) = quant16(y, od.scale, od.inv);
  } else if (n_live == 16 && od.dtype == PMX_F16 && (off & 7) == 0) {
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(od.ptr) + off);
    dst[0] = make_uint4(f16x2_sat(y[0], y[1]), f16x2_sat(y[2], y[3]), f16x2_sat(y[4], y[5]), f16x2_sat(y[6], y[7]));
    dst[1] = make_uint4(f16x2_sat(y[8], y[9]), f16x2_sat(y[10], y[11]), f16x2_sat(y[12], y[13]),
                        f16x2_sat(y[14], y[15]));
  } else if (n_live == 16 && od.dtype == PMX_F32 && (off & 3) == 0) {
    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(od.ptr) + off);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
  } else if (n_live == 16 && od.dtype == PMX_F32X2 && (off & 3) == 0 && (od.c_stride & 7) == 0) {
    store16_f32x2(od, off, y);
  } else {
    for (int j = 0; j < n_live; ++j) store_one(od, pix, c0 + j, y[j]);
  }
}

__host__ pmx_status validate_outs(const pmx_out* outs, int n, int c_needed);

// first-conv input gathered from pillar rows (pmx_conv_gather)
struct GatherIn {
  const void* feats;
  const int32_t* map;
  int32_t pcap;
};

}  // namespace pmx
