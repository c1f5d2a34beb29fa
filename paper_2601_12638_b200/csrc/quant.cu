// K1 quantize / fake_quant / fp16_roundtrip, K2 min/max observers, error plumbing,
// nearest 2x upsample.  All HBM-bound elementwise kernels: grid-stride loops over
// 4-element vectors, grid sized to a multiple of the 148 SMs.
#include <mutex>

#include "pmx_common.cuh"

namespace pmx {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int num_sms() {
  static std::once_flag once[64];
  static int count[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::call_once(once[dev], [dev] {
    int n = 0;
    count[dev] = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0 ? n : 148;
  });
  return count[dev];
}

pmx_status fail(pmx_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

pmx_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PMX_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return PMX_OK;
}

pmx_status validate_outs(const pmx_out* outs, int n, int c_needed) {
  if (n < 1 || n > PMX_MAX_OUTS) return fail(PMX_ERR_INVALID, "n_outs must be 1..3");
  for (int i = 0; i < n; ++i) {
    if (!outs[i].ptr) return fail(PMX_ERR_INVALID, "output pointer is NULL");
    const int dt = outs[i].dtype;
    if (!(dt == PMX_F32 || dt == PMX_F16 || dt == PMX_I8 || dt == PMX_F32X2))
      return fail(PMX_ERR_INVALID, "bad output dtype");
    const int plane = dt == PMX_F32X2 ? outs[i].c_stride / 2 : outs[i].c_stride;
    if (dt == PMX_F32X2 && (outs[i].c_stride & 1)) return fail(PMX_ERR_INVALID, "f32x2 output needs an even c_stride");
    if (outs[i].c_offset < 0 || outs[i].c_offset + c_needed > plane)
      return fail(PMX_ERR_INVALID, "output channel slice exceeds c_stride");
    if (outs[i].dtype == PMX_I8 && !(outs[i].scale > 0.0))
      return fail(PMX_ERR_INVALID, "int8 output needs a positive scale");
  }
  return PMX_OK;
}

static int grid_for(int64_t n, int threads) {
  int64_t blocks = ceil_div(n, threads);
  int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

__global__ void quantize_kernel(const float* __restrict__ x, int64_t n, double s, float inv,
                                int32_t* __restrict__ codes, float* __restrict__ fq) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int c = quantize_exact(x[i], s, inv);
    if (codes) codes[i] = c;
    if (fq) fq[i] = (float)__dmul_rn((double)c, s);
  }
}

__global__ void quantize_f64_kernel(const double* __restrict__ x, int64_t n, double s, int32_t* __restrict__ codes,
                                    float* __restrict__ fq) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = x[i];
    double q = v != v ? 0.0 : rint(__ddiv_rn(v, s));
    q = q < -128.0 ? -128.0 : (q > 127.0 ? 127.0 : q);
    if (codes) codes[i] = (int32_t)q;
    if (fq) fq[i] = (float)__dmul_rn(q, s);
  }
}

__device__ __forceinline__ unsigned long long d2key(double f) {
  unsigned long long b = (unsigned long long)__double_as_longlong(f);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void __launch_bounds__(256) minmax_f64_kernel(const double* __restrict__ x, int64_t n,
                                                         unsigned long long* keys) {
  unsigned long long lo = ~0ull, hi = 0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = x[i];
    unsigned long long kl, kh;
    if (v != v) {  // NaN widens both ends to a non-finite value
      kl = d2key(-__longlong_as_double(0x7ff8000000000000ll));
      kh = d2key(__longlong_as_double(0x7ff8000000000000ll));
    } else {
      kl = kh = d2key(v);
    }
    lo = kl < lo ? kl : lo;
    hi = kh > hi ? kh : hi;
  }
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if ((threadIdx.x & 31) == 0 && lo <= hi) {
    atomicMin(keys + 0, lo);
    atomicMax(keys + 1, hi);
  }
}

__global__ void minmax_f64_init_kernel(unsigned long long* keys) {
  keys[0] = ~0ull;
  keys[1] = 0ull;
}

__global__ void quantize_rows_kernel(const float* __restrict__ w, int64_t rows, int64_t cols,
                                     const double* __restrict__ scales, int8_t* __restrict__ codes,
                                     float* __restrict__ fq) {
  int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = scales[i / cols];
    // weights: the f64 divide is the reference op; tiny tensors, exactness first
    double q = rint(__ddiv_rn((double)w[i], s));
    q = q < -128.0 ? -128.0 : (q > 127.0 ? 127.0 : q);
    if (codes) codes[i] = (int8_t)(int)q;
    if (fq) fq[i] = (float)__dmul_rn(q, s);
  }
}

__global__ void fp16_kernel(const float* __restrict__ x, int64_t n, float* __restrict__ out,
                            __half* __restrict__ out16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    __half h = f16_sat(x[i]);
    if (out) out[i] = __half2float(h);
    if (out16) out16[i] = h;
  }
}

__global__ void minmax_init_kernel(uint32_t* keys, int64_t n_pairs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pairs;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[2 * i] = 0xffffffffu;
    keys[2 * i + 1] = 0u;
  }
}

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_f<int8_t>(int8_t v) { return (float)v; }

template <typename T>
__global__ void __launch_bounds__(256) minmax_kernel(const T* __restrict__ x, int64_t n, uint32_t* keys) {
  float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = to_f<T>(x[i]);
    lo = nmin(lo, v);
    hi = nmax(hi, v);
  }
  // NaN-aware warp reduce: propagate NaN to both ends
  for (int o = 16; o > 0; o >>= 1) {
    lo = nmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = nmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (lo != lo || hi != hi) {  // non-finite marker: NaN key extremes
      atomicMin(keys + 0, f2key(__int_as_float(0xffc00000)));
      atomicMax(keys + 1, f2key(__int_as_float(0x7fc00000)));
    } else if (lo <= hi) {
      atomicMin(keys + 0, f2key(lo));
      atomicMax(keys + 1, f2key(hi));
    }
  }
}

__global__ void __launch_bounds__(256) cast_out_kernel(const float* __restrict__ x, int64_t pixels, int32_t c,
                                                       const Outs outs, uint32_t* keys) {
  float lo = __int_as_float(0x7f800000), hi = -lo;
  const int64_t n = pixels * c;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    store_all(outs, i / c, (int)(i % c), v);
    lo = nmin(lo, v);
    hi = nmax(hi, v);
  }
  if (keys) block_minmax_commit<256>(lo, hi, keys);
}

// fixed partial count (not tied to the SM count): the f64 reduction order, and so the
// result, is the same on every device
constexpr int kErrBlocks = 1184;

__global__ void __launch_bounds__(256) sq_err_partial(const float* __restrict__ a, const float* __restrict__ b,
                                                      int64_t n, double* part) {
  __shared__ double sh[2][8];
  double e = 0.0, r = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)a[i] - (double)b[i];
    e += d * d;
    r += (double)b[i] * (double)b[i];
  }
  for (int o = 16; o > 0; o >>= 1) {
    e += __shfl_xor_sync(0xffffffffu, e, o);
    r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  const int wid = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sh[0][wid] = e;
    sh[1][wid] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double se = 0.0, sr = 0.0;
    for (int w = 0; w < 8; ++w) {
      se += sh[0][w];
      sr += sh[1][w];
    }
    part[2 * blockIdx.x] = se;
    part[2 * blockIdx.x + 1] = sr;
  }
}

__global__ void sq_err_final(const double* __restrict__ part, int nparts, double* out2) {
  if (threadIdx.x != 0) return;
  double e = 0.0, r = 0.0;
  for (int i = 0; i < nparts; ++i) {
    e += part[2 * i];
    r += part[2 * i + 1];
  }
  out2[0] += e;
  out2[1] += r;
}

template <typename T>
__global__ void upsample2x_kernel(const T* __restrict__ x, int32_t b, int32_t h, int32_t w, int32_t c,
                                  T* __restrict__ out) {
  int64_t n = (int64_t)b * (2 * h) * (2 * w) * c;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t ch = i % c;
    int64_t pix = i / c;
    int64_t ox = pix % (2 * w);
    int64_t t = pix / (2 * w);
    int64_t oy = t % (2 * h);
    int64_t bb = t / (2 * h);
    out[i] = x[((bb * h + oy / 2) * w + ox / 2) * c + ch];
  }
}

}  // namespace pmx

using namespace pmx;

extern "C" {

const char* pmx_last_error(void) { return g_last_error.c_str(); }
int32_t pmx_abi_version(void) { return PMX_ABI_VERSION; }

pmx_status pmx_zero(void* ptr, size_t bytes, pmx_stream_t stream) {
  if (bytes == 0) return PMX_OK;
  PMX_REQUIRE(ptr != nullptr, "NULL pointer");
  PMX_CUDA(cudaMemsetAsync(ptr, 0, bytes, stream));
  return PMX_OK;
}

static pmx_status quantize_any(const void* x, int32_t x_dtype, int64_t n, double scale, int32_t* codes, float* fq,
                               pmx_stream_t stream, const char* what) {
  PMX_REQUIRE(n >= 0, "negative length");
  PMX_REQUIRE(scale > 0.0, "scale must be positive and finite");
  PMX_REQUIRE(x_dtype == PMX_F32 || x_dtype == PMX_F64, "quantize input must be f32 or f64");
  if (n == 0) return PMX_OK;
  if (x_dtype == PMX_F32) {
    QScale q = make_qscale(scale);
    quantize_kernel<<<grid_for(n, 256), 256, 0, stream>>>((const float*)x, n, q.s, q.inv, codes, fq);
  } else {
    quantize_f64_kernel<<<grid_for(n, 256), 256, 0, stream>>>((const double*)x, n, scale, codes, fq);
  }
  return check_launch(what);
}

pmx_status pmx_quantize(const void* x, int32_t x_dtype, int64_t n, double scale, int32_t* codes,
                        pmx_stream_t stream) {
  return quantize_any(x, x_dtype, n, scale, codes, nullptr, stream, "pmx_quantize");
}

pmx_status pmx_fake_quant(const void* x, int32_t x_dtype, int64_t n, double scale, float* out, pmx_stream_t stream) {
  return quantize_any(x, x_dtype, n, scale, nullptr, out, stream, "pmx_fake_quant");
}

pmx_status pmx_minmax_f64_init(uint64_t* keys, pmx_stream_t stream) {
  minmax_f64_init_kernel<<<1, 1, 0, stream>>>((unsigned long long*)keys);
  return check_launch("pmx_minmax_f64_init");
}

pmx_status pmx_minmax_f64(const double* x, int64_t n, uint64_t* keys, pmx_stream_t stream) {
  PMX_REQUIRE(n >= 0, "negative length");
  if (n == 0) return PMX_OK;
  minmax_f64_kernel<<<grid_for(n, 256), 256, 0, stream>>>(x, n, (unsigned long long*)keys);
  return check_launch("pmx_minmax_f64");
}

pmx_status pmx_quantize_rows(const float* w, int64_t rows, int64_t cols, const double* scales,
                             int8_t* codes, float* dequant, pmx_stream_t stream) {
  PMX_REQUIRE(rows >= 0 && cols >= 0, "negative extent");
  if (rows * cols == 0) return PMX_OK;
  quantize_rows_kernel<<<grid_for(rows * cols, 256), 256, 0, stream>>>(w, rows, cols, scales, codes, dequant);
  return check_launch("pmx_quantize_rows");
}

pmx_status pmx_fp16_roundtrip(const float* x, int64_t n, float* out_f32, uint16_t* out_f16,
                              pmx_stream_t stream) {
  PMX_REQUIRE(n >= 0, "negative length");
  if (n == 0) return PMX_OK;
  fp16_kernel<<<grid_for(n, 256), 256, 0, stream>>>(x, n, out_f32, reinterpret_cast<__half*>(out_f16));
  return check_launch("pmx_fp16_roundtrip");
}

pmx_status pmx_minmax_init(uint32_t* keys, int64_t n_pairs, pmx_stream_t stream) {
  PMX_REQUIRE(n_pairs >= 0, "negative length");
  if (n_pairs == 0) return PMX_OK;
  minmax_init_kernel<<<grid_for(n_pairs, 256), 256, 0, stream>>>(keys, n_pairs);
  return check_launch("pmx_minmax_init");
}

pmx_status pmx_minmax(const void* x, int64_t n, int32_t dtype, uint32_t* keys, pmx_stream_t stream) {
  PMX_REQUIRE(n >= 0, "negative length");
  if (n == 0) return PMX_OK;
  int g = grid_for(n, 256);
  if (dtype == PMX_F32)
    minmax_kernel<float><<<g, 256, 0, stream>>>((const float*)x, n, keys);
  else if (dtype == PMX_F16)
    minmax_kernel<__half><<<g, 256, 0, stream>>>((const __half*)x, n, keys);
  else if (dtype == PMX_I8)
    minmax_kernel<int8_t><<<g, 256, 0, stream>>>((const int8_t*)x, n, keys);
  else
    return fail(PMX_ERR_INVALID, "bad dtype");
  return check_launch("pmx_minmax");
}

size_t pmx_sq_err_workspace(void) { return 2 * sizeof(double) * kErrBlocks; }

pmx_status pmx_sq_err(const float* a, const float* b, int64_t n, double* out2, double* ws, size_t ws_bytes,
                      pmx_stream_t stream) {
  PMX_REQUIRE(n >= 0, "negative length");
  if (n == 0) return PMX_OK;
  PMX_REQUIRE(a && b && out2 && ws, "NULL operand");
  PMX_REQUIRE(ws_bytes >= pmx_sq_err_workspace(), "pmx_sq_err workspace too small (see pmx_sq_err_workspace)");
  sq_err_partial<<<kErrBlocks, 256, 0, stream>>>(a, b, n, ws);
  sq_err_final<<<1, 32, 0, stream>>>(ws, kErrBlocks, out2);
  return check_launch("pmx_sq_err");
}

pmx_status pmx_cast_out(const float* x, int64_t pixels, int32_t c, const pmx_out* outs, int32_t n_outs,
                        uint32_t* keys, pmx_stream_t stream) {
  PMX_REQUIRE(pixels >= 0 && c >= 1, "bad extents");
  pmx_status st = validate_outs(outs, n_outs, c);
  if (st != PMX_OK) return st;
  if (pixels == 0) return PMX_OK;
  cast_out_kernel<<<grid_for(pixels * c, 256), 256, 0, stream>>>(x, pixels, c, make_outs(outs, n_outs), keys);
  return check_launch("pmx_cast_out");
}

pmx_status pmx_upsample2x(const void* x, int32_t dtype, int32_t batch, int32_t h, int32_t w, int32_t c,
                          void* out, pmx_stream_t stream) {
  PMX_REQUIRE(batch >= 0 && h >= 0 && w >= 0 && c >= 0, "negative extent");
  int64_t n = (int64_t)batch * 4 * h * w * c;
  if (n == 0) return PMX_OK;
  int g = grid_for(n, 256);
  if (dtype == PMX_F32)
    upsample2x_kernel<float><<<g, 256, 0, stream>>>((const float*)x, batch, h, w, c, (float*)out);
  else if (dtype == PMX_F16)
    upsample2x_kernel<__half><<<g, 256, 0, stream>>>((const __half*)x, batch, h, w, c, (__half*)out);
  else if (dtype == PMX_I8)
    upsample2x_kernel<int8_t><<<g, 256, 0, stream>>>((const int8_t*)x, batch, h, w, c, (int8_t*)out);
  else
    return fail(PMX_ERR_INVALID, "bad dtype");
  return check_launch("pmx_upsample2x");
}

}  // extern "C"
