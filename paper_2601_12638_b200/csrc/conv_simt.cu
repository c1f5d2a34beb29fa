// SIMT implicit-GEMM conv / deconv (all precisions, any kernel/stride/padding).
//
// This is the general-shape kernel and the in-tree cross-check for the tcgen05
// path: INT8 accumulates int8 x int8 products in int32 (exact, order-free, so the
// tensor-core accumulators must match it bit for bit); FP16 multiplies binary16
// values in f32 (exact products) and sums in f32; FP32 is plain FFMA.
// GEMM view: M = output pixels (deconv: input pixels), N = Cout (deconv:
// k*k*Cout), K = kh*kw*Cin in (ky, kx, c) order (deconv: Cin).
#include "pmx_common.cuh"

namespace pmx {

// implemented in conv_tc.cu
pmx_status conv_tc_try(const pmx_conv_desc& d, const void* x, const void* w, const float* alpha, const float* bias,
                       const float* bn_post, const Outs& outs, uint32_t* keys, void* ws, size_t ws_bytes,
                       cudaStream_t st, bool* launched, const GatherIn* gin);
size_t conv_tc_workspace(const pmx_conv_desc& d);
bool conv_tc_gather_ok(const pmx_conv_desc& d);
int conv_tc_supported(const pmx_conv_desc& d);
bool conv_tc_heads_ok(const pmx_conv_desc& d);
pmx_status conv_tc_deconv_heads(const pmx_conv_desc& d, const void* x, const void* w, const float* alpha,
                                const float* bias, const pmx_head_fuse& hf, cudaStream_t st);
const char* conv_tc_backend(int dtype, int kind);

// backend override of the CALLING thread (tests): thread-local, so concurrent callers on
// other threads are unaffected and the library holds no shared mutable state
thread_local int g_conv_backend_mode = 0;

namespace {

constexpr int BM = 64, BN = 64, BK = 32;

struct ConvArgs {
  pmx_conv_desc d;
  const void* x;
  const void* w;
  const float* alpha;
  const float* bias;
  const float* bn_post;
  uint32_t* keys;
  int64_t M;
  int N, K;
};

template <int DT>
struct Acc { using T = float; };
template <>
struct Acc<PMX_I8> { using T = int; };

template <int DT>
__device__ __forceinline__ typename Acc<DT>::T load_x(const void* p, int64_t off) {
  if constexpr (DT == PMX_I8) return (int)reinterpret_cast<const int8_t*>(p)[off];
  else if constexpr (DT == PMX_F16) return __half2float(reinterpret_cast<const __half*>(p)[off]);
  else return reinterpret_cast<const float*>(p)[off];
}

// PMX_F32X2 activation: hi + lo reassembles the f32 value exactly
__device__ __forceinline__ float load_x2(const void* p, int64_t off, int plane) {
  const float* f = reinterpret_cast<const float*>(p);
  return __fadd_rn(f[off], f[off + plane]);
}

template <int DT, bool DECONV>
__global__ void __launch_bounds__(256) conv_simt_kernel(const ConvArgs a, const Outs outs) {
  using T = typename Acc<DT>::T;
  __shared__ T As[BK][BM + 4];
  __shared__ T Bs[BK][BN + 4];
  const pmx_conv_desc& d = a.d;
  const int tid = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int tm = tid / 16, tn = tid % 16;
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = T(0);

  for (int k0 = 0; k0 < a.K; k0 += BK) {
    // A tile: BM x BK
    for (int e = tid; e < BM * BK; e += 256) {
      const int mm = e / BK, kk = e % BK;
      const int64_t m = m0 + mm;
      const int k = k0 + kk;
      T v = T(0);
      if (m < a.M && k < a.K) {
        if (DECONV) {
          if constexpr (DT == PMX_F32X2) v = load_x2(a.x, m * d.in_c_stride + d.in_c_offset + k, d.in_c_stride / 2);
          else v = load_x<DT>(a.x, m * d.in_c_stride + d.in_c_offset + k);
        } else {
          const int c = k % d.in_c;
          const int tap = k / d.in_c;
          const int ky = tap / d.k_w, kx = tap % d.k_w;
          const int ox = (int)(m % d.out_w);
          const int64_t t = m / d.out_w;
          const int oy = (int)(t % d.out_h);
          const int64_t bb = t / d.out_h;
          const int iy = oy * d.stride_h - d.pad_h + ky;
          const int ix = ox * d.stride_w - d.pad_w + kx;
          if (iy >= 0 && iy < d.in_h && ix >= 0 && ix < d.in_w) {
            const int64_t off = ((bb * d.in_h + iy) * d.in_w + ix) * d.in_c_stride + d.in_c_offset + c;
            if constexpr (DT == PMX_F32X2) v = load_x2(a.x, off, d.in_c_stride / 2);
            else v = load_x<DT>(a.x, off);
          }
        }
      }
      As[kk][mm] = v;
    }
    for (int e = tid; e < BN * BK; e += 256) {
      const int nn = e / BK, kk = e % BK;
      const int n = n0 + nn, k = k0 + kk;
      T v = T(0);
      if (n < a.N && k < a.K) {
        if constexpr (DT == PMX_F32X2) {
          // prepacked [w_hi | w_hi | w_lo] per tap: w = w_hi + w_lo exactly
          const int tap = k / d.in_c, c = k - tap * d.in_c;
          const float* w = reinterpret_cast<const float*>(a.w) + (int64_t)n * 3 * a.K + (int64_t)tap * 3 * d.in_c;
          v = __fadd_rn(w[c], w[2 * d.in_c + c]);
        } else {
          v = load_x<DT>(a.w, (int64_t)n * a.K + k);
        }
      }
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < BK; ++kk) {
      T av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][tm * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tn * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (DT == PMX_I8) acc[i][j] += av[i] * bv[j];
          else acc[i][j] = __fmaf_rn(av[i], bv[j], acc[i][j]);
        }
    }
    __syncthreads();
  }

  float lo = __int_as_float(0x7f800000), hi = -lo;
  const int cout = d.out_c;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + tm * 4 + i;
    if (m >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tn * 4 + j;
      if (n >= a.N) continue;
      int co;
      int64_t pix;
      if (DECONV) {
        co = n % cout;
        const int tap = n / cout;
        const int dy = tap / d.k_w, dx = tap % d.k_w;
        const int ix = (int)(m % d.in_w);
        const int64_t t = m / d.in_w;
        const int iy = (int)(t % d.in_h);
        const int64_t bb = t / d.in_h;
        pix = (bb * d.out_h + (int64_t)iy * d.stride_h + dy) * d.out_w + (int64_t)ix * d.stride_w + dx;
      } else {
        co = n;
        pix = m;
      }
      float y;
      if constexpr (DT == PMX_I8) y = __fmaf_rn((float)acc[i][j], a.alpha[co], a.bias[co]);
      else y = __fadd_rn(acc[i][j], a.bias[co]);
      if (a.bn_post)
        y = __fadd_rn(__fmul_rn(__fsub_rn(y, a.bn_post[co]), a.bn_post[cout + co]), a.bn_post[2 * cout + co]);
      if (d.relu) y = fmaxf(y, 0.f);
      store_all(outs, pix, co, y);
      lo = nmin(lo, y);
      hi = nmax(hi, y);
    }
  }
  if (a.keys) block_minmax_commit<256>(lo, hi, a.keys);
}

template <int DT>
void launch_simt(const ConvArgs& a, const Outs& o, cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(a.M, BM), (unsigned)ceil_div(a.N, BN));
  if (a.d.kind == PMX_DECONV2D) conv_simt_kernel<DT, true><<<grid, 256, 0, st>>>(a, o);
  else conv_simt_kernel<DT, false><<<grid, 256, 0, st>>>(a, o);
}

pmx_status validate(const pmx_conv_desc& d) {
  PMX_REQUIRE(d.kind == PMX_CONV2D || d.kind == PMX_DECONV2D, "bad conv kind");
  PMX_REQUIRE((d.in_dtype >= PMX_F32 && d.in_dtype <= PMX_I8) || d.in_dtype == PMX_F32X2, "bad conv dtype");
  PMX_REQUIRE(d.batch >= 0 && d.in_h >= 1 && d.in_w >= 1 && d.in_c >= 1 && d.out_c >= 1, "bad conv extents");
  PMX_REQUIRE(d.in_dtype != PMX_F32X2 || d.in_c_stride % 2 == 0, "f32x2 input needs an even in_c_stride");
  PMX_REQUIRE(d.in_c_offset >= 0 &&
                  d.in_c_offset + d.in_c <= (d.in_dtype == PMX_F32X2 ? d.in_c_stride / 2 : d.in_c_stride),
              "input channel slice exceeds stride");
  PMX_REQUIRE(d.k_h >= 1 && d.k_w >= 1 && d.stride_h >= 1 && d.stride_w >= 1 && d.pad_h >= 0 && d.pad_w >= 0,
              "bad kernel/stride/padding");
  if (d.kind == PMX_CONV2D) {
    const int oh = (d.in_h + 2 * d.pad_h - d.k_h) / d.stride_h + 1;
    const int ow = (d.in_w + 2 * d.pad_w - d.k_w) / d.stride_w + 1;
    PMX_REQUIRE(oh >= 1 && ow >= 1 && oh == d.out_h && ow == d.out_w, "conv output extents mismatch");
  } else {
    PMX_REQUIRE(d.k_h == d.stride_h && d.k_w == d.stride_w && d.pad_h == 0 && d.pad_w == 0,
                "deconv2d supports kernel == stride, no padding");
    PMX_REQUIRE(d.out_h == d.in_h * d.stride_h && d.out_w == d.in_w * d.stride_w, "deconv output extents mismatch");
  }
  return PMX_OK;
}

}  // namespace
}  // namespace pmx

using namespace pmx;

extern "C" {

void pmx_set_conv_backend(int32_t mode) { g_conv_backend_mode = mode; }

const char* pmx_conv_backend(int32_t in_dtype, int32_t kind) {
  if (g_conv_backend_mode == 1) return "simt";
  return conv_tc_backend(in_dtype, kind);
}

int32_t pmx_deconv_heads_supported(const pmx_conv_desc* desc) {
  if (!desc || validate(*desc) != PMX_OK) return 0;
  return conv_tc_heads_ok(*desc) ? 1 : 0;
}

pmx_status pmx_deconv_heads(const pmx_conv_desc* desc, const void* x, const void* w, const float* alpha,
                            const float* bias, const pmx_head_fuse* heads, pmx_stream_t stream) {
  PMX_REQUIRE(desc != nullptr && heads != nullptr, "desc/heads is NULL");
  const pmx_conv_desc d = *desc;
  pmx_status st = validate(d);
  if (st != PMX_OK) return st;
  const pmx_head_fuse& hf = *heads;
  PMX_REQUIRE(x && w && bias && hf.w_codes && hf.partial, "NULL deconv/heads operand");
  PMX_REQUIRE(d.in_dtype != PMX_I8 || alpha, "int8 conv needs alpha");
  PMX_REQUIRE(hf.n_heads >= 1 && hf.n_heads <= 20, "n_heads must be 1..20");
  PMX_REQUIRE(hf.stage >= 0 && hf.stage <= 2, "stage must be 0, 1 or 2");
  PMX_REQUIRE(hf.in_scale > 0.0, "heads' activation scale must be positive");
  PMX_REQUIRE(hf.part_stride >= 1 && (hf.part_stride & (hf.part_stride - 1)) == 0 &&
                  d.out_h % hf.part_stride == 0 && d.out_w % hf.part_stride == 0,
              "part_stride must be a power of two dividing the output extents");
  PMX_REQUIRE(hf.stage != 2 || (hf.heads && hf.head_alpha && hf.head_bias && hf.heads_c_stride >= hf.n_heads),
              "the last stage needs heads, head_alpha, head_bias");
  if (d.batch == 0) return PMX_OK;
  return conv_tc_deconv_heads(d, x, w, alpha, bias, hf, stream);
}

int32_t pmx_conv_tc_supported(const pmx_conv_desc* desc) {
  if (!desc || validate(*desc) != PMX_OK) return 0;
  return conv_tc_supported(*desc);
}

size_t pmx_conv_workspace(const pmx_conv_desc* desc) {
  if (!desc) return 0;
  return conv_tc_workspace(*desc);
}

pmx_status pmx_conv(const pmx_conv_desc* desc, const void* x, const void* w, const float* alpha, const float* bias,
                    const float* bn_post, const pmx_out* outs, int32_t n_outs, uint32_t* out_keys, void* ws,
                    size_t ws_bytes, pmx_stream_t stream) {
  PMX_REQUIRE(desc != nullptr, "desc is NULL");
  const pmx_conv_desc d = *desc;
  pmx_status st = validate(d);
  if (st != PMX_OK) return st;
  PMX_REQUIRE(x && w && bias, "NULL conv operand");
  PMX_REQUIRE(d.in_dtype != PMX_I8 || alpha, "int8 conv needs alpha");
  st = validate_outs(outs, n_outs, d.out_c);
  if (st != PMX_OK) return st;
  if (d.batch == 0) return PMX_OK;
  Outs o = make_outs(outs, n_outs);
  if (g_conv_backend_mode == 0) {
    bool launched = false;
    st = conv_tc_try(d, x, w, alpha, bias, bn_post, o, out_keys, ws, ws_bytes, stream, &launched, nullptr);
    if (st != PMX_OK || launched) return st;
  }
  ConvArgs a;
  a.d = d;
  a.x = x;
  a.w = w;
  a.alpha = alpha;
  a.bias = bias;
  a.bn_post = bn_post;
  a.keys = out_keys;
  if (d.kind == PMX_DECONV2D) {
    a.M = (int64_t)d.batch * d.in_h * d.in_w;
    a.N = d.k_h * d.k_w * d.out_c;
    a.K = d.in_c;
  } else {
    a.M = (int64_t)d.batch * d.out_h * d.out_w;
    a.N = d.out_c;
    a.K = d.k_h * d.k_w * d.in_c;
  }
  if (d.in_dtype == PMX_I8) launch_simt<PMX_I8>(a, o, stream);
  else if (d.in_dtype == PMX_F16) launch_simt<PMX_F16>(a, o, stream);
  else if (d.in_dtype == PMX_F32X2) launch_simt<PMX_F32X2>(a, o, stream);
  else launch_simt<PMX_F32>(a, o, stream);
  return check_launch("pmx_conv(simt)");
}

int32_t pmx_conv_gather_supported(const pmx_conv_desc* desc) {
  if (!desc || validate(*desc) != PMX_OK) return 0;
  const int esz = elem_size(desc->in_dtype);
  if (((int64_t)desc->in_c_stride * esz) % 16 != 0 || ((int64_t)desc->in_c_offset * esz) % 16 != 0) return 0;
  return conv_tc_gather_ok(*desc) ? 1 : 0;
}

pmx_status pmx_conv_gather(const pmx_conv_desc* desc, const void* feats, const int32_t* cell_map, int32_t pcap,
                           const void* w, const float* alpha, const float* bias, const float* bn_post,
                           const pmx_out* outs, int32_t n_outs, uint32_t* out_keys, pmx_stream_t stream) {
  PMX_REQUIRE(desc != nullptr, "desc is NULL");
  const pmx_conv_desc d = *desc;
  pmx_status st = validate(d);
  if (st != PMX_OK) return st;
  PMX_REQUIRE(feats && cell_map && w && bias, "NULL conv operand");
  PMX_REQUIRE(pcap >= 1, "pcap must be positive");
  PMX_REQUIRE(d.in_dtype != PMX_I8 || alpha, "int8 conv needs alpha");
  st = validate_outs(outs, n_outs, d.out_c);
  if (st != PMX_OK) return st;
  if (d.batch == 0) return PMX_OK;
  const int esz = elem_size(d.in_dtype);
  PMX_REQUIRE(((int64_t)d.in_c_stride * esz) % 16 == 0 && ((int64_t)d.in_c_offset * esz) % 16 == 0 &&
                  (reinterpret_cast<uintptr_t>(feats) & 15) == 0,
              "gathered pillar rows must be 16-byte aligned");
  if (g_conv_backend_mode == 1) return fail(PMX_ERR_UNSUPPORTED, "pmx_conv_gather: tcgen05 backend disabled");
  Outs o = make_outs(outs, n_outs);
  GatherIn gin{feats, cell_map, pcap};
  bool launched = false;
  st = conv_tc_try(d, feats, w, alpha, bias, bn_post, o, out_keys, nullptr, 0, stream, &launched, &gin);
  if (st != PMX_OK) return st;
  if (!launched) return fail(PMX_ERR_UNSUPPORTED, "pmx_conv_gather: shape outside the tcgen05 halo kernels");
  return PMX_OK;
}

}  // extern "C"
