// QAT (pm/qat.py) on the GPU: the training forward's pre-activation convolutions, the
// backward pass over the tape (conv / deconv / linear data and weight gradients, the
// clipped straight-through estimator, ReLU / max-pool / scatter / upsample / concat
// adjoints), the detection and MSE losses, gradient norm and the SGD step.
//
// Layouts: activations NHWC f32 (a linear layer is a 1x1 conv over rows), weights as
// the model stores them, [Cout, Cin, kh, kw] (deconv: kernel == stride, pm model
// extension).  Every reduction runs in a fixed order (no float atomics), so a
// training run is bit-reproducible on one device.  The shapes QAT fine-tunes are
// small (the toy detector, KITTI smoke grids): thread-per-output SIMT kernels with
// channel-contiguous (coalesced) inner loops; the tensor-core convs are the
// inference path's.
#include <cmath>

#include "pmx_common.cuh"

namespace pmx {

namespace {

constexpr int kRedBlocks = 256;  // fixed partial count of the deterministic reductions

struct Geo {
  int deconv;
  int n, ih, iw, ci, co, kh, kw, sh, sw, ph, pw, oh, ow;
};

Geo geo_of(const pmx_conv_desc& d) {
  return Geo{d.kind == PMX_DECONV2D, d.batch, d.in_h, d.in_w, d.in_c, d.out_c, d.k_h, d.k_w,
             d.stride_h, d.stride_w, d.pad_h, d.pad_w, d.out_h, d.out_w};
}

// out[n, oy, ox, co] = sum_{ci, ki, kj} x[n, iy, ix, ci] * W[co, ci, ki, kj] + b[co]
// (pm/tensor_ops.py:109-131: im2col columns are (ci, ki, kj) -- the same K order here)
__global__ void fwd_kernel(const Geo g, const float* __restrict__ x, const float* __restrict__ w,
                           const float* __restrict__ b, float* __restrict__ out) {
  const int64_t total = (int64_t)g.n * g.oh * g.ow * g.co;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int co = (int)(i % g.co);
    const int64_t pix = i / g.co;
    const int ox = (int)(pix % g.ow), oy = (int)((pix / g.ow) % g.oh), n = (int)(pix / ((int64_t)g.ow * g.oh));
    float acc = 0.f;
    if (g.deconv) {  // pm model extension: out[s*i+dy, s*j+dx] = x[i, j] . W[:, :, dy, dx]
      const int iy = oy / g.sh, ix = ox / g.sw, dy = oy % g.sh, dx = ox % g.sw;
      const float* xr = x + (((int64_t)n * g.ih + iy) * g.iw + ix) * g.ci;
      const float* wr = w + ((int64_t)co * g.ci * g.kh + dy) * g.kw + dx;
      for (int c = 0; c < g.ci; ++c) acc = __fmaf_rn(xr[c], wr[(int64_t)c * g.kh * g.kw], acc);
    } else {
      for (int c = 0; c < g.ci; ++c) {
        const float* wr = w + ((int64_t)co * g.ci + c) * g.kh * g.kw;
        for (int ki = 0; ki < g.kh; ++ki) {
          const int iy = oy * g.sh - g.ph + ki;
          if (iy < 0 || iy >= g.ih) continue;
          for (int kj = 0; kj < g.kw; ++kj) {
            const int ix = ox * g.sw - g.pw + kj;
            if (ix < 0 || ix >= g.iw) continue;
            acc = __fmaf_rn(x[(((int64_t)n * g.ih + iy) * g.iw + ix) * g.ci + c], wr[ki * g.kw + kj], acc);
          }
        }
      }
    }
    out[i] = __fadd_rn(acc, b[co]);
  }
}

// dx[n, y, x, ci] = sum_{co, ki, kj} dout[n, oy, ox, co] * W[co, ci, ki, kj] over the output
// pixels whose window covers (y, x) (pm/qat.py:145-152: dcols = do2 @ W, then col2im)
__global__ void dgrad_kernel(const Geo g, const float* __restrict__ dout, const float* __restrict__ w,
                             float* __restrict__ dx) {
  const int64_t total = (int64_t)g.n * g.ih * g.iw * g.ci;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % g.ci);
    const int64_t pix = i / g.ci;
    const int x = (int)(pix % g.iw), y = (int)((pix / g.iw) % g.ih), n = (int)(pix / ((int64_t)g.iw * g.ih));
    float acc = 0.f;
    if (g.deconv) {
      for (int dy = 0; dy < g.kh; ++dy)
        for (int dxx = 0; dxx < g.kw; ++dxx) {
          const float* dr = dout + (((int64_t)n * g.oh + (y * g.sh + dy)) * g.ow + (x * g.sw + dxx)) * g.co;
          for (int co = 0; co < g.co; ++co)
            acc = __fmaf_rn(dr[co], w[(((int64_t)co * g.ci + c) * g.kh + dy) * g.kw + dxx], acc);
        }
    } else {
      for (int ki = 0; ki < g.kh; ++ki) {
        const int ty = y + g.ph - ki;
        if (ty < 0 || ty % g.sh) continue;
        const int oy = ty / g.sh;
        if (oy >= g.oh) continue;
        for (int kj = 0; kj < g.kw; ++kj) {
          const int tx = x + g.pw - kj;
          if (tx < 0 || tx % g.sw) continue;
          const int ox = tx / g.sw;
          if (ox >= g.ow) continue;
          const float* dr = dout + (((int64_t)n * g.oh + oy) * g.ow + ox) * g.co;
          for (int co = 0; co < g.co; ++co)
            acc = __fmaf_rn(dr[co], w[(((int64_t)co * g.ci + c) * g.kh + ki) * g.kw + kj], acc);
        }
      }
    }
    dx[i] = acc;
  }
}

// dW[co, ci, ki, kj] = sum over output pixels of dout[., co] * x[window pixel, ci]
// (pm/qat.py:142-143: do2.T @ cols).  Block = one (co, ki, kj) and 32 input channels:
// lane = channel (coalesced NHWC reads), the 8 warps stride over pixels, then a
// fixed-order combine of the 8 partials.
__global__ void __launch_bounds__(256) wgrad_kernel(const Geo g, const float* __restrict__ dout,
                                                    const float* __restrict__ x, float* __restrict__ dw) {
  __shared__ float part[8][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int tap = blockIdx.x % (g.kh * g.kw), co = blockIdx.x / (g.kh * g.kw);
  const int ki = tap / g.kw, kj = tap % g.kw;
  const int c = blockIdx.y * 32 + lane;
  float acc = 0.f;
  if (g.deconv) {  // one term per INPUT pixel: dout[s*i+ki, s*j+kj] . x[i, j]
    const int64_t npx = (int64_t)g.n * g.ih * g.iw;
    for (int64_t p = wid; p < npx; p += 8) {
      const int xx = (int)(p % g.iw), yy = (int)((p / g.iw) % g.ih), n = (int)(p / ((int64_t)g.iw * g.ih));
      const float d = dout[(((int64_t)n * g.oh + (yy * g.sh + ki)) * g.ow + (xx * g.sw + kj)) * g.co + co];
      if (c < g.ci) acc = __fmaf_rn(d, x[p * g.ci + c], acc);
    }
  } else {
    const int64_t npx = (int64_t)g.n * g.oh * g.ow;
    for (int64_t p = wid; p < npx; p += 8) {
      const int ox = (int)(p % g.ow), oy = (int)((p / g.ow) % g.oh), n = (int)(p / ((int64_t)g.ow * g.oh));
      const int iy = oy * g.sh - g.ph + ki, ix = ox * g.sw - g.pw + kj;
      if (iy < 0 || iy >= g.ih || ix < 0 || ix >= g.iw) continue;
      const float d = dout[p * g.co + co];
      if (c < g.ci) acc = __fmaf_rn(d, x[(((int64_t)n * g.ih + iy) * g.iw + ix) * g.ci + c], acc);
    }
  }
  part[wid][lane] = acc;
  __syncthreads();
  if (wid == 0 && c < g.ci) {
    float s = part[0][lane];
    for (int k = 1; k < 8; ++k) s = __fadd_rn(s, part[k][lane]);
    dw[(((int64_t)co * g.ci + c) * g.kh + ki) * g.kw + kj] = s;
  }
}

// db[co] = sum over every output pixel of dout[., co] (pm/qat.py:144)
__global__ void __launch_bounds__(256) bgrad_kernel(const float* __restrict__ dout, int64_t npx, int co_n,
                                                    float* __restrict__ db) {
  __shared__ float part[256];
  const int co = blockIdx.x;
  float acc = 0.f;
  for (int64_t p = threadIdx.x; p < npx; p += 256) acc = __fadd_rn(acc, dout[p * co_n + co]);
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) part[threadIdx.x] = __fadd_rn(part[threadIdx.x], part[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) db[co] = part[0];
}

__global__ void relu_kernel(const float* __restrict__ x, int64_t n, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    out[i] = (v != v) ? v : (v > 0.f ? v : 0.f);  // np.maximum(x, 0): NaN propagates
  }
}

// dout * (pre_act > 0) as the reference's f32 product with a 0/1 mask (pm/qat.py:160-161)
__global__ void relu_bwd_kernel(const float* __restrict__ dout, const float* __restrict__ pre, int64_t n,
                                float* __restrict__ dx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dx[i] = __fmul_rn(dout[i], pre[i] > 0.f ? 1.f : 0.f);
}

// clipped STE, per-tensor (pm/qat.py:68-85): the Python-float bounds q_min * scale meet the
// f32 array as f32 scalars (NumPy 2 weak scalar promotion)
__global__ void ste_kernel(const float* __restrict__ x, int64_t n, float lo, float hi, const float* __restrict__ up,
                           float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    out[i] = __fmul_rn(up[i], (v >= lo && v <= hi) ? 1.f : 0.f);
  }
}

// per-channel: the bounds are an f64 array, so the comparison runs in f64 (pm/qat.py:69-71)
__global__ void ste_rows_kernel(const float* __restrict__ x, int64_t rows, int64_t cols,
                                const double* __restrict__ scales, double qmin, double qmax,
                                const float* __restrict__ up, float* __restrict__ out) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double s = scales[i / cols], v = (double)x[i];
    out[i] = __fmul_rn(up[i], (v >= __dmul_rn(qmin, s) && v <= __dmul_rn(qmax, s)) ? 1.f : 0.f);
  }
}

// masked max over points with the winner (first maximal point, np.argmax) per channel
// (pm/model.py:338-345, pm/tensor_ops.py:163-173)
__global__ void maxpool_kernel(const float* __restrict__ x, const uint8_t* __restrict__ mask, int64_t P, int M, int C,
                               float* __restrict__ out, int32_t* __restrict__ arg) {
  const int64_t total = P * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t p = i / C;
    float best = -INFINITY;
    int bi = 0;
    bool nan = false;
    for (int m = 0; m < M; ++m) {
      const float v = mask[p * M + m] ? x[(p * M + m) * C + c] : -INFINITY;
      if (v != v) {  // NaN wins (first one), as in np.max / np.argmax
        if (!nan) best = v, bi = m, nan = true;
      } else if (!nan && v > best) {
        best = v, bi = m;
      }
    }
    out[i] = best;
    if (arg) arg[i] = bi;
  }
}

// dx[p, arg[p, c], c] = dout[p, c], zero elsewhere (pm/qat.py:180-183)
__global__ void maxpool_bwd_kernel(const float* __restrict__ dout, const int32_t* __restrict__ arg, int64_t P, int M,
                                   int C, float* __restrict__ dx) {
  const int64_t total = P * M * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t pm = i / C;
    const int m = (int)(pm % M);
    const int64_t p = pm / M;
    dx[i] = arg[p * C + c] == m ? dout[p * C + c] : 0.f;
  }
}

// canvas[0, y_p, x_p, :] = feat[p, :] (forward) / dx[p, :] = dcanvas[0, y_p, x_p, :]
// (pm/tensor_ops.py:138-160, pm/qat.py:184-186)
__global__ void scatter_kernel(const float* __restrict__ src, const int32_t* __restrict__ coords, int64_t P, int C,
                               int W, float* __restrict__ dst, int bwd) {
  const int64_t total = P * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t p = i / C;
    const int64_t cell = (int64_t)coords[2 * p] * W + coords[2 * p + 1];
    if (bwd) dst[i] = src[cell * C + c];
    else dst[cell * C + c] = src[i];
  }
}

// each input cell sums its 2x2 block (pm/qat.py:188-190)
__global__ void upsample_bwd_kernel(const float* __restrict__ dout, int N, int H, int W, int C, float* __restrict__ dx) {
  const int64_t total = (int64_t)N * H * W * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t pix = i / C;
    const int x = (int)(pix % W), y = (int)((pix / W) % H), n = (int)(pix / ((int64_t)W * H));
    const int64_t r0 = (((int64_t)n * 2 * H + 2 * y) * 2 * W + 2 * x) * C + c, r1 = r0 + (int64_t)2 * W * C;
    dx[i] = __fadd_rn(__fadd_rn(__fadd_rn(dout[r0], dout[r0 + C]), dout[r1]), dout[r1 + C]);
  }
}

__global__ void add_kernel(const float* __restrict__ a, const float* __restrict__ b, int64_t n, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __fadd_rn(a[i], b[i]);
}

// channel-slice copy between NHWC tensors (concat forward / its adjoint)
__global__ void copy_ch_kernel(const float* __restrict__ src, int64_t pixels, int c, int s_stride, int s_off,
                               float* __restrict__ dst, int d_stride, int d_off) {
  const int64_t total = pixels * c;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % c);
    const int64_t p = i / c;
    dst[p * d_stride + d_off + k] = src[p * s_stride + s_off + k];
  }
}

// ---- deterministic f64 reductions: kRedBlocks fixed partials, then one block

__device__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) finish_kernel(const double* __restrict__ part, int n_sums, double* __restrict__ out) {
  __shared__ double sh[256];
  for (int k = 0; k < n_sums; ++k) {
    const double s = block_sum(threadIdx.x < kRedBlocks ? part[k * kRedBlocks + threadIdx.x] : 0.0, sh);
    if (threadIdx.x == 0) out[k] = s;
  }
}

__device__ __forceinline__ double sigmoid64(double x) {  // pm/qat.py:88-89
  return x >= 0.0 ? __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x))) : __ddiv_rn(exp(x), __dadd_rn(1.0, exp(x)));
}

// detection_loss (pm/qat.py:92-116) on NHWC maps: per element the f64 BCE term and the
// f32 gradient, per block the f64 partial sums (cls term, squared box residual)
__global__ void __launch_bounds__(256) det_loss_kernel(const float* __restrict__ z, const double* __restrict__ t,
                                                       const uint8_t* __restrict__ ignore,
                                                       const uint8_t* __restrict__ pos, const float* __restrict__ r,
                                                       const double* __restrict__ rt, int64_t hw, int ncls, int nreg,
                                                       double n_pos, double cls_w, double reg_w, double pos_w,
                                                       float* __restrict__ dcls, float* __restrict__ dreg,
                                                       double* __restrict__ part) {
  __shared__ double sh[256];
  double cls = 0.0, reg = 0.0;
  const int64_t ncl = hw * ncls, nrg = hw * nreg;
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < ncl; i += (int64_t)kRedBlocks * 256) {
    const double zz = (double)z[i], tt = t[i];
    double w = tt > 0.0 ? pos_w : 1.0;
    if (ignore && ignore[i / ncls]) w = __dmul_rn(w, 0.0);
    // left to right as numpy evaluates it, no contraction into FMAs
    const double bce = __dadd_rn(__dsub_rn(fmax(zz, 0.0), __dmul_rn(zz, tt)), log1p(exp(-fabs(zz))));
    cls = __dadd_rn(cls, __dmul_rn(w, bce));
    dcls[i] = (float)__ddiv_rn(__dmul_rn(__dmul_rn(cls_w, w), __dsub_rn(sigmoid64(zz), tt)), n_pos);
  }
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < nrg; i += (int64_t)kRedBlocks * 256) {
    const double m = pos[i / nreg] ? 1.0 : 0.0;
    const double diff = __dmul_rn(__dsub_rn((double)r[i], rt[i]), m);
    reg = __dadd_rn(reg, __dmul_rn(diff, diff));
    dreg[i] = (float)__ddiv_rn(__dmul_rn(__dmul_rn(reg_w, 2.0), diff), __dmul_rn(4.0, n_pos));
  }
  cls = block_sum(cls, sh);
  reg = block_sum(reg, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = cls;
    part[kRedBlocks + blockIdx.x] = reg;
  }
}

// mse_loss (pm/qat.py:119-125): sum of squared f64 residuals, grad = f32(2 diff / n)
__global__ void __launch_bounds__(256) mse_kernel(const float* __restrict__ out, const double* __restrict__ tgt,
                                                  int64_t n, float* __restrict__ grad, double* __restrict__ part) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)kRedBlocks * 256) {
    const double d = __dsub_rn((double)out[i], tgt[i]);
    s = __dadd_rn(s, __dmul_rn(d, d));
    grad[i] = (float)__ddiv_rn(__dmul_rn(2.0, d), (double)n);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// sum of (inv * g)^2 with the f32 product and square of pm/qat.py:285-287
__global__ void __launch_bounds__(256) sumsq_kernel(const float* __restrict__ g, int64_t n, float inv,
                                                    double* __restrict__ part) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)kRedBlocks * 256) {
    const float v = __fmul_rn(inv, g[i]);
    s = __dadd_rn(s, (double)__fmul_rn(v, v));
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// w -= lr * step, step = inv * g (+ momentum: mu * v + step, v = step), f32 as pm/qat.py:290-301
__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g, int64_t n, float inv, float lr, float mu,
                           float* __restrict__ vel) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float step = __fmul_rn(inv, g[i]);
    if (vel) {
      step = __fadd_rn(__fmul_rn(mu, vel[i]), step);
      vel[i] = step;
    }
    w[i] = __fsub_rn(w[i], __fmul_rn(lr, step));
  }
}

int blocks_for(int64_t n) {
  const int64_t b = ceil_div(n > 0 ? n : 1, 256);
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)(b < cap ? b : cap);
}

pmx_status check_desc(const pmx_conv_desc* d) {
  PMX_REQUIRE(d != nullptr, "desc is NULL");
  PMX_REQUIRE(d->kind == PMX_CONV2D || d->kind == PMX_DECONV2D, "kind must be PMX_CONV2D or PMX_DECONV2D");
  PMX_REQUIRE(d->batch >= 0 && d->in_h >= 1 && d->in_w >= 1 && d->in_c >= 1 && d->out_c >= 1, "bad extents");
  PMX_REQUIRE(d->k_h >= 1 && d->k_w >= 1 && d->stride_h >= 1 && d->stride_w >= 1 && d->pad_h >= 0 && d->pad_w >= 0,
              "bad kernel geometry");
  if (d->kind == PMX_DECONV2D) {
    PMX_REQUIRE(d->k_h == d->stride_h && d->k_w == d->stride_w && d->pad_h == 0 && d->pad_w == 0,
                "deconv2d supports kernel == stride, no padding");
    PMX_REQUIRE(d->out_h == d->in_h * d->stride_h && d->out_w == d->in_w * d->stride_w, "deconv output extents");
  } else {
    PMX_REQUIRE(d->out_h == (d->in_h + 2 * d->pad_h - d->k_h) / d->stride_h + 1 &&
                    d->out_w == (d->in_w + 2 * d->pad_w - d->k_w) / d->stride_w + 1 && d->out_h >= 1 && d->out_w >= 1,
                "conv output extents");
  }
  return PMX_OK;
}

}  // namespace

}  // namespace pmx

using namespace pmx;

extern "C" {

pmx_status pmx_train_conv_fwd(const pmx_conv_desc* desc, const float* x, const float* w, const float* bias,
                              float* out, pmx_stream_t stream) {
  pmx_status s = check_desc(desc);
  if (s != PMX_OK) return s;
  const Geo g = geo_of(*desc);
  const int64_t n = (int64_t)g.n * g.oh * g.ow * g.co;
  if (n == 0) return PMX_OK;
  fwd_kernel<<<blocks_for(n), 256, 0, stream>>>(g, x, w, bias, out);
  return check_launch("pmx_train_conv_fwd");
}

pmx_status pmx_train_conv_dgrad(const pmx_conv_desc* desc, const float* dout, const float* w, float* dx,
                                pmx_stream_t stream) {
  pmx_status s = check_desc(desc);
  if (s != PMX_OK) return s;
  const Geo g = geo_of(*desc);
  const int64_t n = (int64_t)g.n * g.ih * g.iw * g.ci;
  if (n == 0) return PMX_OK;
  dgrad_kernel<<<blocks_for(n), 256, 0, stream>>>(g, dout, w, dx);
  return check_launch("pmx_train_conv_dgrad");
}

pmx_status pmx_train_conv_wgrad(const pmx_conv_desc* desc, const float* dout, const float* x, float* dw, float* db,
                                pmx_stream_t stream) {
  pmx_status s = check_desc(desc);
  if (s != PMX_OK) return s;
  const Geo g = geo_of(*desc);
  if (dw) {
    dim3 grid((unsigned)(g.co * g.kh * g.kw), (unsigned)ceil_div(g.ci, 32));
    wgrad_kernel<<<grid, 256, 0, stream>>>(g, dout, x, dw);
  }
  if (db) bgrad_kernel<<<g.co, 256, 0, stream>>>(dout, (int64_t)g.n * g.oh * g.ow, g.co, db);
  return check_launch("pmx_train_conv_wgrad");
}

pmx_status pmx_train_relu(const float* x, int64_t n, float* out, pmx_stream_t stream) {
  PMX_REQUIRE(n >= 0, "negative length");
  if (n) relu_kernel<<<blocks_for(n), 256, 0, stream>>>(x, n, out);
  return check_launch("pmx_train_relu");
}

pmx_status pmx_train_relu_bwd(const float* dout, const float* pre_act, int64_t n, float* dx, pmx_stream_t stream) {
  PMX_REQUIRE(n >= 0, "negative length");
  if (n) relu_bwd_kernel<<<blocks_for(n), 256, 0, stream>>>(dout, pre_act, n, dx);
  return check_launch("pmx_train_relu_bwd");
}

pmx_status pmx_train_ste(const float* x, int64_t n, double scale, int32_t q_min, int32_t q_max, const float* upstream,
                         float* out, pmx_stream_t stream) {
  PMX_REQUIRE(n >= 0, "negative length");
  PMX_REQUIRE(std::isfinite(scale) && scale > 0.0, "scale must be positive and finite");
  const float lo = (float)((double)q_min * scale), hi = (float)((double)q_max * scale);
  if (n) ste_kernel<<<blocks_for(n), 256, 0, stream>>>(x, n, lo, hi, upstream, out);
  return check_launch("pmx_train_ste");
}

pmx_status pmx_train_ste_rows(const float* x, int64_t rows, int64_t cols, const double* scales, int32_t q_min,
                              int32_t q_max, const float* upstream, float* out, pmx_stream_t stream) {
  PMX_REQUIRE(rows >= 0 && cols >= 0, "negative extent");
  if (rows * cols)
    ste_rows_kernel<<<blocks_for(rows * cols), 256, 0, stream>>>(x, rows, cols, scales, (double)q_min, (double)q_max,
                                                                 upstream, out);
  return check_launch("pmx_train_ste_rows");
}

pmx_status pmx_train_maxpool(const float* x, const uint8_t* mask, int64_t pillars, int32_t m, int32_t c, float* out,
                             int32_t* argmax, pmx_stream_t stream) {
  PMX_REQUIRE(pillars >= 0 && m >= 1 && c >= 1, "bad extents");
  if (pillars) maxpool_kernel<<<blocks_for(pillars * c), 256, 0, stream>>>(x, mask, pillars, m, c, out, argmax);
  return check_launch("pmx_train_maxpool");
}

pmx_status pmx_train_maxpool_bwd(const float* dout, const int32_t* argmax, int64_t pillars, int32_t m, int32_t c,
                                 float* dx, pmx_stream_t stream) {
  PMX_REQUIRE(pillars >= 0 && m >= 1 && c >= 1, "bad extents");
  if (pillars) maxpool_bwd_kernel<<<blocks_for(pillars * m * c), 256, 0, stream>>>(dout, argmax, pillars, m, c, dx);
  return check_launch("pmx_train_maxpool_bwd");
}

pmx_status pmx_train_scatter(const float* feats, const int32_t* coords, int64_t pillars, int32_t c, int32_t grid_w,
                             float* canvas, pmx_stream_t stream) {
  PMX_REQUIRE(pillars >= 0 && c >= 1 && grid_w >= 1, "bad extents");
  if (pillars) scatter_kernel<<<blocks_for(pillars * c), 256, 0, stream>>>(feats, coords, pillars, c, grid_w, canvas, 0);
  return check_launch("pmx_train_scatter");
}

pmx_status pmx_train_scatter_bwd(const float* dcanvas, const int32_t* coords, int64_t pillars, int32_t c,
                                 int32_t grid_w, float* dfeats, pmx_stream_t stream) {
  PMX_REQUIRE(pillars >= 0 && c >= 1 && grid_w >= 1, "bad extents");
  if (pillars)
    scatter_kernel<<<blocks_for(pillars * c), 256, 0, stream>>>(dcanvas, coords, pillars, c, grid_w, dfeats, 1);
  return check_launch("pmx_train_scatter_bwd");
}

pmx_status pmx_train_upsample2x_bwd(const float* dout, int32_t batch, int32_t h, int32_t w, int32_t c, float* dx,
                                    pmx_stream_t stream) {
  PMX_REQUIRE(batch >= 0 && h >= 1 && w >= 1 && c >= 1, "bad extents");
  const int64_t n = (int64_t)batch * h * w * c;
  if (n) upsample_bwd_kernel<<<blocks_for(n), 256, 0, stream>>>(dout, batch, h, w, c, dx);
  return check_launch("pmx_train_upsample2x_bwd");
}

pmx_status pmx_train_add(const float* a, const float* b, int64_t n, float* out, pmx_stream_t stream) {
  PMX_REQUIRE(n >= 0, "negative length");
  if (n) add_kernel<<<blocks_for(n), 256, 0, stream>>>(a, b, n, out);
  return check_launch("pmx_train_add");
}

pmx_status pmx_train_copy_channels(const float* src, int64_t pixels, int32_t c, int32_t src_stride, int32_t src_offset,
                                   float* dst, int32_t dst_stride, int32_t dst_offset, pmx_stream_t stream) {
  PMX_REQUIRE(pixels >= 0 && c >= 1 && src_offset >= 0 && dst_offset >= 0 && src_offset + c <= src_stride &&
                  dst_offset + c <= dst_stride,
              "bad channel slice");
  if (pixels)
    copy_ch_kernel<<<blocks_for(pixels * c), 256, 0, stream>>>(src, pixels, c, src_stride, src_offset, dst, dst_stride,
                                                                dst_offset);
  return check_launch("pmx_train_copy_channels");
}

size_t pmx_train_reduce_workspace(void) { return sizeof(double) * 2 * kRedBlocks; }

pmx_status pmx_train_detection_loss(const float* cls, const double* cls_target, const uint8_t* ignore_mask,
                                    const uint8_t* pos_mask, const float* reg, const double* reg_target, int64_t hw,
                                    int32_t n_cls, int32_t n_reg, double n_pos, double cls_weight, double reg_weight,
                                    double pos_weight, float* d_cls, float* d_reg, double* sums, double* ws,
                                    pmx_stream_t stream) {
  PMX_REQUIRE(hw >= 0 && n_cls >= 1 && n_reg >= 1 && n_pos >= 1.0, "bad extents");
  PMX_REQUIRE(sums != nullptr && ws != nullptr, "sums / workspace are NULL");
  det_loss_kernel<<<kRedBlocks, 256, 0, stream>>>(cls, cls_target, ignore_mask, pos_mask, reg, reg_target, hw, n_cls,
                                                  n_reg, n_pos, cls_weight, reg_weight, pos_weight, d_cls, d_reg, ws);
  finish_kernel<<<1, 256, 0, stream>>>(ws, 2, sums);
  return check_launch("pmx_train_detection_loss");
}

pmx_status pmx_train_mse_loss(const float* out, const double* target, int64_t n, float* grad, double* sum, double* ws,
                              pmx_stream_t stream) {
  PMX_REQUIRE(n >= 1, "empty tensor");
  PMX_REQUIRE(sum != nullptr && ws != nullptr, "sum / workspace are NULL");
  mse_kernel<<<kRedBlocks, 256, 0, stream>>>(out, target, n, grad, ws);
  finish_kernel<<<1, 256, 0, stream>>>(ws, 1, sum);
  return check_launch("pmx_train_mse_loss");
}

pmx_status pmx_train_sumsq(const float* g, int64_t n, float inv, double* sum, double* ws, pmx_stream_t stream) {
  PMX_REQUIRE(n >= 0, "negative length");
  PMX_REQUIRE(sum != nullptr && ws != nullptr, "sum / workspace are NULL");
  sumsq_kernel<<<kRedBlocks, 256, 0, stream>>>(g, n, inv, ws);
  finish_kernel<<<1, 256, 0, stream>>>(ws, 1, sum);
  return check_launch("pmx_train_sumsq");
}

pmx_status pmx_train_sgd(float* w, const float* grad, int64_t n, float inv, float lr, float momentum, float* velocity,
                         pmx_stream_t stream) {
  PMX_REQUIRE(n >= 0, "negative length");
  PMX_REQUIRE(momentum == 0.0f || velocity != nullptr, "momentum needs a velocity buffer");
  if (n) sgd_kernel<<<blocks_for(n), 256, 0, stream>>>(w, grad, n, inv, lr, momentum, momentum > 0.0f ? velocity : nullptr);
  return check_launch("pmx_train_sgd");
}

}  // extern "C"
