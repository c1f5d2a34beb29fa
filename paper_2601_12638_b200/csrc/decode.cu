// K11 anchor top-k + box decode (KITTI extension; conventions of
// pm/detector.py:266-307 -- deterministic ordering, lower index wins ties).
//
// Candidates are packed into 64-bit keys (order-preserving f32 logit << 32 |
// ~index) so that "larger key" == "higher logit, then lower index": the ranking
// is a pure integer sort, bit-reproducible.  Reduction: CTAs bitonic-sort chunks
// of 2048 keys in shared memory and keep their top k; repeated until one chunk
// remains (107,136 anchors -> 53 x k -> 3 x k -> k for the KITTI head).  The
// final CTA decodes the k boxes with the SECOND delta coder in IEEE f32.
#include "pmx_common.cuh"

namespace pmx {
namespace {

constexpr int kChunk = 2048;
constexpr int kThreads = 1024;

__device__ __forceinline__ void bitonic_sort_desc(unsigned long long* s) {
  for (int size = 2; size <= kChunk; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < kChunk / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool desc = ((lo & size) == 0);
        unsigned long long a = s[lo], b = s[hi];
        if ((a < b) == desc) {
          s[lo] = b;
          s[hi] = a;
        }
      }
    }
  }
  __syncthreads();
}

// round 0: keys from the cls head map
__global__ void __launch_bounds__(kThreads) topk_first(const float* __restrict__ heads, int c_stride, int cls_off,
                                                       int n_anchors, int64_t ncand, int k,
                                                       unsigned long long* out, int nchunks) {
  __shared__ unsigned long long s[kChunk];
  const int b = blockIdx.y;
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  for (int t = threadIdx.x; t < kChunk; t += blockDim.x) {
    const int64_t i = base + t;
    unsigned long long key = 0ull;
    if (i < ncand) {
      const int64_t pix = i / n_anchors;
      const int a = (int)(i % n_anchors);
      const float logit = heads[((int64_t)b * (ncand / n_anchors) + pix) * c_stride + cls_off + a];
      key = ((unsigned long long)f2key(logit) << 32) | (unsigned long long)(0xffffffffu - (uint32_t)i);
    }
    s[t] = key;
  }
  bitonic_sort_desc(s);
  unsigned long long* dst = out + ((int64_t)b * nchunks + blockIdx.x) * k;
  for (int t = threadIdx.x; t < k; t += blockDim.x) dst[t] = s[t];
}

// later rounds: top-k of chunks of an existing key array [B, n]
__global__ void __launch_bounds__(kThreads) topk_merge(const unsigned long long* __restrict__ in, int64_t n, int k,
                                                       unsigned long long* out, int nchunks) {
  __shared__ unsigned long long s[kChunk];
  const int b = blockIdx.y;
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  for (int t = threadIdx.x; t < kChunk; t += blockDim.x) {
    const int64_t i = base + t;
    s[t] = i < n ? in[(int64_t)b * n + i] : 0ull;
  }
  bitonic_sort_desc(s);
  unsigned long long* dst = out + ((int64_t)b * nchunks + blockIdx.x) * k;
  for (int t = threadIdx.x; t < k; t += blockDim.x) dst[t] = s[t];
}

__global__ void decode_kernel(const pmx_anchor_desc d, const unsigned long long* __restrict__ keys, int64_t n_in,
                              int out_h, int out_w, const float* __restrict__ heads, int c_stride, int box_off,
                              int dir_off, int32_t* topk_idx, float* topk_logit, float* boxes, int32_t* dir_label) {
  const int b = blockIdx.y;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= d.k) return;
  const unsigned long long key = keys[(int64_t)b * n_in + r];
  const int64_t o = (int64_t)b * d.k + r;
  const int64_t ncand = (int64_t)out_h * out_w * d.n_anchors;
  const uint32_t idx = 0xffffffffu - (uint32_t)(key & 0xffffffffull);
  if (key == 0ull || (int64_t)idx >= ncand) {
    topk_idx[o] = -1;
    topk_logit[o] = __int_as_float(0x7fc00000);
    for (int j = 0; j < 7; ++j) boxes[o * 7 + j] = __int_as_float(0x7fc00000);
    dir_label[o] = -1;
    return;
  }
  const int A = d.n_anchors;
  const int a = (int)(idx % A);
  const int64_t pix = idx / A;
  const int xx = (int)(pix % out_w), yy = (int)(pix / out_w);
  const float* hp = heads + ((int64_t)b * out_h * out_w + pix) * c_stride;
  float t[7];
  for (int j = 0; j < 7; ++j) t[j] = hp[box_off + a * 7 + j];
  const float d0 = hp[dir_off + a * 2 + 0], d1 = hp[dir_off + a * 2 + 1];
  const float xa = __fadd_rn(d.x_min, __fmul_rn(__fadd_rn((float)xx, 0.5f), d.stride_x));
  const float ya = __fadd_rn(d.y_min, __fmul_rn(__fadd_rn((float)yy, 0.5f), d.stride_y));
  const float wa = d.anchor_w, la = d.anchor_l, ha = d.anchor_h;
  const float za = __fadd_rn(d.anchor_z, __fdiv_rn(ha, 2.0f));
  const float ra = d.rotations[a];
  const float diag = __fsqrt_rn(__fadd_rn(__fmul_rn(la, la), __fmul_rn(wa, wa)));
  const float xg = __fadd_rn(__fmul_rn(t[0], diag), xa);
  const float yg = __fadd_rn(__fmul_rn(t[1], diag), ya);
  float zg = __fadd_rn(__fmul_rn(t[2], ha), za);
  const float wg = __fmul_rn(expf(t[3]), wa);
  const float lg = __fmul_rn(expf(t[4]), la);
  const float hg = __fmul_rn(expf(t[5]), ha);
  float rg = __fadd_rn(t[6], ra);
  zg = __fsub_rn(zg, __fdiv_rn(hg, 2.0f));
  const int label = d1 > d0 ? 1 : 0;
  const float period = 3.14159265358979323846f;
  const float val = __fsub_rn(rg, d.dir_offset);
  const float rot = __fsub_rn(val, __fmul_rn(floorf(__fdiv_rn(val, period)), period));
  rg = __fadd_rn(__fadd_rn(rot, d.dir_offset), __fmul_rn(period, (float)label));
  topk_idx[o] = (int32_t)idx;
  topk_logit[o] = key2f((uint32_t)(key >> 32));
  float* bx = boxes + o * 7;
  bx[0] = xg; bx[1] = yg; bx[2] = zg; bx[3] = wg; bx[4] = lg; bx[5] = hg; bx[6] = rg;
  dir_label[o] = label;
}

int64_t rounds_bytes(int32_t batch, int64_t ncand, int k) {
  // two ping-pong key buffers sized for the first round's output
  int64_t n1 = ceil_div(ncand, kChunk) * k;
  return 2 * (int64_t)batch * n1 * 8 + 512;
}

}  // namespace
}  // namespace pmx

using namespace pmx;

extern "C" {

size_t pmx_decode_workspace(const pmx_anchor_desc* desc, int32_t batch, int32_t out_h, int32_t out_w) {
  if (!desc) return 0;
  return (size_t)rounds_bytes(batch, (int64_t)out_h * out_w * desc->n_anchors, desc->k);
}

pmx_status pmx_decode_topk(const pmx_anchor_desc* desc, int32_t batch, int32_t out_h, int32_t out_w,
                           const float* heads, int32_t head_c_stride, int32_t cls_off, int32_t box_off,
                           int32_t dir_off, int32_t* topk_idx, float* topk_logit, float* boxes, int32_t* dir_label,
                           void* ws, size_t ws_bytes, pmx_stream_t stream) {
  PMX_REQUIRE(desc != nullptr, "desc is NULL");
  const pmx_anchor_desc d = *desc;
  PMX_REQUIRE(d.n_anchors >= 1 && d.n_anchors <= 4, "n_anchors must be 1..4");
  PMX_REQUIRE(d.k >= 1 && d.k <= 512, "k must be 1..512");
  PMX_REQUIRE(out_h >= 1 && out_w >= 1, "bad head extents");
  PMX_REQUIRE(cls_off + d.n_anchors <= head_c_stride && box_off + 7 * d.n_anchors <= head_c_stride &&
                  dir_off + 2 * d.n_anchors <= head_c_stride,
              "head channel offsets exceed stride");
  if (batch == 0) return PMX_OK;
  const int64_t ncand = (int64_t)out_h * out_w * d.n_anchors;
  PMX_REQUIRE(ncand < 0x7fffffff, "too many anchors");
  const size_t need = (size_t)rounds_bytes(batch, ncand, d.k);
  PMX_REQUIRE(ws && ws_bytes >= need, "decode workspace too small");
  const int64_t n1 = ceil_div(ncand, kChunk) * d.k;
  unsigned long long* buf0 = static_cast<unsigned long long*>(ws);
  unsigned long long* buf1 = buf0 + (int64_t)batch * n1;
  int nch = (int)ceil_div(ncand, kChunk);
  topk_first<<<dim3(nch, batch), kThreads, 0, stream>>>(heads, head_c_stride, cls_off, d.n_anchors, ncand, d.k, buf0,
                                                        nch);
  int64_t n = (int64_t)nch * d.k;
  unsigned long long* cur = buf0;
  unsigned long long* nxt = buf1;
  while (nch > 1) {
    int nn = (int)ceil_div(n, kChunk);
    topk_merge<<<dim3(nn, batch), kThreads, 0, stream>>>(cur, n, d.k, nxt, nn);
    n = (int64_t)nn * d.k;
    nch = nn;
    unsigned long long* t = cur;
    cur = nxt;
    nxt = t;
  }
  decode_kernel<<<dim3((unsigned)ceil_div(d.k, 128), batch), 128, 0, stream>>>(
      d, cur, n, out_h, out_w, heads, head_c_stride, box_off, dir_off, topk_idx, topk_logit, boxes, dir_label);
  return check_launch("pmx_decode_topk");
}

}  // extern "C"
