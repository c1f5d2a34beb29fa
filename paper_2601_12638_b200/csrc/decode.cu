// K11 anchor top-k + box decode (KITTI extension; conventions of
// pm/detector.py:266-307 -- deterministic ordering, lower index wins ties).
//
// Candidates are packed into 64-bit keys (order-preserving f32 logit << 32 |
// ~index) so that "larger key" == "higher logit, then lower index": the ranking
// is a pure integer sort, bit-reproducible.  A per-frame 2048-bin histogram of the
// top key bits finds the bin holding the k-th largest logit; only keys at or above
// it are compacted (a few hundred of 107,136 for the KITTI head), then CTAs
// bitonic-sort 2048-key chunks and keep their top k, repeated until one chunk
// remains (empty chunks skip the sort).  The final kernel decodes the k boxes with
// the SECOND delta coder in IEEE f32.
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

// ---- threshold pre-filter: a per-frame histogram of the top 11 key bits (a quarter
// octave of the logit) locates the bin holding the k-th largest logit; only keys at
// or above that bin (typically a few hundred of 107k) enter the sorting rounds.
constexpr int kBins = 2048;

__device__ __forceinline__ unsigned long long cand_key(const float* __restrict__ heads, int c_stride, int cls_off,
                                                       int n_anchors, int64_t ncand, int b, int64_t i) {
  const int64_t pix = i / n_anchors;
  const int a = (int)(i % n_anchors);
  const float logit = heads[((int64_t)b * (ncand / n_anchors) + pix) * c_stride + cls_off + a];
  return ((unsigned long long)f2key(logit) << 32) | (unsigned long long)(0xffffffffu - (uint32_t)i);
}

__global__ void __launch_bounds__(256) topk_hist(const float* __restrict__ heads, int c_stride, int cls_off,
                                                 int n_anchors, int64_t ncand, int* hist) {
  __shared__ int h[kBins];
  const int b = blockIdx.y;
  for (int t = threadIdx.x; t < kBins; t += blockDim.x) h[t] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  for (int t = threadIdx.x; t < kChunk; t += blockDim.x) {
    const int64_t i = base + t;
    if (i < ncand) atomicAdd(&h[(int)(cand_key(heads, c_stride, cls_off, n_anchors, ncand, b, i) >> 53)], 1);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kBins; t += blockDim.x)
    if (h[t]) atomicAdd(hist + (int64_t)b * kBins + t, h[t]);
}

__global__ void __launch_bounds__(kBins / 2) topk_thresh(const int* __restrict__ hist, int k, uint32_t* thresh) {
  __shared__ int sh[32];
  const int b = blockIdx.x;
  // thread t owns bins (from the top) 2t, 2t+1; inclusive scan of counts from the top
  const int* hb = hist + (int64_t)b * kBins;
  const int t = threadIdx.x;
  const int c0 = hb[kBins - 1 - 2 * t], c1 = hb[kBins - 2 - 2 * t];
  int v = c0 + c1;
  const int lane = t & 31, wid = t >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  if (lane == 31) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int s = sh[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += u;
    }
    sh[lane] = s;
  }
  __syncthreads();
  const int incl = v + (wid > 0 ? sh[wid - 1] : 0);
  const int excl = incl - c0 - c1;
  // the first bin (from the top) whose inclusive count reaches k
  if (excl < k && excl + c0 >= k) thresh[b] = (uint32_t)(kBins - 1 - 2 * t) << 21;
  else if (excl + c0 < k && incl >= k) thresh[b] = (uint32_t)(kBins - 2 - 2 * t) << 21;
  if (t == blockDim.x - 1 && incl < k) thresh[b] = 0u;  // fewer candidates than k: keep all
}

__global__ void __launch_bounds__(256) topk_compact(const float* __restrict__ heads, int c_stride, int cls_off,
                                                    int n_anchors, int64_t ncand, const uint32_t* __restrict__ thresh,
                                                    unsigned long long* buf, int* cnt) {
  const int b = blockIdx.y;
  const uint32_t T = thresh[b];
  const int lane = threadIdx.x & 31;
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  for (int t0 = 0; t0 < kChunk; t0 += blockDim.x) {
    const int64_t i = base + t0 + threadIdx.x;
    unsigned long long key = 0ull;
    bool keep = false;
    if (i < ncand) {
      key = cand_key(heads, c_stride, cls_off, n_anchors, ncand, b, i);
      keep = (uint32_t)(key >> 32) >= T;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (!m) continue;
    int slot = 0;
    if (lane == 0) slot = atomicAdd(cnt + b, __popc(m));
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (keep) buf[(int64_t)b * ncand + slot + __popc(m & ((1u << lane) - 1u))] = key;
  }
}

// sorting rounds: top-k of each 2048-key chunk of a key array [B, n]; entries past
// the per-frame device count (n_dev) are empty, and all-empty chunks skip the sort
__global__ void __launch_bounds__(kThreads) topk_merge(const unsigned long long* __restrict__ in, int64_t n,
                                                       const int* __restrict__ n_dev, int k, unsigned long long* out,
                                                       int nchunks) {
  __shared__ unsigned long long s[kChunk];
  const int b = blockIdx.y;
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  const int64_t nb = n_dev ? (int64_t)n_dev[b] : n;
  unsigned long long* dst = out + ((int64_t)b * nchunks + blockIdx.x) * k;
  int any = 0;
  for (int t = threadIdx.x; t < kChunk; t += blockDim.x) {
    const int64_t i = base + t;
    const unsigned long long v = (i < nb && i < n) ? in[(int64_t)b * n + i] : 0ull;
    s[t] = v;
    any |= v != 0ull;
  }
  if (!__syncthreads_or(any)) {
    for (int t = threadIdx.x; t < k; t += blockDim.x) dst[t] = 0ull;
    return;
  }
  bitonic_sort_desc(s);
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

struct DecodeWs {
  unsigned long long *buf0, *buf1, *cand;
  int* hist;
  int* cnt;
  uint32_t* thresh;
  size_t bytes;
};

DecodeWs carve_ws(void* base, int32_t batch, int64_t ncand, int k) {
  // two ping-pong key buffers sized for the first round's output, the compacted
  // candidate buffer, the per-frame histograms / counts / thresholds
  const int64_t n1 = ceil_div(ncand, kChunk) * k;
  char* p = static_cast<char*>(base);
  DecodeWs w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    void* r = p ? p + off : nullptr;
    off += (bytes + 255) & ~size_t(255);
    return r;
  };
  w.buf0 = (unsigned long long*)take(sizeof(unsigned long long) * batch * n1);
  w.buf1 = (unsigned long long*)take(sizeof(unsigned long long) * batch * n1);
  w.cand = (unsigned long long*)take(sizeof(unsigned long long) * batch * ncand);
  w.hist = (int*)take(sizeof(int) * batch * kBins);
  w.cnt = (int*)take(sizeof(int) * batch);
  w.thresh = (uint32_t*)take(sizeof(uint32_t) * batch);
  w.bytes = off;
  return w;
}

int64_t rounds_bytes(int32_t batch, int64_t ncand, int k) { return (int64_t)carve_ws(nullptr, batch, ncand, k).bytes; }

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
  DecodeWs w = carve_ws(ws, batch, ncand, d.k);
  PMX_CUDA(cudaMemsetAsync(w.hist, 0, sizeof(int) * batch * kBins, stream));
  PMX_CUDA(cudaMemsetAsync(w.cnt, 0, sizeof(int) * batch, stream));
  int nch = (int)ceil_div(ncand, kChunk);
  topk_hist<<<dim3(nch, batch), 256, 0, stream>>>(heads, head_c_stride, cls_off, d.n_anchors, ncand, w.hist);
  topk_thresh<<<batch, kBins / 2, 0, stream>>>(w.hist, d.k, w.thresh);
  topk_compact<<<dim3(nch, batch), 256, 0, stream>>>(heads, head_c_stride, cls_off, d.n_anchors, ncand, w.thresh,
                                                     w.cand, w.cnt);
  // round 1 over the compacted candidates (per-frame count on the device)
  topk_merge<<<dim3(nch, batch), kThreads, 0, stream>>>(w.cand, ncand, w.cnt, d.k, w.buf0, nch);
  int64_t n = (int64_t)nch * d.k;
  unsigned long long* cur = w.buf0;
  unsigned long long* nxt = w.buf1;
  while (nch > 1) {
    int nn = (int)ceil_div(n, kChunk);
    topk_merge<<<dim3(nn, batch), kThreads, 0, stream>>>(cur, n, nullptr, d.k, nxt, nn);
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
