// K11 anchor top-k + box decode (KITTI extension; conventions of
// pm/detector.py:266-307 -- deterministic ordering, lower index wins ties).
//
// Candidates are packed into 64-bit keys (order-preserving f32 logit << 32 |
// ~index) so that "larger key" == "higher logit, then lower index": the ranking
// is a pure integer sort, bit-reproducible.  Two kernels per call:
//   1. topk_hist: per-frame 2048-bin histogram of the top 11 key bits (a quarter
//      octave of the logit); the last CTA of each frame (arrival counter) scans it
//      and stores the bin holding the k-th largest key;
//   2. topk_select: keys at or above that bin (typically a few hundred of 107,136
//      for the KITTI head) are appended to a candidate list; the last CTA of each
//      frame bitonic-sorts the candidates in shared memory (or, when more than
//      kCap survive, finds the exact k-th key by an 8-pass MSD radix select over
//      the list first) and decodes the top k boxes with the SECOND delta coder in
//      IEEE f32.
#include "pmx_common.cuh"

namespace pmx {
namespace {

// anchors per CTA, chosen per call: large batches want few, full CTAs (16384: 7 per
// KITTI frame; batch 32: 0.058 ms vs 0.067 at 4096), batch 1 wants more CTAs per frame
// (2048, 53 CTAs, with the rank-sort finish: b1 p50 mixed 0.2464 -> 0.2458 ms, INT8
// 0.2331 -> 0.2312 vs 4096; 1024 no better, 8192 +6 us), batch 8 sits between (4096:
// 0.673 ms per step vs 0.684 at 16384, 0.675 at 8192)
int decode_chunk(int batch) {
  const char* e = getenv("PMX_DECODE_CHUNK");  // A/B override
  if (e && atoi(e) >= 1024) return atoi(e) & ~1023;
  return batch > 16 ? 16384 : (batch > 8 ? 8192 : (batch >= 2 ? 4096 : 2048));
}
constexpr int kThreads = 1024;

bool fused_enabled() {  // PMX_DECODE_FUSED=0: always the two-kernel path (A/B runs)
  static const bool on = [] {
    const char* e = getenv("PMX_DECODE_FUSED");
    return !(e && e[0] == '0');
  }();
  return on;
}
constexpr int kCap = 4096;    // candidates sorted in shared memory

template <int N>
__device__ __forceinline__ void bitonic_sort_desc(unsigned long long* s, int n) {
  // n: power of two <= N
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < n / 2; t += blockDim.x) {
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

constexpr int kBins = 2048;

__device__ __forceinline__ unsigned long long cand_key(const float* __restrict__ heads, int c_stride, int cls_off,
                                                       int n_anchors, int64_t ncand, int b, int64_t i) {
  const int64_t pix = i / n_anchors;
  const int a = (int)(i % n_anchors);
  const float logit = heads[((int64_t)b * (ncand / n_anchors) + pix) * c_stride + cls_off + a];
  return ((unsigned long long)f2key(logit) << 32) | (unsigned long long)(0xffffffffu - (uint32_t)i);
}

// last CTA of frame b to arrive on counter *ctr: the block barrier orders every thread's
// writes before thread 0's gpu-scope acq_rel add (release is cumulative), and the last
// arriver's acquire + the second barrier make the other CTAs' writes visible to all its
// threads -- one fenced atomic per CTA instead of a membar.gl per thread
__device__ __forceinline__ bool last_arrival(int* ctr, int n_ctas) {
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    int old;
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    last = old == n_ctas - 1;
  }
  __syncthreads();
  return last;
}

// the bin (key >> 53) holding the k-th largest key of the frame's histogram -> *thr as
// a 32-bit key prefix (0: fewer candidates than k, keep all); blockDim.x == kBins / 2
__device__ void hist_threshold(const int* hb, int k, uint32_t* thr) {
  __shared__ int sh[32];
  // thread t owns bins (from the top) 2t, 2t+1; inclusive scan of counts from the top
  const int t = threadIdx.x;
  const int c0 = __ldcg(hb + kBins - 1 - 2 * t), c1 = __ldcg(hb + kBins - 2 - 2 * t);
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
  if (excl < k && excl + c0 >= k) *thr = (uint32_t)(kBins - 1 - 2 * t) << 21;
  else if (excl + c0 < k && incl >= k) *thr = (uint32_t)(kBins - 2 - 2 * t) << 21;
  if (t == blockDim.x - 1 && incl < k) *thr = 0u;  // fewer candidates than k: keep all
}

__global__ void __launch_bounds__(kThreads) topk_hist(const float* __restrict__ heads, int c_stride, int cls_off,
                                                      int n_anchors, int64_t ncand, int k, int* hist, int* arrive,
                                                      uint32_t* thresh, int chunk, unsigned long long* keys) {
  pdl_begin();
  __shared__ int h[kBins];
  __shared__ int sh[32];
  const int b = blockIdx.y;
  for (int t = threadIdx.x; t < kBins; t += blockDim.x) h[t] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * chunk;
  unsigned long long* kb = keys + (int64_t)b * ncand;
  for (int t = threadIdx.x; t < chunk; t += blockDim.x) {
    const int64_t i = base + t;
    if (i < ncand) {
      // the key goes to a dense array: pass 2 reads 8 bytes per anchor, not the heads rows
      const unsigned long long key = cand_key(heads, c_stride, cls_off, n_anchors, ncand, b, i);
      kb[i] = key;
      atomicAdd(&h[(int)(key >> 53)], 1);
    }
  }
  __syncthreads();
  int* hb = hist + (int64_t)b * kBins;
  for (int t = threadIdx.x; t < kBins; t += blockDim.x)
    if (h[t]) atomicAdd(hb + t, h[t]);
  if (!last_arrival(arrive + b, gridDim.x)) return;
  hist_threshold(hb, k, thresh + b);
}

__device__ void decode_one(const pmx_anchor_desc& d, unsigned long long key, int b, int r, int out_h, int out_w,
                           const float* __restrict__ heads, int c_stride, int box_off, int dir_off, int32_t* topk_idx,
                           float* topk_logit, float* boxes, int32_t* dir_label) {
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

// last CTA of frame b: rank the frame's n candidate keys (cb) and decode the top k
__device__ void finish_frame(const pmx_anchor_desc& d, int b, int n, const unsigned long long* cb, unsigned long long* s,
                             const float* __restrict__ heads, int c_stride, int box_off, int dir_off, int out_h,
                             int out_w, int32_t* topk_idx, float* topk_logit, float* boxes, int32_t* dir_label) {
  __shared__ int sh_hist[256];
  __shared__ int sh_n, sh_sel[2];
  const int k = d.k;
  if (n <= (int)blockDim.x && k <= kCap / 2) {
    // few candidates (batch-1 frames: ~200): rank sort -- each key's rank is the number
    // of larger keys (keys are unique), one pass over the list in shared memory instead
    // of a bitonic network of log2(n)^2 / 2 barrier-separated stages
    unsigned long long* out = s + kCap / 2;
    const int t = threadIdx.x;
    const unsigned long long key = t < n ? __ldcg(cb + t) : 0ull;
    if (t < n) s[t] = key;
    for (int r = n + t; r < k; r += blockDim.x) out[r] = 0ull;  // fewer than k candidates: empty ranks
    __syncthreads();
    if (t < n) {
      int rank = 0;
      int j = 0;
      for (; j + 1 < n; j += 2) {
        const ulonglong2 kk2 = *reinterpret_cast<const ulonglong2*>(s + j);
        rank += (kk2.x > key) + (kk2.y > key);
      }
      if (j < n) rank += s[j] > key;
      if (rank < k) out[rank] = key;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < k; r += blockDim.x)
      decode_one(d, out[r], b, r, out_h, out_w, heads, c_stride, box_off, dir_off, topk_idx, topk_logit, boxes,
                 dir_label);
    return;
  }
  if (n <= kCap) {
    int np = 2;
    while (np < n || np < k) np <<= 1;
    for (int t = threadIdx.x; t < np; t += blockDim.x) s[t] = t < n ? __ldcg(cb + t) : 0ull;
    bitonic_sort_desc<kCap>(s, np);
  } else {
    // exact k-th largest key by MSD radix select (8 bits per pass); keys are unique
    unsigned long long prefix = 0ull, mask = 0ull;
    int kk = k;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int t = threadIdx.x; t < 256; t += blockDim.x) sh_hist[t] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const unsigned long long key = __ldcg(cb + i);
        if ((key & mask) == prefix) atomicAdd(&sh_hist[(int)(key >> shift) & 255], 1);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int above = 0, bin = 255;
        for (; bin > 0; --bin) {
          if (above + sh_hist[bin] >= kk) break;
          above += sh_hist[bin];
        }
        sh_sel[0] = above;
        sh_sel[1] = bin;
      }
      __syncthreads();
      kk -= sh_sel[0];
      prefix |= (unsigned long long)sh_sel[1] << shift;
      mask |= 255ull << shift;
      __syncthreads();
    }
    // prefix == the k-th largest key: gather the k keys >= it, then sort them
    if (threadIdx.x == 0) sh_n = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long key = __ldcg(cb + i);
      if (key >= prefix) s[atomicAdd(&sh_n, 1)] = key;
    }
    __syncthreads();
    int np = 2;
    while (np < k) np <<= 1;
    for (int t = k + threadIdx.x; t < np; t += blockDim.x) s[t] = 0ull;
    bitonic_sort_desc<kCap>(s, np);
  }
  for (int r = threadIdx.x; r < k; r += blockDim.x)
    decode_one(d, s[r], b, r, out_h, out_w, heads, c_stride, box_off, dir_off, topk_idx, topk_logit, boxes,
               dir_label);
}

__global__ void __launch_bounds__(kThreads) topk_select(
    const pmx_anchor_desc d, const float* __restrict__ heads, int c_stride, int cls_off, int box_off, int dir_off,
    int out_h, int out_w, const uint32_t* __restrict__ thresh, unsigned long long* cand, int* cnt, int* arrive,
    int32_t* topk_idx, float* topk_logit, float* boxes, int32_t* dir_label, int chunk,
    const unsigned long long* __restrict__ keys) {
  pdl_begin();
  __shared__ __align__(16) unsigned long long s[kCap];
  const int b = blockIdx.y;
  const int n_anchors = d.n_anchors;
  const int64_t ncand = (int64_t)out_h * out_w * n_anchors;
  const uint32_t T = thresh[b];
  const int lane = threadIdx.x & 31;
  unsigned long long* cb = cand + (int64_t)b * ncand;
  const int64_t base = (int64_t)blockIdx.x * chunk;
  for (int t0 = 0; t0 < chunk; t0 += blockDim.x) {
    const int64_t i = base + t0 + threadIdx.x;
    unsigned long long key = 0ull;
    bool keep = false;
    if (i < ncand) {
      key = __ldcs(keys + (int64_t)b * ncand + i);  // written by pass 1 (streaming: read once)
      keep = (uint32_t)(key >> 32) >= T;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (!m) continue;
    int slot = 0;
    if (lane == 0) slot = atomicAdd(cnt + b, __popc(m));
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (keep) cb[slot + __popc(m & ((1u << lane) - 1u))] = key;
  }
  if (!last_arrival(arrive + b, gridDim.x)) return;

  finish_frame(d, b, __ldcg(cnt + b), cb, s, heads, c_stride, box_off, dir_off, out_h, out_w, topk_idx, topk_logit,
               boxes, dir_label);
}

// Small grids (every CTA of the call resident at once, chunk <= kCap): both passes in
// one kernel.  A CTA keeps its chunk's keys in shared memory, adds its histogram, and
// meets the frame's other CTAs at a flag the last arriving one raises after computing
// the threshold; then it appends its candidates and the last CTA to arrive ranks and
// decodes -- one launch and no key round trip through HBM (batch 1: 27 CTAs).
__global__ void __launch_bounds__(kThreads) topk_fused(
    const pmx_anchor_desc d, const float* __restrict__ heads, int c_stride, int cls_off, int box_off, int dir_off,
    int out_h, int out_w, int* hist, int* arrive, int* flag, uint32_t* thresh, unsigned long long* cand, int* cnt,
    int32_t* topk_idx, float* topk_logit, float* boxes, int32_t* dir_label, int chunk) {
  pdl_begin();
#ifdef PMX_DECODE_TRACE
  unsigned long long tt[6];
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt[0]));
#define PMX_DT(i) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt[i]))
#else
#define PMX_DT(i)
#endif
  __shared__ __align__(16) unsigned long long s[kCap];
  __shared__ int h[kBins];
  const int b = blockIdx.y;
  const int n_anchors = d.n_anchors;
  const int64_t ncand = (int64_t)out_h * out_w * n_anchors;
  for (int t = threadIdx.x; t < kBins; t += blockDim.x) h[t] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * chunk;
  for (int t = threadIdx.x; t < chunk; t += blockDim.x) {
    const int64_t i = base + t;
    unsigned long long key = 0ull;
    if (i < ncand) {
      key = cand_key(heads, c_stride, cls_off, n_anchors, ncand, b, i);
      atomicAdd(&h[(int)(key >> 53)], 1);
    }
    s[t] = key;
  }
  __syncthreads();
  PMX_DT(1);
  int* hb = hist + (int64_t)b * kBins;
  for (int t = threadIdx.x; t < kBins; t += blockDim.x)
    if (h[t]) atomicAdd(hb + t, h[t]);
  if (last_arrival(arrive + b, gridDim.x)) {
    hist_threshold(hb, d.k, thresh + b);
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.gpu.b32 [%0], %1;" ::"l"(flag + b), "r"(1) : "memory");
  } else {
    if (threadIdx.x == 0) {
      int f = 0;
      do {
        asm volatile("ld.acquire.gpu.b32 %0, [%1];" : "=r"(f) : "l"(flag + b) : "memory");
        if (!f) __nanosleep(64);
      } while (!f);
    }
    __syncthreads();
  }
  PMX_DT(2);
  const uint32_t T = __ldcg(thresh + b);
  const int lane = threadIdx.x & 31;
  unsigned long long* cb = cand + (int64_t)b * ncand;
  for (int t0 = 0; t0 < chunk; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    const unsigned long long key = t < chunk ? s[t] : 0ull;
    const bool keep = key != 0ull && (uint32_t)(key >> 32) >= T;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (!m) continue;
    int slot = 0;
    if (lane == 0) slot = atomicAdd(cnt + b, __popc(m));
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (keep) cb[slot + __popc(m & ((1u << lane) - 1u))] = key;
  }
  PMX_DT(3);
  if (!last_arrival(arrive + gridDim.y + b, gridDim.x)) return;
  PMX_DT(4);
  finish_frame(d, b, __ldcg(cnt + b), cb, s, heads, c_stride, box_off, dir_off, out_h, out_w, topk_idx, topk_logit,
               boxes, dir_label);
#ifdef PMX_DECODE_TRACE
  __syncthreads();
  PMX_DT(5);
  if (threadIdx.x == 0)
    printf("decode trace b %d cta %d n %d: keys+hist %llu, thresh/flag %llu, append %llu, arrive %llu, finish %llu ns\n", b,
           blockIdx.x, __ldcg(cnt + b), tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3], tt[5] - tt[4]);
#endif
}

// per-call zeroing of the counters as a kernel (keeps the programmatic launch chain,
// which a memset node would break)
__global__ void zero_ws_kernel(int* p, int n) {
  pdl_begin();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = 0;
}

__global__ void pack_records_kernel(int n, const int32_t* __restrict__ idx, const float* __restrict__ logit,
                                    const float* __restrict__ boxes, const int32_t* __restrict__ dir, float* rec) {
  pdl_begin();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float* r = rec + (int64_t)i * 10;
  r[0] = (float)idx[i];
  r[1] = logit[i];
#pragma unroll
  for (int j = 0; j < 7; ++j) r[2 + j] = boxes[(int64_t)i * 7 + j];
  r[9] = (float)dir[i];
}

struct DecodeWs {
  unsigned long long* cand;
  unsigned long long* keys;  // [B, ncand] every anchor's key (pass 1 -> pass 2)
  int* hist;     // [B, kBins]
  int* cnt;      // [B]
  int* arrive;   // [2, B]
  int* flag;     // [B] fused path: threshold ready
  uint32_t* thresh;
  size_t zero_bytes;  // hist .. arrive are contiguous and zeroed per call
  size_t bytes;
};

DecodeWs carve_ws(void* base, int32_t batch, int64_t ncand) {
  char* p = static_cast<char*>(base);
  DecodeWs w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    void* r = p ? p + off : nullptr;
    off += (bytes + 255) & ~size_t(255);
    return r;
  };
  w.cand = (unsigned long long*)take(sizeof(unsigned long long) * batch * ncand);
  w.keys = (unsigned long long*)take(sizeof(unsigned long long) * batch * ncand);
  const size_t z0 = off;
  w.hist = (int*)take(sizeof(int) * batch * kBins);
  w.cnt = (int*)take(sizeof(int) * batch);
  w.arrive = (int*)take(sizeof(int) * 2 * batch);
  w.flag = (int*)take(sizeof(int) * batch);
  w.zero_bytes = off - z0;
  w.thresh = (uint32_t*)take(sizeof(uint32_t) * batch);
  w.bytes = off;
  return w;
}

}  // namespace
}  // namespace pmx

using namespace pmx;

extern "C" {

size_t pmx_decode_workspace(const pmx_anchor_desc* desc, int32_t batch, int32_t out_h, int32_t out_w) {
  if (!desc) return 0;
  return carve_ws(nullptr, batch, (int64_t)out_h * out_w * desc->n_anchors).bytes;
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
  DecodeWs w = carve_ws(ws, batch, ncand);
  PMX_REQUIRE(ws && ws_bytes >= w.bytes, "decode workspace too small");
  const int chunk = decode_chunk(batch);
  const int nch = (int)ceil_div(ncand, chunk);
  const int nz = (int)(w.zero_bytes / sizeof(int));
  PMX_CUDA(launch_pdl(zero_ws_kernel, dim3((unsigned)(nz < 65536 ? ceil_div(nz, 1024) : 64)), dim3(1024), 0, stream,
                      w.hist, nz));
  if (chunk <= kCap && (int64_t)nch * batch <= num_sms() && fused_enabled()) {
    PMX_CUDA(launch_pdl(topk_fused, dim3(nch, batch), dim3(kThreads), 0, stream, d, heads, head_c_stride, cls_off,
                        box_off, dir_off, out_h, out_w, w.hist, w.arrive, w.flag, w.thresh, w.cand, w.cnt, topk_idx,
                        topk_logit, boxes, dir_label, chunk));
    return check_launch("pmx_decode_topk");
  }
  PMX_CUDA(launch_pdl(topk_hist, dim3(nch, batch), dim3(kThreads), 0, stream, heads, head_c_stride, cls_off,
                      d.n_anchors, ncand, d.k, w.hist, w.arrive, w.thresh, chunk, w.keys));
  PMX_CUDA(launch_pdl(topk_select, dim3(nch, batch), dim3(kThreads), 0, stream, d, heads, head_c_stride, cls_off,
                      box_off, dir_off, out_h, out_w, (const uint32_t*)w.thresh, w.cand, w.cnt, w.arrive + batch,
                      topk_idx, topk_logit, boxes, dir_label, chunk, (const unsigned long long*)w.keys));
  return check_launch("pmx_decode_topk");
}

pmx_status pmx_pack_topk_records(int32_t batch, int32_t k, const int32_t* topk_idx, const float* topk_logit,
                                 const float* boxes, const int32_t* dir_label, float* records, pmx_stream_t stream) {
  PMX_REQUIRE(batch >= 0 && k >= 0, "negative extent");
  PMX_REQUIRE((topk_idx && topk_logit && boxes && dir_label && records) || batch * k == 0, "NULL operand");
  const int n = batch * k;
  if (n == 0) return PMX_OK;
  PMX_CUDA(launch_pdl(pack_records_kernel, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, stream, n, topk_idx,
                      topk_logit, boxes, dir_label, records));
  return check_launch("pmx_pack_topk_records");
}

}  // extern "C"
