// K11b: local-peak box decode + per-class greedy NMS on the GPU -- the reference's
// own decode entry point, pm/detector.py:266-307 (decode_and_nms), with
// _sigmoid :251-252, _local_peaks :255-263 and iou_matrix pm/metrics.py:52-66.
//
// One CTA per (frame, class).  The class map's cells are scored in f64 exactly as
// the reference does (where(x >= 0, 1 / (1 + exp(-x)), exp(x) / (1 + exp(x)))),
// a cell is a candidate when its score is >= the NaN-propagating max of its 3 x 3
// neighbourhood (-inf outside the map; ties keep both) and not below the score
// threshold.  Candidates are ordered by score descending, then by row-major cell
// index (the stable sort of the reference over np.argwhere order) with a bitonic
// sort in shared memory, then suppressed greedily: in chunks of 32 candidates,
// every warp tests one candidate against all boxes kept so far, one warp resolves
// the chunk internally in order.  Every f64 operation is written with explicit
// IEEE round-to-nearest intrinsics (no FMA contraction), so boxes, IoUs and
// decisions follow the reference's arithmetic; only exp() is the CUDA libm one
// (<= 1 ulp; the reference's numpy exp is itself host-dependent).
#include "pmx_common.cuh"

namespace pmx {
namespace {

constexpr int kNmsThreads = 1024;
constexpr int kNmsMaxCells = 16384;

__device__ __forceinline__ double sigmoid_ref(double x) {
  // pm/detector.py:251-252
  if (x >= 0.0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-x)));
  const double e = exp(x);
  return __ddiv_rn(e, __dadd_rn(1.0, e));
}

// np.maximum / np.minimum: NaN in either operand -> NaN
__device__ __forceinline__ double np_max(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a > b ? a : b;
}
__device__ __forceinline__ double np_min(double a, double b) {
  if (a != a) return a;
  if (b != b) return b;
  return a < b ? a : b;
}

struct Box {
  double cx, cy, w, h;
};

// pm/metrics.py:52-66 for one pair (symmetric bit for bit: + and max/min commute)
__device__ __forceinline__ double iou_ref(const Box& a, const Box& b) {
  const double ax1 = __dsub_rn(a.cx, __ddiv_rn(a.w, 2.0)), ay1 = __dsub_rn(a.cy, __ddiv_rn(a.h, 2.0));
  const double ax2 = __dadd_rn(a.cx, __ddiv_rn(a.w, 2.0)), ay2 = __dadd_rn(a.cy, __ddiv_rn(a.h, 2.0));
  const double bx1 = __dsub_rn(b.cx, __ddiv_rn(b.w, 2.0)), by1 = __dsub_rn(b.cy, __ddiv_rn(b.h, 2.0));
  const double bx2 = __dadd_rn(b.cx, __ddiv_rn(b.w, 2.0)), by2 = __dadd_rn(b.cy, __ddiv_rn(b.h, 2.0));
  const double iw = np_max(0.0, __dsub_rn(np_min(ax2, bx2), np_max(ax1, bx1)));
  const double ih = np_max(0.0, __dsub_rn(np_min(ay2, by2), np_max(ay1, by1)));
  const double inter = __dmul_rn(iw, ih);
  const double uni = __dsub_rn(__dadd_rn(__dmul_rn(a.w, a.h), __dmul_rn(b.w, b.h)), inter);
  return uni > 0.0 ? __ddiv_rn(inter, uni) : 0.0;
}

// Python's min(4.0, max(-4.0, d)) (a NaN d gives -4.0)
__device__ __forceinline__ double clip4(double d) {
  const double t = d > -4.0 ? d : -4.0;
  return t < 4.0 ? t : 4.0;
}

struct NmsArgs {
  pmx_nms_desc d;
  const float* cls;  // [B, C, H, W]
  const float* reg;  // [B, 4, H, W]
  double* dets;      // [B, C, H*W, 5]
  int32_t* n_dets;   // [B, C]
  int np2;           // sort width (power of two >= H*W)
};

__device__ __forceinline__ Box box_of(const NmsArgs& a, const float* reg, int idx) {
  const int W = a.d.out_w, HW = a.d.out_h * a.d.out_w;
  const int i = idx / W, j = idx - (idx / W) * W;
  const double dx = reg[idx], dy = reg[HW + idx], dw = reg[2 * HW + idx], dh = reg[3 * HW + idx];
  Box b;
  b.cx = __dmul_rn(__dadd_rn(__dadd_rn((double)j, 0.5), dx), a.d.cell_w);
  b.cy = __dmul_rn(__dadd_rn(__dadd_rn((double)i, 0.5), dy), a.d.cell_h);
  b.w = __dmul_rn(a.d.base_size, exp(clip4(dw)));
  b.h = __dmul_rn(a.d.base_size, exp(clip4(dh)));
  return b;
}

// (score desc, cell asc): true when (sa, ia) must come before (sb, ib)
__device__ __forceinline__ bool before(double sa, int ia, double sb, int ib) {
  return sa > sb || (sa == sb && ia < ib);
}

__global__ void __launch_bounds__(kNmsThreads) nms_kernel(const NmsArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  double* ks = reinterpret_cast<double*>(smem);           // [np2] scores
  int* ki = reinterpret_cast<int*>(ks + a.np2);            // [np2] cells
  __shared__ int n_cand, n_kept;
  __shared__ Box cbox[32];
  __shared__ double cscore[32];
  __shared__ int csupp[32];
  const int b = blockIdx.x / a.d.n_classes, c = blockIdx.x - b * a.d.n_classes;
  const int H = a.d.out_h, W = a.d.out_w, HW = H * W;
  const float* logit = a.cls + ((int64_t)b * a.d.n_classes + c) * HW;
  const float* reg = a.reg + (int64_t)b * 4 * HW;
  double* out = a.dets + ((int64_t)b * a.d.n_classes + c) * (int64_t)HW * 5;
  pdl_begin();
  if (threadIdx.x == 0) n_cand = 0, n_kept = 0;
  __syncthreads();
  // candidates: local peaks (pm/detector.py:255-263) at or above the threshold (:289-290)
  for (int idx = threadIdx.x; idx < HW; idx += blockDim.x) {
    const int i = idx / W, j = idx - i * W;
    const double s = sigmoid_ref((double)logit[idx]);
    double nb = -INFINITY;
    for (int di = -1; di <= 1; ++di)
      for (int dj = -1; dj <= 1; ++dj) {
        const int y = i + di, x = j + dj;
        if (y < 0 || y >= H || x < 0 || x >= W) continue;  // -inf padding
        nb = np_max(nb, (di == 0 && dj == 0) ? s : sigmoid_ref((double)logit[y * W + x]));
      }
    if (s >= nb && !(s < a.d.score_thresh)) {
      const int p = atomicAdd(&n_cand, 1);
      ks[p] = s;
      ki[p] = idx;
    }
  }
  __syncthreads();
  const int n = n_cand;
  int m = 1;
  while (m < n) m <<= 1;
  for (int p = n + threadIdx.x; p < m; p += blockDim.x) ks[p] = -INFINITY, ki[p] = 0x7fffffff;
  __syncthreads();
  // bitonic sort of (score, cell) pairs into (score desc, cell asc) order
  for (int k = 2; k <= m; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < m; t += blockDim.x) {
        const int u = t ^ j;
        if (u > t) {
          const bool up = (t & k) == 0;
          const bool swap = up ? before(ks[u], ki[u], ks[t], ki[t]) : before(ks[t], ki[t], ks[u], ki[u]);
          if (swap) {
            const double s0 = ks[t];
            ks[t] = ks[u];
            ks[u] = s0;
            const int i0 = ki[t];
            ki[t] = ki[u];
            ki[u] = i0;
          }
        }
      }
      __syncthreads();
    }
  // greedy NMS (pm/detector.py:293-301): a candidate survives unless a box kept before
  // it overlaps it with IoU >= thr
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int K = n_kept;
    if (c0 + warp < n) {
      const Box bx = box_of(a, reg, ki[c0 + warp]);
      bool sup = false;
      for (int k = lane; k < K && !sup; k += 32) {
        const double* o = out + (int64_t)k * 5;
        const Box kb{o[0], o[1], o[2], o[3]};
        sup = iou_ref(bx, kb) >= a.d.iou_thresh;
      }
      sup = __any_sync(0xffffffffu, sup);
      if (lane == 0) {
        cbox[warp] = bx;
        cscore[warp] = ks[c0 + warp];
        csupp[warp] = sup;
      }
    }
    __syncthreads();
    if (warp == 0) {
      const bool valid = c0 + lane < n;
      uint32_t mask = 0;  // earlier chunk members this candidate overlaps
      if (valid)
        for (int jj = 0; jj < lane; ++jj)
          if (iou_ref(cbox[lane], cbox[jj]) >= a.d.iou_thresh) mask |= 1u << jj;
      const bool free0 = valid && !csupp[lane];
      uint32_t kept = 0;
      for (int ii = 0; ii < 32; ++ii) {
        const bool mine = free0 && (mask & kept) == 0;
        if (__shfl_sync(0xffffffffu, mine ? 1 : 0, ii)) kept |= 1u << ii;
      }
      if ((kept >> lane) & 1u) {
        const int pos = K + __popc(kept & ((1u << lane) - 1u));
        double* o = out + (int64_t)pos * 5;
        o[0] = cbox[lane].cx;
        o[1] = cbox[lane].cy;
        o[2] = cbox[lane].w;
        o[3] = cbox[lane].h;
        o[4] = cscore[lane];
      }
      if (lane == 0) n_kept = K + __popc(kept);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) a.n_dets[(int64_t)b * a.d.n_classes + c] = n_kept;
}

}  // namespace
}  // namespace pmx

using namespace pmx;

extern "C" {

pmx_status pmx_decode_nms(const pmx_nms_desc* desc, int32_t batch, const float* cls, const float* reg, double* dets,
                          int32_t* n_dets, pmx_stream_t stream) {
  PMX_REQUIRE(desc != nullptr, "desc is NULL");
  const pmx_nms_desc& d = *desc;
  if (!(d.score_thresh >= 0.0 && d.score_thresh <= 1.0 && d.iou_thresh >= 0.0 && d.iou_thresh <= 1.0))
    return fail(PMX_ERR_INVALID, "thresholds must lie in [0, 1], got " + std::to_string(d.score_thresh) + ", " +
                                     std::to_string(d.iou_thresh));
  PMX_REQUIRE(batch >= 0 && d.n_classes >= 1 && d.out_h >= 1 && d.out_w >= 1, "bad extents");
  if ((int64_t)d.out_h * d.out_w > kNmsMaxCells)
    return fail(PMX_ERR_UNSUPPORTED, "decode_nms: at most 16384 cells per class map");
  if (batch == 0) return PMX_OK;
  PMX_REQUIRE(cls && reg && dets && n_dets, "NULL operand");
  NmsArgs a{};
  a.d = d;
  a.cls = cls;
  a.reg = reg;
  a.dets = dets;
  a.n_dets = n_dets;
  int np2 = 1;
  while (np2 < d.out_h * d.out_w) np2 <<= 1;
  a.np2 = np2;
  const size_t smem = (size_t)np2 * (sizeof(double) + sizeof(int));
  PMX_CUDA(cudaFuncSetAttribute(nms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PMX_CUDA(launch_pdl(nms_kernel, dim3(batch * d.n_classes), dim3(kNmsThreads), smem, stream, a));
  return check_launch("pmx_decode_nms");
}

}  // extern "C"
