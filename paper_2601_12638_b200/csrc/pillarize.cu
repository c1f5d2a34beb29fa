// K3 pillarize (pm/scenes.py:155-193 + KITTI cap) and feature materialisation.
//
// Deterministic with atomics; six kernels per call (five at batch <= 8):
//  0 init     the per-call workspace counters and cell arrays
//  1 bin      per point: cell (IEEE f32 divide, trunc, clamp), atomicMin(first[cell], i),
//             atomicAdd(cnt[cell], 1)                           -- coalesced float4 loads
//  2 hist     per cell block: occupied cells counted into the 1024-point block of their
//             first point
//  3 thresh   per frame: T = index of the P_max-th first-seen point (cap rule) or
//             INT_MAX -- at small batches done by the hist kernel's last CTA per frame
//  4 emit     per cell block (single pass, decoupled look-back): kept = cnt>0 &&
//             first<=T; pillar id in ascending flat order, coords, segment offsets,
//             n_pillars
//  5 slot     per point: atomic slot in its pillar's CSR segment (arbitrary order)
//  6 select   thread per pillar: the first M points of the segment by scene index
//             (rank counts; the pillar's warp runs a threshold search when a cell holds
//             more than 32 points)
#include <climits>

#include <cooperative_groups.h>

#include "pmx_common.cuh"

namespace pmx {

namespace {

constexpr int kPtBlock = 1024;   // points per flag block
constexpr int kCellPerThr = 4;
constexpr int kCellBlock = 1024 * kCellPerThr;

struct PillarWs {
  int32_t* first;   // [B*HW]
  int32_t* cnt;     // [B*HW]
  int32_t* pid;     // [B*HW] kept pillar slot + 1, 0 = empty
  int32_t* cell;    // [B*Nmax]
  int32_t* ptblk;   // [B*NB]
  int32_t* thresh;  // [B]
  int2* cblk;       // [B*CB]
  int32_t* segoff;  // [B*Pcap]
  int32_t* fill;    // [B*Pcap]
  int32_t* csr;     // [B*Nmax]
  unsigned long long* look;  // [B*CB] single-pass emit: per-block (flag, kept, points) look-back words
  int32_t* ticket;           // [B] single-pass emit: block order per frame
  int32_t* hdone;            // [B] firsthist (small batches): CTAs done per frame
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

size_t carve(const pmx_grid* g, int32_t B, int64_t nmax, int32_t pcap, void* base, PillarWs* ws) {
  int64_t hw = (int64_t)g->grid_h * g->grid_w;
  int64_t nb = ceil_div(nmax > 0 ? nmax : 1, kPtBlock);
  int64_t cb = ceil_div(hw, kCellBlock);
  size_t off = 0;
  char* p = static_cast<char*>(base);
  auto take = [&](size_t bytes) {
    void* r = p ? p + off : nullptr;
    off += align256(bytes);
    return r;
  };
  PillarWs w;
  w.first = (int32_t*)take(sizeof(int32_t) * B * hw);
  w.cnt = (int32_t*)take(sizeof(int32_t) * B * hw);
  w.pid = (int32_t*)take(sizeof(int32_t) * B * hw);
  w.cell = (int32_t*)take(sizeof(int32_t) * B * (nmax > 0 ? nmax : 1));
  w.ptblk = (int32_t*)take(sizeof(int32_t) * B * nb);
  w.thresh = (int32_t*)take(sizeof(int32_t) * B);
  w.cblk = (int2*)take(sizeof(int2) * B * cb);
  w.segoff = (int32_t*)take(sizeof(int32_t) * B * pcap);
  w.fill = (int32_t*)take(sizeof(int32_t) * B * pcap);
  w.csr = (int32_t*)take(sizeof(int32_t) * B * (nmax > 0 ? nmax : 1));
  w.look = (unsigned long long*)take(sizeof(unsigned long long) * B * cb);
  w.ticket = (int32_t*)take(sizeof(int32_t) * B);
  w.hdone = (int32_t*)take(sizeof(int32_t) * B);
  if (ws) *ws = w;
  return off;
}

// first = INT_MAX-ish (0x7f7f7f7f, as the memset it replaces), cnt = fill = 0,
// look-back words, tickets and the overflow counter = 0
__device__ __forceinline__ void init_ws(const PillarWs& w, int64_t n_cells, int64_t n_fill, int64_t n_look, int batch,
                                        int64_t n_ptblk, int64_t tid, int64_t nt) {
  const int4 f4 = make_int4(0x7f7f7f7f, 0x7f7f7f7f, 0x7f7f7f7f, 0x7f7f7f7f), z4 = make_int4(0, 0, 0, 0);
  if ((n_cells & 3) == 0) {
    for (int64_t i = tid; i < n_cells / 4; i += nt) {
      reinterpret_cast<int4*>(w.first)[i] = f4;
      reinterpret_cast<int4*>(w.cnt)[i] = z4;
    }
  } else {
    for (int64_t i = tid; i < n_cells; i += nt) {
      w.first[i] = 0x7f7f7f7f;
      w.cnt[i] = 0;
    }
  }
  for (int64_t i = tid; i < n_fill; i += nt) w.fill[i] = 0;
  for (int64_t i = tid; i < n_look; i += nt) w.look[i] = 0ull;
  for (int64_t i = tid; i < batch; i += nt) w.ticket[i] = 0, w.hdone[i] = 0;
  for (int64_t i = tid; i < n_ptblk; i += nt) w.ptblk[i] = 0;
}

__global__ void init_ws_kernel(PillarWs w, int64_t n_cells, int64_t n_fill, int64_t n_look, int batch,
                               int64_t n_ptblk) {
  pdl_begin();
  init_ws(w, n_cells, n_fill, n_look, batch, n_ptblk, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
          (int64_t)gridDim.x * blockDim.x);
}

__device__ __forceinline__ int bin_cell(float x, float y, const pmx_grid g) {
  // pm/scenes.py:177-178: (f32(p) - origin) / cell in IEEE f32, astype(int64) truncates, clip
  float fy = __fdiv_rn(__fsub_rn(y, g.y_min), g.cell_h);
  float fx = __fdiv_rn(__fsub_rn(x, g.x_min), g.cell_w);
  // truncation toward zero of values far outside the grid: clamp in float first
  fy = fminf(fmaxf(fy, -1.0f), (float)g.grid_h);
  fx = fminf(fmaxf(fx, -1.0f), (float)g.grid_w);
  int r = (int)fy, c = (int)fx;  // (int) truncates toward zero
  if (fy != fy) r = 0;          // NaN: reference behaviour undefined; pin to 0
  if (fx != fx) c = 0;
  r = r < 0 ? 0 : (r > g.grid_h - 1 ? g.grid_h - 1 : r);
  c = c < 0 ? 0 : (c > g.grid_w - 1 ? g.grid_w - 1 : c);
  return r * g.grid_w + c;
}

__device__ __forceinline__ void bin_frame(const float4* __restrict__ pts, const int64_t* __restrict__ offs,
                                          int64_t nmax, const pmx_grid& g, const PillarWs& w, int b, int64_t i0,
                                          int64_t stride) {
  const int64_t base = offs[b];
  const int64_t n = offs[b + 1] - base;
  const int64_t hw = (int64_t)g.grid_h * g.grid_w;
  for (int64_t i = i0; i < n; i += stride) {
    float4 p = __ldg(pts + base + i);
    int cell = bin_cell(p.x, p.y, g);
    w.cell[b * nmax + i] = cell;
    atomicMin(w.first + b * hw + cell, (int)i);
    atomicAdd(w.cnt + b * hw + cell, 1);
  }
}

__global__ void bin_kernel(const float4* __restrict__ pts, const int64_t* __restrict__ offs, int64_t nmax,
                           const pmx_grid g, PillarWs w) {
  pdl_begin();
  bin_frame(pts, offs, nmax, g, w, blockIdx.y, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
            (int64_t)gridDim.x * blockDim.x);
}

__global__ void __launch_bounds__(kPtBlock) flag_kernel(const int64_t* __restrict__ offs, int64_t nmax,
                                                        const pmx_grid g, PillarWs w, int nb) {
  pdl_begin();
  const int b = blockIdx.y;
  const int64_t n = offs[b + 1] - offs[b];
  const int64_t hw = (int64_t)g.grid_h * g.grid_w;
  int64_t i = (int64_t)blockIdx.x * kPtBlock + threadIdx.x;
  int flag = 0;
  if (i < n) flag = w.first[b * hw + w.cell[b * nmax + i]] == (int)i;
  int c = __syncthreads_count(flag);
  if (threadIdx.x == 0) w.ptblk[b * nb + blockIdx.x] = c;
}

// Same counts per cell instead of per point: every occupied cell adds 1 to the
// 1024-point block holding its first point (shared-memory histogram per CTA, then one
// atomic per non-empty bin) -- a coalesced pass over first[] instead of a random
// first[cell[i]] read per point.  ptblk is zeroed by init_ws_kernel.
__device__ void cap_threshold(const int64_t* __restrict__ offs, int64_t nmax, const pmx_grid& g, PillarWs& w, int nb,
                              int b);

// one cell block bx of frame b (blockDim.x == 1024); ncb = cell blocks per frame (the
// last of them to finish computes the cap threshold when fold is set); h: nb ints of
// shared memory
__device__ void firsthist_block(const int64_t* __restrict__ offs, int64_t nmax, const pmx_grid& g, PillarWs& w,
                                int nb, int fold, int bx, int b, int ncb, int* h) {
  const int64_t hw = (int64_t)g.grid_h * g.grid_w;
  for (int t = threadIdx.x; t < nb; t += blockDim.x) h[t] = 0;
  __syncthreads();
  const int64_t c0 = (int64_t)bx * kCellBlock + threadIdx.x * kCellPerThr;
  int f[kCellPerThr];
  if ((hw & 3) == 0 && c0 + kCellPerThr <= hw) {
    const int4 f4 = __ldcg(reinterpret_cast<const int4*>(w.first + b * hw + c0));
    f[0] = f4.x; f[1] = f4.y; f[2] = f4.z; f[3] = f4.w;
  } else {
#pragma unroll
    for (int j = 0; j < kCellPerThr; ++j) f[j] = c0 + j < hw ? w.first[b * hw + c0 + j] : 0x7f7f7f7f;
  }
#pragma unroll
  for (int j = 0; j < kCellPerThr; ++j)
    if (f[j] != 0x7f7f7f7f) atomicAdd(&h[f[j] / kPtBlock], 1);
  __syncthreads();
  for (int t = threadIdx.x; t < nb; t += blockDim.x)
    if (h[t]) atomicAdd(w.ptblk + (int64_t)b * nb + t, h[t]);
  if (!fold) return;
  // small batches: the frame's last CTA to arrive computes the cap threshold (one launch
  // less on the latency path; the block barrier + one acq_rel add per CTA order the counts)
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    int old;
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(w.hdone + b) : "memory");
    s_last = old == ncb - 1;
  }
  __syncthreads();
  if (!s_last) return;
  cap_threshold(offs, nmax, g, w, nb, b);
}

__global__ void __launch_bounds__(1024) firsthist_kernel(const int64_t* __restrict__ offs, int64_t nmax,
                                                        const pmx_grid g, PillarWs w, int nb, int fold) {
  pdl_begin();
  extern __shared__ int h[];  // [nb]
  firsthist_block(offs, nmax, g, w, nb, fold, blockIdx.x, blockIdx.y, gridDim.x, h);
}

// inclusive block scan of one int per thread (blockDim.x == 1024)
__device__ int block_incl_scan(int v, int* sh /*32*/) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int s = sh[lane];
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += t;
    }
    sh[lane] = s;
  }
  __syncthreads();
  if (wid > 0) v += sh[wid - 1];
  __syncthreads();
  return v;
}

// the same for a (kept, points) pair packed as kept << 40 | points in 64 bits: one scan
// (and three barriers) instead of two; returns the inclusive pair, *total = block sum
__device__ unsigned long long block_incl_scan2(unsigned long long v, unsigned long long* sh /*32*/,
                                               unsigned long long* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    unsigned long long x = sh[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    sh[lane] = x;
  }
  __syncthreads();
  if (wid > 0) v += sh[wid - 1];
  *total = sh[31];
  __syncthreads();
  return v;
}

// cap rule: T = index of the P_max-th first-seen point of frame b, or INT_MAX when the
// cap does not bind (block counts of first-seen points, then one block's flags)
__device__ void cap_threshold(const int64_t* __restrict__ offs, int64_t nmax, const pmx_grid& g, PillarWs& w, int nb,
                              int b) {
  __shared__ int sh[32];
  __shared__ int s_blk, s_need;
  const int64_t n = offs[b + 1] - offs[b];
  const int64_t hw = (int64_t)g.grid_h * g.grid_w;
  if (g.max_pillars <= 0) {
    if (threadIdx.x == 0) w.thresh[b] = INT_MAX;
    return;
  }
  // the first point block whose running count of first-seen points exceeds max_pillars
  // (the cap binds only if more than max_pillars cells are occupied): thread t sums a
  // contiguous run of blocks, one block scan, and the thread whose run crosses the cap
  // walks it (a serial walk from block 0 cost ~0.3 us of L2 latency per block)
  if (threadIdx.x == 0) s_blk = -1, s_need = 0;
  const int per = (nb + (int)blockDim.x - 1) / (int)blockDim.x;
  const int k0 = threadIdx.x * per;
  int run = 0;
  for (int k = k0; k < k0 + per && k < nb; ++k) run += __ldcg(w.ptblk + b * nb + k);
  const int incl = block_incl_scan(run, sh);  // (synchronises the s_blk reset too)
  const int excl = incl - run;
  if (excl < g.max_pillars + 1 && incl >= g.max_pillars + 1) {  // exactly one thread
    int cum = excl;
    for (int k = k0; k < k0 + per && k < nb; ++k) {
      const int c = __ldcg(w.ptblk + b * nb + k);
      if (cum + c >= g.max_pillars + 1) {
        s_blk = k;
        s_need = g.max_pillars - cum;  // the need-th first-seen point in this block is the last kept
        break;
      }
      cum += c;
    }
  }
  __syncthreads();
  if (s_blk < 0) {
    if (threadIdx.x == 0) w.thresh[b] = INT_MAX;
    return;
  }
  if (s_need == 0) {  // the cap is reached exactly before this block
    // the last kept first-point lies in an earlier block: T = (first index of blk) - 1
    if (threadIdx.x == 0) w.thresh[b] = s_blk * kPtBlock - 1;
    return;
  }
  int64_t i = (int64_t)s_blk * kPtBlock + threadIdx.x;
  int flag = 0;
  if (i < n) flag = __ldcg(w.first + b * hw + w.cell[b * nmax + i]) == (int)i;
  int inc = block_incl_scan(flag, sh);
  if (flag && inc == s_need) w.thresh[b] = (int)i;
}

__global__ void __launch_bounds__(1024) thresh_kernel(const int64_t* __restrict__ offs, int64_t nmax,
                                                      const pmx_grid g, PillarWs w, int nb) {
  pdl_begin();
  cap_threshold(offs, nmax, g, w, nb, blockIdx.x);
}

// Single pass of cellcount + cellscan + emit: every block reads its 4096 cells
// once (int4 loads), takes its place in the frame's block order from a ticket, and
// gets its exclusive (pillar, point) offsets by decoupled look-back over the blocks
// before it (64-bit words: flag << 62 | kept prefix << 40 | point prefix).
constexpr unsigned long long kLookAgg = 1ull << 62, kLookInc = 2ull << 62;
constexpr unsigned long long kLookPtsMask = (1ull << 40) - 1, kLookKeptMask = (1ull << 22) - 1;

// one cell block of frame b, in ticket order (blockDim.x == 1024)
__device__ void emit_block(const pmx_grid& g, const PillarWs& w, int cb, int32_t pcap, int32_t* coords,
                           int32_t* counts, int32_t* n_pillars, int b) {
  __shared__ unsigned long long sh2[32];
  __shared__ int s_blk;
  __shared__ unsigned long long s_prefix;
  const int64_t hw = (int64_t)g.grid_h * g.grid_w;
  if (threadIdx.x == 0) s_blk = atomicAdd(w.ticket + b, 1);
  __syncthreads();
  const int blk = s_blk;
  const int T = __ldcg(w.thresh + b);
  const int64_t c0 = (int64_t)blk * kCellBlock + threadIdx.x * kCellPerThr;
  int keep[kCellPerThr], n[kCellPerThr], f[kCellPerThr];
  if ((hw & 3) == 0 && c0 + kCellPerThr <= hw) {
    const int4 n4 = __ldcg(reinterpret_cast<const int4*>(w.cnt + b * hw + c0));
    const int4 f4 = __ldcg(reinterpret_cast<const int4*>(w.first + b * hw + c0));
    n[0] = n4.x; n[1] = n4.y; n[2] = n4.z; n[3] = n4.w;
    f[0] = f4.x; f[1] = f4.y; f[2] = f4.z; f[3] = f4.w;
  } else {
#pragma unroll
    for (int j = 0; j < kCellPerThr; ++j) {
      n[j] = c0 + j < hw ? w.cnt[b * hw + c0 + j] : 0;
      f[j] = c0 + j < hw ? w.first[b * hw + c0 + j] : INT_MAX;
    }
  }
  int kept = 0, pts = 0;
#pragma unroll
  for (int j = 0; j < kCellPerThr; ++j) {
    keep[j] = n[j] > 0 && f[j] <= T;
    kept += keep[j];
    pts += keep[j] ? n[j] : 0;
  }
  unsigned long long tot2;
  const unsigned long long mine = ((unsigned long long)kept << 40) | (unsigned long long)pts;
  const unsigned long long incl = block_incl_scan2(mine, sh2, &tot2);
  const int kept_tot = (int)(tot2 >> 40), pts_tot = (int)(tot2 & kLookPtsMask);
  int a = (int)((incl - mine) >> 40);
  int p = (int)((incl - mine) & kLookPtsMask);
  if (threadIdx.x < 32) {
    // warp-wide decoupled look-back: 32 predecessors per round (nearest first in lane
    // order); stop at the nearest one that already holds its inclusive prefix
    const int lane = threadIdx.x;
    unsigned long long* look = w.look + (int64_t)b * cb;
    const unsigned long long agg = ((unsigned long long)kept_tot << 40) | (unsigned long long)pts_tot;
    if (lane == 0) atomicExch(look + blk, (blk == 0 ? kLookInc : kLookAgg) | agg);
    unsigned long long excl = 0;
    for (int j = blk - 1; j >= 0; j -= 32) {
      const int jj = j - lane;
      unsigned long long v = jj >= 0 ? atomicAdd(look + jj, 0ull) : kLookInc;  // before block 0: inclusive 0
      while (__any_sync(0xffffffffu, (v >> 62) == 0)) {
        if ((v >> 62) == 0) v = atomicAdd(look + jj, 0ull);
      }
      const unsigned incl = __ballot_sync(0xffffffffu, (v >> 62) == 2);
      const int stop = incl ? __ffs(incl) - 1 : 31;
      unsigned long long x = lane <= stop ? (v & ~(3ull << 62)) : 0ull;
      for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
      excl += __shfl_sync(0xffffffffu, x, 0);
      if (incl) break;
    }
    if (lane == 0) {
      if (blk > 0) atomicExch(look + blk, kLookInc | (excl + agg));
      s_prefix = excl;
      if (blk == cb - 1) n_pillars[b] = (int)(((excl + agg) >> 40) & kLookKeptMask);
    }
  }
  __syncthreads();
  a += (int)((s_prefix >> 40) & kLookKeptMask);
  p += (int)(s_prefix & kLookPtsMask);
  static_assert(kCellPerThr == 4, "the cell map row store below is one int4");
  int pv[kCellPerThr];
#pragma unroll
  for (int j = 0; j < kCellPerThr; ++j) {
    const int64_t c = c0 + j;
    pv[j] = 0;
    if (c >= hw) break;
    if (keep[j]) {
      const int64_t q = (int64_t)b * pcap + a;
      pv[j] = a + 1;  // slot + 1 (0 = empty)
      *reinterpret_cast<int2*>(coords + 2 * q) = make_int2((int)(c / g.grid_w), (int)(c % g.grid_w));
      counts[q] = n[j] < g.max_points ? n[j] : g.max_points;
      w.segoff[q] = p;
      a += 1;
      p += n[j];
    }
  }
  // the cell map row as one 16-byte store per thread: four 4-byte stores 16 bytes apart
  // per instruction left every L2 sector partially written (ncu: emit read ~2x its bytes)
  if ((hw & 3) == 0 && c0 + kCellPerThr <= hw) {
    *reinterpret_cast<int4*>(w.pid + b * hw + c0) = make_int4(pv[0], pv[1], pv[2], pv[3]);
  } else {
#pragma unroll
    for (int j = 0; j < kCellPerThr; ++j)
      if (c0 + j < hw) w.pid[b * hw + c0 + j] = pv[j];
  }
}

__global__ void __launch_bounds__(1024) emit_fused_kernel(const pmx_grid g, PillarWs w, int cb, int32_t pcap,
                                                          int32_t* coords, int32_t* counts, int32_t* n_pillars) {
  pdl_begin();
  emit_block(g, w, cb, pcap, coords, counts, n_pillars, blockIdx.y);
}

__device__ __forceinline__ void slot_frame(const int64_t* __restrict__ offs, int64_t nmax, const pmx_grid& g,
                                           const PillarWs& w, int32_t pcap, int b, int64_t i0, int64_t stride) {
  const int64_t n = offs[b + 1] - offs[b];
  const int64_t hw = (int64_t)g.grid_h * g.grid_w;
  for (int64_t i = i0; i < n; i += stride) {
    int p = __ldcg(w.pid + b * hw + __ldcg(w.cell + b * nmax + i)) - 1;
    if (p >= 0) {
      int64_t q = (int64_t)b * pcap + p;
      int s = atomicAdd(w.fill + q, 1);
      w.csr[b * nmax + __ldcg(w.segoff + q) + s] = (int)i;
    }
  }
}

__global__ void slot_kernel(const int64_t* __restrict__ offs, int64_t nmax, const pmx_grid g, PillarWs w,
                            int32_t pcap) {
  pdl_begin();
  slot_frame(offs, nmax, g, w, pcap, blockIdx.y, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
             (int64_t)gridDim.x * blockDim.x);
}

// One pillar whose segment holds c > 32 points, warp-cooperatively: the first M points
// by scene index via a threshold search (t = the M-th smallest index; indices are
// distinct), compaction of the indices <= t, then a shuffle rank sort.  buf: 32 ints
// of this warp's shared memory.  All 32 lanes call it.
__device__ void warp_select_long(int64_t n_frame, int64_t nmax, int M, const PillarWs& w, int b, int64_t q,
                                 int32_t* dst, int* buf) {
  const int lane = threadIdx.x & 31;
  const int c = w.fill[q];
  const int* seg = w.csr + b * nmax + w.segoff[q];
  const int kept = c < M ? c : M;
  if (lane < M && lane >= kept) dst[lane] = -1;
  int lo = 0, hi = (int)n_frame - 1;
  while (lo < hi) {
    const int mid = lo + ((hi - lo) >> 1);
    int cntle = 0;
    for (int k = lane; k < c; k += 32) cntle += seg[k] <= mid;
    cntle = __reduce_add_sync(0xffffffffu, cntle);
    if (cntle >= M) hi = mid; else lo = mid + 1;
  }
  const int t = lo;
  int off = 0;
  for (int k0 = 0; k0 < c; k0 += 32) {
    const int k = k0 + lane;
    const int val = k < c ? seg[k] : INT_MAX;
    const bool sel = k < c && val <= t;
    const unsigned m = __ballot_sync(0xffffffffu, sel);
    if (sel) buf[off + __popc(m & ((1u << lane) - 1u))] = val;
    off += __popc(m);
  }
  __syncwarp();
  const int v = lane < M ? buf[lane] : INT_MAX;
  int rank = 0;
  for (int j = 0; j < 32; ++j) rank += __shfl_sync(0xffffffffu, v, j) < v;
  if (v != INT_MAX && rank < M) dst[rank] = v;
  __syncwarp();
}

// Thread per pillar: a KITTI pillar holds 1-3 points, so the first-M-by-scene-index
// selection is a tiny rank count over the segment; a pillar with more than 32 points
// (dense clusters) is handled by its whole warp afterwards (warp_select_long).
__global__ void __launch_bounds__(256) select_small_kernel(const int64_t* __restrict__ offs, int64_t nmax,
                                                           const pmx_grid g, PillarWs w, int32_t pcap,
                                                           const int32_t* __restrict__ n_pillars, int32_t* pt_idx) {
  pdl_begin();
  __shared__ int buf[8][32];
  const int b = blockIdx.y;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int P = n_pillars[b];
  const int M = g.max_points;
  const int64_t q = (int64_t)b * pcap + p;
  const int c = p < P ? w.fill[q] : 0;
  if (p < P && c <= 32) {
    const int* seg = w.csr + b * nmax + w.segoff[q];
    int32_t* dst = pt_idx + q * M;
    if ((M & 3) == 0) {
      for (int s = 0; s < M; s += 4) *reinterpret_cast<int4*>(dst + s) = make_int4(-1, -1, -1, -1);
    } else {
      for (int s = 0; s < M; ++s) dst[s] = -1;
    }
    for (int i = 0; i < c; ++i) {
      const int v = seg[i];
      int r = 0;
      for (int j = 0; j < c; ++j) r += seg[j] < v;
      if (r < M) dst[r] = v;
    }
  }
  unsigned long_m = __ballot_sync(0xffffffffu, p < P && c > 32);
  while (long_m) {
    const int l = __ffs(long_m) - 1;
    long_m &= long_m - 1;
    const int64_t ql = __shfl_sync(0xffffffffu, q, l);
    warp_select_long(offs[b + 1] - offs[b], nmax, M, w, b, ql, pt_idx + ql * M, buf[threadIdx.x >> 5]);
  }
}

// M == 32 variant: lane = pillar builds its 128-byte row in shared memory (16-byte
// chunks XOR-swizzled by lane % 8: conflict-free), then the warp writes 4 whole rows
// per store instruction (a thread-per-row store scatters over 32 lines).
// the 32 pillars p0 .. p0 + 31 of frame b by one warp; rows: this warp's 32 x 8 int4
// of shared memory, buf: its 32 ints
__device__ void select32_warp(const int64_t* __restrict__ offs, int64_t nmax, const PillarWs& w, int32_t pcap,
                              const int32_t* __restrict__ n_pillars, int32_t* pt_idx, int b, int p0,
                              int4 (*rows)[8], int* buf) {
  const int lane = threadIdx.x & 31;
  const int P = __ldcg(n_pillars + b);
  if (p0 >= P) return;  // warp-uniform
  const int p = p0 + lane;
  bool mine = p < P;
  const int64_t q = (int64_t)b * pcap + p;
  const int c = mine ? __ldcg(w.fill + q) : 0;
  const bool longp = mine && c > 32;  // dense cluster: the warp handles it below
  if (longp) mine = false;
  const int sw = lane & 7;
#pragma unroll
  for (int k = 0; k < 8; ++k) rows[lane][k ^ sw] = make_int4(-1, -1, -1, -1);
  if (mine) {
    const int* seg = w.csr + b * nmax + __ldcg(w.segoff + q);
    int* r32 = reinterpret_cast<int*>(rows[lane]);
    for (int i = 0; i < c; ++i) {
      const int v = seg[i];
      int r = 0;
      for (int j = 0; j < c; ++j) r += seg[j] < v;
      r32[(((r >> 2) ^ sw) << 2) + (r & 3)] = v;  // r < c <= 32
    }
  }
  const unsigned keep = __ballot_sync(0xffffffffu, mine);
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int r = 4 * j + (lane >> 3), k = lane & 7;
    if ((keep >> r) & 1)
      reinterpret_cast<int4*>(pt_idx + ((int64_t)b * pcap + p0 + r) * 32)[k] = rows[r][k ^ (r & 7)];
  }
  unsigned long_m = __ballot_sync(0xffffffffu, longp);
  while (long_m) {
    const int l = __ffs(long_m) - 1;
    long_m &= long_m - 1;
    const int64_t ql = (int64_t)b * pcap + p0 + l;
    warp_select_long(offs[b + 1] - offs[b], nmax, 32, w, b, ql, pt_idx + ql * 32, buf);
  }
  __syncwarp();
}

__global__ void __launch_bounds__(256) select_small32_kernel(const int64_t* __restrict__ offs, int64_t nmax,
                                                             const pmx_grid g, PillarWs w, int32_t pcap,
                                                             const int32_t* __restrict__ n_pillars, int32_t* pt_idx) {
  pdl_begin();
  __shared__ int4 rows[8][32][8];  // [warp][pillar][16-byte chunk]
  __shared__ int buf[8][32];
  const int wid = threadIdx.x >> 5;
  select32_warp(offs, nmax, w, pcap, n_pillars, pt_idx, blockIdx.y, (blockIdx.x * 8 + wid) * 32, rows[wid], buf[wid]);
}

// ---------------------------------------------------------------------------
// Small batches (opt-in): all six stages in ONE cooperative (gang-scheduled) persistent kernel,
// grid-wide barriers between them instead of kernel boundaries (batch 1: six launches
// of 3.4-7.6 us each, mostly launch ramp and tail).  Same device functions, same
// results: per-frame work is distributed over virtual blocks / a grid-stride loop.
constexpr int kSelWarps = 32;  // warps per persistent CTA (1024 threads)
constexpr size_t kPersistSmem = (size_t)kSelWarps * 32 * 8 * sizeof(int4) + (size_t)kSelWarps * 32 * sizeof(int);

__global__ void __launch_bounds__(1024, 1)
    pillarize_persistent_kernel(const float4* __restrict__ pts, const int64_t* __restrict__ offs, int64_t nmax,
                                const pmx_grid g, PillarWs w, int nb, int cb, int batch, int32_t pcap,
                                int32_t* coords, int32_t* counts, int32_t* pt_idx, int32_t* n_pillars,
                                int64_t n_cells, int64_t n_fill, int64_t n_look, int64_t n_ptblk) {
  namespace cg = cooperative_groups;
  pdl_begin();
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) uint8_t psm[];
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, gthreads = (int64_t)gridDim.x * blockDim.x;
  init_ws(w, n_cells, n_fill, n_look, batch, n_ptblk, gtid, gthreads);
  grid.sync();
  for (int b = 0; b < batch; ++b) bin_frame(pts, offs, nmax, g, w, b, gtid, gthreads);
  grid.sync();
  for (int v = blockIdx.x; v < cb * batch; v += gridDim.x) {
    firsthist_block(offs, nmax, g, w, nb, 1, v % cb, v / cb, cb, reinterpret_cast<int*>(psm));
    __syncthreads();
  }
  grid.sync();
  for (int v = blockIdx.x; v < cb * batch; v += gridDim.x) {
    emit_block(g, w, cb, pcap, coords, counts, n_pillars, v / cb);  // blocks of a frame in ticket order
    __syncthreads();
  }
  grid.sync();
  for (int b = 0; b < batch; ++b) slot_frame(offs, nmax, g, w, pcap, b, gtid, gthreads);
  grid.sync();
  const int warp = threadIdx.x >> 5;
  int4(*rows)[8] = reinterpret_cast<int4(*)[8]>(psm + (size_t)warp * 32 * 8 * sizeof(int4));
  int* buf = reinterpret_cast<int*>(psm + (size_t)kSelWarps * 32 * 8 * sizeof(int4)) + warp * 32;
  const int nwt = (pcap + 31) / 32;  // 32-pillar warp tasks per frame
  for (int t = blockIdx.x * kSelWarps + warp; t < nwt * batch; t += gridDim.x * kSelWarps)
    select32_warp(offs, nmax, w, pcap, n_pillars, pt_idx, t / nwt, (t % nwt) * 32, rows, buf);
}

// measured (B200, batch 1, 120k points): 34.8 us in the captured step vs 28.3 us for the
// six PDL-chained kernels -- five grid.sync()s cost more than the launches they replace;
// kept as an opt-in experiment (PMX_PILLARIZE_PERSIST=1), bit-identical either way
bool persistent_enabled() {
  static const bool on = [] {
    const char* e = getenv("PMX_PILLARIZE_PERSIST");
    return e && e[0] == '1';
  }();
  return on;
}

// ---------------------------------------------------------------------------
// feature materialisation (PillarSample.features / point_mask)

__global__ void __launch_bounds__(256) features_kernel(const float4* __restrict__ pts, const int64_t* __restrict__ offs,
                                                       const pmx_grid g, int32_t pcap, int nf,
                                                       const int32_t* __restrict__ coords,
                                                       const int32_t* __restrict__ counts,
                                                       const int32_t* __restrict__ pt_idx,
                                                       const int32_t* __restrict__ n_pillars, float* feats,
                                                       uint8_t* mask) {
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int p = blockIdx.x * 8 + wid;
  if (p >= n_pillars[b]) return;
  const int M = g.max_points;
  const int64_t q = (int64_t)b * pcap + p;
  const int k = counts[q];
  float4 pt = make_float4(0.f, 0.f, 0.f, 0.f);
  if (lane < k) pt = __ldg(pts + offs[b] + pt_idx[q * M + lane]);
  // sequential f32 mean over kept points (numpy chunk.mean(axis=0), pm/scenes.py:187)
  float sx = 0.f, sy = 0.f, sz = 0.f;
  for (int s = 0; s < k; ++s) {
    sx = __fadd_rn(sx, __shfl_sync(0xffffffffu, pt.x, s));
    sy = __fadd_rn(sy, __shfl_sync(0xffffffffu, pt.y, s));
    sz = __fadd_rn(sz, __shfl_sync(0xffffffffu, pt.z, s));
  }
  const float fk = (float)(k > 0 ? k : 1);
  const float mx = __fdiv_rn(sx, fk), my = __fdiv_rn(sy, fk), mz = __fdiv_rn(sz, fk);
  if (lane >= M) return;
  float* f = feats + (q * M + lane) * nf;
  const bool live = lane < k;
  mask[q * M + lane] = live ? 1 : 0;
  if (nf == 5) {
    f[0] = live ? pt.x : 0.f;
    f[1] = live ? pt.y : 0.f;
    f[2] = live ? pt.z : 0.f;
    f[3] = live ? __fsub_rn(pt.x, mx) : 0.f;
    f[4] = live ? __fsub_rn(pt.y, my) : 0.f;
  } else {
    const float xoff = (float)((double)g.cell_w * 0.5 + (double)g.x_min);
    const float yoff = (float)((double)g.cell_h * 0.5 + (double)g.y_min);
    const float xc = __fadd_rn(__fmul_rn((float)coords[2 * q + 1], g.cell_w), xoff);
    const float yc = __fadd_rn(__fmul_rn((float)coords[2 * q + 0], g.cell_h), yoff);
    f[0] = live ? pt.x : 0.f;
    f[1] = live ? pt.y : 0.f;
    f[2] = live ? pt.z : 0.f;
    f[3] = live ? pt.w : 0.f;
    f[4] = live ? __fsub_rn(pt.x, mx) : 0.f;
    f[5] = live ? __fsub_rn(pt.y, my) : 0.f;
    f[6] = live ? __fsub_rn(pt.z, mz) : 0.f;
    f[7] = live ? __fsub_rn(pt.x, xc) : 0.f;
    f[8] = live ? __fsub_rn(pt.y, yc) : 0.f;
  }
}

}  // namespace

}  // namespace pmx

using namespace pmx;

extern "C" {

const int32_t* pmx_pillarize_cell_map(const pmx_grid* g, int32_t batch, int64_t max_points_per_frame,
                                      const void* ws) {
  if (!g || !ws || batch < 0) return nullptr;
  int32_t pcap = g->max_pillars > 0 ? g->max_pillars : g->grid_h * g->grid_w;
  PillarWs w;
  carve(g, batch, max_points_per_frame, pcap, const_cast<void*>(ws), &w);
  return w.pid;  // emit_kernel writes every cell: kept pillar slot + 1, or 0
}

size_t pmx_pillarize_workspace(const pmx_grid* g, int32_t batch, int64_t max_points_per_frame) {
  if (!g || batch < 0) return 0;
  int32_t pcap = g->max_pillars > 0 ? g->max_pillars : g->grid_h * g->grid_w;
  return carve(g, batch, max_points_per_frame, pcap, nullptr, nullptr);
}

pmx_status pmx_pillarize(const float* points, const int64_t* frame_offsets, int32_t batch,
                         int64_t max_points_per_frame, const pmx_grid* grid, int32_t pcap, int32_t* coords,
                         int32_t* counts, int32_t* pt_idx, int32_t* n_pillars, void* ws, size_t ws_bytes,
                         pmx_stream_t stream) {
  PMX_REQUIRE(grid != nullptr, "grid is NULL");
  const pmx_grid g = *grid;
  PMX_REQUIRE(g.grid_h >= 1 && g.grid_w >= 1, "grid extents must be positive");
  PMX_REQUIRE(g.max_points >= 1 && g.max_points <= 32, "max_points must be 1..32");
  PMX_REQUIRE(g.cell_w > 0.f && g.cell_h > 0.f, "cell sizes must be positive");
  PMX_REQUIRE(batch >= 0 && max_points_per_frame >= 0, "negative extent");
  PMX_REQUIRE(max_points_per_frame < INT_MAX, "too many points per frame");
  const int64_t hw = (int64_t)g.grid_h * g.grid_w;
  PMX_REQUIRE(hw < (1 << 22), "grid too large (> 4M cells)");
  if (g.max_pillars > 0) {
    PMX_REQUIRE(pcap >= g.max_pillars, "pcap < max_pillars");
  } else {
    PMX_REQUIRE(pcap >= hw, "uncapped pillarize needs pcap >= grid_h * grid_w");
  }
  if (batch == 0) return PMX_OK;
  size_t need = carve(&g, batch, max_points_per_frame, pcap, nullptr, nullptr);
  PMX_REQUIRE(ws != nullptr && ws_bytes >= need, "pillarize workspace too small");
  PillarWs w;
  carve(&g, batch, max_points_per_frame, pcap, ws, &w);
  const int64_t nmax = max_points_per_frame > 0 ? max_points_per_frame : 1;
  const int nb = (int)ceil_div(nmax, kPtBlock);
  const int cb = (int)ceil_div(hw, kCellBlock);
  if (batch <= 8 && g.max_points == 32 && (size_t)nb * 4 <= kPersistSmem && persistent_enabled()) {
    static int occ = -1;  // resident 1024-thread CTAs per SM with the persistent kernel's shared memory
    if (occ < 0) {
      PMX_CUDA(cudaFuncSetAttribute(pillarize_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kPersistSmem));
      PMX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pillarize_persistent_kernel, 1024, kPersistSmem));
    }
    if (occ >= 1) {
      const int64_t need = std::max<int64_t>(ceil_div(nmax, 1024), (int64_t)cb) * batch;
      const int grid_n = (int)std::min<int64_t>(std::max<int64_t>(need, 1), (int64_t)num_sms());
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid_n);
      cfg.blockDim = dim3(1024);
      cfg.dynamicSmemBytes = kPersistSmem;
      cfg.stream = stream;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeCooperative;  // gang-scheduled: every CTA resident (grid.sync)
      attr[0].val.cooperative = 1;
      attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 2;
      PMX_CUDA(cudaLaunchKernelEx(&cfg, pillarize_persistent_kernel, reinterpret_cast<const float4*>(points),
                                  frame_offsets, nmax, g, w, nb, cb, (int)batch, pcap, coords, counts, pt_idx,
                                  n_pillars, (int64_t)batch * hw, (int64_t)batch * pcap, (int64_t)batch * cb,
                                  (int64_t)batch * nb));
      return check_launch("pmx_pillarize");
    }
  }
  // one kernel initialises every per-call workspace array (six memset nodes before)
  {
    const int64_t n4 = batch * hw;  // first / cnt (int4 when hw % 4 == 0)
    const int blocks = (int)std::min<int64_t>(ceil_div(n4, 256 * 4), (int64_t)num_sms() * 8);
    PMX_CUDA(launch_pdl(init_ws_kernel, dim3(blocks), dim3(256), 0, stream, w, n4, (int64_t)batch * pcap,
                        (int64_t)batch * cb, batch, (int64_t)batch * nb));
  }
  const int ptx = (int)std::min<int64_t>(ceil_div(nmax, 256), 4096);
  PMX_CUDA(launch_pdl(bin_kernel, dim3(ptx, batch), dim3(256), 0, stream, reinterpret_cast<const float4*>(points),
                      frame_offsets, nmax, g, w));
  if (nb <= 16384) {  // the per-frame bins fit in shared memory
    PMX_CUDA(cudaFuncSetAttribute(firsthist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, nb * 4));
    // small batches: its last CTA per frame also computes the cap threshold (measured:
    // batch 1 one launch less on the latency path; batch 32 faster as a separate kernel)
    const int fold = batch <= 8 ? 1 : 0;
    PMX_CUDA(launch_pdl(firsthist_kernel, dim3(cb, batch), dim3(1024), (size_t)nb * 4, stream, frame_offsets, nmax,
                        g, w, nb, fold));
    if (!fold)
      PMX_CUDA(launch_pdl(thresh_kernel, dim3(batch), dim3(1024), 0, stream, frame_offsets, nmax, g, w, nb));
  } else {
    PMX_CUDA(launch_pdl(flag_kernel, dim3(nb, batch), dim3(kPtBlock), 0, stream, frame_offsets, nmax, g, w, nb));
    PMX_CUDA(launch_pdl(thresh_kernel, dim3(batch), dim3(1024), 0, stream, frame_offsets, nmax, g, w, nb));
  }
  PMX_CUDA(launch_pdl(emit_fused_kernel, dim3(cb, batch), dim3(1024), 0, stream, g, w, cb, pcap, coords, counts,
                      n_pillars));
  PMX_CUDA(launch_pdl(slot_kernel, dim3(ptx, batch), dim3(256), 0, stream, frame_offsets, nmax, g, w, pcap));
  // (pillars with more than 32 points: their warp, inside the same kernels)
  if (g.max_points == 32)
    PMX_CUDA(launch_pdl(select_small32_kernel, dim3((int)ceil_div(pcap, 256), batch), dim3(256), 0, stream,
                        frame_offsets, nmax, g, w, pcap, n_pillars, pt_idx));
  else
    PMX_CUDA(launch_pdl(select_small_kernel, dim3((int)ceil_div(pcap, 256), batch), dim3(256), 0, stream,
                        frame_offsets, nmax, g, w, pcap, n_pillars, pt_idx));
  return check_launch("pmx_pillarize");
}

pmx_status pmx_pillar_features(const float* points, const int64_t* frame_offsets, int32_t batch,
                               const pmx_grid* grid, int32_t pcap, int32_t n_features, const int32_t* coords,
                               const int32_t* counts, const int32_t* pt_idx, const int32_t* n_pillars,
                               float* features, uint8_t* mask, pmx_stream_t stream) {
  PMX_REQUIRE(grid != nullptr, "grid is NULL");
  PMX_REQUIRE(n_features == 5 || n_features == 9, "n_features must be 5 or 9");
  PMX_REQUIRE(grid->max_points >= 1 && grid->max_points <= 32, "max_points must be 1..32");
  if (batch == 0 || pcap == 0) return PMX_OK;
  features_kernel<<<dim3((int)ceil_div(pcap, 8), batch), 256, 0, stream>>>(
      reinterpret_cast<const float4*>(points), frame_offsets, *grid, pcap, n_features, coords, counts, pt_idx,
      n_pillars, features, mask);
  return check_launch("pmx_pillar_features");
}

}  // extern "C"
