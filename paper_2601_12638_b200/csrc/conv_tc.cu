// tcgen05 implicit-GEMM conv / deconv / 1x1 for sm_100a (K6, K7, K9, K10).
//
// Persistent (grid <= 148, one CTA per SM), warp-specialised, mbarrier-pipelined;
// every role walks the same static tile sequence (tile = 128 output pixels x BN).
// The sub-partition scheduler favours high warp ids, so the single-thread roles
// sit at the top:
//   warps 0-15          epilogue (4 per TMEM lane quarter, warp & 3): tcgen05.ld
//                       (thread = output pixel row), scale + bias (+ unfolded BN) +
//                       ReLU, exact requantisation to every consumer format; NHWC
//                       stores, staged through shared memory for wide int8 rows and
//                       for the f16 half of an (int8, f16) consumer pair;
//   warp 16 (1 thread)  TMA producer: per K-block, one box of the A operand (the
//                       input shifted per 3x3 tap -- implicit im2col, padding by TMA
//                       out-of-bounds zero fill) and one box of B (weights); in HALO
//                       mode one halo box per tile (stride 1: a swizzled
//                       pixel-major 16 x 18 halo) and resident weights instead;
//                       GATHER (first conv): warps 16, 18, 19 fill the halo from
//                       pillar rows with cp.async;
//   warp 17 (1 thread)  TMEM allocator + MMA issuer: tcgen05.mma kind::i8 (s8 x s8 ->
//                       s32) or kind::f16 (f16 x f16 -> f32) into 2-8 TMEM
//                       accumulators; tcgen05.commit frees the stage / signals the
//                       epilogue.
// Stride-2 3x3 convs read the input through four parity-split tensor maps
// (x[2i+p] -> map p at i), so every tap is a plain tiled box.  Launched with
// programmatic dependent launch: the prologue overlaps the previous layer's tail.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "pmx_common.cuh"

namespace pmx {

extern thread_local int g_conv_backend_mode;  // per calling thread (test override)
thread_local unsigned long long* g_trace = nullptr;  // pmx_debug_trace (per calling thread)
thread_local unsigned long long* g_timeline = nullptr;  // pmx_debug_timeline (per calling thread)
thread_local uint32_t g_tl_tag = 0;

namespace {

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

// plain try_wait loop (no suspend-time hint) for the MMA issuer: it must resume the
// moment an operand stage or accumulator frees up
__device__ __forceinline__ void mbar_spin(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}

// Every role waits with the plain try_wait (the hardware suspends the warp inside
// TRYWAIT and resumes it when the phase completes).  The suspend-time-hint form
// compiles to TRYWAIT + NANOSLEEP.SYNCS, whose wake-up was measured (conv_trace) to
// lag the barrier by up to ~6000 cycles -- epilogue warps of one tile started
// thousands of cycles apart.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) { mbar_spin(bar, parity); }

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            int c4, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
      "[%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}

// ---- CTA pairs (cta_group::2): the two CTAs of a 2-CTA cluster compute one M = 256
// tile; each holds its 128 rows of A and half of B, the leader (rank 0) issues the MMAs.
// In the shared::cluster window bit 24 of a CTA's shared address is its rank, so an
// address with bit 24 cleared names the same offset in the leader CTA (as CUTLASS does).
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA into this CTA's shared memory, completing transaction bytes on the LEADER's barrier
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar & kPeerMask)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                                 uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar & kPeerMask)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                                 int c4, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar & kPeerMask)
      : "memory");
}
// MMA completion -> the barrier at this offset in BOTH CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          bar)
      : "memory");
}
// arrive on the leader CTA's barrier at this offset
__device__ __forceinline__ void mbar_arrive_leader(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar & kPeerMask) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int DT>
__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (DT == PMX_I8) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  } else if constexpr (DT == PMX_F32X2) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  }
}

template <int DT>
__device__ __forceinline__ void tc_mma_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (DT == PMX_I8) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  }
}

__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// tcgen05.ld of 16 accumulator columns (thread = TMEM lane) WITHOUT waiting; the
// matching tmem_ld_wait names the destination registers as in/out operands so the
// compiler cannot read them before the wait
__device__ __forceinline__ void tmem_ld16_issue(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait(uint32_t (&v)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
               :
               : "memory");
}

// 16 accumulator columns of this thread's row; 3xTF32 adds its correction accumulator
// (lo_col columns further) in f32, round to nearest
template <int DT>
__device__ __forceinline__ void acc_ld16(uint32_t taddr, int lo_col, uint32_t (&v)[16]) {
  tmem_ld16_issue(taddr, v);
  if constexpr (DT == PMX_F32X2) {
    uint32_t w[16];
    tmem_ld16_issue(taddr + (uint32_t)lo_col, w);
    tmem_ld_wait(v);
    tmem_ld_wait(w);
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(__fadd_rn(__uint_as_float(v[j]), __uint_as_float(w[j])));
  } else {
    tmem_ld_wait(v);
  }
}

// one lane of a converged warp (the lowest active one)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred)
      :
      : "memory");
  return pred != 0;
}

// K-major smem operand descriptor (tcgen05 format: version 1 at bit 46, layout at 61).
// LBO = byte stride between K-adjacent 8x16B core matrices (no-swizzle layouts only),
// SBO = byte stride between M/N-adjacent 8-row core-matrix groups.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t sbo, uint32_t layout, uint32_t lbo = 16) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// ------------------------------------------------------------------ kernel

// CONV3: 3x3 conv, one shifted input box per tap (implicit im2col by TMA coordinates)
// GEMM : 1x1 conv / deconv over flattened pixels
// HALO : stride-1 3x3 conv whose 128-pixel tile (16 rows x 8 cols) is fed from ONE
//        (18 x 10)-pixel halo box per tile stored as un-swizzled 8x16B core matrices,
//        so each tap's A operand is just a descriptor offset (9x less L2 traffic);
//        the weights stay resident in smem for the whole persistent kernel
enum : int { MODE_CONV3 = 0, MODE_GEMM = 1, MODE_HALO = 2 };

struct TcParams {
  // geometry
  int mode, deconv;
  int batch, in_h, in_w, out_h, out_w, out_c;
  int stride;      // conv stride (1 or 2) or deconv k (= s)
  int tw, th;      // conv output tile (tw * th = 128)
  int tiles_x, tiles_y;
  int m_tiles, n_tiles;  // tile grid (tile t -> m = t / n_tiles, n = t % n_tiles)
  int tw_shift;          // log2(tw)
  FastDiv fd_nt, fd_tx, fd_ty, fd_iw, fd_ih, fd_oc;  // / n_tiles, tiles_x, tiles_y, in_w, in_h, out_c
  int oc_shift;          // log2(out_c) when a power of two, else -1 (deconv tap split)
  int st_shift;          // log2(stride) (deconv stride is a power of two)
  int64_t m_total;  // GEMM mode: number of rows (input pixels)
  int n_gemm;       // GEMM N (deconv: k*k*Cout)
  int kc;           // channels per K-block
  // PMX_F32X2 (3xTF32): the K-blocks of a tap run over three segments of seg_n blocks --
  // hi x w_hi, lo x w_hi, hi x w_lo; A channel of block cb = a_off (+ a_lo in segment 1)
  // + (cb mod seg_n) * kc, the map spanning both planes of the pixel.  seg_n = 0: plain.
  int seg_n, a_off, a_lo;
  // TMEM columns per accumulator buffer: bn, or 2 * bn for 3xTF32, whose hi x w_hi
  // products accumulate at column 0 and the small lo x w_hi + hi x w_lo corrections at
  // column lo_col = bn (summed in f32 by the epilogue): the tensor core's accumulation
  // truncates, so the corrections must not be added into the large partial sums
  int acc_stride, lo_col;
  int pair;  // 2-CTA cluster (cta_group::2, M = 256): the kernel's PAIR instantiation
  // HEADS (OUTK 2, deconvs of the neck): the deconv's output tile is never written; its
  // int8 codes (the heads' input format) are staged in shared memory as the A operand of
  // a second kind::i8 MMA against this deconv's 128-channel slice of the three 1x1 heads
  // (N = 32 >= n_heads), and the int32 head partial sums go to hpart (stage 0 writes,
  // 1 accumulates, 2 accumulates and applies the heads' epilogue into hout)
  int hstage_mode, n_heads, hcs;
  // partial layout: [ps][ps][B][out_h / ps][out_w / ps][20] -- the sub-pixel phase of the
  // output pixel outermost (ps = the largest deconv stride), so every deconv's tile (one
  // tap of consecutive input pixels) reads and writes contiguous runs of partials
  int pshift, part_b;
  const int8_t* hwc;     // [32][128] int8 head weight codes of this slice (rows >= n_heads zero)
  int32_t* hpart;        // [pixels][n_heads]
  float* hout;           // stage 2: f32 heads [pixels][hcs]
  const float* halpha;   // stage 2
  const float* hbias;    // stage 2
  double hscale;
  float hinv;
  uint32_t hidesc, hcol0;
  int cblocks;      // K-blocks per tap
  int taps;         // 9 or 1
  int bn;           // N tile
  int stages;
  uint32_t a_bytes, b_bytes;  // per stage
  uint32_t sbo, layout;       // smem descriptor params (same for A and B)
  uint32_t idesc;
  uint32_t tmem_cols;
  int nacc;        // TMEM accumulator buffers (power of two; MMA runs up to nacc tiles ahead)
  int nacc_shift;  // log2(nacc)
  int egroups;     // epilogue tile slots (1, 2 or 4)
  // stride-1 HALO with a swizzled pixel-major halo (16 x 18 pixels, one TMA box
  // whose inner dimension is a whole pixel: 288 requests instead of 180 * groups)
  int hswz;
  int hswz_bo;  // descriptor base-offset rule (experiment): 0 none, 1 (addr>>7)&7, 2 (addr>>7)&3
  // warp-transposed int8 stores (single int8 consumer): each epilogue warp stages its
  // 4 chunks (32 rows x 64 B) in shared memory and every store instruction then
  // writes 8 rows x 64 contiguous bytes (thread-per-row 16-byte stores scatter over
  // 32 lines per instruction and run at ~1/4 of the write bandwidth)
  int estage;
  // the same for the (int8, f16) consumer pair of a block's last conv (next block +
  // its FP16 deblock): the int8 codes go straight out (64-byte rows), the binary16
  // values (128 bytes per row and warp) are staged -- 4 KB per warp
  int estage2;
  // HALO mode
  uint32_t halo_tx;     // halo bytes per tile (TMA transaction size)
  uint32_t hp, hw;      // halo pixels, halo row width (pixels)
  uint32_t cin_bytes;   // bytes of channels per pixel
  uint32_t bblk_bytes;  // resident weight block (one tap, one channel block)
  uint32_t bres_bytes;  // all resident weights
  int relu;
  const float* alpha;
  const float* bias;
  const float* bn_post;
  uint32_t* keys;
  unsigned long long* trace;  // debug: per-role clock64 stamps of CTA 0 (pmx_debug_trace)
  unsigned long long* tl;     // debug: per-CTA globaltimer stamps of every launch (pmx_debug_timeline)
  uint32_t tl_tag;
  // GATHER (first conv on the pillar canvas)
  const void* g_feats;   // [B * pcap, row] pillar features (+ channel offset)
  const int32_t* g_map;  // [B, in_h, in_w] pillar slot per cell, -1 empty
  int g_pcap;
  int g_row_bytes;
};

// per-role timeline of CTA 0 (tools/op_profile.py --trace); compiled in only with
// PMX_TRACE_BUILD=1 (-DPMX_CONV_TRACE) so the production kernels carry no trace code
#ifdef PMX_CONV_TRACE
#define PMX_TRACE(ev, idx)                                                              \
  do {                                                                                  \
    if (p.trace && blockIdx.x == 0 && (idx) < 64) p.trace[(ev) * 64 + (idx)] = clock64(); \
  } while (0)
#else
#define PMX_TRACE(ev, idx) \
  do {                     \
  } while (0)
#endif

// whole-graph timeline (tools/b1_timeline.py): thread 0 of every CTA stamps entry, the
// return of griddepcontrol.wait and exit with %globaltimer (trace builds only)
#ifdef PMX_CONV_TRACE
#define PMX_TL_DECL unsigned long long tl_t0 = 0, tl_t1 = 0
#define PMX_TL_STAMP(v) \
  if (p.tl && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v))
#define PMX_TL_COMMIT()                                                                            \
  do {                                                                                             \
    if (p.tl && threadIdx.x == 0) {                                                                \
      unsigned long long t2;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));                                       \
      const unsigned long long slot = atomicAdd(p.tl, 1ull);                                       \
      unsigned long long* r = p.tl + 1 + 4 * slot;                                                 \
      r[0] = ((unsigned long long)p.tl_tag << 32) | blockIdx.x;                                    \
      r[1] = tl_t0;                                                                                \
      r[2] = tl_t1;                                                                                \
      r[3] = t2;                                                                                   \
    }                                                                                              \
  } while (0)
#else
#define PMX_TL_DECL
#define PMX_TL_STAMP(v)
#define PMX_TL_COMMIT()
#endif

struct TcMaps {
  CUtensorMap a[4];  // conv: [parity] maps (stride 2) or a[0]; GEMM: a[0] 2D
  CUtensorMap b;
};

// Warp roles.  The SM sub-partition scheduler picks the eligible warp with the
// HIGHEST id first, so the latency-critical single-thread roles get the top ids:
// warps 0..15 epilogue (warp & 3 = TMEM lane quarter), 16 TMA producer (GATHER: a
// halo builder), 17 MMA issuer, 18..19 the other GATHER halo builders.
constexpr uint32_t kHaloW = 16;  // swizzled stride-1 halo row width (pixels)
constexpr int kEpiWarps = 16;
constexpr int kProdWarp = 16;
constexpr int kMmaWarp = 17;
constexpr int kThreads = 32 * (2 + kEpiWarps);  // + TMA producer warp + MMA warp
constexpr int kGatherWarps = 3;                 // GATHER: warps 16, 18, 19 build the halo tiles
constexpr int kThreadsGather = kThreads + 32 * (kGatherWarps - 1);

// 16 f32 values -> 16 exact int8 codes WITHOUT clamping: valid (returns true) when
// every |q| < 127 and no q lies within the tie band of a half-integer -- then
// rint(q) is already the code (pm/quant.py:98-103 semantics, no clip needed); NaN /
// Inf / saturation / near-ties return false and the caller takes the exact path.
// RELU: relu(y) then quantize == max(code, 0): negative bytes are zeroed with a
// sign-replicating byte permute.  ~4 instructions per value.
template <bool RELU>
__device__ __forceinline__ bool quant16_noclamp(const float (&y)[16], float inv, uint4& out) {
  const float2 M2 = make_float2(12582912.0f, 12582912.0f), I2 = make_float2(inv, inv);
  uint32_t tb[16];
  float dm = 0.0f, rm = 0.0f;
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    // t = RN(y * inv + M): the exact product rounded once to an integer (ties to even)
    // in the low mantissa bits; r = that integer; d = RN(y * inv - r), the product's
    // distance to it.  |d| < kTieBand => r == rint(y / s) (|y * inv - y / s| < 8e-6 for
    // |y / s| < 128), |r| <= 127 => no clamp.  5 instructions per pair.
    const float2 yy = make_float2(y[j], y[j + 1]);
    const float2 t = __ffma2_rn(yy, I2, M2);
    const float2 r = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
    const float2 d = __ffma2_rn(yy, I2, make_float2(-r.x, -r.y));
    dm = fmax3_nan(dm, fabsf(d.x), fabsf(d.y));
    rm = fmax3_nan(rm, fabsf(r.x), fabsf(r.y));
    tb[j] = __float_as_uint(t.x);
    tb[j + 1] = __float_as_uint(t.y);
  }
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    w[k] = __byte_perm(__byte_perm(tb[4 * k], tb[4 * k + 1], 0x0040), __byte_perm(tb[4 * k + 2], tb[4 * k + 3], 0x0040),
                       0x5410);
    if (RELU) {
      // prmt with the sign-replicate bit (nibble msb) set: 0xFF where the byte is
      // negative (the __byte_perm intrinsic drops that bit)
      uint32_t sm;
      asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(sm) : "r"(w[k]));
      w[k] &= ~sm;
    }
  }
  out = make_uint4(w[0], w[1], w[2], w[3]);
  return dm < kTieBand && rm < 127.5f;
}

// quant16_noclamp finished in place: when a chunk has a near-tie, NaN or saturating
// value (a constant empty-region activation on a tie puts ~5% of a deconv's chunks
// there), only the flagged values are redone on the exact path -- the others keep
// their fast code -- instead of requantising all 16 with clamps and patching again
// (batch 1: every layer's slowest CTA waits for this).  Bit-identical to quant16 with
// lo = 0 (RELU) or -128: every value is clip(rint(f64(relu?(y)) / s)).
template <bool RELU>
__device__ __forceinline__ uint4 quant16_sel(const float (&y)[16], double s, float inv) {
  const float2 M2 = make_float2(12582912.0f, 12582912.0f), I2 = make_float2(inv, inv);
  uint32_t tb[16];
  float dm = 0.0f, rm = 0.0f;
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    const float2 yy = make_float2(y[j], y[j + 1]);
    const float2 t = __ffma2_rn(yy, I2, M2);
    const float2 r = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
    const float2 d = __ffma2_rn(yy, I2, make_float2(-r.x, -r.y));
    dm = fmax3_nan(dm, fabsf(d.x), fabsf(d.y));
    rm = fmax3_nan(rm, fabsf(r.x), fabsf(r.y));
    tb[j] = __float_as_uint(t.x);
    tb[j + 1] = __float_as_uint(t.y);
  }
  if (!(dm < kTieBand && rm < 127.5f)) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float r = __fsub_rn(__uint_as_float(tb[j]), 12582912.0f);
      const float d = __fmaf_rn(y[j], inv, -r);
      if (!(fabsf(d) < kTieBand && fabsf(r) < 127.5f))
        tb[j] = (uint32_t)quantize_exact(RELU ? fmaxf(y[j], 0.0f) : y[j], s, inv);
    }
  }
  uint32_t w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    w[k] = __byte_perm(__byte_perm(tb[4 * k], tb[4 * k + 1], 0x0040), __byte_perm(tb[4 * k + 2], tb[4 * k + 3], 0x0040),
                       0x5410);
    if (RELU) {
      uint32_t sm;
      asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(sm) : "r"(w[k]));
      w[k] &= ~sm;
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// One chunk (16 accumulator columns of one pixel row): y = acc * alpha + bias (int8)
// or acc + bias (f16), optional unfolded BN and ReLU, observer min/max, then every
// consumer format.  alpha / bias come from the shared-memory copies.
template <int DT, int OUTK>
__device__ __forceinline__ void epi_chunk(const TcParams& p, const Outs& outs, const uint32_t (&v)[16], uint32_t pix,
                                          int nbase, int cobase, const float* s_alpha, const float* s_bias, float qlo,
                                          float& lo, float& hi) {
  const bool full16 = (nbase + 16) <= p.n_gemm;
  float y[16];
  if (full16) {
    const float4* b4p = reinterpret_cast<const float4*>(s_bias + cobase);
    const float4* a4p = reinterpret_cast<const float4*>(s_alpha + cobase);
#pragma unroll
    for (int j4 = 0; j4 < 4; ++j4) {
      const float4 b4 = b4p[j4];
      float2 r0, r1;
      if constexpr (DT == PMX_I8) {
        const float4 a4 = a4p[j4];
        r0 = __ffma2_rn(make_float2((float)(int)v[4 * j4], (float)(int)v[4 * j4 + 1]), make_float2(a4.x, a4.y),
                        make_float2(b4.x, b4.y));
        r1 = __ffma2_rn(make_float2((float)(int)v[4 * j4 + 2], (float)(int)v[4 * j4 + 3]), make_float2(a4.z, a4.w),
                        make_float2(b4.z, b4.w));
      } else {
        r0 = __fadd2_rn(make_float2(__uint_as_float(v[4 * j4]), __uint_as_float(v[4 * j4 + 1])),
                        make_float2(b4.x, b4.y));
        r1 = __fadd2_rn(make_float2(__uint_as_float(v[4 * j4 + 2]), __uint_as_float(v[4 * j4 + 3])),
                        make_float2(b4.z, b4.w));
      }
      y[4 * j4] = r0.x;
      y[4 * j4 + 1] = r0.y;
      y[4 * j4 + 2] = r1.x;
      y[4 * j4 + 3] = r1.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int co = cobase + j;
      y[j] = 0.f;
      if ((nbase + j) < p.n_gemm) {
        if constexpr (DT == PMX_I8) y[j] = __fmaf_rn((float)(int)v[j], s_alpha[co], s_bias[co]);
        else y[j] = __fadd_rn(__uint_as_float(v[j]), s_bias[co]);
      }
    }
  }
  if constexpr (OUTK == 1) {
    // single int8 consumer, 16-byte aligned rows (checked on the host); the ReLU folds
    // into the quantizer's lower clamp
    if (full16 && !p.bn_post && !p.keys) {
      const OutDev& od = outs.o[0];
      *reinterpret_cast<uint4*>(reinterpret_cast<int8_t*>(od.ptr) + (size_t)pix * od.c_stride + od.c_offset + cobase) =
          (qlo == 0.0f ? quant16_sel<true>(y, od.scale, od.inv) : quant16_sel<false>(y, od.scale, od.inv));
      return;
    }
  }
  if (p.bn_post) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int co = cobase + j;
      if ((nbase + j) < p.n_gemm)
        y[j] = __fadd_rn(__fmul_rn(__fsub_rn(y[j], p.bn_post[co]), p.bn_post[p.out_c + co]), p.bn_post[2 * p.out_c + co]);
    }
  }
  if (p.relu) {
#pragma unroll
    for (int j = 0; j < 16; ++j) y[j] = fmaxf(y[j], 0.f);
  }
  if (p.keys) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if ((nbase + j) < p.n_gemm) {
        lo = nmin(lo, y[j]);
        hi = nmax(hi, y[j]);
      }
  }
  if constexpr (OUTK == 1) {
    const OutDev& od = outs.o[0];
    if (full16) {
      *reinterpret_cast<uint4*>(reinterpret_cast<int8_t*>(od.ptr) + (size_t)pix * od.c_stride + od.c_offset + cobase) =
          quant16_sel<false>(y, od.scale, od.inv);
    } else {
      for (int j = 0; j < 16; ++j)
        if (nbase + j < p.n_gemm) store_one(od, pix, cobase + j, y[j]);
    }
  } else {
#pragma unroll
    for (int o = 0; o < PMX_MAX_OUTS; ++o) {
      if (o >= outs.n) break;
      const OutDev& od = outs.o[o];
      const int64_t off = (int64_t)pix * od.c_stride + od.c_offset + cobase;
      if (full16 && od.dtype == PMX_I8 && (off & 15) == 0) {
        *reinterpret_cast<uint4*>(reinterpret_cast<int8_t*>(od.ptr) + off) = quant16_sel<false>(y, od.scale, od.inv);
      } else if (full16 && od.dtype == PMX_F16 && (off & 7) == 0) {
        uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(od.ptr) + off);
        dst[0] = make_uint4(f16x2_sat(y[0], y[1]), f16x2_sat(y[2], y[3]), f16x2_sat(y[4], y[5]), f16x2_sat(y[6], y[7]));
        dst[1] = make_uint4(f16x2_sat(y[8], y[9]), f16x2_sat(y[10], y[11]), f16x2_sat(y[12], y[13]),
                            f16x2_sat(y[14], y[15]));
      } else if (full16 && od.dtype == PMX_F32 && (off & 3) == 0) {
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(od.ptr) + off);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) dst[qq] = make_float4(y[4 * qq], y[4 * qq + 1], y[4 * qq + 2], y[4 * qq + 3]);
      } else if (full16 && od.dtype == PMX_F32X2 && (off & 3) == 0 && (od.c_stride & 7) == 0) {
        store16_f32x2(od, off, y);
      } else {
        for (int j = 0; j < 16; ++j)
          if (nbase + j < p.n_gemm) store_one(od, pix, cobase + j, y[j]);
      }
    }
  }
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// GATHER producer (first conv on the pillar canvas, never materialised): the halo
// tile of the (virtual) canvas x[b, y, x, :] = feats[b * pcap + map[b, y, x] - 1, :]
// (0 where map == 0 or outside the grid) is built in shared memory by 96 threads in
// exactly the layout the TMA halo path produces -- per parity plane, [channel
// group][plane pixel][16 B].  Every thread owns kPixPerThr fixed halo pixels and,
// per tile, independently of the others (no barriers, no shared lists):
//   waits for the stage, zeroes its pixels the stage's previous tile filled, copies
//   the feature rows of its occupied pixels (~7% at KITTI density) with cp.async
//   straight into the stage, and arrives on the stage's full barrier through
//   cp.async.mbarrier.arrive (the arrival lands when its copies have); the cell-map
//   entries of its next tile are loaded meanwhile.
// The MMA warp's tcgen05.mma reads the stage through the async proxy: it issues a
// proxy fence after the full-barrier wait.  (The tensor core saturates shared-memory
// bandwidth on this N = 64 layer, so the producer avoids every dependent
// shared-memory round trip.)
// Replaces the canvas write of pm/tensor_ops.py:138-160 + the conv's canvas read.
template <int HS>
struct GatherGeom {
  static constexpr int HPX_TOTAL = HS == 2 ? 561 : 180;
};

constexpr int kPixPerThr = 6;  // ceil(561 / 96)

__host__ __device__ constexpr int plane_w(int hs, int q) { return hs == 2 ? 8 + (q & 1) : 10; }
__host__ __device__ constexpr int plane_hpx(int hs, int q) { return hs == 2 ? (16 + (q >> 1)) * (8 + (q & 1)) : 180; }
__host__ __device__ constexpr int plane_p0(int hs, int q) {
  return hs == 2 ? (q == 0 ? 0 : (q == 1 ? 128 : (q == 2 ? 272 : 408))) : 0;
}

// smem of the gather producer (after alpha / bias): counters, two occupied-pixel
// lists (load side, one per tile in flight) and one clear list per stage
constexpr int kGatherSmem = 0;  // the cp.async gather producer keeps its state in registers

// 16 zero bytes into shared memory through cp.async (src-size 0: nothing is read)
__device__ __forceinline__ void cp_async_zero16(uint32_t dst, const void* any_global) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;" ::"r"(dst), "l"(any_global) : "memory");
}

template <int CINB, int HS, typename FullF, typename EmptyF>
__device__ __forceinline__ void gather_producer(const TcParams& p, uint32_t a_smem, int gt, int total, FullF full,
                                                EmptyF empty) {
  using Geo = GatherGeom<HS>;
  constexpr int G = CINB / 16;  // 16-byte channel groups per pixel
  constexpr int NT = 32 * kGatherWarps;
  static_assert(NT * kPixPerThr >= Geo::HPX_TOTAL, "halo pixels per thread");
  const char* feats = reinterpret_cast<const char*>(p.g_feats);
  // my halo pixels: offset from the tile's input origin and the stage offset of
  // channel group 0 (group g adds g * plane pixels * 16 bytes)
  int ry[kPixPerThr], rx[kPixPerThr];
  uint32_t dst0[kPixPerThr], gstep[kPixPerThr];
  uint32_t have = 0;  // bit j: pixel j exists
#pragma unroll
  for (int j = 0; j < kPixPerThr; ++j) {
    const int hp = gt + NT * j;
    int q = 0;
    if (HS == 2) q = (hp >= 128) + (hp >= 272) + (hp >= 408);
    const int pp = hp - plane_p0(HS, q);
    const int W = plane_w(HS, q);
    const int r = pp / W, c = pp - (pp / W) * W;
    const int py = q >> 1, px = q & 1;
    ry[j] = HS == 2 ? 2 * (r - py) + py : r - 1;  // iy = stride * oy0 + ry
    rx[j] = HS == 2 ? 2 * (c - px) + px : c - 1;
    dst0[j] = (uint32_t)(plane_p0(HS, q) * G + pp) * 16u;
    gstep[j] = (uint32_t)plane_hpx(HS, q) * 16u;
    if (hp < Geo::HPX_TOTAL) have |= 1u << j;
  }
  auto load_map = [&](int t, int (&m)[kPixPerThr]) {
    const int tq = (int)fdiv((uint32_t)t, p.fd_tx), tx = t - tq * p.tiles_x;
    const int tb = (int)fdiv((uint32_t)tq, p.fd_ty);
    const int oy0 = (tq - tb * p.tiles_y) * p.th, ox0 = tx * p.tw;
    const int32_t* map = p.g_map + (int64_t)tb * p.in_h * p.in_w;
#pragma unroll
    for (int j = 0; j < kPixPerThr; ++j) {
      const int iy = HS * oy0 + ry[j], ix = HS * ox0 + rx[j];
      m[j] = 0;
      if (((have >> j) & 1) && (unsigned)iy < (unsigned)p.in_h && (unsigned)ix < (unsigned)p.in_w)
        m[j] = __ldg(map + iy * p.in_w + ix);
    }
  };
  // every thread owns its pixels in every stage: zero them once, afterwards clear only
  // the pixels the stage's previous tile filled (bits in clr, kPixPerThr per stage).
  // Zeros are written by cp.async with a zero source size, so every write to a stage
  // is tracked by the thread's cp.async.mbarrier.arrive on the stage's full barrier.
  for (int st = 0; st < p.stages; ++st)
#pragma unroll
    for (int j = 0; j < kPixPerThr; ++j)
      if ((have >> j) & 1)
        for (int g = 0; g < G; ++g)
          cp_async_zero16(a_smem + st * p.a_bytes + dst0[j] + g * gstep[j], feats);
  uint64_t clr = 0;
  // cell-map entries of this tile and of the next one (loaded a whole tile ahead, so
  // the copies of a stage wait for one L2 round trip, not two)
  int mcur[kPixPerThr], mnext[kPixPerThr];
  if (blockIdx.x < total) load_map(blockIdx.x, mcur);
  if (blockIdx.x + (int)gridDim.x < total) load_map(blockIdx.x + gridDim.x, mnext);
  uint32_t s = 0, ph = 0;
  int it = 0;  // trace index
  (void)it;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int tb = (int)fdiv(fdiv((uint32_t)t, p.fd_tx), p.fd_ty);
    const char* fb = feats + (int64_t)tb * p.g_pcap * p.g_row_bytes;
    if (gt == 0) PMX_TRACE(0, it);
    mbar_wait(empty(s), ph ^ 1);
    if (gt == 0) PMX_TRACE(10, it);
    const uint32_t slot = a_smem + s * p.a_bytes;
    const uint32_t old = (uint32_t)(clr >> (kPixPerThr * s)) & ((1u << kPixPerThr) - 1);
    uint32_t now = 0;
#pragma unroll
    for (int j = 0; j < kPixPerThr; ++j) {
      // a pixel the stage's previous tile filled and this one leaves empty: zero it
      // (st.shared: no L1TEX request; occupied pixels are overwritten by the copies)
      if (((old >> j) & 1) && mcur[j] == 0)
        for (int g = 0; g < G; ++g)
          asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(slot + dst0[j] + g * gstep[j]), "r"(0)
                       : "memory");
      if (mcur[j] != 0) {
        // occupied pixel: its feature row (G x 16 bytes) straight into the stage
        const char* src = fb + (int64_t)(mcur[j] - 1) * p.g_row_bytes;
        for (int g = 0; g < G; ++g)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slot + dst0[j] + g * gstep[j]),
                       "l"(src + 16 * g)
                       : "memory");
        now |= 1u << j;
      }
    }
    clr = (clr & ~((uint64_t)((1u << kPixPerThr) - 1) << (kPixPerThr * s))) | ((uint64_t)now << (kPixPerThr * s));
    // two arrivals per thread on the stage's full barrier: a release arrive ordering its
    // zero fills, the cp.async arrive once its copies have landed
    mbar_arrive(full(s));
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full(s)) : "memory");
    if (gt == 0) PMX_TRACE(1, it);
    ++it;
#pragma unroll
    for (int j = 0; j < kPixPerThr; ++j) mcur[j] = mnext[j];
    const int tn2 = t + 2 * (int)gridDim.x;
    if (tn2 < total) load_map(tn2, mnext);  // in flight for a whole tile
    if (++s == (uint32_t)p.stages) s = 0, ph ^= 1;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Persistent: grid = min(tiles, SMs); every role walks the same static tile sequence.
// Accumulators are double-buffered in TMEM so the epilogue of tile i overlaps the
// TMA + MMA of tile i+1; the smem ring runs across tile boundaries.
template <int DT, int OUTK, int KCB, int CINB, int HS, bool GATHER, bool PAIR = false>
__global__ void __launch_bounds__(GATHER ? kThreadsGather : kThreads, 1)
    conv_tc_kernel(const __grid_constant__ TcMaps maps, const TcParams p, const Outs outs) {
  PMX_TL_DECL;
  PMX_TL_STAMP(tl_t0);
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t a_smem = base;
  const uint32_t b_smem = base + p.stages * p.a_bytes;
  const uint32_t bres = b_smem + p.stages * p.b_bytes;  // HALO: resident weights (1024-aligned)
  const uint32_t bar_base = bres + p.bres_bytes;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (bar_base - base) + 8 * (2 * p.stages + 2 * p.nacc + 1));
  const uint32_t bfull = bar_base + 8u * (2 * p.stages + 2 * p.nacc);
  // per-channel alpha / bias copies (16-byte aligned, after the barriers + TMEM slot)
  float* s_alpha = reinterpret_cast<float*>(gbase + (((bar_base - base) + 8 * (2 * p.stages + 2 * p.nacc + 1) + 4 + 15) & ~15u));
  float* s_bias = s_alpha + ((p.out_c + 3) & ~3);
  // epilogue store staging: 2 KB per epilogue warp (after alpha / bias / gather list)
  const uint32_t s_estage = (smem_u32(s_bias + ((p.out_c + 3) & ~3)) + (GATHER ? (uint32_t)kGatherSmem : 0u) + 15u) & ~15u;
  auto full = [&](int s) { return bar_base + 8u * s; };
  auto empty = [&](int s) { return bar_base + 8u * (p.stages + s); };
  auto tfull = [&](int a) { return bar_base + 8u * (2 * p.stages + a); };
  auto tempty = [&](int a) { return bar_base + 8u * (2 * p.stages + p.nacc + a); };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // PAIR: the 2-CTA cluster walks pair tiles (two adjacent M tiles x one N tile); this
  // CTA's M tile is 2 * (pair tile's M index) + rank
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int total = PAIR ? ((p.m_tiles + 1) / 2) * p.n_tiles : p.m_tiles * p.n_tiles;
  const int tstart = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int tstride = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  auto tile_of = [&](uint32_t t, uint32_t& mt, uint32_t& nt) {
    const uint32_t q = fdiv(t, p.fd_nt);
    nt = t - q * (uint32_t)p.n_tiles;
    mt = PAIR ? 2u * q + rank : q;
  };
  const int nk = p.taps * p.cblocks;
  __shared__ uint64_t hbar_s[4];  // HEADS: head MMA done, per (epilogue tile slot, buffer)

  if (threadIdx.x == 0) {
    PMX_TRACE(8, 0);
    if (OUTK == 2)
      for (int b = 0; b < 4; ++b) mbar_init(smem_u32(&hbar_s[b]), 1);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(full(s), GATHER ? 2 * 32 * kGatherWarps : 1);  // TMA: expect_tx; gather: 2 arrivals per thread
      mbar_init(empty(s), 1);
    }
    for (int a = 0; a < p.nacc; ++a) {
      mbar_init(tfull(a), 1);
      mbar_init(tempty(a), (PAIR ? 2 : 1) * 4 * (4 / p.egroups));  // the warps draining one tile (both CTAs)
    }
    mbar_init(bfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(p.tmem_cols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(p.tmem_cols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // both CTAs' barriers initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) PMX_TRACE(8, 1);
  // Programmatic dependent launch: everything above, the resident-weight TMA and the
  // epilogue's parameter prefetch only touch data no earlier kernel writes, so they
  // overlap the previous layer's tail; the activations are read (and the outputs
  // written) only after griddepcontrol.wait.  The next layer may start launching now.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (p.bres_bytes && warp == kProdWarp && lane == 0) {
    // PAIR: each CTA holds its half of the N tile's weights; both halves complete on the
    // leader's barrier
    if (!PAIR || rank == 0) mbar_expect_tx(bfull, (PAIR ? 2u : 1u) * p.bres_bytes);
    const int nb0 = PAIR ? (int)rank * (p.bn >> 1) : (int)(blockIdx.x % (uint32_t)p.n_tiles) * p.bn;
    for (int kb = 0; kb < nk; ++kb) {
      const int tap = kb / p.cblocks, cb = kb % p.cblocks;
      if constexpr (PAIR) tma_load_2d_pair(bres + kb * p.bblk_bytes, &maps.b, tap * (p.cblocks * p.kc) + cb * p.kc, nb0, bfull);
      else tma_load_2d(bres + kb * p.bblk_bytes, &maps.b, tap * (p.cblocks * p.kc) + cb * p.kc, nb0, bfull);
    }
  }
  if (warp < kEpiWarps) {
    const int n0 = (blockIdx.x % p.n_tiles) * p.bn;
    for (int c = warp >> 2; c < p.bn / 16; c += 4) {
      const int co = n0 + 16 * c < p.out_c ? n0 + 16 * c : 0;
      asm volatile("prefetch.global.L1 [%0];" ::"l"(p.bias + co));
      if (p.alpha) asm volatile("prefetch.global.L1 [%0];" ::"l"(p.alpha + co));
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  PMX_TL_STAMP(tl_t1);

  if (GATHER && (warp == kProdWarp || warp > kMmaWarp)) {
    if constexpr (GATHER) {
      gather_producer<CINB, HS>(p, a_smem, warp == kProdWarp ? lane : 32 * (warp - kMmaWarp) + lane, total, full,
                                empty);
    }
  } else if (warp == kProdWarp) {
    if (lane == 0) {
      // ---------------- TMA producer
      uint32_t it = 0, s = 0, ph = 0;  // ring position, slot, phase
      if (p.mode == MODE_HALO) {
        for (int t = tstart; t < total; t += tstride, ++it) {
          uint32_t mtu, ntu;
          tile_of((uint32_t)t, mtu, ntu);  // N tile: blockIdx.x % n_tiles for every t
          const int mt = (int)mtu;
          const int tq = (int)fdiv((uint32_t)mt, p.fd_tx), tx = mt - tq * p.tiles_x;
          const int tb = (int)fdiv((uint32_t)tq, p.fd_ty);
          const int oy0 = (tq - tb * p.tiles_y) * p.th, ox0 = tx * p.tw;
          PMX_TRACE(0, it);
          mbar_wait(empty(s), ph ^ 1);
#if defined(PMX_ABLATE) && PMX_ABLATE == 4
          // diagnostic: after the first ring of halos, no more TMA traffic (stale data)
          if ((int)it >= p.stages) {
            mbar_arrive(full(s));
            PMX_TRACE(1, it);
            if (++s == (uint32_t)p.stages) s = 0, ph ^= 1;
            continue;
          }
#endif
          // PAIR: both CTAs' halos complete on the leader's barrier
          if (!PAIR || rank == 0) mbar_expect_tx(full(s), (PAIR ? 2u : 1u) * p.halo_tx);
          const uint32_t slot = a_smem + s * p.a_bytes;
          if (p.stride == 1) {
            if (p.hswz) {
              if constexpr (PAIR) tma_load_4d_pair(slot, &maps.a[0], 0, ox0 - 1, oy0 - 1, tb, full(s));
              else tma_load_4d(slot, &maps.a[0], 0, ox0 - 1, oy0 - 1, tb, full(s));
            } else {
              if constexpr (PAIR) tma_load_5d_pair(slot, &maps.a[0], 0, ox0 - 1, oy0 - 1, 0, tb, full(s));
              else tma_load_5d(slot, &maps.a[0], 0, ox0 - 1, oy0 - 1, 0, tb, full(s));
            }
          } else {
            // four parity planes (py, px): (16 + py) x (8 + px) pixels from (oy0 - py, ox0 - px)
            uint32_t off = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int py = q >> 1, px = q & 1;
              if constexpr (PAIR) tma_load_5d_pair(slot + off, &maps.a[q], 0, ox0 - px, oy0 - py, 0, tb, full(s));
              else tma_load_5d(slot + off, &maps.a[q], 0, ox0 - px, oy0 - py, 0, tb, full(s));
              off += (uint32_t)((16 + py) * (8 + px)) * p.cin_bytes;
            }
          }
          PMX_TRACE(1, it);
          if (++s == (uint32_t)p.stages) s = 0, ph ^= 1;
        }
      }
      for (int t = tstart; t < total && p.mode != MODE_HALO; t += tstride) {
        uint32_t mtu, ntu;
        tile_of((uint32_t)t, mtu, ntu);
        const int mt = (int)mtu, nt = (int)ntu;
        // PAIR: this CTA's half of the N tile
        const int n0 = nt * p.bn + (PAIR ? (int)rank * (p.bn >> 1) : 0);
        int tb = 0, oy0 = 0, ox0 = 0, m0 = 0;
        if (p.mode == MODE_CONV3) {
          const int tq = (int)fdiv((uint32_t)mt, p.fd_tx), tx = mt - tq * p.tiles_x;
          tb = (int)fdiv((uint32_t)tq, p.fd_ty);
          oy0 = (tq - tb * p.tiles_y) * p.th;
          ox0 = tx * p.tw;
        } else {
          m0 = mt * 128;
        }
        for (int kb = 0; kb < nk; ++kb, ++it) {
          PMX_TRACE(0, it);
          mbar_wait(empty(s), ph ^ 1);
          // PAIR: the leader's full barrier counts the bytes of both CTAs' loads
          if (!PAIR || rank == 0) mbar_expect_tx(full(s), (PAIR ? 2u : 1u) * (p.a_bytes + p.b_bytes));
          const int tap = kb / p.cblocks, cb = kb % p.cblocks;
          const bool load_b = p.b_bytes != 0;  // 0: the GEMM mode's weights are resident
          const int c0 = cb * p.kc;
          int ac = c0;  // A channel coordinate
          if (p.seg_n) {
            const int seg = cb / p.seg_n;
            ac = p.a_off + (seg == 1 ? p.a_lo : 0) + (cb - seg * p.seg_n) * p.kc;
          }
          const uint32_t adst = a_smem + s * p.a_bytes, bdst = b_smem + s * p.b_bytes;
          if constexpr (PAIR) {
            if (p.mode == MODE_CONV3) {
              const int dy = tap / 3 - 1, dx = tap % 3 - 1;
              if (p.stride == 1) {
                tma_load_4d_pair(adst, &maps.a[0], ac, ox0 + dx, oy0 + dy, tb, full(s));
              } else {
                const int ay = dy < 0 ? -1 : 0, py = dy == 0 ? 0 : 1;
                const int ax = dx < 0 ? -1 : 0, px = dx == 0 ? 0 : 1;
                tma_load_4d_pair(adst, &maps.a[py * 2 + px], ac, ox0 + ax, oy0 + ay, tb, full(s));
              }
            } else {
              tma_load_2d_pair(adst, &maps.a[0], ac, m0, full(s));
            }
            tma_load_2d_pair(bdst, &maps.b, tap * (p.cblocks * p.kc) + c0, n0, full(s));
          } else {
          if (p.mode == MODE_CONV3) {
            const int dy = tap / 3 - 1, dx = tap % 3 - 1;
            if (p.stride == 1) {
              tma_load_4d(adst, &maps.a[0], ac, ox0 + dx, oy0 + dy, tb, full(s));
            } else {  // 2*o + d = 2*(o + a) + par
              const int ay = dy < 0 ? -1 : 0, py = dy == 0 ? 0 : 1;
              const int ax = dx < 0 ? -1 : 0, px = dx == 0 ? 0 : 1;
              tma_load_4d(adst, &maps.a[py * 2 + px], ac, ox0 + ax, oy0 + ay, tb, full(s));
            }
          } else {
            tma_load_2d(adst, &maps.a[0], ac, m0, full(s));
          }
          if (load_b) tma_load_2d(bdst, &maps.b, tap * (p.cblocks * p.kc) + c0, n0, full(s));
          }
          PMX_TRACE(1, it);
          if (++s == (uint32_t)p.stages) s = 0, ph ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer.  The whole warp walks the loop (barrier waits are
    // warp-wide, so the descriptors stay in uniform registers) and one elected lane
    // issues.  Descriptor words: hi = SBO | version | layout (constant), lo = LBO << 16
    // | (address >> 4); the address is always < 256 KB, so every operand's lo word is
    // one uniform add of a compile-time constant to the stage base -- the issue path
    // is ~2 instructions per MMA and never starves behind the epilogue warps.
    const uint32_t idesc = p.idesc;
    const uint32_t bn = (uint32_t)p.bn;
    uint32_t i = 0;
    if constexpr (CINB > 0) {
      constexpr int CB = CINB / KCB;
      const uint32_t bblk = p.bblk_bytes;
      const uint32_t b_hi = (uint32_t)(sdesc(0, p.sbo, p.layout) >> 32), b_lo0 = (uint32_t)sdesc(bres, p.sbo, p.layout);
      // resident weights: the B descriptor of every (tap, 32-byte K step), hoisted out of
      // the tile loop
      // (256-byte rows: 72 descriptors would spill; those are one IMAD each instead)
      constexpr bool kHoistB = CINB <= 128;
      uint32_t b_lo_tap[kHoistB ? 9 * (CINB / 32) : 1];
      const uint32_t bblk16 = bblk >> 4;
      if constexpr (kHoistB) {
#pragma unroll
        for (int tap = 0; tap < 9; ++tap)
#pragma unroll
          for (int k = 0; k < CINB / 32; ++k)
            b_lo_tap[tap * (CINB / 32) + k] =
                b_lo0 + (((uint32_t)(tap * CB + (k * 32) / KCB) * bblk + (uint32_t)((k * 32) % KCB)) >> 4);
      }
      auto b_lo_of = [&](int tap, int k) -> uint32_t {
        if constexpr (kHoistB) return b_lo_tap[tap * (CINB / 32) + k];
        else return b_lo0 + (uint32_t)(tap * CB + (k * 32) / KCB) * bblk16 + (uint32_t)(((k * 32) % KCB) >> 4);
      };
      if (!PAIR || rank == 0) mbar_wait(bfull, 0);  // (PAIR: both halves land on the leader's barrier)
      tc_fence_after();
      if (lane == 0) PMX_TRACE(8, 2);
      uint32_t s = 0, ph = 0, acc = 0, aph = 0;  // smem stage / accumulator and their phases
      // PAIR: only the leader issues (M = 256 over both CTAs' halos, N over both B halves)
      for (int t = tstart; t < total && (!PAIR || rank == 0); t += tstride, ++i) {
        if (lane == 0) PMX_TRACE(9, i);
        mbar_spin(tempty(acc), aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * (uint32_t)p.acc_stride;
        if (lane == 0) PMX_TRACE(2, i);
        mbar_spin(full(s), ph);
        tc_fence_after();
        // GATHER: the stage was written through the generic proxy (st.shared, cp.async)
        if constexpr (GATHER) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (HS == 1 && p.hswz) {
          if (elect_one()) {
            // pixel-major halo rows of CINB bytes (SW128 / SW64, TMA-swizzled by address):
            // tap (dy, dx) starts at halo pixel (dy + 1) * 16 + dx + 1; 8-row groups are
            // 16 pixels = whole swizzle patterns apart (the swizzle follows the absolute
            // address, base offset 0).  Every descriptor is the stage's base plus a
            // compile-time offset: the issue path is one add per MMA (the per-MMA address
            // arithmetic it replaced made the MMA warp issue-bound, ~80 cycles per MMA)
            constexpr uint32_t lay = CINB == 128 ? 2u : 4u;
            constexpr uint32_t a_hi = (kHaloW * CINB) >> 4 | (1u << 14) | (lay << 29);
            const uint32_t a_lo = (1u << 16) + ((a_smem + s * p.a_bytes) >> 4);  // smem < 256 KB
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) {
              const int dy = tap / 3 - 1, dx = tap % 3 - 1;
#pragma unroll
              for (int k = 0; k < CINB / 32; ++k) {
                const uint32_t aoff = (uint32_t)((((dy + 1) * (int)kHaloW + dx + 1) * CINB + 32 * k) >> 4);
                const uint64_t ad = ((uint64_t)a_hi << 32) | (a_lo + aoff);
                const uint64_t bd = ((uint64_t)b_hi << 32) | b_lo_of(tap, k);
                if constexpr (PAIR) tc_mma_pair<DT>(d, ad, bd, idesc, (tap | k) != 0);
                else tc_mma<DT>(d, ad, bd, idesc, (tap | k) != 0);
              }
            }
            if constexpr (PAIR) {
              tc_commit_pair(empty(s));
              tc_commit_pair(tfull(acc));
            } else {
              tc_commit(empty(s));
              tc_commit(tfull(acc));
            }
          }
        } else if (elect_one()) {
          PMX_TRACE(3, i);
          const uint32_t alo = (a_smem + s * p.a_bytes) >> 4;
          // (256-byte rows: a tap loop, not 72 unrolled descriptors held in registers)
          constexpr int kTapUnroll = CINB <= 128 ? 9 : 1;
#pragma unroll kTapUnroll
          for (int tap = 0; tap < 9; ++tap) {
            // A operand of this tap inside the halo: plane base, pixel offset, row width
            const int dy = tap / 3 - 1, dx = tap % 3 - 1;
            const int py = HS == 2 ? (dy != 0) : 0, px = HS == 2 ? (dx != 0) : 0;
            const int HW = HS == 2 ? 8 + px : 10;            // halo row width (pixels)
            const int HPX = HS == 2 ? (16 + py) * HW : 180;  // pixels in this plane
            const int q = py * 2 + px;
            const int plane_px = HS == 2 ? (q == 0 ? 0 : (q == 1 ? 128 : (q == 2 ? 272 : 408))) : 0;
            const int pix0 = HS == 2 ? (dy == 1) * HW + (dx == 1) : (dy + 1) * HW + (dx + 1);
            const uint32_t a_hi = (uint32_t)(HW * 16) >> 4 | (1u << 14);  // SBO | version (layout 0)
            const uint32_t a_lbo = (uint32_t)(HPX * 16) >> 4;
#pragma unroll
            for (int k = 0; k < CINB / 32; ++k) {
              // two 16-byte channel groups per instruction (core matrices at +LBO)
              const uint32_t aoff = (uint32_t)(plane_px * CINB + ((2 * k) * HPX + pix0) * 16);
              const uint64_t ad = ((uint64_t)a_hi << 32) | (alo + ((a_lbo << 16) + (aoff >> 4)));
              const uint64_t bd = ((uint64_t)b_hi << 32) | b_lo_of(tap, k);
              if constexpr (PAIR) tc_mma_pair<DT>(d, ad, bd, idesc, (tap | k) != 0);
              else tc_mma<DT>(d, ad, bd, idesc, (tap | k) != 0);
            }
          }
          if constexpr (PAIR) {
            tc_commit_pair(empty(s));
            tc_commit_pair(tfull(acc));
          } else {
            tc_commit(empty(s));
            tc_commit(tfull(acc));
          }
          PMX_TRACE(4, i);
        }
        __syncwarp();
        if (++s == (uint32_t)p.stages) s = 0, ph ^= 1;
        if (++acc == (uint32_t)p.nacc) acc = 0, aph ^= 1;
      }
    } else {
      constexpr int ksteps = KCB / 32;  // 32 bytes of K per instruction
      const uint32_t hi = (uint32_t)(sdesc(0, p.sbo, p.layout) >> 32), lo0 = (uint32_t)sdesc(0, p.sbo, p.layout);
      uint32_t s = 0, ph = 0, acc = 0, aph = 0;
      // GEMM with resident weights (b_bytes == 0): K-block kb of this CTA's N tile sits
      // at bres + kb * bblk_bytes for the whole kernel
      const bool bres_on = p.b_bytes == 0;
      if (bres_on) {
        mbar_wait(bfull, 0);
        tc_fence_after();
      }
      // PAIR: only the leader issues (M = 256 over both CTAs' A, N over both B halves)
      for (int t = tstart; t < total && (!PAIR || rank == 0); t += tstride, ++i) {
        if (lane == 0) PMX_TRACE(9, i);
        mbar_spin(tempty(acc), aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * (uint32_t)p.acc_stride;
        if (lane == 0) PMX_TRACE(2, i);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_spin(full(s), ph);
          tc_fence_after();
          if (elect_one()) {
            if (kb == 0) PMX_TRACE(3, i);
            const uint32_t alo = lo0 + ((a_smem + s * p.a_bytes) >> 4);
            const uint32_t blo = lo0 + ((bres_on ? bres + (uint32_t)kb * p.bblk_bytes : b_smem + s * p.b_bytes) >> 4);
            uint32_t dk = d;
            bool first = kb == 0;
            if constexpr (DT == PMX_F32X2) {
              // segments 1, 2 (the lo corrections) go to the second accumulator
              const int cb = kb % p.cblocks;
              if (cb >= p.seg_n) {
                dk = d + (uint32_t)p.lo_col;
                first = kb == p.seg_n;
              }
            }
#pragma unroll
            for (int k = 0; k < ksteps; ++k) {
              const uint64_t ad = ((uint64_t)hi << 32) | (alo + 2u * k);
              const uint64_t bd = ((uint64_t)hi << 32) | (blo + 2u * k);
              if constexpr (PAIR) tc_mma_pair<DT>(dk, ad, bd, idesc, !(first && k == 0));
              else tc_mma<DT>(dk, ad, bd, idesc, !(first && k == 0));
            }
            if constexpr (PAIR) tc_commit_pair(empty(s));
            else tc_commit(empty(s));
          }
          __syncwarp();
          if (++s == (uint32_t)p.stages) s = 0, ph ^= 1;
        }
        if (elect_one()) {
          if constexpr (PAIR) tc_commit_pair(tfull(acc));
          else tc_commit(tfull(acc));
          PMX_TRACE(4, i);
        }
        __syncwarp();
        if (++acc == (uint32_t)p.nacc) acc = 0, aph ^= 1;
      }
    }
  } else {
    // ---------------- epilogue warps: thread = accumulator row (TMEM lane).  The 16
    // warps form `egroups` tile slots (consecutive tiles are drained concurrently by
    // different slots) x 4 / egroups column ranges per tile; a warp owns a contiguous
    // range of up to 4 chunks of 16 accumulator columns and double-buffers its TMEM
    // loads.  Per-channel alpha / bias are staged once in shared memory.
    const int q = warp & 3;         // TMEM lane quarter this warp may access
    const int e = warp >> 2;  // 0..3
    const int egn = p.egroups, colsplit = 4 / egn;
    const int eg = e / colsplit, cg = e - eg * colsplit;
    const int row = q * 32 + lane;
    const int nchunks = p.bn / 16;
    const int cpw = (nchunks + colsplit - 1) / colsplit;
    const int c_begin = cg * cpw, c_end = min(nchunks, c_begin + cpw);
    {
      const int et = threadIdx.x;
      for (int j = et; j < p.out_c; j += 32 * kEpiWarps) {
        s_alpha[j] = p.alpha ? p.alpha[j] : 0.0f;
        s_bias[j] = p.bias[j];
      }
      if constexpr (OUTK == 2) {
        // head weights -> the B operand: 32 rows x 128 B, SW128 (16-byte chunk j of row r
        // at chunk j ^ (r & 7))
        const uint32_t hb = (s_estage + 1023u) & ~1023u;
        const uint32_t s_hw = hb + 4u * 16384u;
        if (et < 32 * 8) {
          const int r = et >> 3, j = et & 7;
          const uint4 wv = *reinterpret_cast<const uint4*>(p.hwc + r * 128 + 16 * j);
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(s_hw + r * 128 + ((j ^ (r & 7)) << 4)),
                       "r"(wv.x), "r"(wv.y), "r"(wv.z), "r"(wv.w)
                       : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * kEpiWarps) : "memory");
    }
    float lo = __int_as_float(0x7f800000), hi = -lo;
    const float qlo = p.relu ? 0.0f : -128.0f;
    // OUTK 1 fast path: consumer parameters in registers, kernel-uniform eligibility
    const double o_scale = outs.o[0].scale;
    const float o_inv = outs.o[0].inv;
    const bool fast = OUTK == 1 && !p.bn_post && !p.keys && (p.n_gemm % 16) == 0;
    // HEADS: wait for the head MMA of the slot's tile `ti`, then its partial sums (and the
    // heads' epilogue in the last stage); every warp of the slot waits (its code stage is
    // rewritten two tiles later), the column-half-0 warps do the memory work
    auto heads_finish = [&](uint32_t ti) {
      if constexpr (OUTK == 2) {
        const uint32_t ilx = ti / (uint32_t)egn, bx = ilx & 1u;
        mbar_wait(smem_u32(&hbar_s[eg * 2 + bx]), (ilx >> 1) & 1u);
        tc_fence_after();
        if (cg != 0) return;
        const uint32_t t = blockIdx.x + ti * gridDim.x;
        const uint32_t mt = fdiv(t, p.fd_nt), nt = t - mt * (uint32_t)p.n_tiles;
        const uint32_t pin = mt * 128u + row;
        const bool ok = pin < (uint32_t)p.m_total;
        const uint32_t tt = fdiv(pin, p.fd_iw);
        const uint32_t ixx = pin - tt * (uint32_t)p.in_w;
        const uint32_t ibb = fdiv(tt, p.fd_ih);
        const uint32_t iyy = tt - ibb * (uint32_t)p.in_h;
        const uint32_t oy = iyy * (uint32_t)p.stride + (nt >> p.st_shift);
        const uint32_t ox = ixx * (uint32_t)p.stride + (nt & (uint32_t)(p.stride - 1));
        const uint32_t pm = (1u << p.pshift) - 1u;
        const uint32_t ppix =
            ((((oy & pm) << p.pshift | (ox & pm)) * (uint32_t)p.part_b + ibb) * ((uint32_t)p.out_h >> p.pshift) +
             (oy >> p.pshift)) * ((uint32_t)p.out_w >> p.pshift) + (ox >> p.pshift);
        int4 o4[5];
        int4* pp = reinterpret_cast<int4*>(p.hpart + (size_t)ppix * 20u);
        if (ok && p.hstage_mode != 0) {
#pragma unroll
          for (int u = 0; u < 5; ++u) o4[u] = pp[u];
        }
        const uint32_t hcol = tmem + p.hcol0 + 32u * ((uint32_t)eg * 2u + bx) + ((uint32_t)(q * 32) << 16);
        uint32_t h0[16], h1[16];
        tmem_ld16_issue(hcol, h0);
        tmem_ld16_issue(hcol + 16u, h1);
        tmem_ld_wait(h0);
        tmem_ld_wait(h1);
        tc_fence_before();
        if (!ok) return;
        int hs[20];
#pragma unroll
        for (int n = 0; n < 16; ++n) hs[n] = (int)h0[n];
#pragma unroll
        for (int n = 16; n < 20; ++n) hs[n] = (int)h1[n - 16];
        if (p.hstage_mode != 0) {
#pragma unroll
          for (int u = 0; u < 5; ++u) {
            hs[4 * u] += o4[u].x;
            hs[4 * u + 1] += o4[u].y;
            hs[4 * u + 2] += o4[u].z;
            hs[4 * u + 3] += o4[u].w;
          }
        }
        if (p.hstage_mode != 2) {
#pragma unroll
          for (int u = 0; u < 5; ++u) pp[u] = make_int4(hs[4 * u], hs[4 * u + 1], hs[4 * u + 2], hs[4 * u + 3]);
        } else {
          // the heads' epilogue: f32(acc) * alpha + bias in one rounding (the fused-heads
          // kernel's formula, so the result is bit-identical)
          const uint32_t opix = (ibb * (uint32_t)p.out_h + oy) * (uint32_t)p.out_w + ox;
          float* ho = p.hout + (size_t)opix * (uint32_t)p.hcs;
#pragma unroll
          for (int n = 0; n < 20; ++n)
            if (n < p.n_heads) ho[n] = __fmaf_rn((float)hs[n], __ldg(p.halpha + n), __ldg(p.hbias + n));
        }
      }
    };
    uint32_t i_last = 0xffffffffu;
    auto release_acc = [&](uint32_t a) {
      if constexpr (PAIR) mbar_arrive_leader(tempty(a));
      else mbar_arrive(tempty(a));
    };
    for (uint32_t i = (uint32_t)eg;; i += (uint32_t)egn) {
      const uint32_t t = (uint32_t)tstart + i * (uint32_t)tstride;
      if (t >= (uint32_t)total) break;
      i_last = i;
      const uint32_t acc = i & (uint32_t)(p.nacc - 1), aph = (i >> p.nacc_shift) & 1;
      uint32_t mt, nt;
      tile_of(t, mt, nt);
      const int n0 = (int)nt * p.bn;
      bool valid;
      uint32_t pix_in;  // < 2^31 (checked on the host)
      uint32_t iy = 0, ix = 0, ib = 0;
      if (p.mode != MODE_GEMM) {
        const uint32_t tq = fdiv(mt, p.fd_tx), tx = mt - tq * (uint32_t)p.tiles_x;
        const uint32_t tb = fdiv(tq, p.fd_ty), ty = tq - tb * (uint32_t)p.tiles_y;
        const uint32_t oy = ty * p.th + ((uint32_t)row >> p.tw_shift);
        const uint32_t ox = tx * p.tw + ((uint32_t)row & (uint32_t)(p.tw - 1));
        valid = oy < (uint32_t)p.out_h && ox < (uint32_t)p.out_w && mt < (uint32_t)p.m_tiles;
        pix_in = (tb * p.out_h + oy) * p.out_w + ox;
      } else {
        pix_in = mt * 128u + row;
        valid = pix_in < (uint32_t)p.m_total && mt < (uint32_t)p.m_tiles;
        if (p.deconv) {
          const uint32_t tt = fdiv(pix_in, p.fd_iw);
          ix = pix_in - tt * (uint32_t)p.in_w;
          ib = fdiv(tt, p.fd_ih);
          iy = tt - ib * (uint32_t)p.in_h;
        }
      }
      if (warp == 0 && lane == 0) PMX_TRACE(5, i);
      mbar_wait(tfull(acc), aph);
      tc_fence_after();
      if (warp == 0 && lane == 0) PMX_TRACE(6, i);
      if (lane == 0 && i == 6) PMX_TRACE(8, 8 + 2 * warp);  // per-warp view of one steady-state tile
      const uint32_t trow = tmem + acc * (uint32_t)p.acc_stride + ((uint32_t)(q * 32) << 16);
      // deconv: output pixel of tap (0, 0); tap (dy, dx) adds dy * out_w + dx
      const uint32_t pbase = (ib * p.out_h + iy * p.stride) * p.out_w + ix * p.stride;
      if constexpr (OUTK == 2) {
        // ---- deconv + heads: one tile = one tap (bn = Cout = 128) of 128 input pixels.
        // Software-pipelined per tile slot: the codes of tile i go to code stage (i & 1) and
        // its head MMA to head accumulator (i & 1); the head results of the slot's previous
        // tile are finished while that MMA runs
        const uint32_t il = i / (uint32_t)egn, buf = il & 1u;
        const uint32_t hb = (s_estage + 1023u) & ~1023u;
        const uint32_t st = hb + ((uint32_t)eg * 2u + buf) * 16384u, s_hw = hb + 4u * 16384u;
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
          uint32_t v[16];
          acc_ld16<DT>(trow + 16 * (c_begin + k), p.lo_col, v);
          const int cobase = 16 * (c_begin + k);
          float y[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float t;
            if constexpr (DT == PMX_I8) t = __fmaf_rn((float)(int)v[j], s_alpha[cobase + j], s_bias[cobase + j]);
            else t = __fadd_rn(__uint_as_float(v[j]), s_bias[cobase + j]);
            y[j] = p.relu ? fmaxf(t, 0.f) : t;
          }
          uint4 code = valid ? quant16_sel<false>(y, p.hscale, p.hinv) : make_uint4(0, 0, 0, 0);
          const uint32_t jj = (uint32_t)(c_begin + k);  // 16-byte chunk of the 128-byte row
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(st + (uint32_t)row * 128u +
                                                                         ((jj ^ ((uint32_t)row & 7u)) << 4)),
                       "r"(code.x), "r"(code.y), "r"(code.z), "r"(code.w)
                       : "memory");
        }
        // main accumulator drained: release it to the MMA warp
        tc_fence_before();
        __syncwarp();
        if (lane == 0) release_acc(acc);
        // codes -> async proxy, the slot's 8 warps meet, one thread issues the head MMA
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync %0, 256;" ::"r"(2 + eg) : "memory");
        if (cg == 0 && q == 0) {
          tc_fence_after();
          if (elect_one()) {
            const uint32_t ahi = (uint32_t)(sdesc(0, 1024u, 2u) >> 32);
            const uint32_t hcol = tmem + p.hcol0 + 32u * ((uint32_t)eg * 2u + buf);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = ((uint64_t)ahi << 32) | (uint32_t)sdesc(st + 32u * k, 1024u, 2u);
              const uint64_t bd = ((uint64_t)ahi << 32) | (uint32_t)sdesc(s_hw + 32u * k, 1024u, 2u);
              tc_mma<PMX_I8>(hcol, ad, bd, p.hidesc, k != 0);
            }
            tc_commit(smem_u32(&hbar_s[eg * 2 + buf]));
          }
          __syncwarp();
        }
        if (il > 0) heads_finish(i - (uint32_t)egn);
        continue;
      }
      if constexpr (OUTK == 0) {
        if (p.estage2) {
          // int8 consumer and f16 consumer (no dynamic indexing of the parameter struct)
          const bool i8first = outs.o[0].dtype == PMX_I8;
          int8_t* const p8 = reinterpret_cast<int8_t*>(i8first ? outs.o[0].ptr : outs.o[1].ptr) +
                             (i8first ? outs.o[0].c_offset : outs.o[1].c_offset);
          const uint32_t cs8 = (uint32_t)(i8first ? outs.o[0].c_stride : outs.o[1].c_stride);
          const double sc8 = i8first ? outs.o[0].scale : outs.o[1].scale;
          const float inv8 = i8first ? outs.o[0].inv : outs.o[1].inv;
          __half* const ph = reinterpret_cast<__half*>(i8first ? outs.o[1].ptr : outs.o[0].ptr) +
                             (i8first ? outs.o[1].c_offset : outs.o[0].c_offset);
          const uint32_t csh = (uint32_t)(i8first ? outs.o[1].c_stride : outs.o[0].c_stride);
          const int nbase0 = n0 + 16 * c_begin;
          const bool live = nbase0 < p.n_gemm;  // warp-uniform (n_gemm % 64 == 0)
          // y = epilogue of chunk k of this row; int8 codes stored directly
          auto chunk = [&](int k, const uint32_t (&v)[16], float (&y)[16]) {
            const int cobase = nbase0 + 16 * k;
            const float4* b4p = reinterpret_cast<const float4*>(s_bias + cobase);
            const float4* a4p = reinterpret_cast<const float4*>(s_alpha + cobase);
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
              const float4 b4 = b4p[j4];
              float2 r0, r1;
              if constexpr (DT == PMX_I8) {
                const float4 a4 = a4p[j4];
                r0 = __ffma2_rn(make_float2((float)(int)v[4 * j4], (float)(int)v[4 * j4 + 1]),
                                make_float2(a4.x, a4.y), make_float2(b4.x, b4.y));
                r1 = __ffma2_rn(make_float2((float)(int)v[4 * j4 + 2], (float)(int)v[4 * j4 + 3]),
                                make_float2(a4.z, a4.w), make_float2(b4.z, b4.w));
              } else {
                r0 = __fadd2_rn(make_float2(__uint_as_float(v[4 * j4]), __uint_as_float(v[4 * j4 + 1])),
                                make_float2(b4.x, b4.y));
                r1 = __fadd2_rn(make_float2(__uint_as_float(v[4 * j4 + 2]), __uint_as_float(v[4 * j4 + 3])),
                                make_float2(b4.z, b4.w));
              }
              y[4 * j4] = r0.x;
              y[4 * j4 + 1] = r0.y;
              y[4 * j4 + 2] = r1.x;
              y[4 * j4 + 3] = r1.y;
            }
            if (p.relu) {
#pragma unroll
              for (int j = 0; j < 16; ++j) y[j] = fmaxf(y[j], 0.f);
            }
            // clamp-free fast quantizer (y is already ReLU'd when relu is set); ties,
            // saturation and NaN take the exact path
            uint4 code8;
            code8 = quant16_sel<false>(y, sc8, inv8);
            *reinterpret_cast<uint4*>(p8 + (size_t)pix_in * cs8 + cobase) = code8;
          };
          auto sts_f16 = [&](uint32_t a0, uint32_t a1, const float (&y)[16]) {
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a0), "r"(f16x2_sat(y[0], y[1])),
                         "r"(f16x2_sat(y[2], y[3])), "r"(f16x2_sat(y[4], y[5])), "r"(f16x2_sat(y[6], y[7]))
                         : "memory");
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a1), "r"(f16x2_sat(y[8], y[9])),
                         "r"(f16x2_sat(y[10], y[11])), "r"(f16x2_sat(y[12], y[13])), "r"(f16x2_sat(y[14], y[15]))
                         : "memory");
          };
          if (p.estage2 == 2) {
            // small staging (1 KB per warp): each chunk's 32 bytes per row go out right away
            // as 16 rows x 32 bytes (full sectors) per store instruction
            const uint32_t wstage = s_estage + (uint32_t)warp * 1024u;
            const uint32_t sw = ((uint32_t)lane >> 2) & 1u;  // 16-byte slot swizzle (row / 4)
#pragma unroll 1
            for (int k = 0; k < 4; ++k) {
              uint32_t v[16];
              acc_ld16<DT>(trow + 16 * (c_begin + k), p.lo_col, v);
              if (valid && live) {
                float y[16];
                chunk(k, v, y);
                sts_f16(wstage + (uint32_t)lane * 32u + (sw << 4), wstage + (uint32_t)lane * 32u + ((1u ^ sw) << 4), y);
              }
              __syncwarp();
              {
                const uint32_t mp = (valid && live) ? pix_in : 0xffffffffu;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                  const int r = 16 * j + (lane >> 1);
                  const uint32_t sl = (uint32_t)lane & 1u;
                  const uint32_t rp = __shfl_sync(0xffffffffu, mp, r);
                  uint4 w;
                  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                               : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                               : "r"(wstage + (uint32_t)r * 32u + ((sl ^ (((uint32_t)r >> 2) & 1u)) << 4))
                               : "memory");
                  if (rp != 0xffffffffu)
                    *reinterpret_cast<uint4*>(ph + (size_t)rp * csh + nbase0 + 16 * k + 8 * sl) = w;
                }
              }
              __syncwarp();
            }
          } else {
            // 4 KB per warp: the warp's 64 channels of f16 (128 bytes per row), slots
            // (2k, 2k + 1) XOR-swizzled by row % 8; then 4 rows x 128 bytes per store
            const uint32_t wstage = s_estage + (uint32_t)warp * 4096u;
            const uint32_t rb = wstage + (uint32_t)lane * 128u, sw = (uint32_t)lane & 7u;
#pragma unroll 1
            for (int k = 0; k < 4; ++k) {
              uint32_t v[16];
              acc_ld16<DT>(trow + 16 * (c_begin + k), p.lo_col, v);
              if (!valid || !live) continue;
              float y[16];
              chunk(k, v, y);
              sts_f16(rb + (((2u * k) ^ sw) << 4), rb + (((2u * k + 1u) ^ sw) << 4), y);
            }
            __syncwarp();
            {
              const uint32_t mp = (valid && live) ? pix_in : 0xffffffffu;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int r = 4 * j + (lane >> 3);
                const uint32_t sl = (uint32_t)lane & 7u;
                const uint32_t rp = __shfl_sync(0xffffffffu, mp, r);
                uint4 w;
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                             : "r"(wstage + (uint32_t)r * 128u + ((sl ^ ((uint32_t)r & 7u)) << 4))
                             : "memory");
                if (rp != 0xffffffffu) *reinterpret_cast<uint4*>(ph + (size_t)rp * csh + nbase0 + 8 * sl) = w;
              }
            }
            __syncwarp();
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) release_acc(acc);
          continue;
        }
      }
      if constexpr (OUTK == 1) {
        if (fast && p.estage) {
          // this warp's 4 chunks = 64 consecutive output channels of its 32 rows: stage
          // the codes (row-major, 16-byte slots XOR-swizzled by row / 2: conflict-free),
          // then 4 store instructions of 8 rows x 64 bytes each
          const uint32_t wstage = s_estage + (uint32_t)warp * 2048u;
          const int nbase0 = n0 + 16 * c_begin;
          const bool live = nbase0 < p.n_gemm;  // warp-uniform (n_gemm % 64 == 0)
          int cob0 = nbase0;
          uint32_t mypix = pix_in;
          if (p.deconv) {
            const int tap = nbase0 >> p.oc_shift;
            cob0 = nbase0 & (p.out_c - 1);
            mypix = pbase + (uint32_t)(tap >> p.st_shift) * (uint32_t)p.out_w + (uint32_t)(tap & (p.stride - 1));
          }
#pragma unroll 1
          for (int k = 0; k < 4; ++k) {
            uint32_t v[16];
            acc_ld16<DT>(trow + 16 * (c_begin + k), p.lo_col, v);
            if (!valid || !live) continue;
#if defined(PMX_ABLATE) && PMX_ABLATE == 1
            continue;
#endif
            const int cobase = cob0 + 16 * k;
#if defined(PMX_ABLATE) && PMX_ABLATE == 3
            {
              const uint32_t sa3 = wstage + (uint32_t)lane * 64u + (((uint32_t)k ^ (((uint32_t)lane >> 1) & 3u)) << 4);
              asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sa3), "r"(v[0]), "r"(v[5]), "r"(v[10]),
                           "r"(v[15])
                           : "memory");
              continue;
            }
#endif
            float y[16];
            const float4* b4p = reinterpret_cast<const float4*>(s_bias + cobase);
            const float4* a4p = reinterpret_cast<const float4*>(s_alpha + cobase);
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
              const float4 b4 = b4p[j4];
              float2 r0, r1;
              if constexpr (DT == PMX_I8) {
                const float4 a4 = a4p[j4];
                r0 = __ffma2_rn(make_float2((float)(int)v[4 * j4], (float)(int)v[4 * j4 + 1]),
                                make_float2(a4.x, a4.y), make_float2(b4.x, b4.y));
                r1 = __ffma2_rn(make_float2((float)(int)v[4 * j4 + 2], (float)(int)v[4 * j4 + 3]),
                                make_float2(a4.z, a4.w), make_float2(b4.z, b4.w));
              } else {
                r0 = __fadd2_rn(make_float2(__uint_as_float(v[4 * j4]), __uint_as_float(v[4 * j4 + 1])),
                                make_float2(b4.x, b4.y));
                r1 = __fadd2_rn(make_float2(__uint_as_float(v[4 * j4 + 2]), __uint_as_float(v[4 * j4 + 3])),
                                make_float2(b4.z, b4.w));
              }
              y[4 * j4] = r0.x;
              y[4 * j4 + 1] = r0.y;
              y[4 * j4 + 2] = r1.x;
              y[4 * j4 + 3] = r1.y;
            }
            const uint4 code = p.relu ? quant16_sel<true>(y, o_scale, o_inv) : quant16_sel<false>(y, o_scale, o_inv);
            const uint32_t sa = wstage + (uint32_t)lane * 64u + (((uint32_t)k ^ (((uint32_t)lane >> 1) & 3u)) << 4);
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sa), "r"(code.x), "r"(code.y), "r"(code.z),
                         "r"(code.w)
                         : "memory");
          }
          __syncwarp();
          {
            // (converged: shuffles unconditional, one shuffle per row -- ~0 marks an
            // invalid row; the output base is re-read from the parameter bank)
            const uint32_t mp = (valid && live) ? mypix : 0xffffffffu;
            int8_t* const obase = reinterpret_cast<int8_t*>(outs.o[0].ptr) + outs.o[0].c_offset + cob0;
            const uint32_t ocs = (uint32_t)outs.o[0].c_stride;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int r = 8 * j + (lane >> 2);
              const uint32_t cc = (uint32_t)lane & 3u;
              const uint32_t rp = __shfl_sync(0xffffffffu, mp, r);
              uint4 w;
              const uint32_t la = wstage + (uint32_t)r * 64u + ((cc ^ (((uint32_t)r >> 1) & 3u)) << 4);
              asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                           : "r"(la)
                           : "memory");
#if defined(PMX_ABLATE) && PMX_ABLATE == 2
              if ((w.x & w.y & w.z & w.w) == 0x7f7f7f7fu)
#endif
              if (rp != 0xffffffffu) *reinterpret_cast<uint4*>(obase + (size_t)rp * ocs + 16 * cc) = w;
            }
          }
          __syncwarp();
          // release this accumulator buffer to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) release_acc(acc);
          continue;
        }
      }
#pragma unroll 1
      for (int c = c_begin; c < c_end; ++c) {
        // 5 warps share one SM sub-partition: 96 registers per thread leave no room
        // to double-buffer the TMEM loads; the other tile slots hide the latency
        uint32_t v[16];
        acc_ld16<DT>(trow + 16 * c, p.lo_col, v);
        const int nbase = n0 + 16 * c;
        if (!valid || nbase >= p.n_gemm) continue;
        // deconv: 16 consecutive GEMM columns share one tap (Cout % 16 == 0)
        uint32_t pix = pix_in;
        int cobase = nbase;
        if (p.deconv) {
          int tap;
          if (p.oc_shift >= 0) {
            tap = nbase >> p.oc_shift;
            cobase = nbase & (p.out_c - 1);
          } else {
            tap = (int)fdiv((uint32_t)nbase, p.fd_oc);
            cobase = nbase - tap * p.out_c;
          }
          const uint32_t ddy = (uint32_t)tap >> p.st_shift, ddx = (uint32_t)tap & (uint32_t)(p.stride - 1);
          pix = pbase + ddy * (uint32_t)p.out_w + ddx;
        }
        if constexpr (OUTK == 1) {
          if (fast) {
            // one aligned int8 consumer, no unfolded BN / observer, full 16-column run
#if defined(PMX_ABLATE) && (PMX_ABLATE == 1 || PMX_ABLATE == 4)
            continue;
#elif defined(PMX_ABLATE) && PMX_ABLATE == 3
            *reinterpret_cast<uint4*>(reinterpret_cast<int8_t*>(outs.o[0].ptr) + outs.o[0].c_offset +
                                      (size_t)pix * (uint32_t)outs.o[0].c_stride + cobase) = make_uint4(v[0], v[5], v[10], v[15]);
            continue;
#endif
            float y[16];
            const float4* b4p = reinterpret_cast<const float4*>(s_bias + cobase);
            const float4* a4p = reinterpret_cast<const float4*>(s_alpha + cobase);
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
              const float4 b4 = b4p[j4];
              float2 r0, r1;
              if constexpr (DT == PMX_I8) {
                const float4 a4 = a4p[j4];
                r0 = __ffma2_rn(make_float2((float)(int)v[4 * j4], (float)(int)v[4 * j4 + 1]),
                                make_float2(a4.x, a4.y), make_float2(b4.x, b4.y));
                r1 = __ffma2_rn(make_float2((float)(int)v[4 * j4 + 2], (float)(int)v[4 * j4 + 3]),
                                make_float2(a4.z, a4.w), make_float2(b4.z, b4.w));
              } else {
                r0 = __fadd2_rn(make_float2(__uint_as_float(v[4 * j4]), __uint_as_float(v[4 * j4 + 1])),
                                make_float2(b4.x, b4.y));
                r1 = __fadd2_rn(make_float2(__uint_as_float(v[4 * j4 + 2]), __uint_as_float(v[4 * j4 + 3])),
                                make_float2(b4.z, b4.w));
              }
              y[4 * j4] = r0.x;
              y[4 * j4 + 1] = r0.y;
              y[4 * j4 + 2] = r1.x;
              y[4 * j4 + 3] = r1.y;
            }
            const uint4 code = p.relu ? quant16_sel<true>(y, o_scale, o_inv) : quant16_sel<false>(y, o_scale, o_inv);
#if defined(PMX_ABLATE) && PMX_ABLATE == 2
            if ((code.x & code.y & code.z & code.w) == 0x7f7f7f7fu)
#endif
            // (output base / stride from the parameter bank at the store: never spilled)
            *reinterpret_cast<uint4*>(reinterpret_cast<int8_t*>(outs.o[0].ptr) + outs.o[0].c_offset +
                                      (size_t)pix * (uint32_t)outs.o[0].c_stride + cobase) = code;
            continue;
          }
        }
        epi_chunk<DT, OUTK>(p, outs, v, pix, nbase, cobase, s_alpha, s_bias, qlo, lo, hi);
      }
      // release this accumulator buffer to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) release_acc(acc);
      if (warp == 0 && lane == 0) PMX_TRACE(7, i);
      if (lane == 0 && i == 6) PMX_TRACE(8, 9 + 2 * warp);
    }
    if constexpr (OUTK == 2) {
      if (i_last != 0xffffffffu) heads_finish(i_last);
    }
    if (p.keys) block_minmax_commit<kThreads>(lo, hi, p.keys);
  }
  tc_fence_before();
  __syncthreads();
  // PAIR: neither CTA leaves (or frees its TMEM) while the leader's MMAs may still read
  // the peer's shared memory or write its accumulators
  if constexpr (PAIR) cluster_sync_all();
  if (threadIdx.x == 0) PMX_TRACE(8, 3);
  PMX_TL_COMMIT();
  if (warp == kMmaWarp) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
  }
}

// ------------------------------------------------------------------ host side

// programmatic dependent launch on the tcgen05 convs (PMX_PDL=0 turns it off for A/B runs)
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("PMX_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

pmx_status get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) return fail(PMX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return PMX_OK;
}

pmx_status encode(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* addr, const cuuint64_t* dims,
                  const cuuint64_t* strides_bytes, const cuuint32_t* box, CUtensorMapSwizzle sw) {
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(m, dt, rank, const_cast<void*>(addr), dims, strides_bytes, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PMX_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return PMX_OK;
}

struct Plan {
  bool ok;
  TcParams p;
  int grid_x, grid_y;
  size_t smem;
};

// Can the tensor-core path run this layer?  (shape / alignment rules)
// warp-transposed epilogue stores (PMX_ESTAGE=0 turns them off for A/B runs)
bool halo_swz_enabled() {
  static const bool on = [] {
    const char* e = getenv("PMX_HALO_SWZ");
    return !(e && e[0] == '0');
  }();
  return on;
}

uint32_t halo_swz_width() { return kHaloW; }  // swizzled halo row width (16 px; 10 measured slower)

bool halo_pair_enabled() {  // PMX_HALO_PAIR=1: 2-CTA pairs in the halo mode (experiment, off)
  static const bool on = [] {
    const char* e = getenv("PMX_HALO_PAIR");
    return e && e[0] == '1';
  }();
  return on;
}

int gemm_res_mode() {  // PMX_GEMM_RES=1: resident weights in the GEMM mode (experiment, measured neutral: off)
  static const int v = [] {
    const char* e = getenv("PMX_GEMM_RES");
    return e ? atoi(e) : 0;
  }();
  return v;
}
bool small_halo_enabled() {  // PMX_SMALL_HALO=0: no halo for N-split / 256-byte layers (A/B runs)
  static const bool on = [] {
    const char* e = getenv("PMX_SMALL_HALO");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool one_slot_enabled() {  // PMX_ONE_SLOT=0: keep the tile slots at one tile per CTA (A/B runs)
  static const bool on = [] {
    const char* e = getenv("PMX_ONE_SLOT");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool pair_enabled() {  // PMX_PAIR=0: no 2-CTA clusters (A/B runs)
  static const bool on = [] {
    const char* e = getenv("PMX_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

int lat_tiles() {
  static const int v = [] {
    const char* e = getenv("PMX_LAT_TILES");
    return e ? atoi(e) : 0;
  }();
  return v;
}

bool estage_enabled() {
  static const bool on = [] {
    const char* e = getenv("PMX_ESTAGE");
    return !(e && e[0] == '0');
  }();
  return on;
}
int estage_min_row() {  // PMX_ESTAGE=2: stage every eligible layer (experiments)
  static const int v = [] {
    const char* e = getenv("PMX_ESTAGE");
    return (e && e[0] == '2') ? 0 : 128;
  }();
  return v;
}

constexpr uint32_t kHeadsSmem = 1024u + 4u * 16384u + 4096u;  // alignment + 2 x 2 code stages + head weights

Plan plan_for(const pmx_conv_desc& d, bool gather = false, bool want_stage = false, int out_row_bytes = 0,
              bool want_stage2 = false, bool heads = false) {
  Plan pl{};
  pl.ok = false;
  if (heads && !(d.kind == PMX_DECONV2D && d.out_c == 128 && (d.in_dtype == PMX_I8 || d.in_dtype == PMX_F16)))
    return pl;
  if (d.in_dtype != PMX_I8 && d.in_dtype != PMX_F16 && d.in_dtype != PMX_F32X2) return pl;
  const bool x3 = d.in_dtype == PMX_F32X2;
  if (x3 && (gather || d.in_c % 32 != 0 || d.in_c_stride % 2 != 0)) return pl;
  const int esz = d.in_dtype == PMX_I8 ? 1 : (x3 ? 4 : 2);
  TcParams& p = pl.p;
  p.deconv = d.kind == PMX_DECONV2D;
  const bool conv3 = d.kind == PMX_CONV2D && d.k_h == 3 && d.k_w == 3 && d.pad_h == 1 && d.pad_w == 1 &&
                     d.stride_h == d.stride_w && (d.stride_h == 1 || d.stride_h == 2);
  const bool conv1 = d.kind == PMX_CONV2D && d.k_h == 1 && d.k_w == 1 && d.stride_h == 1 && d.stride_w == 1 &&
                     d.pad_h == 0 && d.pad_w == 0;
  if (!(conv3 || conv1 || p.deconv)) return pl;
  // K-block = 128 bytes of channels (SW128) or 64 bytes (SW64); 3xTF32 runs 3 * Cin
  // "channels" per tap (the hi / lo / hi segments)
  const int cin_bytes = (x3 ? 3 : 1) * d.in_c * esz;
  int kc_bytes;
  if (cin_bytes % 128 == 0) kc_bytes = 128;
  else if (cin_bytes == 64) kc_bytes = 64;
  else return pl;
  if ((d.in_c_stride * esz) % 16 != 0 || (d.in_c_offset * esz) % 16 != 0) return pl;
  p.kc = kc_bytes / esz;
  p.cblocks = (x3 ? 3 : 1) * d.in_c / p.kc;
  p.seg_n = x3 ? d.in_c / p.kc : 0;
  p.a_off = x3 ? d.in_c_offset : 0;
  p.a_lo = x3 ? d.in_c_stride / 2 : 0;
  p.layout = kc_bytes == 128 ? 2u : 4u;
  p.sbo = 8u * kc_bytes;
  p.batch = d.batch;
  p.in_h = d.in_h;
  p.in_w = d.in_w;
  p.out_h = d.out_h;
  p.out_w = d.out_w;
  p.out_c = d.out_c;
  p.relu = d.relu;
  if (conv3) {
    p.mode = MODE_CONV3;
    p.taps = 9;
    p.stride = d.stride_h;
    if (p.stride == 2 && ((d.in_h & 1) || (d.in_w & 1))) return pl;
    p.n_gemm = d.out_c;
    // output tile: tw * th = 128 pixels (216 -> 27 x 8, 108 -> 27 x 4, 54 -> 27 x 2 columns)
    const int tw = d.out_w >= 128 ? 8 : (d.out_w >= 64 ? 4 : 2);
    p.tw = tw;
    p.th = 128 / tw;
    p.tiles_x = (int)ceil_div(d.out_w, p.tw);
    p.tiles_y = (int)ceil_div(d.out_h, p.th);
    p.m_tiles = d.batch * p.tiles_x * p.tiles_y;
  } else {
    p.mode = MODE_GEMM;
    p.taps = 1;
    p.stride = p.deconv ? d.k_h : 1;
    p.n_gemm = p.deconv ? d.k_h * d.k_w * d.out_c : d.out_c;
    if (p.deconv && (d.out_c % 16 != 0)) return pl;
    p.m_total = (int64_t)d.batch * d.in_h * d.in_w;
    p.m_tiles = (int)ceil_div(p.m_total, 128);
    if (p.deconv && (p.stride & (p.stride - 1))) return pl;  // stride must be a power of two
  }
  // the epilogue indexes pixels in 32 bits
  if ((int64_t)d.batch * d.out_h * d.out_w >= (int64_t)1 << 31 ||
      (int64_t)d.batch * d.in_h * d.in_w >= (int64_t)1 << 31)
    return pl;
  p.oc_shift = (d.out_c & (d.out_c - 1)) == 0 ? __builtin_ctz((unsigned)d.out_c) : -1;
  p.st_shift = __builtin_ctz((unsigned)(p.stride > 0 ? p.stride : 1));
  // N tile: the whole GEMM N up to 256 (the A tile is then read once); TMEM holds two
  int bn = (int)(ceil_div(p.n_gemm, 16) * 16);
  if (bn > 256) bn = 256;
  if (x3 && bn > 128) bn = 128;  // two accumulators (hi, corrections) per buffer
  {
    const char* e = getenv("PMX_DECONV_BN");  // experiment: cap the deconv N tile
    if (e && p.deconv && bn > atoi(e)) bn = atoi(e);
  }
  // small M (batch-1 blocks.2: 27 M tiles): split N while the tile count still fits
  // one wave -- each CTA then streams a quarter of the weights and issues N=64 MMAs
  while (bn > 64 && bn % 32 == 0 && (int64_t)p.m_tiles * ceil_div(p.n_gemm, bn / 2) <= num_sms()) bn /= 2;
  if (heads) bn = 128;  // one tile = one deconv tap = one head MMA of K = 128
  p.bn = bn;
  p.n_tiles = (int)ceil_div(p.n_gemm, bn);
  const int64_t tiles = (int64_t)p.m_tiles * p.n_tiles;
  pl.grid_x = (int)(tiles < num_sms() ? tiles : num_sms());
  pl.grid_y = 1;
  // warp-transposed int8 stores: every epilogue warp owns exactly 4 chunks (64
  // channels) of a tile, groups never straddle a deconv tap
  p.acc_stride = x3 ? 2 * bn : bn;
  p.lo_col = x3 ? bn : 0;
  p.nacc = 2;
  while (!heads && p.nacc < 8 && 2 * p.nacc * p.acc_stride <= 512) p.nacc *= 2;
  p.nacc_shift = __builtin_ctz((unsigned)p.nacc);
  p.egroups = bn <= 64 ? 4 : (bn <= 128 ? 2 : 1);
  if (p.egroups > p.nacc) p.egroups = p.nacc;
  // one tile per CTA (batch-1 layers): every epilogue warp works on that tile instead of
  // one slot's 4 or 8 warps (the other slots would have nothing to drain)
  if (!heads && tiles <= num_sms() && one_slot_enabled()) p.egroups = 1;
  p.hcol0 = (uint32_t)(p.nacc * p.acc_stride);  // HEADS: 2 x 32 columns per tile slot after the accumulators
  if (heads) want_stage = want_stage2 = false;
  // (measured: a win for 128- and 384-byte output rows -- deconvs into the concat,
  // blocks.1.0 -- a loss for the 64-byte rows of block 0, which are MMA-bound)
  p.estage = want_stage && estage_enabled() && out_row_bytes >= estage_min_row() && (bn / 16) == 4 * (4 / p.egroups) &&
             p.n_gemm % 64 == 0 &&
             (!p.deconv || (p.oc_shift >= 0 && d.out_c % 64 == 0));
  p.estage2 = want_stage2 && estage_enabled() && !p.deconv && (bn / 16) == 4 * (4 / p.egroups) &&
              p.n_gemm % 64 == 0;
  auto estage_bytes_of = [&] {
    return p.estage ? (uint32_t)kEpiWarps * 2048u
                    : (p.estage2 == 1 ? (uint32_t)kEpiWarps * 4096u : (p.estage2 == 2 ? (uint32_t)kEpiWarps * 1024u : 0u));
  };
  uint32_t estage_bytes = estage_bytes_of();
  p.a_bytes = 128u * kc_bytes;
  p.b_bytes = (uint32_t)bn * kc_bytes;
  const uint32_t stage = p.a_bytes + p.b_bytes;
  int stages = (int)((200u * 1024u - 8u * (uint32_t)d.out_c - estage_bytes - (heads ? kHeadsSmem : 0u)) /
                     stage);  // one persistent CTA per SM
  if (stages > 12) stages = 12;
  if (stages < 2) stages = 2;
  p.stages = stages;
  p.bres_bytes = 0;
  // few tiles per CTA (small batches): the resident-weight halo kernel loads every tap's
  // weights before its first MMA; the per-K-block ring streams them behind the MMAs
  // instead.  PMX_LAT_TILES = the tiles-per-SM threshold (0: always the halo kernel)
  const bool latency_mode = !gather && (int64_t)p.m_tiles * p.n_tiles <= (int64_t)lat_tiles() * num_sms();
  // at most one tile per CTA (small batches): the halo also serves 256-byte channel rows
  // and N-split layers -- every CTA keeps one N tile's weights resident for all its tiles
  // (grid a multiple of n_tiles) and one halo stage is enough
  const bool one_tile = tiles <= num_sms() && !gather && small_halo_enabled();
  if (conv3 && !x3 && !latency_mode && g_conv_backend_mode != 2 &&
      (cin_bytes == kc_bytes || (one_tile && p.stride == 1 && cin_bytes == 256 && kc_bytes == 128)) &&
      (p.n_tiles == 1 || one_tile) && d.out_w >= 8) {
    // stride 1: one (16 + 2) x (8 + 2) halo; stride 2: four parity planes of
    // (16 + py) x (8 + px) pixels (561 in total) -- see the producer
    // stride 1, 64 / 128 channel bytes: swizzled pixel-major halo 16 x 18 (PMX_HALO_SWZ=0: off)
    // (not for a 128-channel (int8, f16) pair: its larger halo would evict the f16 staging)
    p.hswz = (p.stride == 1 && !gather && (cin_bytes == 64 || cin_bytes == 128) && halo_swz_enabled() &&
              !(p.estage2 && cin_bytes == 128)) ? 1 : 0;
    {
      const char* e = getenv("PMX_HSWZ_BO");
      p.hswz_bo = e ? atoi(e) : 0;  // measured: the swizzle follows the absolute address
    }
    const uint32_t swz_w = halo_swz_width();
    const uint32_t hw = p.hswz ? swz_w : 10, hp = p.stride == 1 ? (p.hswz ? 18u * swz_w : 180u) : 561u;
    const uint32_t halo = hp * (uint32_t)cin_bytes;
    const uint32_t halo_al = (halo + 1023u) & ~1023u;
    // CTA pairs (cta_group::2, M = 256, int8): each CTA keeps half of the N tile's
    // weights resident and reads its halo plus half of B per MMA
    // (measured slower on blocks 0 / 1 -- 79 -> 89 us, 54 -> 61 us -- except the (int8, f16)
    // pair-output layer 1.15; opt-in PMX_HALO_PAIR=1)
    const bool hpair = halo_pair_enabled() && !gather && !heads && d.in_dtype == PMX_I8 && pair_enabled() && !one_tile &&
                       p.n_tiles == 1 && bn % 32 == 0 && tiles >= 2LL * num_sms() && num_sms() >= 2;
    const uint32_t bblk = (uint32_t)(hpair ? bn / 2 : bn) * kc_bytes;
    const uint32_t bres_total = 9u * p.cblocks * bblk;
    // dynamic smem minus alignment, barriers and the alpha / bias copies
    const uint32_t budget0 = 227u * 1024u - 2048u - 8u * (uint32_t)((d.out_c + 3) & ~3) - (gather ? (uint32_t)kGatherSmem : 0u);
    uint32_t budget = budget0 - estage_bytes;
    const uint32_t two_stages = (one_tile ? 1u : 2u) * halo_al;  // (one tile per CTA: one stage)
    if (p.estage2 == 1 && bres_total + two_stages > budget &&
        bres_total + two_stages <= budget0 - (uint32_t)kEpiWarps * 1024u) {
      p.estage2 = 2;  // resident weights + two halo stages fit next to the 1 KB-per-warp staging
      estage_bytes = estage_bytes_of();
      budget = budget0 - estage_bytes;
    }
    if ((p.estage || p.estage2) && bres_total + two_stages > budget && bres_total + two_stages <= budget0) {
      p.estage = p.estage2 = 0;  // resident weights + two halo stages win over the store staging
      estage_bytes = 0;
      budget = budget0;
    }
    if (bres_total + two_stages <= budget) {
      p.mode = MODE_HALO;
      p.tw = 8;
      p.th = 16;
      p.tiles_x = (int)ceil_div(d.out_w, 8);
      p.tiles_y = (int)ceil_div(d.out_h, 16);
      p.m_tiles = d.batch * p.tiles_x * p.tiles_y;
      const int64_t t2 = (int64_t)p.m_tiles * p.n_tiles;
      const int gmax = (num_sms() / p.n_tiles) * p.n_tiles;  // CTA b keeps N tile b % n_tiles
      pl.grid_x = (int)(t2 < gmax ? t2 : gmax);
      if (hpair) {
        p.pair = 1;
        const int64_t pt = (int64_t)((p.m_tiles + 1) / 2);
        const int gm2 = num_sms() & ~1;
        pl.grid_x = (int)(2 * pt < gm2 ? 2 * pt : gm2);
      }
      p.a_bytes = halo_al;
      p.b_bytes = 0;
      int hs = (int)((budget - bres_total) / halo_al);
      p.stages = hs > 6 ? 6 : hs;
      p.halo_tx = halo;
      p.hp = hp;
      p.hw = hw;
      p.cin_bytes = (uint32_t)cin_bytes;
      p.bblk_bytes = bblk;
      p.bres_bytes = bres_total;
    } else {
      p.hswz = 0;
    }
  }
  // GEMM (1x1 convs, deconvs): one N tile's weights for all K resident in shared memory
  // (CTA b keeps N tile b % n_tiles, grid a multiple of n_tiles) and the ring carries
  // only A: the same shared memory then holds about twice the A bytes in flight (the
  // deconvs' producer otherwise waits on stages their weight re-loads keep occupied)
  if (p.mode == MODE_GEMM && !x3 && !heads && gemm_res_mode() != 0 && g_conv_backend_mode != 2) {
    const uint32_t bblk = (uint32_t)bn * kc_bytes;
    const uint32_t bslice = bblk * (uint32_t)p.cblocks;
    const uint32_t budget = 227u * 1024u - 2048u - 8u * (uint32_t)((d.out_c + 3) & ~3) - estage_bytes;
    const int gmax = (num_sms() / p.n_tiles) * p.n_tiles;
    const int sa = bslice < budget ? (int)((budget - bslice) / p.a_bytes) : 0;
    if (gmax >= 1 && sa >= 2 && (sa >= 2 * p.cblocks || sa >= 4 || gemm_res_mode() == 2)) {
      p.b_bytes = 0;
      p.bblk_bytes = bblk;
      p.bres_bytes = bslice;
      p.stages = sa > 16 ? 16 : sa;
      pl.grid_x = (int)(tiles < gmax ? tiles : gmax);
    }
  }
  p.tw_shift = p.tw > 0 ? __builtin_ctz((unsigned)p.tw) : 0;
  p.fd_nt = make_fastdiv((uint32_t)p.n_tiles);
  p.fd_tx = make_fastdiv((uint32_t)(p.tiles_x > 0 ? p.tiles_x : 1));
  p.fd_ty = make_fastdiv((uint32_t)(p.tiles_y > 0 ? p.tiles_y : 1));
  p.fd_iw = make_fastdiv((uint32_t)d.in_w);
  p.fd_ih = make_fastdiv((uint32_t)d.in_h);
  p.fd_oc = make_fastdiv((uint32_t)d.out_c);
  // as many TMEM accumulators as fit (a power of two, 2..8): the MMA warp runs ahead
  // of the epilogue; the epilogue drains up to 4 tiles at once (tile slots)
  const int cols = p.nacc * p.acc_stride + (heads ? 128 : 0);
  p.tmem_cols = cols <= 32 ? 32 : (cols <= 64 ? 64 : (cols <= 128 ? 128 : (cols <= 256 ? 256 : 512)));
  const uint32_t m_enc = 128u >> 4, n_enc = (uint32_t)bn >> 3;
  if (d.in_dtype == PMX_I8)
    p.idesc = (2u << 4) | (1u << 7) | (1u << 10) | (n_enc << 17) | (m_enc << 24);
  else if (x3)  // f32 <- tf32 x tf32
    p.idesc = (1u << 4) | (2u << 7) | (2u << 10) | (n_enc << 17) | (m_enc << 24);
  else
    p.idesc = (1u << 4) | (0u << 7) | (0u << 10) | (n_enc << 17) | (m_enc << 24);
  // CTA pairs for the TMA-ring modes with a wide N tile: each SM then reads its own A and
  // HALF of B from shared memory per MMA (operand bandwidth is what limits these layers)
  // (the halo mode decided its own pairing above)
  if (!gather && !heads && !x3 && p.mode == MODE_CONV3 && bn >= 128 && bn % 32 == 0 && pair_enabled() &&
      (int64_t)p.m_tiles * p.n_tiles >= 2LL * num_sms() && num_sms() >= 2) {
    p.pair = 1;
    p.b_bytes = (uint32_t)(bn / 2) * kc_bytes;
    int st2 = (int)((200u * 1024u - 8u * (uint32_t)d.out_c - estage_bytes) / (p.a_bytes + p.b_bytes));
    p.stages = st2 > 12 ? 12 : (st2 < 2 ? 2 : st2);
    const int64_t pair_tiles = (int64_t)((p.m_tiles + 1) / 2) * p.n_tiles;
    const int gmax = num_sms() & ~1;
    pl.grid_x = (int)(2 * pair_tiles < gmax ? 2 * pair_tiles : gmax);
  }
  if (p.pair) p.idesc = (p.idesc & ~(0x1Fu << 24)) | ((256u >> 4) << 24);  // M = 256 over the pair
  pl.smem = 1024 + (size_t)p.stages * (p.a_bytes + p.b_bytes) + p.bres_bytes + (2 * p.stages + 2 * p.nacc + 1) * 8 + 32 +
            8 * (size_t)((d.out_c + 3) & ~3) + (gather ? kGatherSmem : 0) + (estage_bytes ? 16 + estage_bytes : 0) +
            (heads ? 16 + kHeadsSmem : 0);
  p.hidesc = (2u << 4) | (1u << 7) | (1u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);  // s32 <- s8 x s8, N 32
  // experiment (PMX_GRID_DIV=d): at small tile counts use num_sms / d persistent CTAs, so
  // the next layer's CTAs find free SMs and run their prologue under this layer
  {
    static const int div = [] {
      const char* e = getenv("PMX_GRID_DIV");
      return e ? atoi(e) : 1;
    }();
    const int64_t tl = (int64_t)p.m_tiles * p.n_tiles;
    if (div > 1 && !gather && !p.pair && tl <= 4LL * num_sms() && pl.grid_x > num_sms() / div) pl.grid_x = num_sms() / div;
  }
  pl.ok = true;
  return pl;
}

pmx_status build_maps(const pmx_conv_desc& d, const Plan& pl, const void* x, const void* w, TcMaps* maps) {
  const TcParams& p = pl.p;
  const bool x3 = d.in_dtype == PMX_F32X2;
  const int esz = d.in_dtype == PMX_I8 ? 1 : (x3 ? 4 : 2);
  const CUtensorMapDataType dt = d.in_dtype == PMX_I8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : (x3 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  const CUtensorMapSwizzle sw = p.layout == 2u ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  // 3xTF32: the A map spans the whole pixel (both planes); the producer's channel
  // coordinate carries the offsets
  const char* xb = static_cast<const char*>(x) + (x3 ? 0 : (size_t)d.in_c_offset * esz);
  const cuuint64_t a_ch = x3 ? (cuuint64_t)d.in_c_stride : (cuuint64_t)d.in_c;
  const cuuint64_t cs = (cuuint64_t)d.in_c_stride * esz;
  pmx_status st;
  if (x == nullptr) {
    // GATHER: the A operand is built in shared memory by the producer warps
  } else if (p.mode == MODE_HALO && p.stride == 2) {
    // parity plane (py, px) of the input: x[2i + py, 2j + px] -> plane[i, j];
    // [channel group][plane pixel][16 bytes], box (16 + py) x (8 + px)
    const cuuint32_t cpg = 16 / esz;
    for (int q = 0; q < 4; ++q) {
      const int py = q >> 1, px = q & 1;
      cuuint64_t dims[5] = {cpg, (cuuint64_t)(d.in_w / 2), (cuuint64_t)(d.in_h / 2), (cuuint64_t)(p.cin_bytes / 16),
                            (cuuint64_t)d.batch};
      cuuint64_t str[4] = {2 * cs, 2 * cs * d.in_w, 16, cs * d.in_w * d.in_h};
      cuuint32_t box[5] = {cpg, (cuuint32_t)(8 + px), (cuuint32_t)(16 + py), p.cin_bytes / 16, 1};
      const char* basep = xb + (size_t)(py * d.in_w + px) * cs;
      st = encode(&maps->a[q], dt, 5, basep, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE);
      if (st != PMX_OK) return st;
    }
  } else if (p.mode == MODE_HALO && p.hswz) {
    // pixel-major swizzled halo: dims {channels, W, H, B}, box {channels, 16, 18, 1}
    cuuint64_t dims[4] = {(cuuint64_t)d.in_c, (cuuint64_t)d.in_w, (cuuint64_t)d.in_h, (cuuint64_t)d.batch};
    cuuint64_t str[3] = {cs, cs * d.in_w, cs * d.in_w * d.in_h};
    cuuint32_t box[4] = {(cuuint32_t)d.in_c, p.hw, p.hp / p.hw, 1};
    st = encode(&maps->a[0], dt, 4, xb, dims, str, box,
                p.cin_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
    if (st != PMX_OK) return st;
  } else if (p.mode == MODE_HALO) {
    // [channel group][halo pixel][16 bytes]: dims {16B of channels, W, H, channel groups, B}
    const cuuint32_t cpg = 16 / esz;
    cuuint64_t dims[5] = {cpg, (cuuint64_t)d.in_w, (cuuint64_t)d.in_h, (cuuint64_t)(p.cin_bytes / 16),
                          (cuuint64_t)d.batch};
    cuuint64_t str[4] = {cs, cs * d.in_w, 16, cs * d.in_w * d.in_h};
    cuuint32_t box[5] = {cpg, p.hw, p.hp / p.hw, p.cin_bytes / 16, 1};
    st = encode(&maps->a[0], dt, 5, xb, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE);
    if (st != PMX_OK) return st;
  } else if (p.mode == MODE_CONV3) {
    if (p.stride == 1) {
      cuuint64_t dims[4] = {a_ch, (cuuint64_t)d.in_w, (cuuint64_t)d.in_h, (cuuint64_t)d.batch};
      cuuint64_t str[3] = {cs, cs * d.in_w, cs * d.in_w * d.in_h};
      cuuint32_t box[4] = {(cuuint32_t)p.kc, (cuuint32_t)p.tw, (cuuint32_t)p.th, 1};
      st = encode(&maps->a[0], dt, 4, xb, dims, str, box, sw);
      if (st != PMX_OK) return st;
    } else {
      for (int py = 0; py < 2; ++py)
        for (int px = 0; px < 2; ++px) {
          cuuint64_t dims[4] = {a_ch, (cuuint64_t)(d.in_w / 2), (cuuint64_t)(d.in_h / 2), (cuuint64_t)d.batch};
          cuuint64_t str[3] = {2 * cs, 2 * cs * d.in_w, cs * d.in_w * d.in_h};
          cuuint32_t box[4] = {(cuuint32_t)p.kc, (cuuint32_t)p.tw, (cuuint32_t)p.th, 1};
          const char* basep = xb + (size_t)(py * d.in_w + px) * cs;
          st = encode(&maps->a[py * 2 + px], dt, 4, basep, dims, str, box, sw);
          if (st != PMX_OK) return st;
        }
    }
  } else {
    cuuint64_t dims[2] = {a_ch, (cuuint64_t)p.m_total};
    cuuint64_t str[1] = {cs};
    cuuint32_t box[2] = {(cuuint32_t)p.kc, 128};
    st = encode(&maps->a[0], dt, 2, xb, dims, str, box, sw);
    if (st != PMX_OK) return st;
  }
  const int K = p.taps * p.cblocks * p.kc;  // 3xTF32: taps * 3 * Cin
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)p.n_gemm};
  cuuint64_t str[1] = {(cuuint64_t)K * esz};
  cuuint32_t box[2] = {(cuuint32_t)p.kc, (cuuint32_t)(p.pair ? p.bn / 2 : p.bn)};  // PAIR: half of N per CTA
  return encode(&maps->b, dt, 2, w, dims, str, box, sw);
}

}  // namespace

const char* conv_tc_backend(int dtype, int) {
  if (g_conv_backend_mode == 1) return "simt";  // 2 = tcgen05 without the halo variant (tests)
  return (dtype == PMX_I8 || dtype == PMX_F16 || dtype == PMX_F32X2) ? "tcgen05" : "simt";
}

int conv_tc_supported(const pmx_conv_desc& d) {
  if (g_conv_backend_mode == 1) return 0;
  const Plan pl = plan_for(d);
  return pl.ok ? 1 | (pl.p.pair << 1) | (pl.p.mode << 2) : 0;
}

size_t conv_tc_workspace(const pmx_conv_desc&) { return 0; }

bool conv_tc_gather_ok(const pmx_conv_desc& d) {
  if (g_conv_backend_mode == 1) return false;
  const Plan pl = plan_for(d, true);
  return pl.ok && pl.p.mode == MODE_HALO;
}

pmx_status conv_tc_try(const pmx_conv_desc& d, const void* x, const void* w, const float* alpha, const float* bias,
                       const float* bn_post, const Outs& outs, uint32_t* keys, void*, size_t, cudaStream_t st,
                       bool* launched, const GatherIn* gin) {
  *launched = false;
  const bool gather = gin != nullptr;
  // OUTK 1: the common single int8 consumer with 16-byte aligned pixel rows
  const bool one_i8 = outs.n == 1 && outs.o[0].dtype == PMX_I8 && outs.o[0].c_stride % 16 == 0 &&
                      outs.o[0].c_offset % 16 == 0 && (reinterpret_cast<uintptr_t>(outs.o[0].ptr) & 15) == 0;
  // (int8, f16) consumer pair with 16-byte aligned rows: staged f16 stores
  bool pair = outs.n == 2 && !bn_post && !keys && (outs.o[0].dtype == PMX_I8) != (outs.o[1].dtype == PMX_I8);
  for (int i = 0; pair && i < 2; ++i) {
    const int esz = outs.o[i].dtype == PMX_I8 ? 1 : 2;
    pair = (outs.o[i].dtype == PMX_I8 || outs.o[i].dtype == PMX_F16) && (outs.o[i].c_stride * esz) % 16 == 0 &&
           (outs.o[i].c_offset * esz) % 16 == 0 && (reinterpret_cast<uintptr_t>(outs.o[i].ptr) & 15) == 0;
  }
  Plan pl = plan_for(d, gather, one_i8 && !bn_post && !keys, outs.o[0].c_stride, pair);
  if (!pl.ok) return PMX_OK;
  if (gather && pl.p.mode != MODE_HALO) return PMX_OK;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(w) & 15)) return PMX_OK;
  pmx_status s = get_encode();
  if (s != PMX_OK) return s;
  TcMaps maps;
  memset(&maps, 0, sizeof(maps));
  if (gather && gin->pcap > (1 << 20)) return PMX_OK;
  s = build_maps(d, pl, gather ? nullptr : x, w, &maps);
  if (s != PMX_OK) return s;
  pl.p.alpha = alpha;
  pl.p.bias = bias;
  pl.p.bn_post = bn_post;
  pl.p.keys = keys;
  pl.p.trace = g_trace;
  pl.p.tl = g_timeline;
  pl.p.tl_tag = g_timeline ? g_tl_tag++ : 0u;
  if (gather) {
    const int esz = d.in_dtype == PMX_I8 ? 1 : 2;
    pl.p.g_feats = static_cast<const char*>(gin->feats) + (size_t)d.in_c_offset * esz;
    pl.p.g_map = gin->map;
    pl.p.g_pcap = gin->pcap;
    pl.p.g_row_bytes = d.in_c_stride * esz;
  }
  dim3 grid(pl.grid_x, pl.grid_y);
  auto launch = [&](auto kern, int threads) -> pmx_status {
    PMX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (pl.p.pair) {  // 2-CTA clusters
      attr[1].id = cudaLaunchAttributeClusterDimension;
      attr[1].val.clusterDim.x = 2;
      attr[1].val.clusterDim.y = 1;
      attr[1].val.clusterDim.z = 1;
      cfg.numAttrs = 2;
    }
    PMX_CUDA(cudaLaunchKernelEx(&cfg, kern, maps, pl.p, outs));
    return PMX_OK;
  };
  const int kcb = (int)(pl.p.sbo / 8);  // K-block bytes (64 or 128)
  const int cinb = pl.p.mode == MODE_HALO ? (int)pl.p.cin_bytes : 0;
  const int hs = pl.p.mode == MODE_HALO ? pl.p.stride : 0;
#define PMX_TC_LAUNCH(DTV, KB, CB, HSV)                                                                        \
  if (gather)                                                                                                  \
    s = one_i8 ? launch(conv_tc_kernel<DTV, 1, KB, CB, HSV, true>, kThreadsGather)                            \
               : launch(conv_tc_kernel<DTV, 0, KB, CB, HSV, true>, kThreadsGather);                           \
  else                                                                                                         \
    s = one_i8 ? launch(conv_tc_kernel<DTV, 1, KB, CB, HSV, false>, kThreads)                                 \
               : launch(conv_tc_kernel<DTV, 0, KB, CB, HSV, false>, kThreads)
#define PMX_TC_LAUNCH_NG(DTV, KB)                                                                              \
  if (pl.p.pair)                                                                                               \
    s = one_i8 ? launch(conv_tc_kernel<DTV, 1, KB, 0, 0, false, true>, kThreads)                              \
               : launch(conv_tc_kernel<DTV, 0, KB, 0, 0, false, true>, kThreads);                             \
  else                                                                                                         \
    s = one_i8 ? launch(conv_tc_kernel<DTV, 1, KB, 0, 0, false>, kThreads)                                    \
               : launch(conv_tc_kernel<DTV, 0, KB, 0, 0, false>, kThreads)
#define PMX_TC_HPAIR(DTV, KB, CB, HSV)                                                                         \
  s = one_i8 ? launch(conv_tc_kernel<DTV, 1, KB, CB, HSV, false, true>, kThreads)                              \
             : launch(conv_tc_kernel<DTV, 0, KB, CB, HSV, false, true>, kThreads)
#define PMX_TC_SHAPES(DTV)                                          \
  if (cinb == 64 && hs == 1) { PMX_TC_LAUNCH(DTV, 64, 64, 1); }     \
  else if (cinb == 64) { PMX_TC_LAUNCH(DTV, 64, 64, 2); }           \
  else if (cinb == 128 && hs == 1) { PMX_TC_LAUNCH(DTV, 128, 128, 1); } \
  else if (cinb == 128) { PMX_TC_LAUNCH(DTV, 128, 128, 2); }        \
  else if (cinb == 256 && hs == 1) {                                \
    s = one_i8 ? launch(conv_tc_kernel<DTV, 1, 128, 256, 1, false>, kThreads) \
               : launch(conv_tc_kernel<DTV, 0, 128, 256, 1, false>, kThreads); }  \
  else if (kcb == 64) { PMX_TC_LAUNCH_NG(DTV, 64); }                \
  else { PMX_TC_LAUNCH_NG(DTV, 128); }
  if (d.in_dtype == PMX_I8 && pl.p.pair && pl.p.mode == MODE_HALO) {
    if (cinb == 64 && hs == 1) { PMX_TC_HPAIR(PMX_I8, 64, 64, 1); }
    else if (cinb == 64) { PMX_TC_HPAIR(PMX_I8, 64, 64, 2); }
    else if (cinb == 128 && hs == 1) { PMX_TC_HPAIR(PMX_I8, 128, 128, 1); }
    else { PMX_TC_HPAIR(PMX_I8, 128, 128, 2); }
  } else if (d.in_dtype == PMX_I8) {
    PMX_TC_SHAPES(PMX_I8)
  } else if (d.in_dtype == PMX_F32X2) {
    PMX_TC_LAUNCH_NG(PMX_F32X2, 128);  // 3xTF32: TMA per K-block (no halo variants)
  } else {
    PMX_TC_SHAPES(PMX_F16)
  }
#undef PMX_TC_SHAPES
#undef PMX_TC_HPAIR
#undef PMX_TC_LAUNCH
#undef PMX_TC_LAUNCH_NG
  if (s != PMX_OK) return s;
  *launched = true;
  return check_launch(gather ? "pmx_conv_gather(tcgen05)" : "pmx_conv(tcgen05)");
}

bool conv_tc_heads_ok(const pmx_conv_desc& d) {
  if (g_conv_backend_mode == 1) return false;
  return plan_for(d, false, false, 0, false, true).ok;
}

// deconv with the three 1x1 heads fused into its epilogue (OUTK 2): see TcParams::hstage_mode
pmx_status conv_tc_deconv_heads(const pmx_conv_desc& d, const void* x, const void* w, const float* alpha,
                                const float* bias, const pmx_head_fuse& hf, cudaStream_t st) {
  Plan pl = plan_for(d, false, false, 0, false, true);
  if (!pl.ok || g_conv_backend_mode == 1)
    return fail(PMX_ERR_UNSUPPORTED, "pmx_deconv_heads: deconv shape outside the fused tcgen05 kernel");
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(w) & 15) ||
      (reinterpret_cast<uintptr_t>(hf.w_codes) & 15) || (reinterpret_cast<uintptr_t>(hf.partial) & 15))
    return fail(PMX_ERR_INVALID, "pmx_deconv_heads: operands must be 16-byte aligned");
  pmx_status s = get_encode();
  if (s != PMX_OK) return s;
  TcMaps maps;
  memset(&maps, 0, sizeof(maps));
  s = build_maps(d, pl, x, w, &maps);
  if (s != PMX_OK) return s;
  TcParams p = pl.p;
  p.alpha = alpha;
  p.bias = bias;
  p.bn_post = nullptr;
  p.keys = nullptr;
  p.trace = g_trace;
  p.tl = g_timeline;
  p.tl_tag = g_timeline ? g_tl_tag++ : 0u;
  p.hstage_mode = hf.stage;
  p.n_heads = hf.n_heads;
  p.hcs = hf.heads_c_stride;
  p.hwc = hf.w_codes;
  p.hpart = hf.partial;
  p.hout = hf.heads;
  p.halpha = hf.head_alpha;
  p.hbias = hf.head_bias;
  p.hscale = hf.in_scale;
  p.hinv = (float)(1.0 / hf.in_scale);
  p.part_b = d.batch;
  p.pshift = __builtin_ctz((unsigned)hf.part_stride);
  Outs outs{};
  outs.n = 0;
  auto launch = [&](auto kern) -> pmx_status {
    PMX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(pl.grid_x, pl.grid_y);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PMX_CUDA(cudaLaunchKernelEx(&cfg, kern, maps, p, outs));
    return PMX_OK;
  };
  const int kcb = (int)(pl.p.sbo / 8);
  if (d.in_dtype == PMX_I8)
    s = kcb == 64 ? launch(conv_tc_kernel<PMX_I8, 2, 64, 0, 0, false>) : launch(conv_tc_kernel<PMX_I8, 2, 128, 0, 0, false>);
  else
    s = kcb == 64 ? launch(conv_tc_kernel<PMX_F16, 2, 64, 0, 0, false>)
                  : launch(conv_tc_kernel<PMX_F16, 2, 128, 0, 0, false>);
  if (s != PMX_OK) return s;
  return check_launch("pmx_deconv_heads(tcgen05)");
}

}  // namespace pmx

extern "C" void pmx_debug_trace(unsigned long long* buf) { pmx::g_trace = buf; }

extern "C" void pmx_debug_timeline(unsigned long long* buf) {
  pmx::g_timeline = buf;
  pmx::g_tl_tag = 0;
}
