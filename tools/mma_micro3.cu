// Microbenchmark 3: per-tile issue structure of the conv MMA warp.  18 MMAs (N=64 i8)
// per "tile"; variants add a tcgen05.commit per tile, the elect/syncwarp structure,
// and a try_wait on an already-completed mbarrier.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t sbo, uint32_t layout, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred)::"memory");
  return pred != 0;
}

template <int V>
__global__ void bench(int tiles, uint32_t idesc, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  for (int i = threadIdx.x; i < 100 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 4; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    const uint32_t abase = base, bbase = base + 65536;
    const uint32_t a_hi = (uint32_t)(sdesc(0, 160, 0, 2880) >> 32), b_hi = (uint32_t)(sdesc(0, 512, 4, 16) >> 32);
    const uint32_t b_lo0 = (uint32_t)sdesc(bbase, 512, 4, 16);
    long long t0 = clock64();
    uint32_t acc = 0;
    for (int t = 0; t < tiles; ++t) {
      if (V >= 3) {  // try_wait on a completed phase (parity 1 of a fresh barrier)
        uint32_t ok;
        do {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&bar[3])) : "memory");
        } while (!ok);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      const bool leader = V >= 2 ? elect_one() : (threadIdx.x == 0);
      if (leader) {
        const uint32_t alo = (abase + (t & 1) * 16384) >> 4;
        const uint32_t d = tmem + acc * 64;
#pragma unroll
        for (int tap = 0; tap < 9; ++tap)
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int dy = tap / 3 - 1, dx = tap % 3 - 1;
            const uint32_t aoff = ((2 * k) * 180 + (dy + 1) * 10 + (dx + 1)) * 16;
            const uint32_t boff = tap * 4096 + 32 * k;
            const uint64_t ad = ((uint64_t)a_hi << 32) | (alo + ((180u << 16) + (aoff >> 4)));
            const uint64_t bd = ((uint64_t)b_hi << 32) | (b_lo0 + (boff >> 4));
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                "l"(ad), "l"(bd), "r"(idesc), "r"(tap | k));
          }
        if (V >= 1) {
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[1])) : "memory");
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[2])) : "memory");
        }
      }
      if (V >= 2) __syncwarp();
      if (++acc == 8) acc = 0;
    }
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[0])));
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar[0])));
      long long t2 = clock64();
      if (blockIdx.x == 0) out[0] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  const int tiles = 100;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      kern<<<148, 128, 110 * 1024>>>(tiles, idesc, d);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    }
    printf("%-44s: %.1f cyc/tile (%.1f /mma) %s\n", name, (double)h / tiles, (double)h / tiles / 18,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(bench<0>, "18 MMAs per tile, thread 0");
  run(bench<1>, "+ 2 commits per tile");
  run(bench<2>, "+ elect / syncwarp (whole warp)");
  run(bench<3>, "+ try_wait on a completed barrier");
  return 0;
}
