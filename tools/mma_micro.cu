// Microbenchmark: tcgen05.mma issue/execution cost per instruction (one CTA per SM,
// operands in smem, same descriptors every iteration).  nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o mma_micro tools/mma_micro.cu
#include <cstdio>
#include <cstdint>
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

#ifndef RANDOM_FILL
#define RANDOM_FILL 1
#endif
template <int KIND>
__global__ void mma_bench(int n_mma, uint32_t idesc, uint32_t layout, uint32_t sbo, uint32_t lbo, int vary,
                          long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ 0x9e3779b9u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    reinterpret_cast<uint32_t*>(sm)[i] = (RANDOM_FILL) ? (KIND == 1 ? (h & 0x3BFF3BFFu) : h) : 0u;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t step = vary == 1 ? 32u : (vary == 2 ? 16u : (vary == 3 ? 512u : (vary == 5 ? 64u : (vary == 6 ? 128u : 1024u))));
    uint64_t ad[9], bd[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      uint32_t off = vary ? (uint32_t)j * step : 0u;
      if (vary == 7) off = (uint32_t)(((j / 3) * 16 + (j % 3)) * 64 + (j & 1) * 32);
      ad[j] = sdesc(base + off, sbo, layout, lbo);
      bd[j] = sdesc(base + 32768 + (off & ~1023u), sbo, layout, lbo);
    }
    long long t0 = clock64();
    for (int i = 0; i < n_mma; i += 9) {
#pragma unroll
      for (int j = 0; j < 9; ++j) {
      if (KIND == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(ad[j]), "l"(bd[j]), "r"(idesc), "r"(i + j));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(ad[j]), "l"(bd[j]), "r"(idesc), "r"(i + j));
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  const int n = 504;
  cudaFuncSetAttribute(mma_bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(mma_bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  struct Cfg { int lay; uint32_t sbo, lbo; int vary; const char* name; };
  Cfg cfgs[] = {{2, 1024, 16, 0, "SW128 fixed"}, {2, 1024, 16, 1, "SW128 vary+32B"}, {4, 512, 16, 0, "SW64 fixed"},
                {0, 128, 2048, 0, "NONE sbo128"}, {0, 160, 2880, 0, "NONE sbo160 lbo2880"},
                {0, 160, 2880, 2, "NONE sbo160 vary+16B"},
                {4, 512, 16, 3, "SW64 vary+512B"}, {2, 1024, 16, 4, "SW128 vary+1024B"}, {0, 128, 1024, 3, "NONE sbo128 vary+512B"},
                {4, 512, 16, 5, "SW64 vary+64B (row)"}, {4, 1024, 16, 5, "SW64 sbo1024 vary+64B"},
                {2, 1024, 16, 6, "SW128 vary+128B (row)"}, {2, 2048, 16, 6, "SW128 sbo2048 vary+128B"},
                {4, 512, 16, 1, "SW64 vary+32B (K)"}, {4, 1024, 16, 1, "SW64 sbo1024 vary+32B"},
                {4, 1024, 16, 7, "SW64 sbo1024 halo taps"}};
  for (int kind = 0; kind < 1; ++kind)
    for (int N : {64, 128})
      for (const Cfg& c : cfgs) {
        const int lay = c.lay;
        uint32_t idesc = kind == 0 ? ((2u << 4) | (1u << 7) | (1u << 10)) : (1u << 4);
        idesc |= ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
        uint32_t sbo = c.sbo, lbo = c.lbo;
        long long h[2] = {0, 0};
        for (int rep = 0; rep < 2; ++rep) {
          if (kind == 0) mma_bench<0><<<148, 128, 100 * 1024>>>(n, idesc, lay, sbo, lbo, c.vary, d);
          else mma_bench<1><<<148, 128, 100 * 1024>>>(n, idesc, lay, sbo, lbo, c.vary, d);
          cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        }
        cudaError_t e = cudaGetLastError();
        double ideal = 128.0 * N / 256.0;  // cycles per MMA at full rate (K = 32 bytes)
        printf("%s N=%3d %-22s: issue %.1f cyc/mma, complete %.1f cyc/mma (ideal %.0f) %s\n",
               kind == 0 ? "i8 " : "f16", N, c.name, (double)h[0] / n, (double)h[1] / n, ideal,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
