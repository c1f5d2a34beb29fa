// Microbenchmark 2: the exact tcgen05 operand sequences of the conv kernels, one CTA
// per SM, one thread issuing back-to-back MMAs (no TMA / epilogue traffic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_micro2 tools/mma_micro2.cu
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

// MODE 0: halo A (no swizzle, tap offsets) + resident SW64 B (stepping per tap / k)
// MODE 1: halo A + fixed B
// MODE 2: fixed A (SW64) + stepping B
// MODE 3: fixed A + fixed B
// MODE 4: SW64 A stepping by 512 B per tap (3-box layout) + stepping B
// LOAD (warps 1..16 while warp 0 issues): 0 none, 1 tcgen05.ld loop on other TMEM
// columns, 2 shared-memory LDS.128 loop, 3 global STG.128 stream, 4 tcgen05.ld of the
// columns the MMAs accumulate into
template <int MODE, int LOAD>
__global__ void bench(int reps, uint32_t idesc, long long* out, int4* gbuf) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ uint32_t stopflag;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  for (int i = threadIdx.x; i < 150 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) stopflag = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
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
  if (threadIdx.x == 0) {
    uint64_t ad[18], bd[18];
    const uint32_t abase = base, bbase = base + 65536;
#pragma unroll
    for (int tap = 0; tap < 9; ++tap)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int dy = tap / 3 - 1, dx = tap % 3 - 1;
        const uint32_t pix0 = (dy + 1) * 10 + (dx + 1);
        const uint32_t aoff = ((2 * k) * 180 + pix0) * 16;
        if (MODE <= 1) ad[tap * 2 + k] = sdesc(abase + aoff, 160, 0, 2880);
        else if (MODE == 4) ad[tap * 2 + k] = sdesc(abase + (dx + 1) * 9216 + (dy + 1) * 512 + 32 * k, 512, 4, 16);
        else ad[tap * 2 + k] = sdesc(abase, 512, 4, 16);
        if (MODE == 0 || MODE == 2 || MODE == 4) bd[tap * 2 + k] = sdesc(bbase + tap * 4096 + 32 * k, 512, 4, 16);
        else bd[tap * 2 + k] = sdesc(bbase, 512, 4, 16);
      }
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int j = 0; j < 18; ++j)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(
                tmem + (r & 3) * 64),
            "l"(ad[j]), "l"(bd[j]), "r"(idesc), "r"(j));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar)));
    long long t2 = clock64();
    if (blockIdx.x == 0) out[0] = t2 - t0;
    asm volatile("st.volatile.shared.u32 [%0], 1;" ::"r"(smem_u32(&stopflag)));
  } else if (LOAD != 0 && threadIdx.x >= 32) {
    const int w = threadIdx.x >> 5, q = w & 3;
    uint32_t acc = 0;
    volatile uint32_t* stop = &stopflag;
    int it = 0;
    while (true) {
      if ((it & 15) == 0 && *stop == 1) break;
      ++it;
      if (LOAD == 1 || LOAD == 4) {
        uint32_t v[16];
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (LOAD == 1 ? 256u : 0u) + 16u * (it & 15);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
      } else if (LOAD == 2) {
        const uint32_t sa = smem_u32(sm) + 100 * 1024 + ((threadIdx.x * 16 + it * 512) & 32767);
        uint32_t x0, x1, x2, x3;
        asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"(sa));
        acc += x0 + x1 + x2 + x3;
      } else {
        gbuf[((size_t)blockIdx.x * 512 + threadIdx.x + (size_t)(it & 255) * 148 * 512) & ((1u << 24) - 1)] =
            make_int4(it, acc, 0, 0);
      }
    }
    if (acc == 0x12345) out[1] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  const int reps = 200;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  int4* gbuf;
  cudaMalloc(&gbuf, (size_t)16 << 24);
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      kern<<<148, 544, 160 * 1024>>>(reps, idesc, d, gbuf);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    }
    printf("i8 N=64 %-48s: %.1f cyc/mma %s\n", name, (double)h / (reps * 18), cudaGetErrorString(cudaGetLastError()));
  };
  run(bench<0, 0>, "halo A + stepping SW64 B (kernel)");
  run(bench<3, 0>, "fixed A + fixed B");
  run(bench<4, 0>, "3-box SW64 A + stepping B");
  run(bench<0, 1>, "kernel + 16 warps tcgen05.ld other cols");
  run(bench<0, 4>, "kernel + 16 warps tcgen05.ld same cols");
  run(bench<0, 2>, "kernel + 16 warps LDS.128");
  run(bench<0, 3>, "kernel + 16 warps STG.128");
  run(bench<4, 1>, "3-box + 16 warps tcgen05.ld other cols");
  return 0;
}
