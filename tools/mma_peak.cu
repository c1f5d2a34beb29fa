// Dense tcgen05 MMA peak on this B200 (the roofline denominators bench.py uses for the
// INT8 / FP16 / TF32 conv layers).  One CTA per SM; one elected thread issues
// back-to-back cta_group::1 MMAs, M = 128, N = 256, K = 32 bytes, from SW128 smem
// operands holding random bytes (data toggling matters for power), alternating two
// TMEM accumulators.  "burst" = one ~10 ms launch after warm-up; "sustained" = launches
// back to back for --seconds, rate over the second half.  Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_peak tools/mma_peak.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  // K-major SW128: SBO = 1024 B (8 rows x 128 B), version 1, layout 2
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

template <int KIND>  // 0 = i8, 1 = f16, 2 = tf32
__global__ void __launch_bounds__(128, 1) peak_kernel(int iters, uint32_t idesc, unsigned seed) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  uint32_t* w = reinterpret_cast<uint32_t*>(sm + (base - smem_u32(sm)));
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed ^ (blockIdx.x * 40503u);
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    if (KIND == 1) h &= 0x3BFF3BFFu;  // finite f16 in (-1, 1)
    if (KIND == 2) h = (h & 0x807FFFFFu) | 0x3F000000u;  // f32 in +-[0.5, 1)
    w[i] = h;
  }
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
    // A: 128 rows x 128 B (16 KB), B: 256 rows x 128 B (32 KB); 4 K-steps of 32 B per atom
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ad[k] = sdesc(base + 32u * k);
      bd[k] = sdesc(base + 16384u + 32u * k);
    }
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (uint32_t)(i & 1) * 256u;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (KIND == 0)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, "
              "p;\n\t}" ::"r"(d),
              "l"(ad[k]), "l"(bd[k]), "r"(idesc), "r"(k));
        else if (KIND == 1)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, "
              "p;\n\t}" ::"r"(d),
              "l"(ad[k]), "l"(bd[k]), "r"(idesc), "r"(k));
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, "
              "p;\n\t}" ::"r"(d),
              "l"(ad[k]), "l"(bd[k]), "r"(idesc), "r"(k));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

struct Result {
  double burst, sustained;
};

template <int KIND>
Result measure(int sms, double seconds, int n = 256) {
  const uint32_t m_enc = 128u >> 4, n_enc = (uint32_t)n >> 3;
  uint32_t idesc = (n_enc << 17) | (m_enc << 24);
  if (KIND == 0) idesc |= (2u << 4) | (1u << 7) | (1u << 10);  // s32 <- s8 x s8
  if (KIND == 1) idesc |= (1u << 4);                           // f32 <- f16 x f16
  if (KIND == 2) idesc |= (1u << 4) | (2u << 7) | (2u << 10);  // f32 <- tf32 x tf32
  const size_t smem = 50 * 1024;
  cudaFuncSetAttribute(peak_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // K elements per 32-byte step: i8 32, f16 16, tf32 8
  const double k_el = KIND == 0 ? 32.0 : (KIND == 1 ? 16.0 : 8.0);
  const double ops_per_iter = 4.0 * 2.0 * 128.0 * (double)n * k_el;
  const int iters = 40000;  // ~10 ms at full rate
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  peak_kernel<KIND><<<sms, 128, smem>>>(iters / 10, idesc, 1u);
  cudaDeviceSynchronize();
  double best = 0.0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    peak_kernel<KIND><<<sms, 128, smem>>>(iters, idesc, 7u + r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double rate = ops_per_iter * iters * sms / (ms * 1e-3) / 1e12;
    if (rate > best) best = rate;
  }
  if (seconds <= 0.0) return Result{best, 0.0};  // burst only (--by-n)
  // sustained: back to back for `seconds`, rate over the second half
  const auto t0 = std::chrono::steady_clock::now();
  double ops2 = 0.0, t_half = 0.0;
  bool second = false;
  cudaEvent_t s2;
  cudaEventCreate(&s2);
  for (;;) {
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el >= seconds) break;
    if (!second && el >= seconds / 2) {
      cudaDeviceSynchronize();
      cudaEventRecord(s2);
      second = true;
      t_half = el;
    }
    for (int j = 0; j < 8; ++j) peak_kernel<KIND><<<sms, 128, smem>>>(iters, idesc, 11u + j);
    if (second) ops2 += 8.0 * ops_per_iter * iters * sms;
    cudaDeviceSynchronize();
  }
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms2 = 0.f;
  cudaEventElapsedTime(&ms2, s2, b);
  (void)t_half;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "kernel error: %s\n", cudaGetErrorString(e));
    exit(1);
  }
  return Result{best, ops2 / (ms2 * 1e-3) / 1e12};
}

int main(int argc, char** argv) {
  double seconds = 4.0;
  for (int i = 1; i + 1 < argc; ++i)
    if (!strcmp(argv[i], "--seconds")) seconds = atof(argv[i + 1]);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int i = 1; i < argc; ++i)
    if (!strcmp(argv[i], "--by-n")) {
      // burst rate of one instruction shape per N (the conv layers' N tiles: 64, 128, 256)
      printf("{\"how\": \"tools/mma_peak.cu --by-n: burst (best of 5) back-to-back M=128 K=32B MMAs per N\"");
      for (int n : {64, 128, 256}) {
        const Result a = measure<0>(sms, 0.0, n), b = measure<1>(sms, 0.0, n);
        printf(", \"int8_n%d_tops\": %.1f, \"f16_n%d_tflops\": %.1f", n, a.burst, n, b.burst);
      }
      printf("}\n");
      return 0;
    }
  const Result i8 = measure<0>(sms, seconds);
  const Result f16 = measure<1>(sms, seconds);
  const Result tf32 = measure<2>(sms, seconds);
  printf(
      "{\"how\": \"tools/mma_peak.cu: %d CTAs (1/SM), back-to-back tcgen05.mma cta_group::1 M=128 N=256 K=32B from "
      "SW128 smem (random operands), 2 TMEM accumulators; burst = best of 5 ~10 ms launches, sustained = launches "
      "back to back for %.1f s, second half\", \"sms\": %d, \"int8_tops_burst\": %.1f, \"int8_tops_sustained\": %.1f, "
      "\"f16_tflops_burst\": %.1f, \"f16_tflops_sustained\": %.1f, \"tf32_tflops_burst\": %.1f, "
      "\"tf32_tflops_sustained\": %.1f}\n",
      sms, seconds, sms, i8.burst, i8.sustained, f16.burst, f16.sustained, tf32.burst, tf32.sustained);
  return 0;
}
