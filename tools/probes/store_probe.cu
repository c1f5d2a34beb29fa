// Store-pattern probe (experiments only): 219 MB of int8 rows written (a) dense,
// (b) as 128-byte slices of 384-byte rows, thread-per-16B coalesced or
// thread-per-pixel (the conv epilogue's pattern).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void coalesced(uint4* dst, long rows, int stride16) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;  // one 16-byte piece
  for (; i < rows * 8; i += (long)gridDim.x * blockDim.x) {
    long r = i >> 3, c = i & 7;
    dst[r * stride16 + c] = make_uint4((uint32_t)i, 1, 2, 3);
  }
}

__global__ void per_pixel(uint4* dst, long rows, int stride16) {
  long r = blockIdx.x * (long)blockDim.x + threadIdx.x;  // one pixel row, 8 stores
  for (; r < rows; r += (long)gridDim.x * blockDim.x) {
#pragma unroll
    for (int c = 0; c < 8; ++c) dst[r * stride16 + c] = make_uint4((uint32_t)r, c, 2, 3);
  }
}

// 8 pixels x 64 B per warp instruction (4 lanes per pixel), two instructions per 128 B
__global__ void seg64(uint4* dst, long rows, int stride16) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  for (; i < rows * 8; i += (long)gridDim.x * blockDim.x) {
    long w = i >> 5, l = i & 31;                       // warp-sized group of 32 pieces
    long grp = w >> 1, half = w & 1;                   // 8 pixels x (2 halves of 64 B)
    long r = grp * 8 + (l >> 2), c = half * 4 + (l & 3);
    if (r < rows) dst[r * stride16 + c] = make_uint4((uint32_t)i, 1, 2, 3);
  }
}

extern "C" float probe(int kind, int stride16, int reps) {
  const long rows = 53568L * 32;
  uint4* d;
  cudaMalloc(&d, rows * stride16 * 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&] {
    if (kind == 0) coalesced<<<148 * 8, 256>>>(d, rows, stride16);
    else if (kind == 1) per_pixel<<<148 * 8, 256>>>(d, rows, stride16);
    else seg64<<<148 * 8, 256>>>(d, rows, stride16);
  };
  for (int i = 0; i < 3; ++i) run();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) run();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(d);
  return ms * 1000.0f / reps;
}
