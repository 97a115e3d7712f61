// Microbenchmark: legacy mma.sync.m16n8k16 (bf16, fp32 accumulate) issue rate per SM on sm_100a, as a function of the
// warps per SM. Decides whether a warp-level MMA formulation of the attention consumer can beat the SIMT kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hmma_rate_bench tools/hmma_rate_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__global__ void hmma_loop(int iters, float* sink) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 11u}, b[2] = {threadIdx.x + 5u, 13u};
  float d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0}, d2[4] = {0, 0, 0, 0}, d3[4] = {0, 0, 0, 0};
  for (int i = 0; i < iters; ++i) {  // four independent accumulator chains per warp
    mma16816(d0, a, b);
    mma16816(d1, a, b);
    mma16816(d2, a, b);
    mma16816(d3, a, b);
  }
  if (d0[0] + d1[1] + d2[2] + d3[3] == 12345.f) sink[0] = 1.f;
}

int main() {
  float* sink;
  cudaMalloc(&sink, 4);
  const int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    hmma_loop<<<148, warps * 32>>>(100, sink);
    cudaEventRecord(e0);
    hmma_loop<<<148, warps * 32>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 148.0 * warps * iters * 4 * (16.0 * 8 * 16 * 2);
    printf("warps/SM %2d: %.3f ms  %.0f TFLOP/s (m16n8k16 bf16)\n", warps, ms, flop / ms / 1e9);
  }
  return cudaGetLastError() != cudaSuccess;
}
