// Microbenchmark: L2 -> SM gather rate for the access pattern of the attention consumer (csrc/attend.cu): every warp
// reads whole 256-byte rows of an L2-resident table at random row indices, ROWS rows in flight per warp, and does
// nothing else with them (one XOR per loaded word). This is the ceiling the consumer's gather can be held against.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_gather_bench tools/l2_gather_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

template <int ROWS>
__global__ void __launch_bounds__(32, 16) gather_rows(const uint2* __restrict__ table, const int* __restrict__ idx, int per_warp,
                                                      uint32_t* sink) {
  const int lane = threadIdx.x;
  const int* my = idx + size_t(blockIdx.x) * per_warp;
  uint32_t acc = 0;
  for (int b = 0; b < per_warp; b += ROWS) {
    const int tok = lane < ROWS ? my[b + lane] : 0;
    uint2 v[ROWS];
#pragma unroll
    for (int i = 0; i < ROWS; ++i) v[i] = __ldg(table + size_t(__shfl_sync(0xffffffffu, tok, i)) * 32 + lane);
#pragma unroll
    for (int i = 0; i < ROWS; ++i) acc ^= v[i].x ^ v[i].y;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int ROWS>
float run(const uint2* table, const int* idx, int warps, int per_warp, uint32_t* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  gather_rows<ROWS><<<warps, 32>>>(table, idx, per_warp, sink);
  float best = 1e9f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    gather_rows<ROWS><<<warps, 32>>>(table, idx, per_warp, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  const int L = 65536, warps = 65536, per_warp = 2048;  // the consumer's C3 shape: 64K rows x 2048 picks of 256 B
  uint2* table;
  int* idx;
  uint32_t* sink;
  cudaMalloc(&table, size_t(L) * 256);
  cudaMemset(table, 1, size_t(L) * 256);
  cudaMalloc(&sink, 4);
  std::vector<int> h(size_t(warps) * per_warp);
  uint64_t s = 88172645463325252ull;
  for (auto& v : h) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    v = int(s % L);
  }
  cudaMalloc(&idx, h.size() * 4);
  cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  const double bytes = double(warps) * per_warp * 256;
  const float t8 = run<8>(table, idx, warps, per_warp, sink), t16 = run<16>(table, idx, warps, per_warp, sink),
              t32 = run<32>(table, idx, warps, per_warp, sink);
  printf("gather of %.1f GB in 256-B rows from a %d MiB table, one warp per CTA, 16 CTAs/SM\n", bytes / 1e9, L * 256 >> 20);
  printf("rows in flight per warp  8: %.3f ms  %.0f GB/s\n", t8, bytes / t8 / 1e6);
  printf("rows in flight per warp 16: %.3f ms  %.0f GB/s\n", t16, bytes / t16 / 1e6);
  printf("rows in flight per warp 32: %.3f ms  %.0f GB/s\n", t32, bytes / t32 / 1e6);
  return cudaGetLastError() != cudaSuccess;
}
