// Microbenchmark: issue rate of tcgen05.mma (kind::f16, bf16 -> fp32) on sm_100a in isolation.
// Each CTA streams MMAs (K = 16 each) from resident shared-memory tiles; everything that could cost issue
// slots (descriptors, accumulator choice, commit cadence) is compile-time.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_bench umma_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2603_28458_b200/csrc/ptx.cuh"
using namespace hisa_dev;

// A_TMEM: A operand from tensor memory; N: MMA N; CHAINS: independent accumulators interleaved MMA by MMA
template <int A_TMEM, int N, int CHAINS>
__global__ void __launch_bounds__(128, 1) umma_rate(int outer, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); fence_proxy_async(); }
  if (threadIdx.x < 32) { tmem_alloc(&tmem_slot, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (threadIdx.x < 32) {
    const uint64_t a_desc = umma_smem_desc_sw128(smem_u32(smem));
    const uint64_t b_desc = umma_smem_desc_sw128(smem_u32(smem) + 16384);
    constexpr uint32_t idesc = umma_idesc_bf16(128, N);
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int it = 0; it < outer; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int u = 0; u < 32; ++u) {  // 32 MMAs per commit
          const uint32_t d = tmem + (u % CHAINS) * N;
          if (A_TMEM) umma_bf16_ts(d, tmem + 448 + (u % 4) * 8, b_desc + 2 * (u % 4), idesc, 1);
          else umma_bf16(d, a_desc + 2 * (u % 4), b_desc + 2 * (u % 4), idesc, 1);
        }
        umma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, phase);
      phase ^= 1;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int A_TMEM, int N, int CHAINS>
void run(int grid, unsigned long long* d_out) {
  const int outer = 2000;
  const size_t smem = 16384 + 32768 + 1024;
  auto k = umma_rate<A_TMEM, N, CHAINS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k<<<grid, 128, smem>>>(outer, d_out);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("CUDA error: %s\n", cudaGetErrorString(err)); exit(1); }
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(grid);
  cudaMemcpy(h.data(), d_out, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0; for (auto c : h) mx = c > mx ? c : mx;
  const double mmas = double(outer) * 32;
  const double flops = mmas * 2.0 * 128 * N * 16 * grid;
  printf("%-5s %-5d %-4d %-6d %10.1f %9.3f %10.1f %8.3f\n", A_TMEM ? "tmem" : "smem", grid, N, CHAINS, mx / mmas, ms,
         flops / (ms * 1e-3) / 1e12, mx / (ms * 1e-3) / 1e9);
}

int main() {
  unsigned long long* d_out; cudaMalloc(&d_out, 148 * sizeof(unsigned long long));
  printf("%-5s %-5s %-4s %-6s %10s %9s %10s %8s\n", "A", "grid", "N", "chains", "cyc/MMA", "ms", "TFLOP/s", "GHz");
  run<0, 256, 1>(1, d_out);  run<0, 256, 1>(148, d_out); run<0, 256, 2>(148, d_out);
  run<0, 192, 1>(148, d_out); run<0, 192, 2>(148, d_out);
  run<0, 128, 1>(148, d_out); run<0, 128, 2>(148, d_out); run<0, 128, 4>(148, d_out);
  run<0, 64, 1>(148, d_out);  run<0, 64, 4>(148, d_out);
  run<1, 256, 1>(1, d_out);  run<1, 256, 1>(148, d_out);
  run<1, 192, 1>(148, d_out); run<1, 192, 2>(148, d_out);
  run<1, 128, 1>(148, d_out); run<1, 128, 2>(148, d_out); run<1, 128, 3>(148, d_out);
  run<1, 64, 1>(148, d_out);  run<1, 64, 4>(148, d_out);
  return 0;
}
