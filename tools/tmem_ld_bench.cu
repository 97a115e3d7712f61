// Microbenchmark: TMEM -> register readout rate (tcgen05.ld) per SM as a function of the number of warps.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2603_28458_b200/csrc/ptx.cuh"
using namespace hisa_dev;

template <int SHAPE>  // 0: 32x32b.x32 (4 KB / warp-instr), 1: 16x256b.x8 (4 KB / warp-instr)
__global__ void __launch_bounds__(1024, 1) tmem_ld_rate(int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t tmem_slot;
  if (threadIdx.x < 32) { tmem_alloc(&tmem_slot, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t quarter = warp & 3;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  uint32_t acc2 = 0, acc3 = 0, acc4 = 0;
  for (int it = 0; it < iters; it += 4) {
    uint32_t v[32], u[32], x[32], y[32];
    const uint32_t taddr = tmem + ((quarter * 32u) << 16) + ((warp >> 2) * 128u & 255u);
    if (SHAPE == 0) { tmem_ld_32x32b_x32(taddr, v); tmem_ld_32x32b_x32(taddr + 32, u); tmem_ld_32x32b_x32(taddr + 64, x); tmem_ld_32x32b_x32(taddr + 96, y); }
    else { tmem_ld_16x256b_x8(taddr, v); tmem_ld_16x256b_x8(taddr + (16u << 16), u); tmem_ld_16x256b_x8(taddr + 64, x); tmem_ld_16x256b_x8(taddr + 64 + (16u << 16), y); }
    tmem_ld_wait();
    acc ^= v[0] ^ v[31]; acc2 ^= u[0] ^ u[31]; acc3 ^= x[0] ^ x[31]; acc4 ^= y[0] ^ y[31];
  }
  acc ^= acc2 ^ acc3 ^ acc4;
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 0x12345678u) sink[0] = acc;
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int SHAPE>
void run(int grid, int warps, unsigned long long* d_out, uint32_t* d_sink) {
  const int iters = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    tmem_ld_rate<SHAPE><<<grid, warps * 32>>>(iters, d_out, d_sink);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("CUDA error: %s\n", cudaGetErrorString(err)); exit(1); }
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> h(grid);
  cudaMemcpy(h.data(), d_out, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0; for (auto c : h) mx = c > mx ? c : mx;
  const double bytes_per_sm = double(iters) * warps * 4096.0;
  printf("%-10s grid=%-4d warps=%-3d  %8.1f cyc/iter  %8.1f B/clk/SM  %7.3f ms\n", SHAPE ? "16x256b.x8" : "32x32b.x32",
         grid, warps, double(mx) / iters, bytes_per_sm / double(mx), ms);
}

int main() {
  unsigned long long* d_out; cudaMalloc(&d_out, 148 * sizeof(unsigned long long));
  uint32_t* d_sink; cudaMalloc(&d_sink, 4);
  for (int warps : {1, 4, 8, 16, 32}) run<0>(148, warps, d_out, d_sink);
  for (int warps : {1, 4, 8, 16, 32}) run<1>(148, warps, d_out, d_sink);
  return 0;
}
