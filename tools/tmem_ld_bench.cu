// Microbenchmark: TMEM -> register readout rate (tcgen05.ld) per SM as a function of the number of warps.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2603_28458_b200/csrc/ptx.cuh"
using namespace hisa_dev;

#define TMEM_LD32(NAME, SHAPE)                                                                                   \
  __device__ __forceinline__ void NAME(uint32_t taddr, uint32_t (&r)[32]) {                                     \
    asm volatile("tcgen05.ld.sync.aligned." SHAPE ".b32 "                                                       \
                 "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "                      \
                 "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"      \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),      \
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),    \
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),    \
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                        \
                 : "r"(taddr)                                                                                   \
                 : "memory");                                                                                   \
  }
TMEM_LD32(ld_16x128b_x16, "16x128b.x16")
TMEM_LD32(ld_16x64b_x32, "16x64b.x32")

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
    else if (SHAPE == 2) { ld_16x128b_x16(taddr, v); ld_16x128b_x16(taddr + (16u << 16), u); ld_16x128b_x16(taddr + 64, x); ld_16x128b_x16(taddr + 64 + (16u << 16), y); }
    else if (SHAPE == 3) { ld_16x64b_x32(taddr, v); ld_16x64b_x32(taddr + (16u << 16), u); ld_16x64b_x32(taddr + 64, x); ld_16x64b_x32(taddr + 64 + (16u << 16), y); }
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
  printf("%-10s grid=%-4d warps=%-3d  %8.1f cyc/iter  %8.1f B/clk/SM  %7.3f ms\n", SHAPE == 0 ? "32x32b.x32" : SHAPE == 1 ? "16x256b.x8" : SHAPE == 2 ? "16x128b.x16" : "16x64b.x32",
         grid, warps, double(mx) / iters, bytes_per_sm / double(mx), ms);
}

int main() {
  unsigned long long* d_out; cudaMalloc(&d_out, 148 * sizeof(unsigned long long));
  uint32_t* d_sink; cudaMalloc(&d_sink, 4);
  for (int warps : {1, 4, 8, 16, 32}) run<0>(148, warps, d_out, d_sink);
  for (int warps : {1, 4, 8, 16, 32}) run<1>(148, warps, d_out, d_sink);
  for (int warps : {1, 4, 8, 16}) run<2>(148, warps, d_out, d_sink);
  for (int warps : {1, 4, 8, 16}) run<3>(148, warps, d_out, d_sink);
  return 0;
}
