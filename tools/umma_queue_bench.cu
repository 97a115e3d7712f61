// Microbenchmark: how far can the issuing thread of tcgen05.mma run ahead of the tensor pipe?
// One warp pushes batches of 4 MMAs (128 x 256 x 16, ~136 cycles each on the pipe), then idles GAP cycles before the
// next batch. While the time per batch stays at 4 x 136 the queued MMAs covered the gap; the GAP at which it starts to
// grow is the slack the MMA warp has for barrier waits between batches.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2603_28458_b200/csrc/ptx.cuh"
using namespace hisa_dev;

__global__ void __launch_bounds__(128, 1) umma_gap(int outer, int gap, int batch, unsigned long long* out) {
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
    constexpr uint32_t idesc = umma_idesc_bf16(128, 256);
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int it = 0; it < outer; ++it) {
      for (int b = 0; b < 16; ++b) {
        if (elect_one()) {
          for (int u = 0; u < batch; ++u) umma_bf16(tmem + (b & 1) * 256, a_desc + 2 * (u % 4), b_desc + 2 * (u % 4), idesc, 1);
        }
        __syncwarp();
        const long long c0 = clock64();
        while (clock64() - c0 < gap) {}
      }
      if (elect_one()) umma_commit(&bar);
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

int main() {
  unsigned long long* d_out; cudaMalloc(&d_out, 148 * sizeof(unsigned long long));
  const size_t smem = 16384 + 32768 + 1024;
  cudaFuncSetAttribute(umma_gap, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int outer = 300;
  for (int batch : {4, 8}) {
    for (int gap : {0, 100, 200, 300, 400, 500, 600, 800, 1000}) {
      umma_gap<<<148, 128, smem>>>(outer, gap, batch, d_out);
      umma_gap<<<148, 128, smem>>>(outer, gap, batch, d_out);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("CUDA error\n"); return 1; }
      std::vector<unsigned long long> h(148);
      cudaMemcpy(h.data(), d_out, 148 * 8, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0; for (auto c : h) mx = c > mx ? c : mx;
      printf("batch=%d gap=%-5d cycles per batch = %8.1f  (pipe time %d)\n", batch, gap, double(mx) / (outer * 16.0), batch * 136);
    }
  }
  return 0;
}
