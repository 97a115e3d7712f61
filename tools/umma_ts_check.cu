// Correctness check: tcgen05.cp.128x256b (smem -> TMEM) + tcgen05.mma with the A operand in tensor memory against the
// shared-memory-descriptor form and a CPU product. One CTA, A = 128 x 128 bf16 (two 64-element K slabs, 128B swizzle),
// B = 192 x 128 bf16 (same layout), D = A * B^T in fp32.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_ts_check umma_ts_check.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_bf16.h>
#include "../paper_2603_28458_b200/csrc/ptx.cuh"
using namespace hisa_dev;

constexpr int M = 128, N = 192, K = 128;
constexpr uint32_t kSlabA = M * 128, kSlabB = N * 128;  // bytes of one 64-element K slab

__device__ __host__ inline uint32_t sw128_off(uint32_t r, uint32_t k) {  // byte offset of element (r, k), k < 64
  return r * 128 + ((((k * 2) >> 4) ^ (r & 7)) << 4) + ((k * 2) & 15);
}

__global__ void __launch_bounds__(128, 1) check(const __nv_bfloat16* A, const __nv_bfloat16* B, float* Dss, float* Dts) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sA = smem;                 // 2 slabs
  unsigned char* sB = smem + 2 * kSlabA;    // 2 slabs
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sA + (k / 64) * kSlabA + sw128_off(r, k % 64)) = A[i];
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sB + (k / 64) * kSlabB + sw128_off(r, k % 64)) = B[i];
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async();
  if (threadIdx.x < 32) { tmem_alloc(&tmem_slot, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t d_ss = tmem, d_ts = tmem + 192, a_tm = tmem + 448;
  if (threadIdx.x < 32) {
    if (elect_one()) {
      constexpr uint32_t idesc = umma_idesc_bf16(M, N);
      const uint64_t a_desc = umma_smem_desc_sw128(smem_u32(sA));
      const uint64_t b_desc = umma_smem_desc_sw128(smem_u32(sB));
      for (int ks = 0; ks < 8; ++ks) {  // K = 16 per instruction
        const uint64_t ad = a_desc + uint64_t((ks / 4) * (kSlabA >> 4) + 2 * (ks % 4));
        const uint64_t bd = b_desc + uint64_t((ks / 4) * (kSlabB >> 4) + 2 * (ks % 4));
        umma_bf16(d_ss, ad, bd, idesc, ks ? 1u : 0u);
      }
      for (int ks = 0; ks < 8; ++ks) {  // 128 rows x 32 bytes of K per copy = 8 TMEM columns
        const uint64_t ad = a_desc + uint64_t((ks / 4) * (kSlabA >> 4) + 2 * (ks % 4));
        tmem_cp_128x256b(a_tm + 8 * ks, ad);
      }
      for (int ks = 0; ks < 8; ++ks) {
        const uint64_t bd = b_desc + uint64_t((ks / 4) * (kSlabB >> 4) + 2 * (ks % 4));
        umma_bf16_ts(d_ts, a_tm + 8 * ks, bd, idesc, ks ? 1u : 0u);
      }
      umma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t row = threadIdx.x;
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(d_ss + ((warp * 32u) << 16) + c0, v);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) Dss[row * N + c0 + j] = __uint_as_float(v[j]);
    tmem_ld_32x32b_x32(d_ts + ((warp * 32u) << 16) + c0, v);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) Dts[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  std::vector<__nv_bfloat16> hA(M * K), hB(N * K);
  std::vector<float> fA(M * K), fB(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) { hA[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < N * K; ++i) { hB[i] = __float2bfloat16((rand() % 13 - 6) / 4.0f); fB[i] = __bfloat162float(hB[i]); }
  __nv_bfloat16 *dA, *dB; float *dss, *dts;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dss, M * N * 4); cudaMalloc(&dts, M * N * 4);
  cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
  cudaMemset(dss, 0xff, M * N * 4); cudaMemset(dts, 0xff, M * N * 4);
  const size_t smem = 2 * kSlabA + 2 * kSlabB + 1024;
  cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  check<<<1, 128, smem>>>(dA, dB, dss, dts);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("CUDA error: %s\n", cudaGetErrorString(err)); return 1; }
  std::vector<float> hss(M * N), hts(M * N);
  cudaMemcpy(hss.data(), dss, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hts.data(), dts, M * N * 4, cudaMemcpyDeviceToHost);
  int bad_ss = 0, bad_ts = 0;
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < N; ++c) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += double(fA[r * K + k]) * fB[c * K + k];
      if (hss[r * N + c] != float(s)) { if (bad_ss++ < 3) printf("ss mismatch (%d,%d): %g vs %g\n", r, c, hss[r * N + c], s); }
      if (hts[r * N + c] != float(s)) { if (bad_ts++ < 3) printf("ts mismatch (%d,%d): %g vs %g\n", r, c, hts[r * N + c], s); }
    }
  printf("smem-A form: %d mismatches; TMEM-A form (tcgen05.cp + .ts): %d mismatches of %d\n", bad_ss, bad_ts, M * N);
  return bad_ss || bad_ts;
}
