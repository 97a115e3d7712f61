// Microbenchmark: issue rates of the epilogue's candidate instruction mixes (per SM sub-partition) on sm_100a.
//   0 FMNMX only            r = max(x, 0) folded into an FADD-free chain (max chain)
//   1 FFMA (3 registers)    acc += x * w
//   2 FFMA2                 acc2 += x2 * w2
//   3 FFMA |x|              acc += |x| * w
//   4 FMNMX + FFMA2         current epilogue: acc2 += max(x2, 0) * w2          (1.5 instr / element)
//   5 FFMA2 + 2 FFMA|x|     relu(x) = (x + |x|) / 2: acc2 += x2 * w2; acc += |x| * w   (1.5 instr / element, FMA pipe only)
//   6 half / half           elements alternate between mixes 4 and 5
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ void ffma2(float2& acc, float a0, float a1, float b0, float b1) {
  uint64_t av, bv, cv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(av) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bv) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(cv) : "f"(acc.x), "f"(acc.y));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(cv) : "l"(av), "l"(bv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(acc.x), "=f"(acc.y) : "l"(cv));
}

template <int MIX>
__global__ void __launch_bounds__(512, 1) mix_kernel(const float* __restrict__ in, float* out, int iters,
                                                      unsigned long long* cycles) {
  float x[32], w[16];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = in[threadIdx.x * 32 + i];
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = in[4096 + threadIdx.x % 64 + i];
  float2 a[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  float s[4] = {0, 0, 0, 0};
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const int c = (i / 2) & 3;
      const float wx = w[i / 2], wy = w[(i / 2 + 1) & 15];
      if (MIX == 0) {
        s[c] = fmaxf(s[c], x[i]);
        s[(c + 1) & 3] = fmaxf(s[(c + 1) & 3], x[i + 1]);
      } else if (MIX == 1) {
        s[c] = fmaf(x[i], wx, s[c]);
        s[(c + 2) & 3] = fmaf(x[i + 1], wy, s[(c + 2) & 3]);
      } else if (MIX == 2) {
        ffma2(a[c], x[i], x[i + 1], wx, wy);
      } else if (MIX == 3) {
        s[c] = fmaf(fabsf(x[i]), wx, s[c]);
        s[(c + 2) & 3] = fmaf(fabsf(x[i + 1]), wy, s[(c + 2) & 3]);
      } else if (MIX == 4) {
        ffma2(a[c], fmaxf(x[i], 0.f), fmaxf(x[i + 1], 0.f), wx, wy);
      } else if (MIX == 5) {
        ffma2(a[c], x[i], x[i + 1], wx, wy);
        s[c] = fmaf(fabsf(x[i]), wx, s[c]);
        s[(c + 2) & 3] = fmaf(fabsf(x[i + 1]), wy, s[(c + 2) & 3]);
      } else {
        if (i & 2) {
          ffma2(a[c], fmaxf(x[i], 0.f), fmaxf(x[i + 1], 0.f), wx, wy);
        } else {
          ffma2(a[c], x[i], x[i + 1], wx, wy);
          s[c] = fmaf(fabsf(x[i]), wx, s[c]);
          s[(c + 2) & 3] = fmaf(fabsf(x[i + 1]), wy, s[(c + 2) & 3]);
        }
      }
    }
    // perturb the inputs so the loop body cannot be hoisted
    x[0] = __int_as_float(__float_as_int(x[0]) ^ (it << 3)); x[17] = __int_as_float(__float_as_int(x[17]) ^ (it << 4));
  }
  const long long t1 = clock64();
  float r = 0;
  for (int c = 0; c < 4; ++c) r += a[c].x + a[c].y + s[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int MIX>
void run(const char* name, double instr_per_elem, float* d_in, float* d_out, unsigned long long* d_cyc) {
  const int iters = 2000;
  for (int warps : {4, 8, 16}) {
    mix_kernel<MIX><<<148, warps * 32>>>(d_in, d_out, iters, d_cyc);
    mix_kernel<MIX><<<148, warps * 32>>>(d_in, d_out, iters, d_cyc);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("CUDA error\n"); exit(1); }
    unsigned long long h[148];
    cudaMemcpy(h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (auto c : h) mx = c > mx ? c : mx;
    const double elems_per_smsp = double(iters) * 32 * (warps / 4);  // warp-elements (32 lanes each)
    printf("%-22s warps/SMSP=%d  %6.3f cycles per warp-element  (%.2f per warp-instr)\n", name, warps / 4,
           double(mx) / elems_per_smsp, double(mx) / elems_per_smsp / instr_per_elem);
  }
}

int main() {
  float *d_in, *d_out;
  unsigned long long* d_cyc;
  cudaMalloc(&d_in, (1024 * 32 + 8192) * 4);
  cudaMemset(d_in, 0x3c, (1024 * 32 + 8192) * 4);
  cudaMalloc(&d_out, 148 * 1024 * 4);
  cudaMalloc(&d_cyc, 148 * 8);
  run<0>("FMNMX", 1, d_in, d_out, d_cyc);
  run<1>("FFMA", 1, d_in, d_out, d_cyc);
  run<2>("FFMA2", 0.5, d_in, d_out, d_cyc);
  run<3>("FFMA|x|", 1, d_in, d_out, d_cyc);
  run<4>("FMNMX+FFMA2", 1.5, d_in, d_out, d_cyc);
  run<5>("FFMA2+FFMA|x|", 1.5, d_in, d_out, d_cyc);
  run<6>("half/half", 1.5, d_in, d_out, d_cyc);
  return 0;
}
