// Downstream consumer of the indexer: softmax attention restricted to the selected token set, over shared
// key/value latent vectors (reference: proj/core/include/hisa/attention.hpp:48-59, Eq.3).
//
//   u_t = sum_{s in T_t} softmax_s(scale * h_t . c_s) * c_s          softmax normalised over T_t only
//
// One query has one state vector, so this is a gathered matrix-vector product: 2 * |T_t| * d_model MACs against
// |T_t| * d_model gathered elements. It is bound by the L2 -> SM gather (the latent table, 16 MiB at L = 64K and
// d_model = 128 in bf16, stays L2-resident), not by the tensor pipe; the kernel is plain SIMT and organised around
// that gather:
//   * one warp per query row; lane l owns elements [l*EPL, (l+1)*EPL) of the model dimension, so a latent row is one
//     fully coalesced warp load (256 B for d_model = 128 in bf16);
//   * TB rows are loaded back to back and kept in registers (TB x row-slice = 64 fp32 registers): TB independent loads in
//     flight per warp, and each gathered byte crosses L2 -> SM once although it is used twice (logit, then weighted sum);
//   * the TB partial dot products are combined with a transposed butterfly (31 shuffles for 32 rows instead of 160):
//     afterwards lane j holds the logit of row j, so the exponentials are evaluated one per lane;
//   * online softmax across batches (running maximum, rescaled accumulators), fp32 throughout.
// The optional weights output first receives the logits and is normalised by the same lanes at the end.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <algorithm>

#include "kernels.cuh"

namespace hisa_dev {
namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kAttnWarps = 1;  // one warp per CTA: the row index comes from blockIdx, so the compiler knows every loop bound is warp-uniform

template <int WORDS>
__device__ __forceinline__ void load_words(const uint32_t* __restrict__ p, uint32_t (&w)[WORDS]) {
  if constexpr (WORDS % 4 == 0) {
#pragma unroll
    for (int i = 0; i < WORDS / 4; ++i) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + i);
      w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
    }
  } else if constexpr (WORDS == 2) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    w[0] = v.x; w[1] = v.y;
  } else {
    static_assert(WORDS == 1, "unsupported row slice");
    w[0] = __ldg(p);
  }
}

// element e of a lane's row slice, widened to fp32 (bf16 -> fp32 is a 16-bit shift: exact)
template <bool BF16>
__device__ __forceinline__ float elem(const uint32_t* w, int e) {
  if constexpr (BF16) return __uint_as_float((e & 1) ? (w[e >> 1] & 0xFFFF0000u) : (w[e >> 1] << 16));
  else return __uint_as_float(w[e]);
}

// v[i] holds this lane's partial sum for row i; returns the full sum of row (lane / (32 / TB)).
template <int TB>
__device__ __forceinline__ float transposed_reduce(float (&v)[TB], uint32_t lane) {
  int n = TB;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    if (n > 1) {
      n >>= 1;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < TB / 2; ++i) {
        if (i < n) {
          const float send = up ? v[i] : v[i + n];
          const float keep = up ? v[i + n] : v[i];
          v[i] = keep + __shfl_xor_sync(kFull, send, o);
        }
      }
    } else {
      v[0] += __shfl_xor_sync(kFull, v[0], o);
    }
  }
  return v[0];
}

// EPL elements of the (padded) model dimension per lane, TB rows per batch.
template <int EPL, int TB, bool BF16>
__global__ void __launch_bounds__(kAttnWarps * 32, 16) sparse_attend_kernel(const AttendArgs a) {
  constexpr int WORDS = BF16 ? EPL / 2 : EPL;
  constexpr int LPR = 32 / TB;  // lanes that end up holding the same row's logit
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w = blockIdx.x * kAttnWarps + (threadIdx.x >> 5);
  if (w >= a.num_rows) return;
  // dense mode: rows differ in length by orders of magnitude; hand out the long ones first
  const uint32_t row = a.idx ? w : a.num_rows - 1 - w;
  const uint32_t t = a.pos[row];
  const bool bad_pos = t >= a.seq_len;  // AttentionInputs: every position < L (attention.hpp:19-20)
  const uint32_t n = a.idx ? (a.count ? min(a.count[row], uint32_t(a.idx_stride)) : uint32_t(a.idx_stride))
                           : (bad_pos ? 0u : t + 1u);
  const int32_t* idx = a.idx ? a.idx + uint64_t(row) * a.idx_stride : nullptr;
  float* wout = a.weights ? a.weights + uint64_t(row) * a.weights_stride : nullptr;
  const uint32_t* lat = static_cast<const uint32_t*>(a.latents);
  const uint32_t row_words = a.dm_pad / (BF16 ? 2 : 1);

  float q[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) q[e] = a.queries[uint64_t(row) * a.dm_pad + lane * EPL + e];

  float acc[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) acc[e] = 0.f;
  float m = -CUDART_INF_F, l = 0.f;
  uint32_t flags = bad_pos ? 4u : 0u;
  const float scale2 = a.scale * 1.4426950408889634f;  // logits in base 2

  for (uint32_t b0 = 0; b0 < n; b0 += TB) {
    int32_t my_tok = -1;
    if (lane < TB && b0 + lane < n) my_tok = idx ? idx[b0 + lane] : int32_t(b0 + lane);
    if (my_tok >= 0 && (uint32_t(my_tok) > t || uint32_t(my_tok) >= a.seq_len)) {
      flags |= 2u;  // CausalViolation (attention.hpp:52)
      my_tok = -1;
    }
    uint32_t raw[TB][WORDS];
#pragma unroll
    for (int i = 0; i < TB; ++i) {
      const int32_t tok = __shfl_sync(kFull, my_tok, i);
      if (tok >= 0) {
        load_words<WORDS>(lat + uint64_t(tok) * row_words + lane * WORDS, raw[i]);
      } else {
#pragma unroll
        for (int x = 0; x < WORDS; ++x) raw[i][x] = 0u;
      }
    }
    float part[TB];
#pragma unroll
    for (int i = 0; i < TB; ++i) {
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < EPL; ++e) s = fmaf(q[e], elem<BF16>(raw[i], e), s);
      part[i] = s;
    }
    const float dot = transposed_reduce<TB>(part, lane);
    const uint32_t mine = lane / LPR;  // row of the batch whose logit this lane holds
    const bool valid = __shfl_sync(kFull, my_tok, mine) >= 0;
    const float x = valid ? dot * scale2 : -CUDART_INF_F;
    if (wout && (lane % LPR) == 0 && b0 + mine < n) wout[b0 + mine] = x;
    float bm = x;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) bm = fmaxf(bm, __shfl_xor_sync(kFull, bm, o));
    const float m_new = fmaxf(m, bm);
    float corr = 1.f, p = 0.f;
    if (m_new > -CUDART_INF_F) {
      corr = exp2f(m - m_new);  // first batch: exp2(-inf) = 0
      p = valid ? exp2f(x - m_new) : 0.f;
    }
    m = m_new;
    l = l * corr + p;
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[e] *= corr;
#pragma unroll
    for (int i = 0; i < TB; ++i) {
      const float pi = __shfl_sync(kFull, p, i * LPR);
#pragma unroll
      for (int e = 0; e < EPL; ++e) acc[e] = fmaf(pi, elem<BF16>(raw[i], e), acc[e]);
    }
  }
  // every row's weight was counted by its LPR lanes
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) l += __shfl_xor_sync(kFull, l, o);
  l *= 1.f / float(LPR);
  if (!(l > 0.f)) flags |= 1u;  // EmptySelection (attention.hpp:51): nothing to normalise over
  const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const uint32_t c = lane * EPL + e;
    if (c < a.d_model) a.out[uint64_t(row) * a.d_model + c] = acc[e] * inv;
  }
  if (wout) {
    // the lane that stored a logit turns it into the weight (same thread: no fence needed)
    for (uint32_t b0 = 0; b0 < a.weights_stride; b0 += TB) {
      const uint32_t j = b0 + lane / LPR;
      if ((lane % LPR) == 0 && j < a.weights_stride) wout[j] = (j < n && l > 0.f) ? exp2f(wout[j] - m) * inv : 0.f;
    }
  }
  const uint32_t report = lane == 0 ? flags : (flags & 2u);  // bits 0 and 2 are warp-uniform
  if (report) atomicOr(a.flag, report);
}

// src [rows, dim] (f32 | bf16) -> dst [rows, dim_pad] (f32 | bf16), zero filled beyond dim
template <typename Src, typename Dst>
__global__ void pad_rows_kernel(const Src* __restrict__ src, uint64_t rows, uint32_t dim, uint32_t dim_pad,
                                Dst* __restrict__ dst) {
  const uint64_t total = rows * dim_pad;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / dim_pad;
    const uint32_t c = uint32_t(i - r * dim_pad);
    float v = 0.f;
    if (c < dim) {
      if constexpr (sizeof(Src) == 2) v = __bfloat162float(src[r * dim + c]);
      else v = src[r * dim + c];
    }
    if constexpr (sizeof(Dst) == 2) dst[i] = __float2bfloat16_rn(v);
    else dst[i] = v;
  }
}

template <int EPL, bool BF16>
int launch_attend_epl(const AttendArgs& a, cudaStream_t stream) {
  // TB x EPL = 64 fp32 values per lane (the compiler widens bf16 slices once and keeps them for both uses)
  constexpr int TB = EPL <= 2 ? 32 : 64 / EPL;
  const uint32_t grid = (a.num_rows + kAttnWarps - 1) / kAttnWarps;
  sparse_attend_kernel<EPL, TB, BF16><<<grid, kAttnWarps * 32, 0, stream>>>(a);
  return 1;
}

}  // namespace

uint32_t attend_padded_dim(uint32_t d_model, bool bf16) {
  uint32_t p = bf16 ? 64u : 32u;
  while (p < d_model) p <<= 1;
  return p <= 512u ? p : 0u;
}

int launch_sparse_attend(const AttendArgs& a, cudaStream_t stream) {
  if (a.num_rows == 0) return 0;
  const int epl = int(a.dm_pad / 32);
  if (a.latents_bf16) {
    switch (epl) {
      case 2: return launch_attend_epl<2, true>(a, stream);
      case 4: return launch_attend_epl<4, true>(a, stream);
      case 8: return launch_attend_epl<8, true>(a, stream);
      case 16: return launch_attend_epl<16, true>(a, stream);
    }
  } else {
    switch (epl) {
      case 1: return launch_attend_epl<1, false>(a, stream);
      case 2: return launch_attend_epl<2, false>(a, stream);
      case 4: return launch_attend_epl<4, false>(a, stream);
      case 8: return launch_attend_epl<8, false>(a, stream);
      case 16: return launch_attend_epl<16, false>(a, stream);
    }
  }
  return 0;
}

int launch_pad_rows(const void* src, bool src_bf16, uint64_t rows, uint32_t dim, uint32_t dim_pad, void* dst,
                    bool dst_bf16, cudaStream_t stream) {
  if (rows == 0) return 0;
  const uint64_t total = rows * dim_pad;
  const uint32_t grid = uint32_t(std::min<uint64_t>((total + 255) / 256, 148 * 16));
  if (src_bf16 && dst_bf16)
    pad_rows_kernel<<<grid, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(src), rows, dim, dim_pad, static_cast<__nv_bfloat16*>(dst));
  else if (src_bf16)
    pad_rows_kernel<<<grid, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(src), rows, dim, dim_pad, static_cast<float*>(dst));
  else if (dst_bf16)
    pad_rows_kernel<<<grid, 256, 0, stream>>>(static_cast<const float*>(src), rows, dim, dim_pad, static_cast<__nv_bfloat16*>(dst));
  else
    pad_rows_kernel<<<grid, 256, 0, stream>>>(static_cast<const float*>(src), rows, dim, dim_pad, static_cast<float*>(dst));
  return 1;
}

}  // namespace hisa_dev
