// Downstream consumer of the indexer: softmax attention restricted to the selected token set, over shared
// key/value latent vectors (reference: proj/core/include/hisa/attention.hpp:48-59, Eq.3).
//
//   u_t = sum_{s in T_t} softmax_s(scale * h_t . c_s) * c_s          softmax normalised over T_t only
//
// One query has one state vector, so this is a gathered matrix-vector product: 2 * |T_t| * d_model MACs against
// |T_t| * d_model gathered elements. It is bound by the L2 -> SM gather (the latent table, 16 MiB at L = 64K and
// d_model = 128 in bf16, stays L2-resident), not by the tensor pipe; the kernel is plain SIMT and organised around
// that gather:
//   * one warp per query row; R lanes share a latent row and each loads 16 bytes of it (R = 16 for d_model = 128 in
//     bf16), so one warp-wide load instruction fetches 32 / R whole rows, fully coalesced;
//   * TB rows are loaded back to back and kept in registers (TB x row-slice = 64 fp32 registers): TB independent loads in
//     flight per warp, and each gathered byte crosses L2 -> SM once although it is used twice (logit, then weighted sum);
//   * the TB partial dot products of a lane are combined with a transposed butterfly inside the R-lane group (TB - 1
//     shuffles per batch instead of TB * log2 R): afterwards every lane holds the logit of one row, so the
//     exponentials are evaluated one per lane; padding entries load row 0 unpredicated and are masked in the softmax;
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

// v[i] holds this lane's partial sum for row slot i, over the R lanes (a contiguous, R-aligned lane group) that share
// the slot's row; returns the full sum of slot (lane % R) / (R / TB). TB <= R, both powers of two.
template <int TB, int R>
__device__ __forceinline__ float transposed_reduce(float (&v)[TB], uint32_t lane) {
  int n = TB;
#pragma unroll
  for (int o = R / 2; o >= 1; o >>= 1) {
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

// R lanes share a latent row, EPL elements of the (padded) model dimension per lane: dm_pad = R * EPL. A warp-wide
// load instruction ("slot") therefore fetches 32 / R rows; TB slots form a batch.
template <int EPL, int R, bool BF16>
__global__ void __launch_bounds__(kAttnWarps * 32, 16) sparse_attend_kernel(const AttendArgs a) {
  constexpr int WORDS = BF16 ? EPL / 2 : EPL;
  constexpr int RPS = 32 / R;                                   // rows per slot
  constexpr int TB0 = EPL <= 2 ? 32 : 64 / EPL;                 // TB x EPL = 64 fp32 values per lane
  constexpr int TB = TB0 < 32 / RPS ? TB0 : 32 / RPS;           // a batch holds at most 32 rows (one index per lane)
  constexpr int ROWS = TB * RPS;                                // rows per batch
  constexpr int LPR = R / TB;                                   // lanes that end up holding the same row's logit
  static_assert(TB <= R && LPR >= 1, "transposed_reduce needs TB <= R");
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t sub = lane / R, rl = lane % R;                 // which row of a slot, which slice of the row
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
  // byte arithmetic: row address = lane base + token * row bytes is ONE 32x32+64 multiply-add per load
  const char* lane_base = static_cast<const char*>(a.latents) + rl * (WORDS * 4);
  const uint32_t row_bytes = a.dm_pad * (BF16 ? 2u : 4u);

  float q[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) q[e] = a.queries[uint64_t(row) * a.dm_pad + rl * EPL + e];

  float acc[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) acc[e] = 0.f;
  float m = -CUDART_INF_F, l = 0.f;
  uint32_t flags = bad_pos ? 4u : 0u;
  const float scale2 = a.scale * 1.4426950408889634f;  // logits in base 2
  const uint32_t mine = (rl / LPR) * RPS + sub;          // row of the batch whose logit this lane ends up holding

  for (uint32_t b0 = 0; b0 < n; b0 += ROWS) {
    int32_t my_tok = -1;
    if (lane < ROWS && b0 + lane < n) my_tok = idx ? idx[b0 + lane] : int32_t(b0 + lane);
    if (my_tok >= 0 && (uint32_t(my_tok) > t || uint32_t(my_tok) >= a.seq_len)) {
      flags |= 2u;  // CausalViolation (attention.hpp:52)
      my_tok = -1;
    }
    // padding and rejected entries load row 0 (always there) and are masked out of the softmax below: the loads of
    // a batch carry no predicates
    const uint32_t load_tok = uint32_t(max(my_tok, 0));
    uint32_t raw[TB][WORDS];
#pragma unroll
    for (int i = 0; i < TB; ++i) {
      const uint32_t tok = __shfl_sync(kFull, load_tok, i * RPS + sub);
      load_words<WORDS>(reinterpret_cast<const uint32_t*>(lane_base + uint64_t(tok) * row_bytes), raw[i]);
    }
    float part[TB];
#pragma unroll
    for (int i = 0; i < TB; ++i) {
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < EPL; ++e) s = fmaf(q[e], elem<BF16>(raw[i], e), s);
      part[i] = s;
    }
    const float dot = transposed_reduce<TB, R>(part, lane);
    const bool valid = __shfl_sync(kFull, my_tok, mine) >= 0;
    const float x = valid ? dot * scale2 : -CUDART_INF_F;
    if (wout && (rl % LPR) == 0 && b0 + mine < n) wout[b0 + mine] = x;
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
      const float pi = __shfl_sync(kFull, p, sub * R + i * LPR);  // the lane of this row group that holds slot i
#pragma unroll
      for (int e = 0; e < EPL; ++e) acc[e] = fmaf(pi, elem<BF16>(raw[i], e), acc[e]);
    }
  }
  // every row's weight was counted by its LPR lanes; the RPS row groups hold partial outputs of disjoint rows
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) l += __shfl_xor_sync(kFull, l, o);
  l *= 1.f / float(LPR);
#pragma unroll
  for (int o = R; o < 32; o <<= 1)
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[e] += __shfl_xor_sync(kFull, acc[e], o);
  if (!(l > 0.f)) flags |= 1u;  // EmptySelection (attention.hpp:51): nothing to normalise over
  const float inv = l > 0.f ? 1.f / l : 0.f;
  if (sub == 0) {
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const uint32_t c = rl * EPL + e;
      if (c < a.d_model) a.out[uint64_t(row) * a.d_model + c] = acc[e] * inv;
    }
  }
  if (wout) {
    // the lane that stored a logit turns it into the weight (same thread: no fence needed)
    for (uint32_t b0 = 0; b0 < a.weights_stride; b0 += ROWS) {
      const uint32_t j = b0 + mine;
      if ((rl % LPR) == 0 && j < a.weights_stride) wout[j] = (j < n && l > 0.f) ? exp2f(wout[j] - m) * inv : 0.f;
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

template <int EPL, int R, bool BF16>
int launch_attend_shape(const AttendArgs& a, cudaStream_t stream) {
  const uint32_t grid = (a.num_rows + kAttnWarps - 1) / kAttnWarps;
  sparse_attend_kernel<EPL, R, BF16><<<grid, kAttnWarps * 32, 0, stream>>>(a);
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
  // a lane loads 16 bytes of a row where the row is long enough for that (8 bf16 / 4 f32 elements); R = lanes per row
  if (a.latents_bf16) {
    switch (a.dm_pad) {
      case 64: return launch_attend_shape<8, 8, true>(a, stream);
      case 128: return launch_attend_shape<8, 16, true>(a, stream);
      case 256: return launch_attend_shape<8, 32, true>(a, stream);
      case 512: return launch_attend_shape<16, 32, true>(a, stream);
    }
  } else {
    switch (a.dm_pad) {
      case 32: return launch_attend_shape<4, 8, false>(a, stream);
      case 64: return launch_attend_shape<4, 16, false>(a, stream);
      case 128: return launch_attend_shape<4, 32, false>(a, stream);
      case 256: return launch_attend_shape<8, 32, false>(a, stream);
      case 512: return launch_attend_shape<16, 32, false>(a, stream);
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
