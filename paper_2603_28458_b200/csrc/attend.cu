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
#include "ptx.cuh"

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

// ---------------------------------------------------------------------------------------------------------------
// Warp-level tensor-core formulation for bf16 latents (d_model padded to 64 / 128 / 256). The SIMT kernel above spends
// ~22 warp-instructions per gathered row (8 FMA + 4 widenings + shuffles); here a batch of 16 gathered rows is staged
// once in shared memory (cp.async, 16 bytes per lane, double-buffered) and used by two sets of mma.sync.m16n8k16:
//   logits   D[16 rows x 8]  = C[16 rows x d] . Q[d x 8]         A = the tile (ldmatrix), B = the query
//   output   U[d x 8]       += C^T[d x 16 rows] . P[16 rows x 8]  A = the tile transposed (ldmatrix.trans), B = weights
// An MMA has eight N columns and one query needs one: columns 0..2 carry the exact three-term bf16 split of the fp32
// operand (query state for the logits, softmax weight for the output) and the three result columns are added, so both
// products keep fp32 accuracy (bf16 weights alone would cost 2^-9 relative, far above the 1e-5 tolerance).
// Measured mma.sync rate on B200 (tools/hmma_rate_bench.cu): 550 TFLOP/s, i.e. the 16 MMAs a batch needs cost ~1 ms
// over the whole C3 workload, well under the gather ceiling.
// ---------------------------------------------------------------------------------------------------------------
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void cp_async_16(uint32_t smem_addr, const void* gptr) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Term `which` (0, 1, 2) of an exact three-term bf16 expansion x = t0 + t1 + t2 by TRUNCATION: t0 is the leading 8
// significand bits of x, x - t0 is exact, and so on (8 + 8 + 8 = the 24 bits of an fp32 significand). Masks and two
// subtractions instead of three round-to-nearest conversions; which >= 3 gives zero.
__device__ __forceinline__ uint32_t pack_terms(float lo, float hi, uint32_t which) {
  uint32_t a = __float_as_uint(lo), b = __float_as_uint(hi);
  if (which >= 1) {
    a = __float_as_uint(lo - __uint_as_float(a & 0xFFFF0000u));
    b = __float_as_uint(hi - __uint_as_float(b & 0xFFFF0000u));
  }
  if (which >= 2) {
    a = __float_as_uint(__uint_as_float(a) - __uint_as_float(a & 0xFFFF0000u));
    b = __float_as_uint(__uint_as_float(b) - __uint_as_float(b & 0xFFFF0000u));
  }
  if (which >= 3) a = b = 0u;
  return (a >> 16) | (b & 0xFFFF0000u);
}

constexpr int kMmaRows = 16;  // gathered rows per batch = the M (logits) / K (output) extent of one MMA

template <int DM>  // padded model dimension: 64, 128 or 256
__global__ void __launch_bounds__(32, DM <= 128 ? 24 : 12) sparse_attend_mma_kernel(const AttendArgs a) {
  constexpr int KS = DM / 16;                   // k-steps of the logits = 16-dim output blocks
  constexpr uint32_t ROW_BYTES = DM * 2 + 16;   // 16 bytes of padding: ldmatrix rows land in distinct banks
  constexpr uint32_t TILE_BYTES = kMmaRows * ROW_BYTES;
  constexpr int CPR = DM * 2 / 16;              // 16-byte chunks per row
  constexpr int RPI = 32 / CPR;                 // rows covered by one warp-wide cp.async (DM = 256: 1, 128: 2, 64: 4)
  // two batches resident: one being reduced, one in flight (a third stage costs 28 registers of ring bookkeeping and
  // the occupancy that goes with them: 4.76 ms against 3.83)
  __shared__ __align__(16) unsigned char tiles[2 * TILE_BYTES];
  const uint32_t lane = threadIdx.x;
  const uint32_t g = lane >> 2, t = lane & 3u;
  const uint32_t w = blockIdx.x;
  const uint32_t row = a.idx ? w : a.num_rows - 1 - w;
  const uint32_t tq = a.pos[row];
  const bool bad_pos = tq >= a.seq_len;
  const uint32_t n = a.idx ? (a.count ? min(a.count[row], uint32_t(a.idx_stride)) : uint32_t(a.idx_stride))
                           : (bad_pos ? 0u : tq + 1u);
  const int32_t* idx = a.idx ? a.idx + uint64_t(row) * a.idx_stride : nullptr;
  float* wout = a.weights ? a.weights + uint64_t(row) * a.weights_stride : nullptr;
  const char* lat = static_cast<const char*>(a.latents);
  const uint32_t tile0 = smem_u32(tiles);
  uint32_t flags = bad_pos ? 4u : 0u;
  const float scale2 = a.scale * 1.4426950408889634f;

  // B operand of the logits: column n = g holds term g of the query state (n >= 3: zero)
  uint32_t qb[KS][2];
  {
    const float* qrow = a.queries + uint64_t(row) * DM;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const float2 lo = *reinterpret_cast<const float2*>(qrow + ks * 16 + 2 * t);
      const float2 hi = *reinterpret_cast<const float2*>(qrow + ks * 16 + 2 * t + 8);
      qb[ks][0] = pack_terms(lo.x, lo.y, g);
      qb[ks][1] = pack_terms(hi.x, hi.y, g);
    }
  }
  // per-lane pieces of the ldmatrix addresses: matrix j = lane / 8, row r = lane % 8 inside it
  const uint32_t lj = lane >> 3, lr = lane & 7u;
  const uint32_t a_off = (lr + (lj & 1u) * 8u) * ROW_BYTES + (lj >> 1) * 16u;        // logits: rows 0-7 / 8-15, k 0-7 / 8-15
  const uint32_t at_off = (lr + (lj >> 1) * 8u) * ROW_BYTES + (lj & 1u) * 16u;        // output: dims 0-7 / 8-15, rows 0-7 / 8-15
  // cp.async role: chunk c of row r0 + i * RPI
  const uint32_t cp_chunk = lane % CPR, cp_row = lane / CPR;

  auto fetch = [&](uint32_t b0, uint32_t buf, int32_t& tok_out) {
    int32_t my = -1;
    if (lane < kMmaRows && b0 + lane < n) my = idx ? idx[b0 + lane] : int32_t(b0 + lane);
    if (my >= 0 && (uint32_t(my) > tq || uint32_t(my) >= a.seq_len)) {
      flags |= 2u;
      my = -1;
    }
    tok_out = my;
    const uint32_t load_tok = uint32_t(max(my, 0));  // padding reads row 0 and is masked in the softmax
    const uint32_t base = tile0 + buf * TILE_BYTES + cp_chunk * 16u;
#pragma unroll
    for (int i = 0; i < kMmaRows / RPI; ++i) {
      const uint32_t r = i * RPI + cp_row;
      const uint32_t tok = __shfl_sync(kFull, load_tok, r);
      cp_async_16(base + r * ROW_BYTES, lat + uint64_t(tok) * (DM * 2) + cp_chunk * 16u);
    }
    cp_async_commit();
  };

  float u[KS][4];
#pragma unroll
  for (int d = 0; d < KS; ++d)
#pragma unroll
    for (int x = 0; x < 4; ++x) u[d][x] = 0.f;
  float m = -CUDART_INF_F, l = 0.f;
  int32_t next_tok = -1;
  if (n) fetch(0, 0, next_tok);
  uint32_t buf = 0;
  for (uint32_t b0 = 0; b0 < n; b0 += kMmaRows, buf ^= 1u) {
    const int32_t my_tok = next_tok;
    if (b0 + kMmaRows < n) {
      fetch(b0 + kMmaRows, buf ^ 1u, next_tok);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const uint32_t tile = tile0 + buf * TILE_BYTES;
    // ---- logits of the 16 rows: columns 0..2 are the three query terms
    float d4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      uint32_t af[4];
      ldmatrix_x4(af, tile + a_off + ks * 32u);
      mma_bf16_16816(d4, af, qb[ks][0], qb[ks][1]);
    }
    // lane (g, 0) holds columns 0, 1 of rows g and g + 8, lane (g, 1) column 2
    float x_lo = d4[0] + d4[1] + __shfl_down_sync(kFull, d4[0], 1);
    float x_hi = d4[2] + d4[3] + __shfl_down_sync(kFull, d4[2], 1);
    x_lo = __shfl_sync(kFull, x_lo, lane & ~3u);
    x_hi = __shfl_sync(kFull, x_hi, lane & ~3u);
    const bool v_lo = __shfl_sync(kFull, my_tok, g) >= 0, v_hi = __shfl_sync(kFull, my_tok, g + 8) >= 0;
    x_lo = v_lo ? x_lo * scale2 : -CUDART_INF_F;
    x_hi = v_hi ? x_hi * scale2 : -CUDART_INF_F;
    if (wout && t == 0) {
      if (b0 + g < n) wout[b0 + g] = x_lo;
      if (b0 + g + 8 < n) wout[b0 + g + 8] = x_hi;
    }
    float bm = fmaxf(x_lo, x_hi);
#pragma unroll
    for (int o = 4; o <= 16; o <<= 1) bm = fmaxf(bm, __shfl_xor_sync(kFull, bm, o));
    const float m_new = fmaxf(m, bm);
    float p_lo = 0.f, p_hi = 0.f;
    if (m_new > -CUDART_INF_F) {
      if (m_new != m) {  // warp-uniform: the running maximum settles after a few batches
        const float corr = exp2f(m - m_new);
        l *= corr;
#pragma unroll
        for (int d = 0; d < KS; ++d)
#pragma unroll
          for (int x = 0; x < 4; ++x) u[d][x] *= corr;
      }
      p_lo = v_lo ? exp2f(x_lo - m_new) : 0.f;
      p_hi = v_hi ? exp2f(x_hi - m_new) : 0.f;
    }
    m = m_new;
    l += p_lo + p_hi;  // every row is counted by the 4 lanes of its group
    // ---- B operand of the output: B[k = row][n = g] = term g of that row's weight
    const float w0 = __shfl_sync(kFull, p_lo, (2 * t) * 4), w1 = __shfl_sync(kFull, p_lo, (2 * t + 1) * 4);
    const float w8 = __shfl_sync(kFull, p_hi, (2 * t) * 4), w9 = __shfl_sync(kFull, p_hi, (2 * t + 1) * 4);
    const uint32_t pb0 = pack_terms(w0, w1, g), pb1 = pack_terms(w8, w9, g);
#pragma unroll
    for (int d = 0; d < KS; ++d) {
      uint32_t af[4];
      ldmatrix_x4_trans(af, tile + at_off + d * 32u);
      mma_bf16_16816(u[d], af, pb0, pb1);
    }
    __syncwarp();  // the tile is free for the copy that the next iteration issues into it
  }
#pragma unroll
  for (int o = 4; o <= 16; o <<= 1) l += __shfl_xor_sync(kFull, l, o);  // groups hold disjoint rows; lanes of a group agree
  if (!(l > 0.f)) flags |= 1u;
  const float inv = l > 0.f ? 1.f / l : 0.f;
  // U[dim][0..2] -> out: lane (g, 0) has columns 0, 1 of dims g and g + 8 of every 16-dim block, lane (g, 1) column 2
#pragma unroll
  for (int d = 0; d < KS; ++d) {
    const float o_lo = u[d][0] + u[d][1] + __shfl_down_sync(kFull, u[d][0], 1);
    const float o_hi = u[d][2] + u[d][3] + __shfl_down_sync(kFull, u[d][2], 1);
    if (t == 0) {
      const uint32_t c0 = d * 16 + g, c1 = c0 + 8;
      if (c0 < a.d_model) a.out[uint64_t(row) * a.d_model + c0] = o_lo * inv;
      if (c1 < a.d_model) a.out[uint64_t(row) * a.d_model + c1] = o_hi * inv;
    }
  }
  if (wout && t == 0) {
    for (uint32_t b0 = 0; b0 < a.weights_stride; b0 += kMmaRows) {
      const uint32_t j0 = b0 + g, j1 = b0 + g + 8;
      if (j0 < a.weights_stride) wout[j0] = (j0 < n && l > 0.f) ? exp2f(wout[j0] - m) * inv : 0.f;
      if (j1 < a.weights_stride) wout[j1] = (j1 < n && l > 0.f) ? exp2f(wout[j1] - m) * inv : 0.f;
    }
  }
  const uint32_t report = lane == 0 ? flags : (flags & 2u);
  if (report) atomicOr(a.flag, report);
}

template <int DM>
int launch_attend_mma(const AttendArgs& a, cudaStream_t stream) {
  sparse_attend_mma_kernel<DM><<<a.num_rows, 32, 0, stream>>>(a);
  return 1;
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
  if (a.latents_bf16 && !a.force_simt) {
    switch (a.dm_pad) {
      case 64: return launch_attend_mma<64>(a, stream);
      case 128: return launch_attend_mma<128>(a, stream);
      case 256: return launch_attend_mma<256>(a, stream);
    }
  }
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
