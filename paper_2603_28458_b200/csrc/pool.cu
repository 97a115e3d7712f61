// Operand preparation and block mean-pooling kernels (north-star kernel 1).
//
// Reference semantics reproduced: hisa::BlockSummaryCache::append / pooled and build_block_summaries
// (proj/core/include/hisa/block_summary.hpp:23-59): per-block sums accumulated in
// DOUBLE in position order, counts, pooled(b) = sum / count, last block partial. The batch build and the
// incremental tail update run the same per-column sequential double accumulation, so they agree bit for
// bit with each other and with a CPU loop in the same order.
#include "kernels.cuh"
#include "ptx.cuh"

#include <cuda_fp8.h>

namespace hisa_dev {

namespace {

__device__ __forceinline__ float e4m3_to_float(uint8_t b) {
  return __half2float(__half(__nv_cvt_fp8_to_halfraw(b, __NV_E4M3)));  // exact: every e4m3 value is a half value
}
// element `i` of a source array of type code 0 = f32, 1 = bf16, 2 = e4m3
__device__ __forceinline__ float load_elem(const void* src, uint32_t type, uint64_t i) {
  if (type == 1) return __bfloat162float(static_cast<const __nv_bfloat16*>(src)[i]);
  if (type == 2) return e4m3_to_float(static_cast<const uint8_t*>(src)[i]);
  return static_cast<const float*>(src)[i];
}

__device__ __forceinline__ void split_bf16(float x, int nseg, __nv_bfloat16* parts) {
  // exact multi-term bf16 expansion of an fp32 value: x == parts[0] + parts[1] + parts[2] for nseg = 3
  float r = x;
#pragma unroll
  for (int s = 0; s < kMaxSeg; ++s) {
    if (s < nseg) {
      parts[s] = __float2bfloat16_rn(r);
      r -= __bfloat162float(parts[s]);
    }
  }
}

// Pooled key of block b, column c (one thread per column, all kDim threads of the CTA call this together).
// pool_scale == null: bf16 segments hi | lo [| lo2] of the f32 value. pool_scale != null (e4m3 storage): four e4m3 terms
// t0 | t1 | t2 | t3 with p = (t0 + t1 + t2 + t3) * 2^e, 2^e = pool_scale[b] chosen from the row's largest magnitude so that t0
// uses the top of the e4m3 range: each term keeps 4 significant bits of what the terms before it left over (the subtraction
// is exact), so the row is represented to 2^-16 of its largest element, and exactly when the values need <= 15 bits (lattice
// inputs). A power-of-two scale keeps p / 2^e and the final multiply in the scorer's epilogue exact.
__device__ __forceinline__ void store_pooled(uint64_t b, uint32_t c, float p, __nv_bfloat16* pooled_op, uint32_t nseg_p,
                                             float* pool_scale) {
  if (pool_scale == nullptr) {
    __nv_bfloat16 parts[kMaxSeg];
    split_bf16(p, int(nseg_p), parts);
    for (uint32_t g = 0; g < nseg_p; ++g) pooled_op[b * (uint64_t(nseg_p) * kDim) + g * kDim + c] = parts[g];
    return;
  }
  __shared__ float s_max[kDim / 32];
  float m = fabsf(p);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __syncthreads();  // s_max may still be read by a previous use in this CTA
  if ((c & 31u) == 0) s_max[c >> 5] = m;
  __syncthreads();
  m = fmaxf(fmaxf(s_max[0], s_max[1]), fmaxf(s_max[2], s_max[3]));
  // smallest power of two with m / 2^e <= 448 (the largest e4m3 value); an all-zero row keeps scale 1
  int e = 0;
  if (m > 0.f) {
    frexpf(m / 448.0f, &e);                      // m / 448 = f * 2^e, f in [0.5, 1)
    if (ldexpf(448.0f, e - 1) >= m) e -= 1;      // f == 0.5 exactly: one power less still fits
  }
  const float scale = ldexpf(1.0f, e);
  if (c == 0) pool_scale[b] = scale;
  float r = ldexpf(p, -e);
  uint8_t* row = reinterpret_cast<uint8_t*>(pooled_op) + b * (uint64_t(kPool8Seg) * kDim);
#pragma unroll
  for (int g = 0; g < kPool8Seg; ++g) {
    const uint8_t t = uint8_t(__nv_cvt_float_to_fp8(r, __NV_SATFINITE, __NV_E4M3));
    row[g * kDim + c] = t;
    r -= e4m3_to_float(t);
  }
}

// dst row (o*dst_heads + h) <- src row (o*src_heads + h) for h < src_heads, zero rows otherwise;
// columns >= src_dim are zero. One thread per (dst row, 8-column group).
__global__ void convert_rows_kernel(const void* __restrict__ src, uint32_t src_type, uint64_t outer,
                                    uint32_t src_heads, uint32_t src_dim, uint32_t nseg,
                                    __nv_bfloat16* __restrict__ dst, uint32_t dst_heads) {
  const uint64_t gid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t total = outer * dst_heads * (kDim / 8);
  if (gid >= total) return;
  const uint32_t cg = uint32_t(gid % (kDim / 8));
  const uint64_t drow = gid / (kDim / 8);
  const uint32_t h = uint32_t(drow % dst_heads);
  const uint64_t o = drow / dst_heads;
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = 0.f;
  if (h < src_heads) {
    const uint64_t srow = o * src_heads + h;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t c = cg * 8 + i;
      if (c < src_dim) {
        v[i] = load_elem(src, src_type, srow * src_dim + c);
      }
    }
  }
  __align__(16) __nv_bfloat16 seg[kMaxSeg][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    __nv_bfloat16 parts[kMaxSeg];
    split_bf16(v[i], int(nseg), parts);
#pragma unroll
    for (int s = 0; s < kMaxSeg; ++s)
      if (s < int(nseg)) seg[s][i] = parts[s];
  }
  __nv_bfloat16* drow_ptr = dst + drow * (uint64_t(nseg) * kDim);
#pragma unroll
  for (int s = 0; s < kMaxSeg; ++s)
    if (s < int(nseg)) *reinterpret_cast<uint4*>(drow_ptr + s * kDim + cg * 8) = *reinterpret_cast<const uint4*>(seg[s]);
}

// e4m3 -> bf16 for full rows of 128 elements (the fp8 production shape: no padding, one segment): 16 bytes in,
// 32 bytes out per thread, fully coalesced. Every e4m3 value is exact in bf16.
__global__ void __launch_bounds__(256) convert_e4m3_rows_kernel(const uint4* __restrict__ src, uint64_t n16,
                                                                uint4* __restrict__ dst) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n16) return;
  const uint4 v = src[i];
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t o[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const __half2_raw hr = __nv_cvt_fp8x2_to_halfraw2(__nv_fp8x2_storage_t((w[j] >> (16 * h)) & 0xFFFFu), __NV_E4M3);
      const float2 f = __half22float2(__half2(hr));
      const __nv_bfloat162 b = __floats2bfloat162_rn(f.x, f.y);
      o[2 * j + h] = *reinterpret_cast<const uint32_t*>(&b);
    }
  }
  dst[2 * i] = make_uint4(o[0], o[1], o[2], o[3]);
  dst[2 * i + 1] = make_uint4(o[4], o[5], o[6], o[7]);
}

// pads the gates of a row to 64 heads and stores head j at gate_slot(j) (see kernels.cuh)
__global__ void permute_gates_kernel(const float* __restrict__ src, uint64_t rows, uint32_t heads,
                                     float* __restrict__ dst) {
  const uint64_t gid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= rows * kHeads) return;
  const uint32_t h = uint32_t(gid % kHeads);
  const uint64_t r = gid / kHeads;
  dst[r * kHeads + gate_slot(h)] = h < heads ? src[r * heads + h] : 0.f;
}

__global__ void check_finite_kernel(const void* __restrict__ src, uint32_t src_type, uint64_t n,
                                    uint32_t* __restrict__ flag) {
  bool bad = false;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    bad |= !isfinite(load_elem(src, src_type, i));  // e4m3 has no infinities; S.1111.111 decodes to NaN
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

__global__ void check_positions_kernel(const uint32_t* __restrict__ pos, uint64_t n, uint32_t seq_len,
                                       uint32_t* __restrict__ flag) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && pos[i] > seq_len) atomicOr(flag, 1u);
}

// One CTA per touched block, one thread per operand column. Sequential (position-order) accumulation.
__global__ void __launch_bounds__(kDim)
pool_update_kernel(const __nv_bfloat16* __restrict__ key_op, uint32_t nseg_k, uint64_t first, uint64_t n,
                   uint32_t block_size, uint32_t pool_max, double* __restrict__ sums,
                   uint32_t* __restrict__ counts, __nv_bfloat16* __restrict__ pooled_op, uint32_t nseg_p,
                   uint32_t* __restrict__ len_out) {
  const uint64_t b = first / block_size + blockIdx.x;
  const uint32_t c = threadIdx.x;
  if (len_out && blockIdx.x == 0 && c == 0) *len_out = uint32_t(first + n);
  const uint64_t blk_lo = b * block_size;
  const uint64_t s_lo = first > blk_lo ? first : blk_lo;
  const uint64_t blk_hi = blk_lo + block_size;
  const uint64_t s_hi = (first + n) < blk_hi ? (first + n) : blk_hi;
  const bool fresh = (s_lo == blk_lo);
  double acc = fresh ? 0.0 : sums[b * kDim + c];
  const uint64_t row_elems = uint64_t(nseg_k) * kDim;
  // the adds stay in position order (bit-for-bit agreement with the incremental update and the CPU loop); the loads of
  // eight rows are issued together so that one DRAM latency covers eight rows instead of one
  constexpr int kAhead = 8;
  for (uint64_t s0 = s_lo; s0 < s_hi; s0 += kAhead) {
    double v[kAhead];
#pragma unroll
    for (int i = 0; i < kAhead; ++i) {
      v[i] = 0.0;
      if (s0 + i < s_hi) {
        const __nv_bfloat16* row = key_op + (s0 + i) * row_elems + c;
        for (uint32_t g = 0; g < nseg_k; ++g) v[i] += double(__bfloat162float(row[g * kDim]));
      }
    }
#pragma unroll
    for (int i = 0; i < kAhead; ++i) {
      if (s0 + i < s_hi) {
        if (pool_max) acc = (fresh && s0 + i == s_lo) ? v[i] : (v[i] > acc ? v[i] : acc);
        else acc += v[i];
      }
    }
  }
  sums[b * kDim + c] = acc;
  const uint32_t cnt = uint32_t(s_hi - blk_lo);
  if (c == 0) counts[b] = cnt;
  const double p = pool_max ? acc : acc / double(cnt);
  store_pooled(b, c, float(p), pooled_op, nseg_p, nullptr);
}

// Same accumulation for e4m3 keys with a per-key scale: the summed value is float(k8) * scale (one f32 rounding),
// exactly what the CPU oracle is given as the dequantised key.
__global__ void __launch_bounds__(kDim)
pool_update_fp8_kernel(const uint8_t* __restrict__ key8, const float* __restrict__ key_scale, uint64_t first, uint64_t n,
                       uint32_t block_size, uint32_t pool_max, double* __restrict__ sums,
                       uint32_t* __restrict__ counts, __nv_bfloat16* __restrict__ pooled_op, uint32_t nseg_p,
                       float* __restrict__ pool_scale, uint32_t* __restrict__ len_out) {
  const uint64_t b = first / block_size + blockIdx.x;
  const uint32_t c = threadIdx.x;
  if (len_out && blockIdx.x == 0 && c == 0) *len_out = uint32_t(first + n);
  const uint64_t blk_lo = b * block_size;
  const uint64_t s_lo = first > blk_lo ? first : blk_lo;
  const uint64_t blk_hi = blk_lo + block_size;
  const uint64_t s_hi = (first + n) < blk_hi ? (first + n) : blk_hi;
  const bool fresh = (s_lo == blk_lo);
  double acc = fresh ? 0.0 : sums[b * kDim + c];
  constexpr int kAhead = 8;  // loads of eight rows in flight, adds in position order (see pool_update_kernel)
  for (uint64_t s0 = s_lo; s0 < s_hi; s0 += kAhead) {
    double v[kAhead];
#pragma unroll
    for (int i = 0; i < kAhead; ++i)
      v[i] = s0 + i < s_hi ? double(e4m3_to_float(key8[(s0 + i) * kDim + c]) * key_scale[s0 + i]) : 0.0;
#pragma unroll
    for (int i = 0; i < kAhead; ++i) {
      if (s0 + i < s_hi) {
        if (pool_max) acc = (fresh && s0 + i == s_lo) ? v[i] : (v[i] > acc ? v[i] : acc);
        else acc += v[i];
      }
    }
  }
  sums[b * kDim + c] = acc;
  const uint32_t cnt = uint32_t(s_hi - blk_lo);
  if (c == 0) counts[b] = cnt;
  const double p = pool_max ? acc : acc / double(cnt);
  store_pooled(b, c, float(p), pooled_op, nseg_p, pool_scale);
}

// Batch build (north-star kernel 1): the same per-column, position-ordered double accumulation, fed from shared
// memory. One CTA per block; the block's rows are contiguous in HBM, so they arrive as bulk copies (cp.async.bulk,
// 64 rows = 16 KB per copy for bf16 storage, two copies in flight per CTA, ~4 CTAs per SM): the whole key array is
// requested within the first microsecond and streams at DRAM speed, while the one-thread-per-column kernel above
// fetched 256 bytes per warp-instruction with eight rows in flight (45 us for 16 MiB: 6 % of the HBM roofline). The
// adds, their order and the rounding are unchanged, so the summaries stay bit-identical to the incremental update and
// to the CPU loop. FP8: rows are 128 bytes; the per-key scales of a chunk are fetched with plain loads.
constexpr int kPoolChunkRows = 64;

template <bool FP8>
__global__ void __launch_bounds__(kDim)
pool_update_staged_kernel(const void* __restrict__ key_op, const float* __restrict__ key_scale, uint32_t nseg_k,
                          uint64_t first, uint64_t n, uint32_t block_size, uint32_t pool_max, double* __restrict__ sums,
                          uint32_t* __restrict__ counts, __nv_bfloat16* __restrict__ pooled_op, uint32_t nseg_p,
                          float* __restrict__ pool_scale, uint32_t* __restrict__ len_out) {
  extern __shared__ __align__(128) unsigned char pool_smem[];
  if (len_out && blockIdx.x == 0 && threadIdx.x == 0) *len_out = uint32_t(first + n);
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ float s_scale[2][kPoolChunkRows];
  const uint64_t b = first / block_size + blockIdx.x;
  const uint32_t c = threadIdx.x;
  const uint64_t blk_lo = b * block_size;
  const uint64_t s_lo = first > blk_lo ? first : blk_lo;
  const uint64_t blk_hi = blk_lo + block_size;
  const uint64_t s_hi = (first + n) < blk_hi ? (first + n) : blk_hi;
  const bool fresh = (s_lo == blk_lo);
  double acc = fresh ? 0.0 : sums[b * kDim + c];
  const uint32_t row_bytes = FP8 ? uint32_t(kDim) : nseg_k * uint32_t(kDim) * 2u;
  const uint32_t buf_bytes = kPoolChunkRows * row_bytes;
  const uint32_t nrows = uint32_t(s_hi - s_lo);
  const uint32_t nchunks = (nrows + kPoolChunkRows - 1) / kPoolChunkRows;
  if (c == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](uint32_t ch) {
    const uint32_t buf = ch & 1u;
    const uint64_t r0 = s_lo + uint64_t(ch) * kPoolChunkRows;
    const uint32_t nr = min(uint32_t(kPoolChunkRows), uint32_t(s_hi - r0));
    mbar_arrive_expect_tx(&bar[buf], nr * row_bytes);
    bulk_load_1d(pool_smem + buf * buf_bytes, static_cast<const unsigned char*>(key_op) + r0 * row_bytes, nr * row_bytes,
                 &bar[buf]);
  };
  if (c == 0) {
    issue(0);
    if (nchunks > 1) issue(1);
  }
  for (uint32_t ch = 0; ch < nchunks; ++ch) {
    const uint32_t buf = ch & 1u;
    const uint64_t r0 = s_lo + uint64_t(ch) * kPoolChunkRows;
    const uint32_t nr = min(uint32_t(kPoolChunkRows), uint32_t(s_hi - r0));
    if (FP8) {
      if (c < nr) s_scale[buf][c] = key_scale[r0 + c];
      __syncthreads();
    }
    mbar_wait(&bar[buf], (ch >> 1) & 1u);
    const unsigned char* rows = pool_smem + buf * buf_bytes;
    // eight rows are read and widened together (independent work), then added in position order (the dependent chain)
    for (uint32_t i0 = 0; i0 < nr; i0 += 8) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t i = min(i0 + j, nr - 1);  // rows past the chunk repeat the last one and are not added
        if (FP8) {
          v[j] = double(e4m3_to_float(rows[i * kDim + c]) * s_scale[buf][i]);
        } else {
          const __nv_bfloat16* row = reinterpret_cast<const __nv_bfloat16*>(rows + i * row_bytes) + c;
          if (nseg_k == 1) {
            v[j] = double(__bfloat162float(row[0]));
          } else {
            v[j] = 0.0;
            for (uint32_t g = 0; g < nseg_k; ++g) v[j] += double(__bfloat162float(row[g * kDim]));
          }
        }
      }
      if (!pool_max && i0 + 8 <= nr) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += v[j];
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (i0 + j < nr) {
            if (pool_max) acc = (fresh && r0 + i0 + j == s_lo) ? v[j] : (v[j] > acc ? v[j] : acc);
            else acc += v[j];
          }
        }
      }
    }
    __syncthreads();  // every thread is done with this buffer
    if (c == 0 && ch + 2 < nchunks) issue(ch + 2);
  }
  sums[b * kDim + c] = acc;
  const uint32_t cnt = uint32_t(s_hi - blk_lo);
  if (c == 0) counts[b] = cnt;
  const double p = pool_max ? acc : acc / double(cnt);
  store_pooled(b, c, float(p), pooled_op, nseg_p, FP8 ? pool_scale : nullptr);
}

template <bool FP8>
bool launch_pool_staged(const void* key_op, const float* key_scale, uint32_t nseg_k, uint64_t first, uint64_t n,
                        uint32_t block_size, uint32_t pool_max, double* sums, uint32_t* counts, __nv_bfloat16* pooled_op,
                        uint32_t nseg_p, float* pool_scale, uint32_t* len_out, cudaStream_t stream) {
  // decode-sized appends stay on the direct kernel: nothing to stage for a handful of rows
  if (n < 32 || reinterpret_cast<uintptr_t>(key_op) % 16 != 0) return false;
  const uint32_t row_bytes = FP8 ? uint32_t(kDim) : nseg_k * uint32_t(kDim) * 2u;
  const size_t smem = size_t(2) * kPoolChunkRows * row_bytes;
  auto kern = pool_update_staged_kernel<FP8>;
  if (smem > 48 * 1024 && !smem_opt_in(reinterpret_cast<const void*>(kern), smem)) return false;
  const uint64_t b0 = first / block_size, b1 = (first + n - 1) / block_size;
  kern<<<uint32_t(b1 - b0 + 1), kDim, smem, stream>>>(key_op, key_scale, nseg_k, first, n, block_size, pool_max, sums, counts,
                                                      pooled_op, nseg_p, pool_scale, len_out);
  return true;
}

__global__ void fill_f32_kernel(float* __restrict__ dst, uint64_t n, float v) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = v;
}

__global__ void pool_export_kernel(const double* __restrict__ sums, const uint32_t* __restrict__ counts,
                                   uint32_t num_blocks, uint32_t dim, uint32_t pool_max,
                                   double* __restrict__ out_sums, double* __restrict__ out_pooled) {
  const uint64_t gid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= uint64_t(num_blocks) * dim) return;
  const uint32_t c = uint32_t(gid % dim);
  const uint32_t b = uint32_t(gid / dim);
  const double s = sums[uint64_t(b) * kDim + c];
  if (out_sums) out_sums[gid] = s;
  if (out_pooled) out_pooled[gid] = pool_max ? s : s / double(counts[b]);
}

// caller-provided summaries (BlockSummaryCache contents, block_summary.hpp:16-18): sums [M, dim] -> the context's padded
// f64 sums, counts and the pooled operand, with the same sum / count -> f32 -> bf16 split as the pooling kernels
__global__ void __launch_bounds__(kDim)
pool_import_kernel(const double* __restrict__ src_sums, const uint32_t* __restrict__ src_counts, uint32_t dim,
                   uint32_t pool_max, double* __restrict__ sums, uint32_t* __restrict__ counts,
                   __nv_bfloat16* __restrict__ pooled_op, uint32_t nseg_p, float* __restrict__ pool_scale) {
  const uint32_t b = blockIdx.x, c = threadIdx.x;
  const uint32_t cnt = src_counts[b];
  const double s = c < dim ? src_sums[uint64_t(b) * dim + c] : 0.0;
  sums[uint64_t(b) * kDim + c] = s;
  if (c == 0) counts[b] = cnt;
  const double p = pool_max ? s : (cnt ? s / double(cnt) : 0.0);
  store_pooled(b, c, float(p), pooled_op, nseg_p, pool_scale);
}

inline uint32_t blocks_for(uint64_t n, uint32_t threads) { return uint32_t((n + threads - 1) / threads); }

}  // namespace

int launch_convert_rows(const void* src, uint32_t src_type, uint64_t outer, uint32_t src_heads, uint32_t src_dim,
                        uint32_t nseg, __nv_bfloat16* dst, uint32_t dst_heads, cudaStream_t stream) {
  const uint64_t total = outer * dst_heads * (kDim / 8);
  if (total == 0) return 0;
  if (src_type == 2 && nseg == 1 && src_dim == uint32_t(kDim) && src_heads == dst_heads &&
      reinterpret_cast<uintptr_t>(src) % 16 == 0) {
    const uint64_t n16 = outer * dst_heads * (kDim / 16);
    convert_e4m3_rows_kernel<<<blocks_for(n16, 256), 256, 0, stream>>>(static_cast<const uint4*>(src), n16,
                                                                      reinterpret_cast<uint4*>(dst));
    return 1;
  }
  convert_rows_kernel<<<blocks_for(total, 256), 256, 0, stream>>>(src, src_type, outer, src_heads, src_dim, nseg,
                                                                  dst, dst_heads);
  return 1;
}

int launch_permute_gates(const float* src, uint64_t rows, uint32_t heads, float* dst, cudaStream_t stream) {
  if (rows == 0) return 0;
  permute_gates_kernel<<<blocks_for(rows * kHeads, 256), 256, 0, stream>>>(src, rows, heads, dst);
  return 1;
}

int launch_check_finite(const void* src, uint32_t src_type, uint64_t n, uint32_t* flag, cudaStream_t stream) {
  if (n == 0) return 0;
  const uint32_t grid = uint32_t(n / 256 + 1 < 148 * 16 ? n / 256 + 1 : 148 * 16);
  check_finite_kernel<<<grid, 256, 0, stream>>>(src, src_type, n, flag);
  return 1;
}

int launch_check_positions(const uint32_t* pos, uint64_t n, uint32_t seq_len, uint32_t* flag, cudaStream_t stream) {
  if (n == 0) return 0;
  check_positions_kernel<<<blocks_for(n, 256), 256, 0, stream>>>(pos, n, seq_len, flag);
  return 1;
}

int launch_pool_update(const __nv_bfloat16* key_op, uint32_t nseg_k, uint64_t first, uint64_t n, uint32_t block_size,
                       uint32_t /*dim*/, uint32_t pool_max, double* sums, uint32_t* counts, __nv_bfloat16* pooled_op,
                       uint32_t nseg_p, uint32_t* len_out, cudaStream_t stream) {
  if (n == 0) return 0;
  if (launch_pool_staged<false>(key_op, nullptr, nseg_k, first, n, block_size, pool_max, sums, counts, pooled_op, nseg_p, nullptr, len_out, stream))
    return 1;
  const uint64_t b0 = first / block_size, b1 = (first + n - 1) / block_size;
  pool_update_kernel<<<uint32_t(b1 - b0 + 1), kDim, 0, stream>>>(key_op, nseg_k, first, n, block_size, pool_max, sums,
                                                                 counts, pooled_op, nseg_p, len_out);
  return 1;
}

int launch_pool_update_fp8(const uint8_t* key8, const float* key_scale, uint64_t first, uint64_t n, uint32_t block_size,
                           uint32_t pool_max, double* sums, uint32_t* counts, __nv_bfloat16* pooled_op, uint32_t nseg_p,
                           float* pool_scale, uint32_t* len_out, cudaStream_t stream) {
  if (n == 0) return 0;
  if (launch_pool_staged<true>(key8, key_scale, 1, first, n, block_size, pool_max, sums, counts, pooled_op, nseg_p, pool_scale, len_out, stream))
    return 1;
  const uint64_t b0 = first / block_size, b1 = (first + n - 1) / block_size;
  pool_update_fp8_kernel<<<uint32_t(b1 - b0 + 1), kDim, 0, stream>>>(key8, key_scale, first, n, block_size, pool_max, sums,
                                                                     counts, pooled_op, nseg_p, pool_scale, len_out);
  return 1;
}

int launch_pool_import(const double* src_sums, const uint32_t* src_counts, uint32_t num_blocks, uint32_t dim,
                       uint32_t pool_max, double* sums, uint32_t* counts, __nv_bfloat16* pooled_op, uint32_t nseg_p,
                       float* pool_scale, cudaStream_t stream) {
  if (num_blocks == 0) return 0;
  pool_import_kernel<<<num_blocks, kDim, 0, stream>>>(src_sums, src_counts, dim, pool_max, sums, counts, pooled_op, nseg_p,
                                                      pool_scale);
  return 1;
}

int launch_fill_f32(float* dst, uint64_t n, float v, cudaStream_t stream) {
  if (n == 0) return 0;
  fill_f32_kernel<<<blocks_for(n, 256), 256, 0, stream>>>(dst, n, v);
  return 1;
}

int launch_pool_export(const double* sums, const uint32_t* counts, uint32_t num_blocks, uint32_t dim, uint32_t pool_max,
                       double* out_sums, double* out_pooled, cudaStream_t stream) {
  const uint64_t total = uint64_t(num_blocks) * dim;
  if (total == 0) return 0;
  pool_export_kernel<<<blocks_for(total, 256), 256, 0, stream>>>(sums, counts, num_blocks, dim, pool_max, out_sums,
                                                                 out_pooled);
  return 1;
}

}  // namespace hisa_dev
