// Selection kernels (north-star kernels 3 and 5) and the work-list builders that feed the scorer.
//
// select_rows_kernel reproduces hisa::top_k_tokens (proj/core/include/hisa/dsa.hpp:22-27)
// and hisa::select_blocks (hisa/hisa.hpp:23-28) on fp32 scores:
//   total order = (score descending, then position ascending for SmallestIndex / descending for
//   LargestIndex), keep the first `keep` entries of that order, emit them in ascending position order;
//   +0 and -0 compare equal. For blocks, the first eligible block and the block containing the query are
//   added on top (force_first_last), or placed first inside the budget (forced_in_budget).
// Method: scores -> order-preserving u32 keys in shared memory; the keep-th largest key T is found by a
// range-adaptive radix select (11-bit digits over [min,max], so fp32 scores that share sign/exponent do
// not pile into one bin); then ONE ordered compaction in position order emits keys > T plus the required
// number of keys == T picked from the front (SmallestIndex) or the back (LargestIndex). That yields the
// reference's tie-break and its ascending output without sorting.
//
// candidate_union (hisa/hisa.hpp:30-33) never materialises: stage-2 candidates are addressed as
// (slot, offset) inside the row's selected-block list and mapped to token positions on output.
#include "kernels.cuh"
#include "ptx.cuh"

#include <cstdlib>

namespace hisa_dev {

namespace {

constexpr int kBins = 2048;
constexpr int kBinBits = 11;
constexpr int kListCap = 1024;  // survivors of the first radix level are compacted when they fit here

// Sequence length / number of summarised blocks of a launch: by value, or read from device memory when the launch is
// part of a replayed CUDA graph (decode: the sequence grows by one key per step while the graph stays the same).
__device__ __forceinline__ uint32_t seq_len_of(const SelectArgs& a) { return a.dyn_len ? __ldg(a.dyn_len) : a.seq_len; }
__device__ __forceinline__ uint32_t num_blocks_of(const SelectArgs& a) {
  return a.dyn_len ? (__ldg(a.dyn_len) + a.block_size - 1) / a.block_size : a.num_blocks;
}

__device__ __forceinline__ uint32_t score_key(float f) {
  uint32_t b = __float_as_uint(f);
  if (b == 0x80000000u) b = 0u;  // -0 == +0
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// exclusive prefix sum over the block; `total` receives the block sum. scratch: >= 33 words.
template <int THREADS>
__device__ __forceinline__ uint32_t block_scan_excl(uint32_t v, uint32_t* scratch, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  __syncthreads();  // scratch reuse across calls
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    constexpr int NW = THREADS / 32;
    uint32_t w = lane < NW ? scratch[lane] : 0u;
    uint32_t winc = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, winc, o);
      if (lane >= o) winc += y;
    }
    if (lane < NW) scratch[lane] = winc - w;
    if (lane == NW - 1) scratch[32] = winc;
  }
  __syncthreads();
  total = scratch[32];
  return scratch[warp] + inc - v;
}

template <int THREADS>
__device__ __forceinline__ uint32_t block_reduce_min(uint32_t v, uint32_t* scratch) {
  v = __reduce_min_sync(0xffffffffu, v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t r = scratch[0];
  for (int w = 1; w < THREADS / 32; ++w) r = min(r, scratch[w]);
  return r;
}
template <int THREADS>
__device__ __forceinline__ uint32_t block_reduce_max(uint32_t v, uint32_t* scratch) {
  v = __reduce_max_sync(0xffffffffu, v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t r = scratch[0];
  for (int w = 1; w < THREADS / 32; ++w) r = max(r, scratch[w]);
  return r;
}

template <int THREADS, bool SMEM_KEYS>
__global__ void __launch_bounds__(THREADS, THREADS == 1024 ? 2 : 1) select_rows_kernel(SelectArgs a) {
  extern __shared__ __align__(16) uint32_t smem_u[];
  uint32_t* hist = smem_u;                // [kBins]
  uint32_t* scratch = smem_u + kBins;     // [64]
  uint32_t* list = smem_u + kBins + 64;   // [kListCap]
  uint32_t* ssel = list + kListCap;       // [sel_stride] the row's selected blocks (candidate mode)
  uint32_t* skey = ssel + a.sel_stride;   // [n_cap] when SMEM_KEYS (16-byte aligned: sel_stride is padded to 4)

  const uint32_t row = blockIdx.x;
  const uint32_t tid = threadIdx.x;
  const bool block_mode = (a.mode == kSelBlocks || a.mode == kSelBlocksGeneric);
  const uint32_t B = a.block_size;

  // ---- how many candidates does this row have, and where do they live -------------------------
  uint32_t n = 0;
  const int32_t* sel_row = nullptr;
  if (a.mode == kSelFlat) {
    const uint32_t t = min(a.pos[row], seq_len_of(a) - 1);
    n = t + 1;
  } else if (a.mode == kSelBlocks) {
    const uint32_t t = min(a.pos[row], seq_len_of(a) - 1);
    n = min(t / B, num_blocks_of(a) - 1) + 1;
  } else if (a.mode == kSelCand) {
    const uint32_t t = min(a.pos[row], seq_len_of(a) - 1);
    const uint32_t ns = a.nsel[row];
    sel_row = a.sel + uint64_t(row) * a.sel_row_stride;
    const uint32_t lastb = uint32_t(sel_row[ns - 1]);
    n = (ns - 1) * B + min(B, t - lastb * B + 1);
    for (uint32_t i = tid; i < ns; i += THREADS) ssel[i] = uint32_t(sel_row[i]);
    __syncthreads();
  } else {
    n = a.n_in[row];
  }
  const float* srow = a.scores + uint64_t(row) * a.stride;
  const uint32_t orow_i = a.out_rows ? a.out_rows[row] : row;  // where this row's result lives in the output arrays
  int32_t* orow = a.out_idx + uint64_t(orow_i) * a.out_stride;
  const uint32_t keep = a.keep;
  const bool forced = block_mode && a.force_first_last && n > 0;

  const uint32_t bshift = a.block_shift;  // log2(B) when B is a power of two, else 32
  auto position_of = [&](uint32_t i) -> int32_t {
    if (a.mode == kSelCand) {
      const uint32_t slot = bshift < 32 ? i >> bshift : i / B;
      return int32_t(ssel[slot] * B + (i - slot * B));
    }
    return int32_t(i);
  };

  if (a.out_cand && tid == 0) a.out_cand[orow_i] = n;

  // ---- everything fits: dense regime ------------------------------------
  if (n <= keep) {
    for (uint32_t i = tid; i < a.out_width; i += THREADS) orow[i] = i < n ? position_of(i) : -1;
    if (a.out_count && tid == 0) a.out_count[orow_i] = n;
    return;
  }

  auto raw_key = [&](uint32_t i) -> uint32_t {
    uint32_t key = score_key(srow[i]);
    if (forced && a.forced_in_budget && (i == 0 || i == n - 1)) key = 0xFFFFFFFFu;
    return key;
  };
  auto key_at = [&](uint32_t i) -> uint32_t {
    if constexpr (SMEM_KEYS) return skey[i];
    else return raw_key(i);
  };

  // ---- keys, min, max ---------------------------------------------------------------------------
  uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
  const bool boost = forced && a.forced_in_budget;
  if (SMEM_KEYS && a.vec_ok && !boost) {
    // 16-byte loads: four scores per request keep enough bytes in flight at 5 CTAs per SM
    const float4* s4 = reinterpret_cast<const float4*>(srow);
    const uint32_t n4 = n >> 2;
    for (uint32_t i = tid; i < n4; i += THREADS) {
      const float4 v = __ldg(s4 + i);
      uint4 kq;
      kq.x = score_key(v.x); kq.y = score_key(v.y); kq.z = score_key(v.z); kq.w = score_key(v.w);
      reinterpret_cast<uint4*>(skey)[i] = kq;
      kmin = min(min(kmin, kq.x), min(min(kq.y, kq.z), kq.w));
      kmax = max(max(kmax, kq.x), max(max(kq.y, kq.z), kq.w));
    }
    for (uint32_t i = (n4 << 2) + tid; i < n; i += THREADS) {
      const uint32_t key = score_key(srow[i]);
      skey[i] = key;
      kmin = min(kmin, key);
      kmax = max(kmax, key);
    }
  } else if (!SMEM_KEYS && a.vec_ok && !boost) {
    // rows too long for shared memory: every pass streams the row from L2 / HBM. 16-byte loads (four scores per request):
    // the scalar version spent 70 % of its stall samples waiting for 4-byte loads (long scoreboard + LSU queue throttle)
    const float4* s4 = reinterpret_cast<const float4*>(srow);
    const uint32_t n4 = n >> 2;
    for (uint32_t i = tid; i < n4; i += THREADS) {
      const float4 v = __ldg(s4 + i);
      const uint32_t kx = score_key(v.x), ky = score_key(v.y), kz = score_key(v.z), kw = score_key(v.w);
      kmin = min(min(kmin, kx), min(min(ky, kz), kw));
      kmax = max(max(kmax, kx), max(max(ky, kz), kw));
    }
    for (uint32_t i = (n4 << 2) + tid; i < n; i += THREADS) {
      const uint32_t key = score_key(srow[i]);
      kmin = min(kmin, key);
      kmax = max(kmax, key);
    }
  } else {
    for (uint32_t i = tid; i < n; i += THREADS) {
      const uint32_t key = raw_key(i);
      if constexpr (SMEM_KEYS) skey[i] = key;
      kmin = min(kmin, key);
      kmax = max(kmax, key);
    }
  }
  const bool vec_g = !SMEM_KEYS && a.vec_ok && !boost;  // the passes below read the row with 16-byte loads as well
  // f(i, key) for every candidate, lanes on consecutive 16-byte chunks (order across threads is irrelevant to the caller)
  auto for_each_strided = [&](auto&& f) {
    if (vec_g) {
      const float4* s4 = reinterpret_cast<const float4*>(srow);
      const uint32_t n4 = n >> 2;
      for (uint32_t i = tid; i < n4; i += THREADS) {
        const float4 v = __ldg(s4 + i);
        f(4 * i + 0, score_key(v.x));
        f(4 * i + 1, score_key(v.y));
        f(4 * i + 2, score_key(v.z));
        f(4 * i + 3, score_key(v.w));
      }
      for (uint32_t i = (n4 << 2) + tid; i < n; i += THREADS) f(i, score_key(srow[i]));
    } else {
      for (uint32_t i = tid; i < n; i += THREADS) f(i, key_at(i));
    }
  };
  uint32_t lo = block_reduce_min<THREADS>(kmin, scratch);
  uint32_t hi = block_reduce_max<THREADS>(kmax, scratch);
  __syncthreads();

  // ---- range-adaptive radix select of the keep-th largest key ------------------------------------
  // (tried and measured on B200, both dropped: a compare-and-count bisection instead of the histogram was 45 %
  //  slower — ~30 block-wide count steps per row cost more than three 11-bit levels, two of them on the survivor
  //  list; a sample-guided bracket that restricts the first level to ~20 % of the keys changed nothing — the
  //  kernel is spread over many short phases, not bound by the shared-memory atomics)
  uint32_t kk = keep;  // still to take from [lo, hi]
  bool use_list = false;
  uint32_t list_n = 0;
  while (lo != hi) {
    const uint32_t range = hi - lo;
    const uint32_t nb = 32 - __clz(range);
    const uint32_t shift = nb > kBinBits ? nb - kBinBits : 0u;
    for (uint32_t i = tid; i < kBins; i += THREADS) hist[i] = 0u;
    __syncthreads();
    if (use_list) {
      for (uint32_t i = tid; i < list_n; i += THREADS) {
        const uint32_t key = list[i];
        if (key >= lo && key <= hi) atomicAdd(&hist[(key - lo) >> shift], 1u);
      }
    } else {
      for_each_strided([&](uint32_t, uint32_t key) {
        if (key >= lo && key <= hi) atomicAdd(&hist[(key - lo) >> shift], 1u);
      });
    }
    __syncthreads();
    constexpr int BPT = kBins / THREADS;
    uint32_t loc = 0;
#pragma unroll
    for (int j = 0; j < BPT; ++j) loc += hist[tid * BPT + j];
    uint32_t total;
    const uint32_t before = block_scan_excl<THREADS>(loc, scratch, total);
    const uint32_t above = total - before - loc;  // keys in bins owned by higher threads
    if (above < kk && kk <= above + loc) {
      uint32_t c = above;
      int j = BPT - 1;
      for (; j > 0; --j) {
        const uint32_t h = hist[tid * BPT + j];
        if (c + h >= kk) break;
        c += h;
      }
      scratch[40] = tid * BPT + j;
      scratch[41] = c;
      scratch[42] = hist[tid * BPT + j];
      scratch[43] = 0;
    }
    __syncthreads();
    const uint32_t bin = scratch[40];
    const uint32_t in_bin = scratch[42];
    kk -= scratch[41];
    lo = lo + (bin << shift);
    const uint32_t width = (shift == 0) ? 0u : ((1u << shift) - 1u);
    hi = lo + min(hi - lo, width);  // (lo + width may pass 2^32 in the top bin: boosted keys are 0xFFFFFFFF)
    if (!use_list && lo != hi && in_bin <= uint32_t(kListCap)) {
      // the remaining levels only concern the keys of this bin: compact them once (order is irrelevant here)
      for_each_strided([&](uint32_t, uint32_t key) {
        if (key >= lo && key <= hi) list[atomicAdd(&scratch[43], 1u)] = key;
      });
      use_list = true;
      list_n = in_bin;
    }
    __syncthreads();
  }
  const uint32_t T = lo;
  const uint32_t need = kk;  // ties (key == T) to take

  // ---- ordered compaction over blocked segments ---------------------------------------------------
  // thread t owns the contiguous candidates [s0, s1); global rows: whole 16-byte chunks per thread, the ragged tail (< 4
  // candidates) goes to the last thread, whose segment is the last one anyway
  uint32_t s0, s1;
  if (vec_g) {
    const uint32_t n4 = n >> 2, q4 = (n4 + THREADS - 1) / THREADS;
    s0 = 4u * min(n4, tid * q4);
    s1 = tid == THREADS - 1 ? n : 4u * min(n4, tid * q4 + q4);
  } else {
    const uint32_t ipt = ((n + THREADS - 1) / THREADS) | 1u;  // odd: conflict-free strided smem walks
    s0 = min(n, tid * ipt);
    s1 = min(n, s0 + ipt);
  }
  // f(i, key) for the thread's candidates in ascending order
  auto for_each_owned = [&](auto&& f) {
    if (vec_g) {
      const uint32_t v1 = s0 + ((s1 - s0) & ~3u);  // end of the whole chunks (s0 is a multiple of 4)
      for (uint32_t i = s0; i < v1; i += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(srow + i));
        f(i + 0, score_key(v.x));
        f(i + 1, score_key(v.y));
        f(i + 2, score_key(v.z));
        f(i + 3, score_key(v.w));
      }
      for (uint32_t i = v1; i < s1; ++i) f(i, score_key(srow[i]));
    } else {
      for (uint32_t i = s0; i < s1; ++i) f(i, key_at(i));
    }
  };
  uint32_t cG = 0, cE = 0;
  for_each_owned([&](uint32_t, uint32_t key) {
    cG += key > T;
    cE += key == T;
  });
  uint32_t totG, totE;
  const uint32_t gBefore = block_scan_excl<THREADS>(cG, scratch, totG);
  const uint32_t eBefore = block_scan_excl<THREADS>(cE, scratch, totE);
  const uint32_t skip = a.tie_break ? totE - need : 0u;  // LargestIndex takes the last `need` ties

  // forced blocks that the score order did not pick are added on top (select_blocks)
  uint32_t add_first = 0, add_last = 0;
  if (forced) {
    const uint32_t k0 = key_at(0), kl = key_at(n - 1);
    const bool sel0 = k0 > T || (k0 == T && skip == 0);
    const bool sell = kl > T || (kl == T && (totE - 1 >= skip) && (totE - 1 < skip + need));
    add_first = sel0 ? 0u : 1u;
    add_last = sell ? 0u : 1u;
  }
  const uint32_t tiesBefore = eBefore > skip ? min(eBefore - skip, need) : 0u;
  uint32_t o = gBefore + tiesBefore + add_first;
  uint32_t e = eBefore;
  for_each_owned([&](uint32_t i, uint32_t key) {
    bool emit = key > T;
    if (key == T) {
      emit = (e >= skip) && (e < skip + need);
      ++e;
    }
    if (emit) orow[o++] = position_of(i);
  });
  const uint32_t count = totG + need + add_first + add_last;
  if (add_first && tid == 0) orow[0] = position_of(0);
  if (add_last && tid == 0) orow[count - 1] = position_of(n - 1);
  for (uint32_t i = count + tid; i < a.out_width; i += THREADS) orow[i] = -1;
  if (a.out_count && tid == 0) a.out_count[orow_i] = count;
}

// ---------------------------------------------------------------------------------------------------
// Warp-per-row selection for short rows (n_cap <= 32 * KPL): select_blocks at prefill sizes (<= 512 blocks)
// and small top-k problems. Keys live in registers (element i = lane + 32 j); the keep-th largest key is found
// by a bitwise radix descent that starts at the highest bit in which min and max differ (one warp-wide
// REDUX per bit), and the ordered compaction uses ballots. No shared memory, no block barriers.
// ---------------------------------------------------------------------------------------------------
constexpr int kWarpSelThreads = 256;

template <int KPL>
__global__ void __launch_bounds__(kWarpSelThreads, KPL <= 16 ? 5 : 4) select_warp_kernel(SelectArgs a, uint32_t rows) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t row = blockIdx.x * (kWarpSelThreads / 32) + (threadIdx.x >> 5);
  if (row >= rows) return;  // warp-uniform
  constexpr uint32_t FULL = 0xffffffffu;
  const bool block_mode = (a.mode == kSelBlocks || a.mode == kSelBlocksGeneric);
  const uint32_t B = a.block_size;
  uint32_t n = 0;
  const int32_t* sel_row = nullptr;
  if (a.mode == kSelFlat) {
    n = min(a.pos[row], seq_len_of(a) - 1) + 1;
  } else if (a.mode == kSelBlocks) {
    n = min(min(a.pos[row], seq_len_of(a) - 1) / B, num_blocks_of(a) - 1) + 1;
  } else if (a.mode == kSelCand) {
    const uint32_t t = min(a.pos[row], seq_len_of(a) - 1);
    const uint32_t ns = a.nsel[row];
    sel_row = a.sel + uint64_t(row) * a.sel_row_stride;
    const uint32_t lastb = uint32_t(sel_row[ns - 1]);
    n = (ns - 1) * B + min(B, t - lastb * B + 1);
  } else {
    n = a.n_in[row];
  }
  const float* srow = a.scores + uint64_t(row) * a.stride;
  const uint32_t orow_i = a.out_rows ? a.out_rows[row] : row;  // where this row's result lives in the output arrays
  int32_t* orow = a.out_idx + uint64_t(orow_i) * a.out_stride;
  const uint32_t keep = a.keep;
  const bool forced = block_mode && a.force_first_last && n > 0;
  const uint32_t bshift = a.block_shift;
  auto position_of = [&](uint32_t i) -> int32_t {
    if (a.mode == kSelCand) {
      const uint32_t slot = bshift < 32 ? i >> bshift : i / B;
      return int32_t(uint32_t(sel_row[slot]) * B + (i - slot * B));
    }
    return int32_t(i);
  };
  if (a.out_cand && lane == 0) a.out_cand[orow_i] = n;
  if (n <= keep) {  // dense regime
    for (uint32_t i = lane; i < a.out_width; i += 32) orow[i] = i < n ? position_of(i) : -1;
    if (a.out_count && lane == 0) a.out_count[orow_i] = n;
    return;
  }
  const bool boost = forced && a.forced_in_budget;
  uint32_t key[KPL];
  uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
#pragma unroll
  for (int j = 0; j < KPL; ++j) {
    const uint32_t i = lane + 32u * j;
    uint32_t k = 0u;  // 0 = not a candidate (no finite score maps to key 0)
    if (i < n) {
      k = score_key(srow[i]);
      if (boost && (i == 0 || i == n - 1)) k = 0xFFFFFFFFu;
      kmin = min(kmin, k);
      kmax = max(kmax, k);
    }
    key[j] = k;
  }
  const uint32_t lo = __reduce_min_sync(FULL, kmin), hi = __reduce_max_sync(FULL, kmax);
  // keep-th largest key: range-adaptive 8-bit radix levels on a warp-private shared-memory histogram (256 bins over the
  // range the threshold is known to lie in), finished by ranking the survivors with shuffles once 32 or fewer remain.
  // Distinct scores take one level (n / 256 keys fall into the threshold bin) and the ranking; the bitwise descent this
  // replaces paid ~3 instructions per key for each of ~log2(n) + 4 bits (1670 warp instructions per 512-score row).
  __shared__ __align__(16) uint32_t whist[kWarpSelThreads / 32][256];
  __shared__ uint32_t wlist[kWarpSelThreads / 32][33];  // [32] = fill counter
  uint32_t T = hi, kk = keep;  // after the search: kk = how many keys EQUAL to T are still to take
  const bool all_ties = false;
  if (lo != hi) {
    uint32_t* hist = whist[threadIdx.x >> 5];
    uint32_t* list = wlist[threadIdx.x >> 5];
    uint32_t l = lo, h = hi, in_range = n;
    for (;;) {
      if (l == h) {  // every remaining key is the threshold value
        T = l;
        break;
      }
      const uint32_t span = h - l;
      if (in_range <= 32u) {
        // lane i receives one of the keys of [l, h], in any order (non-candidates are key 0: 0 - l wraps past every span)
        if (lane == 0) list[32] = 0u;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < KPL; ++j)
          if (key[j] - l <= span) list[atomicAdd(&list[32], 1u)] = key[j];
        __syncwarp();
        const uint32_t mine = lane < in_range ? list[lane] : 0u;
        uint32_t g = 0, eq = 0;
        for (uint32_t i = 0; i < in_range; ++i) {
          const uint32_t o = __shfl_sync(FULL, mine, int(i));
          g += o > mine;
          eq += o == mine;
        }
        const bool is_t = lane < in_range && g < kk && kk <= g + eq;  // true for every lane holding the threshold value
        const int src = __ffs(__ballot_sync(FULL, is_t)) - 1;
        T = __shfl_sync(FULL, mine, src);
        kk -= __shfl_sync(FULL, g, src);
        break;
      }
      const uint32_t nb = 32 - __clz(span);
      const uint32_t shift = nb > 8u ? nb - 8u : 0u;
      reinterpret_cast<uint4*>(hist)[lane * 2] = make_uint4(0u, 0u, 0u, 0u);
      reinterpret_cast<uint4*>(hist)[lane * 2 + 1] = make_uint4(0u, 0u, 0u, 0u);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        const uint32_t d = key[j] - l;
        if (d <= span) atomicAdd(&hist[d >> shift], 1u);
      }
      __syncwarp();
      // lane owns bins 8 lane .. 8 lane + 7; suffix sums over lanes find the bin that holds the kk-th largest key
      const uint4 ha = reinterpret_cast<const uint4*>(hist)[lane * 2], hb4 = reinterpret_cast<const uint4*>(hist)[lane * 2 + 1];
      const uint32_t hb[8] = {ha.x, ha.y, ha.z, ha.w, hb4.x, hb4.y, hb4.z, hb4.w};
      const uint32_t loc = ha.x + ha.y + ha.z + ha.w + hb4.x + hb4.y + hb4.z + hb4.w;
      uint32_t inc = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_down_sync(FULL, inc, o);
        if (lane + o < 32u) inc += y;
      }
      const uint32_t above = inc - loc;  // keys in bins owned by higher lanes
      const bool owner = above < kk && kk <= above + loc;
      uint32_t c = above, bj = 7u, cnt = hb[7];
#pragma unroll
      for (int jj = 7; jj > 0; --jj) {
        if (bj == uint32_t(jj) && c + hb[jj] < kk) {
          c += hb[jj];
          bj = uint32_t(jj - 1);
          cnt = hb[jj - 1];
        }
      }
      const int src = __ffs(__ballot_sync(FULL, owner)) - 1;  // exactly one lane owns the threshold bin
      const uint32_t bin = __shfl_sync(FULL, lane * 8u + bj, src);
      kk -= __shfl_sync(FULL, c, src);
      in_range = __shfl_sync(FULL, cnt, src);
      l += bin << shift;
      h = l + min(h - l, (1u << shift) - 1u);  // (l + width may pass 2^32 in the top bin: boosted keys are 0xFFFFFFFF)
    }
  }
  uint32_t cG = 0, cE = 0;
#pragma unroll
  for (int j = 0; j < KPL; ++j) {
    cG += key[j] > T;
    cE += key[j] == T;
  }
  const uint32_t totG = __reduce_add_sync(FULL, cG), totE = __reduce_add_sync(FULL, cE);
  const uint32_t need = all_ties ? totE : kk;  // ties (key == T) to take
  const uint32_t skip = a.tie_break ? totE - need : 0u;
  uint32_t add_first = 0, add_last = 0;
  if (forced) {
    const uint32_t k0 = __shfl_sync(FULL, key[0], 0);
    uint32_t kl_local = 0;
#pragma unroll
    for (int j = 0; j < KPL; ++j)
      if (lane + 32u * j == n - 1) kl_local = key[j];
    const uint32_t kl = __reduce_max_sync(FULL, kl_local);
    const bool sel0 = k0 > T || (k0 == T && skip == 0);
    const bool sell = kl > T || (kl == T && (totE - 1 >= skip) && (totE - 1 < skip + need));
    add_first = sel0 ? 0u : 1u;
    add_last = sell ? 0u : 1u;
  }
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t o_run = add_first, e_run = 0;
  if (need == totE) {  // every key equal to T is kept (the usual case): one ballot per 32 keys
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      if (32u * j >= n) break;  // warp-uniform
      const bool emit = key[j] >= T;
      const uint32_t bm = __ballot_sync(FULL, emit);
      if (emit) orow[o_run + __popc(bm & lt)] = position_of(lane + 32u * j);
      o_run += __popc(bm);
    }
  } else {
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      if (32u * j >= n) break;  // warp-uniform
      const bool g = key[j] > T, e = key[j] == T;
      const uint32_t be = __ballot_sync(FULL, e);
      const uint32_t erank = e_run + __popc(be & lt);
      const bool emit = g || (e && erank >= skip && erank < skip + need);
      const uint32_t bm = __ballot_sync(FULL, emit);
      if (emit) orow[o_run + __popc(bm & lt)] = position_of(lane + 32u * j);
      o_run += __popc(bm);
      e_run += __popc(be);
    }
  }
  const uint32_t count = totG + need + add_first + add_last;
  if (lane == 0) {
    if (add_first) orow[0] = position_of(0);
    if (add_last) orow[count - 1] = position_of(n - 1);
    if (a.out_count) a.out_count[orow_i] = count;
  }
  for (uint32_t i = count + lane; i < a.out_width; i += 32) orow[i] = -1;
}

// ---------------------------------------------------------------------------------------------------
// CTA-per-row selection for medium rows (n_cap <= THREADS * PER4 * 4; the stage-2 candidate pool of
// (m+2)*B = 8448 scores is the case it is sized for). Same result as select_rows_kernel, built for fewer
// instructions and barriers per row:
//   * the score row arrives by ONE bulk copy (cp.async.bulk -> mbarrier), no register staging;
//   * every pass over the keys is 128-bit (LDS.128), strided for the histogram passes, blocked (each thread
//     owns PER4*4 consecutive keys; PER4 odd keeps the 128-bit accesses conflict-free) for the ordered output;
//   * after the first 11-bit range-adaptive level the few survivors are ranked directly (all-pairs count),
//     which replaces the two remaining radix levels in the common case;
//   * one packed block scan (greater | equal << 16) instead of two; ties only take the slow per-key path
//     when the threshold value really is shared;
//   * indices are staged in shared memory (the dead histogram) and leave as coalesced 128-bit stores
//     together with the -1 padding.
// ---------------------------------------------------------------------------------------------------
template <int THREADS>
__device__ __forceinline__ uint32_t block_scan_excl_packed(uint32_t v, uint32_t* wsum, uint32_t& total) {
  // wsum: THREADS/32 words, must not be in use by a previous call without an intervening barrier
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  uint32_t before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < THREADS / 32; ++w) {
    const uint32_t x = wsum[w];
    before += w < warp ? x : 0u;
    tot += x;
  }
  total = tot;
  return before + inc - v;
}

template <int THREADS, int PER4>
__global__ void __launch_bounds__(THREADS) select_cta_kernel(SelectArgs a) {
  constexpr uint32_t CAP = THREADS * PER4 * 4;
  constexpr uint32_t CAP4 = CAP / 4;
  constexpr int NW = THREADS / 32;
  extern __shared__ __align__(16) uint32_t smem_u[];
  uint32_t* skey = smem_u;                   // [CAP] scores, then keys
  uint32_t* hist = skey + CAP;               // [kBins]; reused as the index staging [<= kBins]
  uint32_t* list = hist + kBins;             // [kListCap]
  uint32_t* ssel = list + kListCap;          // [sel_stride]
  uint32_t* scratch = ssel + a.sel_stride;   // [96]
  __shared__ __align__(8) uint64_t bar;

  const uint32_t row = blockIdx.x;
  const uint32_t tid = threadIdx.x;
  const uint32_t lane = tid & 31u;
  const bool block_mode = (a.mode == kSelBlocks || a.mode == kSelBlocksGeneric);
  const uint32_t B = a.block_size;

  uint32_t n = 0;
  const int32_t* sel_row = nullptr;
  uint32_t ns = 0;
  if (a.mode == kSelFlat) {
    n = min(a.pos[row], seq_len_of(a) - 1) + 1;
  } else if (a.mode == kSelBlocks) {
    n = min(min(a.pos[row], seq_len_of(a) - 1) / B, num_blocks_of(a) - 1) + 1;
  } else if (a.mode == kSelCand) {
    const uint32_t t = min(a.pos[row], seq_len_of(a) - 1);
    ns = a.nsel[row];
    sel_row = a.sel + uint64_t(row) * a.sel_row_stride;
    const uint32_t lastb = uint32_t(sel_row[ns - 1]);
    n = (ns - 1) * B + min(B, t - lastb * B + 1);
  } else {
    n = a.n_in[row];
  }
  const float* srow = a.scores + uint64_t(row) * a.stride;
  const uint32_t orow_i = a.out_rows ? a.out_rows[row] : row;  // where this row's result lives in the output arrays
  int32_t* orow = a.out_idx + uint64_t(orow_i) * a.out_stride;
  const uint32_t keep = a.keep;
  const bool forced = block_mode && a.force_first_last && n > 0;
  const uint32_t bshift = a.block_shift;
  auto position_of = [&](uint32_t i) -> int32_t {
    if (a.mode == kSelCand) {
      const uint32_t slot = bshift < 32 ? i >> bshift : i / B;
      return int32_t(ssel[slot] * B + (i - slot * B));
    }
    return int32_t(i);
  };
  if (a.out_cand && tid == 0) a.out_cand[orow_i] = n;

  const bool dense = n <= keep;
  const uint32_t n4 = (n + 3u) >> 2;  // 16-byte chunks that hold candidates
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    if (!dense) {
      mbar_arrive_expect_tx(&bar, n4 * 16u);
      bulk_load_1d(skey, srow, n4 * 16u, &bar);  // may read up to 3 floats past n: still inside the row's stride
    }
    scratch[0] = 0xFFFFFFFFu;  // min key
    scratch[1] = 0u;           // max key
    scratch[2] = 0u;           // list fill
  }
  for (uint32_t i = tid; i < ns; i += THREADS) ssel[i] = uint32_t(sel_row[i]);
  for (uint32_t i = tid; i < kBins / 4; i += THREADS) reinterpret_cast<uint4*>(hist)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();

  if (dense) {  // everything fits
    for (uint32_t i = tid; i < a.out_width; i += THREADS) orow[i] = i < n ? position_of(i) : -1;
    if (a.out_count && tid == 0) a.out_count[orow_i] = n;
    return;
  }
  mbar_wait(&bar, 0);

  // ---- scores -> keys in place, min / max ------------------------------------------------------------
  const bool boost = forced && a.forced_in_budget;
  uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
  for (uint32_t c = tid; c < CAP4; c += THREADS) {
    uint4 kq = make_uint4(0u, 0u, 0u, 0u);  // 0 = not a candidate (no finite score maps to key 0)
    if (c < n4) {
      const float4 v = reinterpret_cast<const float4*>(skey)[c];
      const uint32_t i0 = c << 2;
      kq.x = score_key(v.x);
      kq.y = i0 + 1 < n ? score_key(v.y) : 0u;
      kq.z = i0 + 2 < n ? score_key(v.z) : 0u;
      kq.w = i0 + 3 < n ? score_key(v.w) : 0u;
      if (boost) {
        if (i0 == 0) kq.x = 0xFFFFFFFFu;
        if (i0 == ((n - 1) & ~3u)) {
          const uint32_t e = (n - 1) & 3u;
          if (e == 0) kq.x = 0xFFFFFFFFu; else if (e == 1) kq.y = 0xFFFFFFFFu; else if (e == 2) kq.z = 0xFFFFFFFFu; else kq.w = 0xFFFFFFFFu;
        }
      }
      kmax = max(max(kmax, kq.x), max(max(kq.y, kq.z), kq.w));
      kmin = min(kmin, kq.x);
      if (kq.y) kmin = min(kmin, kq.y);
      if (kq.z) kmin = min(kmin, kq.z);
      if (kq.w) kmin = min(kmin, kq.w);
    }
    reinterpret_cast<uint4*>(skey)[c] = kq;
  }
  kmin = __reduce_min_sync(0xffffffffu, kmin);
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  if (lane == 0) {
    atomicMin(&scratch[0], kmin);
    atomicMax(&scratch[1], kmax);
  }
  __syncthreads();
  uint32_t lo = scratch[0], hi = scratch[1];

  // ---- threshold: range-adaptive radix levels, finished by direct ranking of the survivors -------------
  uint32_t kk = keep;
  bool use_list = false;
  uint32_t list_n = 0;
  uint32_t T = 0, need = 0;
  bool done = false;
  uint32_t* wsum = scratch + 8;  // [NW] x 2, alternating so consecutive scans need no extra barrier
  uint32_t scan_flip = 0;
  while (!done) {
    if (lo == hi) {
      T = lo;
      need = kk;
      break;
    }
    if (use_list && list_n <= uint32_t(THREADS)) {
      // rank the survivors directly: the kk-th largest of the list is the threshold
      uint32_t mine = 0, g = 0, e = 0;
      if (tid < list_n) {
        mine = list[tid];
        for (uint32_t j = 0; j < list_n; ++j) {
          const uint32_t other = list[j];
          g += other > mine;
          e += other == mine;
        }
        if (g < kk && kk <= g + e) {  // all threads holding this value write the same words
          scratch[4] = mine;
          scratch[5] = kk - g;
        }
      }
      __syncthreads();
      T = scratch[4];
      need = scratch[5];
      break;
    }
    const uint32_t range = hi - lo;
    const uint32_t nb = 32 - __clz(range);
    const uint32_t shift = nb > kBinBits ? nb - kBinBits : 0u;
    if (use_list) {
      for (uint32_t i = tid; i < list_n; i += THREADS) {
        const uint32_t key = list[i];
        if (key >= lo && key <= hi) atomicAdd(&hist[(key - lo) >> shift], 1u);
      }
    } else {
      for (uint32_t c = tid; c < n4; c += THREADS) {
        const uint4 kq = reinterpret_cast<const uint4*>(skey)[c];
        if (kq.x >= lo && kq.x <= hi) atomicAdd(&hist[(kq.x - lo) >> shift], 1u);
        if (kq.y >= lo && kq.y <= hi) atomicAdd(&hist[(kq.y - lo) >> shift], 1u);
        if (kq.z >= lo && kq.z <= hi) atomicAdd(&hist[(kq.z - lo) >> shift], 1u);
        if (kq.w >= lo && kq.w <= hi) atomicAdd(&hist[(kq.w - lo) >> shift], 1u);
      }
    }
    __syncthreads();
    constexpr int BPT = kBins / THREADS;
    uint32_t hb[BPT];
    uint32_t loc = 0;
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      hb[j] = hist[tid * BPT + j];
      loc += hb[j];
    }
    uint32_t total;
    const uint32_t before = block_scan_excl_packed<THREADS>(loc, wsum + scan_flip * NW, total);
    scan_flip ^= 1u;
    const uint32_t above = total - before - loc;  // keys in bins owned by higher threads
    if (above < kk && kk <= above + loc) {
      uint32_t c = above;
      int j = BPT - 1;
#pragma unroll
      for (int jj = BPT - 1; jj > 0; --jj) {
        if (j == jj && c + hb[jj] < kk) {
          c += hb[jj];
          j = jj - 1;
        }
      }
      scratch[80] = tid * BPT + j;
      scratch[81] = c;
      scratch[82] = hb[j];
    }
    __syncthreads();
    const uint32_t bin = scratch[80];
    const uint32_t in_bin = scratch[82];
    kk -= scratch[81];
    lo = lo + (bin << shift);
    const uint32_t width = (shift == 0) ? 0u : ((1u << shift) - 1u);
    hi = lo + min(hi - lo, width);  // (lo + width may pass 2^32 in the top bin: boosted keys are 0xFFFFFFFF)
    if (lo == hi) continue;  // exits at the top of the loop
    if (!use_list && in_bin <= uint32_t(kListCap)) {
      // the remaining work only concerns the keys of this bin: compact them once (order is irrelevant here)
      for (uint32_t c = tid; c < n4; c += THREADS) {
        const uint4 kq = reinterpret_cast<const uint4*>(skey)[c];
        if (kq.x >= lo && kq.x <= hi) list[atomicAdd(&scratch[2], 1u)] = kq.x;
        if (kq.y >= lo && kq.y <= hi) list[atomicAdd(&scratch[2], 1u)] = kq.y;
        if (kq.z >= lo && kq.z <= hi) list[atomicAdd(&scratch[2], 1u)] = kq.z;
        if (kq.w >= lo && kq.w <= hi) list[atomicAdd(&scratch[2], 1u)] = kq.w;
      }
      use_list = true;
      list_n = in_bin;
      if (list_n > uint32_t(THREADS))
        for (uint32_t i = tid; i < kBins / 4; i += THREADS) reinterpret_cast<uint4*>(hist)[i] = make_uint4(0u, 0u, 0u, 0u);
    } else {
      for (uint32_t i = tid; i < kBins / 4; i += THREADS) reinterpret_cast<uint4*>(hist)[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
  }

  // ---- ordered compaction: each thread owns PER4*4 consecutive keys ----------------------------------------
  uint4 kq[PER4];
  uint32_t cG = 0, cE = 0;
#pragma unroll
  for (int j = 0; j < PER4; ++j) {
    kq[j] = reinterpret_cast<const uint4*>(skey)[tid * PER4 + j];
    cG += (kq[j].x > T) + (kq[j].y > T) + (kq[j].z > T) + (kq[j].w > T);
    cE += (kq[j].x == T) + (kq[j].y == T) + (kq[j].z == T) + (kq[j].w == T);
  }
  uint32_t tot;
  const uint32_t pre = block_scan_excl_packed<THREADS>(cG | (cE << 16), wsum + scan_flip * NW, tot);
  const uint32_t totG = tot & 0xFFFFu, totE = tot >> 16;
  const uint32_t gBefore = pre & 0xFFFFu, eBefore = pre >> 16;
  const uint32_t skip = a.tie_break ? totE - need : 0u;
  uint32_t add_first = 0, add_last = 0;
  if (forced) {
    const uint32_t k0 = skey[0], kl = skey[n - 1];
    const bool sel0 = k0 > T || (k0 == T && skip == 0);
    const bool sell = kl > T || (kl == T && (totE - 1 >= skip) && (totE - 1 < skip + need));
    add_first = sel0 ? 0u : 1u;
    add_last = sell ? 0u : 1u;
  }
  const uint32_t count = totG + need + add_first + add_last;
  const bool staged = count <= uint32_t(kBins);  // the histogram is dead: stage the indices there
  const uint32_t tiesBefore = eBefore > skip ? min(eBefore - skip, need) : 0u;
  uint32_t o = gBefore + tiesBefore + add_first;
  uint32_t e = eBefore;
  const bool all_ties = need == totE;
  auto put = [&](uint32_t where, int32_t v) {
    if (staged) hist[where] = uint32_t(v);
    else orow[where] = v;
  };
#pragma unroll
  for (int j = 0; j < PER4; ++j) {
    const uint32_t i0 = (tid * PER4 + j) << 2;
    const uint32_t ks[4] = {kq[j].x, kq[j].y, kq[j].z, kq[j].w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t key = ks[u];
      bool emit = key > T;
      if (key == T) {
        emit = all_ties || ((e >= skip) && (e < skip + need));
        ++e;
      }
      if (emit) put(o++, position_of(i0 + u));
    }
  }
  if (tid == 0) {
    if (add_first) put(0, position_of(0));
    if (add_last) put(count - 1, position_of(n - 1));
    if (a.out_count) a.out_count[orow_i] = count;
  }
  if (staged) {
    __syncthreads();
    if (a.vec_out) {
      const uint32_t w4 = a.out_width >> 2;
      for (uint32_t c = tid; c < w4; c += THREADS) {
        const uint32_t i0 = c << 2;
        int4 v;
        v.x = i0 + 0 < count ? int32_t(hist[i0 + 0]) : -1;
        v.y = i0 + 1 < count ? int32_t(hist[i0 + 1]) : -1;
        v.z = i0 + 2 < count ? int32_t(hist[i0 + 2]) : -1;
        v.w = i0 + 3 < count ? int32_t(hist[i0 + 3]) : -1;
        reinterpret_cast<int4*>(orow)[c] = v;
      }
      for (uint32_t i = (w4 << 2) + tid; i < a.out_width; i += THREADS) orow[i] = i < count ? int32_t(hist[i]) : -1;
    } else {
      for (uint32_t i = tid; i < a.out_width; i += THREADS) orow[i] = i < count ? int32_t(hist[i]) : -1;
    }
  } else {
    for (uint32_t i = count + tid; i < a.out_width; i += THREADS) orow[i] = -1;
  }
}

// ---------------------------------------------------------------------------------------------------
// CTA-per-row top-k over token candidates with the keys held in REGISTERS (modes kSelFlat / kSelCand /
// kSelGeneric, n_cap <= THREADS * PER4 * 4; sized for the stage-2 pool of (m+2)*B = 8448 scores, k = 2048).
// select_cta_kernel re-read its shared-memory keys in every pass and spent ~85 thread-instructions per key;
// this kernel touches shared memory once per key (blocked LDS.128: thread t owns keys [36 t, 36 t + 36)) and
// every later pass is register arithmetic:
//   * histogram level: key - lo, one unsigned compare (also rejects the zero keys of non-candidates), shift,
//     RED.shared;
//   * levels repeat on the registers until the threshold bin holds <= THREADS keys, which are compacted and
//     ranked all-pairs: that yields the threshold T, how many keys equal to T are kept, and how many exist;
//   * ordered output: one bit per key (key >= T when every tie is kept, the common case), popc + one block scan,
//     then a loop over the SET bits only; a thread's 36 consecutive candidates span at most two selected blocks,
//     so their token positions are idx + one of two per-thread deltas;
//   * indices are staged in the dead histogram and leave as coalesced 128-bit stores with the -1 padding.
// ---------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t score_key_fast(float f) {
  const uint32_t b = __float_as_uint(f + 0.0f);  // -0 + +0 = +0: both zeros share a key
  return b ^ (uint32_t(int32_t(b) >> 31) | 0x80000000u);
}

// hist[(d >> shift)] += 1 when d <= span, as ONE predicated RED on a 32-bit shared address (the generic-pointer
// atomicAdd cost ten instructions per key: a branch pair and a re-derived shared window base around every ATOMS)
__device__ __forceinline__ void hist_inc_if_le(uint32_t hist_addr, uint32_t d, uint32_t span, uint32_t shift) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .u32 t;\n\t"
      "setp.le.u32 p, %1, %2;\n\t"
      "shr.u32 t, %1, %3;\n\t"
      "shl.b32 t, t, 2;\n\t"
      "add.u32 t, t, %0;\n\t"
      "@p red.shared.add.u32 [t], 1;\n\t}"
      ::"r"(hist_addr), "r"(d), "r"(span), "r"(shift)
      : "memory");
}
// mask |= bit when d <= span
__device__ __forceinline__ void or_bit_if_le(uint32_t& mask, uint32_t d, uint32_t span, uint32_t bit) {
  asm("{\n\t.reg .pred p;\n\t"
      "setp.le.u32 p, %1, %2;\n\t"
      "@p or.b32 %0, %0, %3;\n\t}"
      : "+r"(mask)
      : "r"(d), "r"(span), "r"(bit));
}
__device__ __forceinline__ uint32_t atom_shared_inc(uint32_t addr) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(addr) : "memory");
  return old;
}

// k[e] for a run-time e: a switch over the (compile-time sized) register array; a few cycles, no memory access
template <int KPT>
__device__ __forceinline__ uint32_t pick_key(const uint32_t (&k)[KPT], uint32_t e) {
  uint32_t v = 0;
#define HISA_PICK4(b) \
  case (b): v = k[(b) < KPT ? (b) : 0]; break; case (b) + 1: v = k[(b) + 1 < KPT ? (b) + 1 : 0]; break; \
  case (b) + 2: v = k[(b) + 2 < KPT ? (b) + 2 : 0]; break; case (b) + 3: v = k[(b) + 3 < KPT ? (b) + 3 : 0]; break;
  switch (e) {
    HISA_PICK4(0) HISA_PICK4(4) HISA_PICK4(8) HISA_PICK4(12) HISA_PICK4(16) HISA_PICK4(20) HISA_PICK4(24) HISA_PICK4(28)
    HISA_PICK4(32) HISA_PICK4(36) HISA_PICK4(40) HISA_PICK4(44) HISA_PICK4(48) HISA_PICK4(52) HISA_PICK4(56) HISA_PICK4(60)
    default: break;
  }
#undef HISA_PICK4
  return v;
}

template <int THREADS, int PER4>
// 64 registers per thread: four 256-thread CTAs per SM (at 72 registers three fit, and the kernel is latency-bound per
// warp: 1.36 -> 1.17 ms at C3 from the fourth CTA alone)
__global__ void __launch_bounds__(THREADS, THREADS == 256 ? 4 : 2) select_tok_kernel(SelectArgs a) {
  constexpr int KPT = PER4 * 4;
  constexpr uint32_t CAP = THREADS * KPT;
  constexpr int NW = THREADS / 32;
  constexpr int BPT = kBins / THREADS;
  static_assert(KPT <= 64, "two 32-bit emit masks per thread");
  static_assert(BPT % 4 == 0, "each thread owns whole 16-byte groups of histogram bins");
  extern __shared__ __align__(16) uint32_t smem_u[];
  uint32_t* skey = smem_u;                  // [CAP] scores as delivered by the bulk copy
  uint32_t* hist = skey + CAP;              // [kBins]; reused as the index staging
  uint32_t* list = hist + kBins;            // [THREADS] survivors of the last radix level
  uint32_t* ssel = list + THREADS;          // [sel_stride]
  uint32_t* scratch = ssel + a.sel_stride;  // [96]
  __shared__ __align__(8) uint64_t bar;
  const uint32_t hist_addr = smem_u32(hist), list_addr = smem_u32(list), fill_addr = smem_u32(scratch + 2);

  const uint32_t row = blockIdx.x;
  const uint32_t tid = threadIdx.x;
  const uint32_t lane = tid & 31u;
  const uint32_t B = a.block_size;
  const bool cand = a.mode == kSelCand;

  uint32_t n = 0, ns = 0;
  const int32_t* sel_row = nullptr;
  if (a.mode == kSelFlat) {
    n = min(a.pos[row], seq_len_of(a) - 1) + 1;
  } else if (cand) {
    const uint32_t t = min(a.pos[row], seq_len_of(a) - 1);
    ns = a.nsel[row];
    sel_row = a.sel + uint64_t(row) * a.sel_row_stride;
    // the last selected block: with force_first_last it is the local block (the last block the summaries cover at or
    // before t), known without reading the list: one dependent global load less before the row's copy can be requested
    const uint32_t lastb = a.force_first_last ? min(t / B, num_blocks_of(a) - 1) : uint32_t(sel_row[ns - 1]);
    n = (ns - 1) * B + min(B, t - lastb * B + 1);
  } else {
    n = a.n_in[row];
  }
  const float* srow = a.scores + uint64_t(row) * a.stride;
  const uint32_t orow_i = a.out_rows ? a.out_rows[row] : row;  // where this row's result lives in the output arrays
  int32_t* orow = a.out_idx + uint64_t(orow_i) * a.out_stride;
  const uint32_t keep = a.keep;
  const uint32_t bshift = a.block_shift;
  auto position_of = [&](uint32_t i) -> int32_t {
    if (cand) {
      const uint32_t slot = bshift < 32 ? i >> bshift : i / B;
      return int32_t(ssel[slot] * B + (i - slot * B));
    }
    return int32_t(i);
  };
  if (a.out_cand && tid == 0) a.out_cand[orow_i] = n;

  const bool dense = n <= keep;
  const uint32_t n4 = (n + 3u) >> 2;  // 16-byte chunks that hold candidates
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    if (!dense) {
      mbar_arrive_expect_tx(&bar, n4 * 16u);
      bulk_load_1d(skey, srow, n4 * 16u, &bar);  // may read up to 3 floats past n: still inside the row's stride
    }
    scratch[0] = 0xFFFFFFFFu;  // min key
    scratch[1] = 0u;           // max key
    scratch[2] = 0u;           // list fill
  }
  for (uint32_t i = tid; i < ns; i += THREADS) ssel[i] = uint32_t(sel_row[i]);
#pragma unroll
  for (int j = 0; j < BPT / 4; ++j) reinterpret_cast<uint4*>(hist)[tid * (BPT / 4) + j] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();

  if (dense) {  // everything fits
    for (uint32_t i = tid; i < a.out_width; i += THREADS) {
      const int32_t v = i < n ? position_of(i) : -1;
      orow[i] = v;
      for (uint32_t r = 0; r < a.n_rep; ++r) a.rep_out[r][uint64_t(orow_i) * a.out_stride + i] = v;
    }
    if (tid == 0) {
      if (a.out_count) a.out_count[orow_i] = n;
      for (uint32_t r = 0; r < a.n_rep; ++r)
        if (a.rep_count[r]) a.rep_count[r][orow_i] = n;
    }
    return;
  }
  mbar_wait(&bar, 0);

  // ---- scores -> keys in registers (0 = not a candidate: no finite score maps to key 0), min / max ------
  uint32_t k[KPT];
  const uint32_t first = tid * KPT;
  {
    const uint32_t c0 = tid * PER4;
#pragma unroll
    for (int j = 0; j < PER4; ++j) {
      // chunks past the copied range hold stale shared memory: never read them as scores
      const float4 v = c0 + j < n4 ? reinterpret_cast<const float4*>(skey)[c0 + j] : make_float4(0.f, 0.f, 0.f, 0.f);
      k[4 * j + 0] = score_key_fast(v.x);
      k[4 * j + 1] = score_key_fast(v.y);
      k[4 * j + 2] = score_key_fast(v.z);
      k[4 * j + 3] = score_key_fast(v.w);
    }
  }
  // One code path for every thread (a warp that runs a "full" and a "partial" variant side by side arrives late at the
  // next barrier): non-candidates are key 0, which max() ignores and which k - 1 turns into the largest value for min()
  if (first + KPT > n) {
#pragma unroll
    for (int e = 0; e < KPT; ++e)
      if (first + e >= n) k[e] = 0u;
  }
  uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
#pragma unroll
  for (int e = 0; e < KPT; ++e) {
    kmin = min(kmin, k[e] - 1u);
    kmax = max(kmax, k[e]);
  }
  kmin = first < n ? kmin + 1u : 0xFFFFFFFFu;
  kmin = __reduce_min_sync(0xffffffffu, kmin);
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  if (lane == 0) {
    atomicMin(&scratch[0], kmin);
    atomicMax(&scratch[1], kmax);
  }
  __syncthreads();
  uint32_t lo = scratch[0], hi = scratch[1];

  // ---- threshold: range-adaptive radix levels on the registers, finished by ranking the survivors -------
  uint32_t kk = keep;        // rank of the threshold among the keys still in [lo, hi]
  uint32_t in_range = n;     // number of keys in [lo, hi]
  uint32_t T = 0, need = 0, totE = 0;
  uint32_t* wsum = scratch + 8;  // [NW] x 2, alternating so consecutive scans need no extra barrier
  uint32_t scan_flip = 0;
  for (;;) {
    if (lo == hi) {  // every remaining key is the threshold value
      T = lo;
      need = kk;
      totE = in_range;
      break;
    }
    const uint32_t span = hi - lo;
    if (in_range <= uint32_t(THREADS)) {
      // compact the keys of the threshold range (order is irrelevant) and rank them all-pairs
      {
        uint32_t h0 = 0, h1 = 0;  // bit e <=> key e lies in the threshold range (few threads have any)
#pragma unroll
        for (int e = 0; e < KPT; ++e) {  // subtract, compare, predicated OR with an immediate
          if (e < 32) or_bit_if_le(h0, k[e] - lo, span, 1u << e);
          else or_bit_if_le(h1, k[e] - lo, span, 1u << (e - 32));
        }
        // few threads own a key of the threshold range: they fetch it from the register file with a jump over the KPT
        // cases (pick_key) instead of every warp walking a KPT-way predicated sequence (154 instructions per warp and row)
        for (uint32_t hh = h0; hh; hh &= hh - 1)
          sts_u32(list_addr + atom_shared_inc(fill_addr) * 4u, pick_key<KPT>(k, uint32_t(__ffs(hh)) - 1u));
        for (uint32_t hh = h1; hh; hh &= hh - 1)
          sts_u32(list_addr + atom_shared_inc(fill_addr) * 4u, pick_key<KPT>(k, 31u + uint32_t(__ffs(hh))));
      }
      __syncthreads();
      if (tid < in_range) {
        const uint32_t mine = list[tid];
        uint32_t g = 0, eq = 0;
        for (uint32_t j = 0; j < in_range; ++j) {
          const uint32_t other = list[j];
          g += other > mine;
          eq += other == mine;
        }
        if (g < kk && kk <= g + eq) {  // all threads holding this value write the same words
          scratch[4] = mine;
          scratch[5] = kk - g;
          scratch[6] = eq;
        }
      }
      __syncthreads();
      T = scratch[4];
      need = scratch[5];
      totE = scratch[6];
      break;
    }
    const uint32_t nb = 32 - __clz(span);
    const uint32_t shift = nb > kBinBits ? nb - kBinBits : 0u;
#pragma unroll
    for (int e = 0; e < KPT; ++e) hist_inc_if_le(hist_addr, k[e] - lo, span, shift);  // zero keys wrap to a huge value
    __syncthreads();
    uint32_t hb[BPT];
    uint32_t loc = 0;
    {
      const uint4* h4 = reinterpret_cast<const uint4*>(hist) + tid * (BPT / 4);
#pragma unroll
      for (int j = 0; j < BPT / 4; ++j) {
        const uint4 h = h4[j];
        hb[4 * j + 0] = h.x; hb[4 * j + 1] = h.y; hb[4 * j + 2] = h.z; hb[4 * j + 3] = h.w;
        loc += h.x + h.y + h.z + h.w;
      }
    }
    uint32_t total;
    const uint32_t before = block_scan_excl_packed<THREADS>(loc, wsum + scan_flip * NW, total);
    scan_flip ^= 1u;
    const uint32_t above = total - before - loc;  // keys in bins owned by higher threads
    if (above < kk && kk <= above + loc) {
      uint32_t c = above;
      int j = BPT - 1;
#pragma unroll
      for (int jj = BPT - 1; jj > 0; --jj) {
        if (j == jj && c + hb[jj] < kk) {
          c += hb[jj];
          j = jj - 1;
        }
      }
      scratch[80] = tid * BPT + j;
      scratch[81] = c;
      scratch[82] = hb[j];
    }
    // the histogram words this thread owns are dead now: clear them for the next level / keep them clean
#pragma unroll
    for (int j = 0; j < BPT / 4; ++j) reinterpret_cast<uint4*>(hist)[tid * (BPT / 4) + j] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    const uint32_t bin = scratch[80];
    in_range = scratch[82];
    kk -= scratch[81];
    lo = lo + (bin << shift);
    const uint32_t width = (shift == 0) ? 0u : ((1u << shift) - 1u);
    hi = lo + min(hi - lo, width);  // (lo + width may pass 2^32 in the top bin: boosted keys are 0xFFFFFFFF)
  }

  // ---- ordered output -------------------------------------------------------------------------------------
  // bit e of (m0, m1) <=> key e of this thread is emitted
  uint32_t m0 = 0, m1 = 0;
  const bool all_ties = need == totE;
  uint32_t cE = 0;
  if (all_ties) {
#pragma unroll
    for (int e = 0; e < KPT; ++e) {  // k >= T  <=>  k - T <= ~T as unsigned (k < T wraps above ~T)
      if (e < 32) or_bit_if_le(m0, k[e] - T, ~T, 1u << e);
      else or_bit_if_le(m1, k[e] - T, ~T, 1u << (e - 32));
    }
  } else {
#pragma unroll
    for (int e = 0; e < KPT; ++e) {
      if (k[e] > T) {
        if (e < 32) m0 |= 1u << e; else m1 |= 1u << (e - 32);
      }
      cE += k[e] == T;
    }
  }
  uint32_t tot;
  uint32_t pre = block_scan_excl_packed<THREADS>((__popc(m0) + __popc(m1)) | (cE << 16), wsum + scan_flip * NW, tot);
  scan_flip ^= 1u;
  uint32_t o = pre & 0xFFFFu;
  if (!all_ties) {
    // only `need` of the totE keys equal to T are kept: the first ones (SmallestIndex) or the last ones
    const uint32_t skip = a.tie_break ? totE - need : 0u;
    uint32_t eidx = pre >> 16;
    o += eidx > skip ? min(eidx - skip, need) : 0u;
#pragma unroll
    for (int e = 0; e < KPT; ++e) {
      if (k[e] == T) {
        if (eidx >= skip && eidx < skip + need) {
          if (e < 32) m0 |= 1u << e; else m1 |= 1u << (e - 32);
        }
        ++eidx;
      }
    }
  }
  const uint32_t count = keep;  // n > keep here, so exactly `keep` candidates are selected
  const bool staged = count <= uint32_t(kBins);  // the histogram is dead: stage the indices there
  // candidate mode: the thread's KPT consecutive candidates lie in at most two selected blocks when B >= KPT
  int32_t delta0 = 0, delta1 = 0;
  uint32_t boundary = 0xFFFFFFFFu;
  const bool two_block = cand && bshift < 32 && B >= uint32_t(KPT);
  if (two_block) {
    const uint32_t slot0 = first >> bshift;
    boundary = (slot0 + 1) << bshift;
    delta0 = slot0 < ns ? int32_t((ssel[slot0] - slot0) << bshift) : 0;
    delta1 = slot0 + 1 < ns ? int32_t((ssel[slot0 + 1] - (slot0 + 1)) << bshift) : 0;
  }
  if (staged && (two_block || !cand)) {
    // common case, branch-free body: position = idx + per-thread delta, staged through shared memory
    if (!cand) boundary = 0xFFFFFFFFu;  // identity mapping: delta0 = delta1 = 0
    uint32_t oaddr = hist_addr + o * 4u;
    while (m0) {
      const uint32_t idx = first + __ffs(m0) - 1;
      m0 &= m0 - 1;
      sts_u32(oaddr, idx + uint32_t(idx < boundary ? delta0 : delta1));
      oaddr += 4;
    }
    while (m1) {
      const uint32_t idx = first + 31 + __ffs(m1);
      m1 &= m1 - 1;
      sts_u32(oaddr, idx + uint32_t(idx < boundary ? delta0 : delta1));
      oaddr += 4;
    }
  } else {
    auto emit = [&](uint32_t idx) {
      const int32_t v = position_of(idx);
      if (staged) hist[o] = uint32_t(v);
      else orow[o] = v;
      ++o;
    };
    while (m0) {
      const uint32_t e = __ffs(m0) - 1;
      m0 &= m0 - 1;
      emit(first + e);
    }
    while (m1) {
      const uint32_t e = __ffs(m1) - 1;
      m1 &= m1 - 1;
      emit(first + 32 + e);
    }
  }
  if (tid == 0 && a.out_count) a.out_count[orow_i] = count;
  if (tid == 0)
    for (uint32_t r = 0; r < a.n_rep; ++r)
      if (a.rep_count[r]) a.rep_count[r][orow_i] = count;
  if (staged) {
    __syncthreads();
    if (a.vec_out) {
      const uint32_t w4 = a.out_width >> 2;
      for (uint32_t c = tid; c < w4; c += THREADS) {
        const uint32_t i0 = c << 2;
        int4 v;
        if (i0 + 3 < count) {
          v = reinterpret_cast<const int4*>(hist)[c];
        } else {
          v.x = i0 + 0 < count ? int32_t(hist[i0 + 0]) : -1;
          v.y = i0 + 1 < count ? int32_t(hist[i0 + 1]) : -1;
          v.z = i0 + 2 < count ? int32_t(hist[i0 + 2]) : -1;
          v.w = i0 + 3 < count ? int32_t(hist[i0 + 3]) : -1;
        }
        reinterpret_cast<int4*>(orow)[c] = v;
        // fused all-gather: the same 16 bytes go to the row's place in every peer GPU's [Q, k] matrix (NVLink stores
        // to peer memory), so the selection kernel IS the collective and no staging copy or permutation follows it
        for (uint32_t r = 0; r < a.n_rep; ++r)
          reinterpret_cast<int4*>(a.rep_out[r] + uint64_t(orow_i) * a.out_stride)[c] = v;
      }
      for (uint32_t i = (w4 << 2) + tid; i < a.out_width; i += THREADS) orow[i] = i < count ? int32_t(hist[i]) : -1;
    } else {
      for (uint32_t i = tid; i < a.out_width; i += THREADS) orow[i] = i < count ? int32_t(hist[i]) : -1;
    }
  } else {
    for (uint32_t i = count + tid; i < a.out_width; i += THREADS) orow[i] = -1;
  }
}

// ---------------------------------------------------------------------------------------------------
// dense work list (stage 1 and the flat indexer): chunk-major items, only tiles a chunk can need.
// ---------------------------------------------------------------------------------------------------
constexpr int kDenseThreads = 1024;
constexpr int kDenseMaxChunks = 4096;

__global__ void __launch_bounds__(kDenseThreads)
build_dense_work_kernel(const uint32_t* __restrict__ pos, uint32_t nq, uint32_t chunk, uint32_t seq_len,
                        uint32_t unit_div, uint32_t ntiles, WorkItem* __restrict__ work,
                        uint32_t* __restrict__ work_count, uint32_t* __restrict__ work_cursor,
                        const uint32_t* __restrict__ dyn_len, uint32_t* __restrict__ zero_a, uint32_t* __restrict__ zero_b) {
  __shared__ uint32_t offs[kDenseMaxChunks + 1];
  __shared__ uint32_t scratch[64];
  if (dyn_len) {  // graph replay: the sequence length lives in device memory; tiles of the operand follow from it
    seq_len = *dyn_len;
    ntiles = min(ntiles, ((seq_len + unit_div - 1) / unit_div + kTileRows - 1) / kTileRows);
  }
  if (threadIdx.x == 0 && zero_a) {  // the counters of the stage-2 work list, cleared here instead of by a launch of their own
    *zero_a = 0;
    *zero_b = 0;
  }
  const uint32_t nchunks = (nq + chunk - 1) / chunk;
  const uint32_t tid = threadIdx.x;
  // tiles needed by each chunk
  uint32_t carry = 0;
  for (uint32_t base = 0; base < nchunks; base += kDenseThreads) {
    const uint32_t c = base + tid;
    uint32_t need = 0;
    if (c < nchunks) {
      uint32_t mp = 0;
      const uint32_t q1 = min(nq, (c + 1) * chunk);
      for (uint32_t q = c * chunk; q < q1; ++q) mp = max(mp, pos[q]);
      mp = min(mp, seq_len - 1);
      need = min(ntiles, (mp / unit_div) / kTileRows + 1);
    }
    uint32_t total;
    const uint32_t before = block_scan_excl<kDenseThreads>(need, scratch, total);
    if (c < nchunks) offs[c] = carry + before;
    carry += total;
    __syncthreads();
  }
  if (tid == 0) {
    offs[nchunks] = carry;
    *work_count = carry;
    *work_cursor = 0;
  }
  __syncthreads();
  const uint32_t total_items = offs[nchunks];
  for (uint32_t it = tid; it < total_items; it += kDenseThreads) {
    uint32_t lo_c = 0, hi_c = nchunks;  // largest c with offs[c] <= it
    while (hi_c - lo_c > 1) {
      const uint32_t mid = (lo_c + hi_c) >> 1;
      if (offs[mid] <= it) lo_c = mid; else hi_c = mid;
    }
    WorkItem w;
    w.tile = it - offs[lo_c];
    w.first = lo_c * chunk;
    w.count = min(nq, (lo_c + 1) * chunk) - lo_c * chunk;
    w.reserved = 0;
    work[it] = w;
  }
}

// ---------------------------------------------------------------------------------------------------
// list work (stage 2): per chunk of queries, group the (query, slot) pairs by selected block.
// One CTA per chunk. pairs for chunk c live at [c*chunk*sel_stride, ...).
// ---------------------------------------------------------------------------------------------------
constexpr int kInvThreads = 256;

__global__ void __launch_bounds__(kInvThreads)
invert_selection_kernel(const int32_t* __restrict__ sel, const uint32_t* __restrict__ nsel, uint32_t sel_stride,
                        uint32_t nq, uint32_t chunk, uint32_t num_blocks, uint32_t block_size,
                        uint32_t segs_per_block, uint32_t split, WorkItem* __restrict__ work,
                        uint32_t* __restrict__ work_count, uint2* __restrict__ pairs, uint32_t* __restrict__ gcount) {
  extern __shared__ __align__(16) uint32_t smem_u[];
  // per-block counters live in shared memory; sequences with more blocks than fit there (gcount != null: 1M tokens at
  // B = 32, or the degenerate B = 1) keep them in a per-chunk slice of global memory instead
  const uint32_t c = blockIdx.x, tid = threadIdx.x;
  uint32_t* cnt = gcount ? gcount + uint64_t(c) * 2u * num_blocks : smem_u + 64;  // [num_blocks]
  uint32_t* off = cnt + num_blocks;                                               // [num_blocks]
  uint32_t* scratch = smem_u;                                                     // [64]
  const uint32_t q0 = c * chunk, q1 = min(nq, q0 + chunk);
  for (uint32_t b = tid; b < num_blocks; b += kInvThreads) cnt[b] = 0;
  __syncthreads();
  for (uint32_t q = q0 + tid; q < q1; q += kInvThreads) {
    const uint32_t ns = nsel[q];
    for (uint32_t s = 0; s < ns; ++s) atomicAdd(&cnt[uint32_t(sel[uint64_t(q) * sel_stride + s])], 1u);
  }
  __syncthreads();
  // exclusive scan of counts and of the non-empty indicator, blocked over threads
  const uint32_t per = (num_blocks + kInvThreads - 1) / kInvThreads;
  const uint32_t b0 = min(num_blocks, tid * per), b1 = min(num_blocks, b0 + per);
  uint32_t lsum = 0, lne = 0;
  // a block's query list becomes ceil(n / split) work items: the forced blocks (sink, local) are selected by EVERY query
  // of the chunk, and in a call with few rows one such list is a large share of an SM's whole work (decode: 16 of the
  // ~10 groups an SM gets on average), so the host caps the list length per item for small calls
  for (uint32_t b = b0; b < b1; ++b) { lsum += cnt[b]; lne += cnt[b] ? (cnt[b] - 1) / split + 1 : 0u; }
  uint32_t tot_pairs, tot_ne;
  uint32_t pre = block_scan_excl<kInvThreads>(lsum, scratch, tot_pairs);
  uint32_t pne = block_scan_excl<kInvThreads>(lne, scratch, tot_ne);
  if (tid == 0) scratch[48] = atomicAdd(work_count, tot_ne * segs_per_block);
  __syncthreads();
  const uint32_t item_base = scratch[48];
  const uint32_t pair_base = q0 * sel_stride;
  for (uint32_t b = b0; b < b1; ++b) {
    const uint32_t n = cnt[b];
    off[b] = pre;
    for (uint32_t done = 0; done < n; done += split) {
      for (uint32_t j = 0; j < segs_per_block; ++j) {
        WorkItem w;
        w.tile = b * segs_per_block + j;
        w.first = pair_base + pre + done;
        w.count = min(split, n - done);
        w.reserved = 0;
        work[item_base + pne * segs_per_block + j] = w;
      }
      ++pne;
      if (split >= n) break;  // split may be 2^32 - 1: do not let `done += split` wrap
    }
    pre += n;
  }
  __syncthreads();
  for (uint32_t q = q0 + tid; q < q1; q += kInvThreads) {
    const uint32_t ns = nsel[q];
    for (uint32_t s = 0; s < ns; ++s) {
      const uint32_t b = uint32_t(sel[uint64_t(q) * sel_stride + s]);
      const uint32_t idx = atomicAdd(&off[b], 1u);
      pairs[pair_base + idx] = make_uint2(q, s * block_size);
    }
  }
}

// Same list work for a call that is ONE chunk of few queries (decode: 64 queries). The kernel above gives every query one
// thread, which then walks its ~66 selected blocks twice with a dependent global load per step: 14.6 us for 64 queries.
// Here the whole selection (nq x sel_stride entries) is first staged in shared memory by one coalesced pass of independent
// loads, and 1024 threads count and place the (query, slot) pairs from there: one global round trip instead of ~130.
constexpr int kInvSmallThreads = 1024;

__global__ void __launch_bounds__(kInvSmallThreads)
invert_small_kernel(const int32_t* __restrict__ sel, const uint32_t* __restrict__ nsel, uint32_t sel_stride, uint32_t nq,
                    uint32_t num_blocks, uint32_t block_size, uint32_t segs_per_block, uint32_t split,
                    WorkItem* __restrict__ work, uint32_t* __restrict__ work_count, uint2* __restrict__ pairs) {
  extern __shared__ __align__(16) uint32_t smem_u[];
  uint32_t* scratch = smem_u;              // [64]
  uint32_t* cnt = smem_u + 64;             // [num_blocks]
  uint32_t* off = cnt + num_blocks;        // [num_blocks]
  uint32_t* ssel = off + num_blocks;       // [nq * sel_stride]
  uint32_t* sns = ssel + nq * sel_stride;  // [nq]
  const uint32_t tid = threadIdx.x;
  const uint32_t total = nq * sel_stride;
  for (uint32_t i = tid; i < total; i += kInvSmallThreads) ssel[i] = uint32_t(sel[i]);
  for (uint32_t q = tid; q < nq; q += kInvSmallThreads) sns[q] = nsel[q];
  for (uint32_t b = tid; b < num_blocks; b += kInvSmallThreads) cnt[b] = 0;
  __syncthreads();
  for (uint32_t i = tid; i < total; i += kInvSmallThreads) {
    const uint32_t q = i / sel_stride, sl = i - q * sel_stride;
    if (sl < sns[q]) atomicAdd(&cnt[ssel[i]], 1u);
  }
  __syncthreads();
  const uint32_t per = (num_blocks + kInvSmallThreads - 1) / kInvSmallThreads;
  const uint32_t b0 = min(num_blocks, tid * per), b1 = min(num_blocks, b0 + per);
  uint32_t lsum = 0, lne = 0;
  for (uint32_t b = b0; b < b1; ++b) { lsum += cnt[b]; lne += cnt[b] ? (cnt[b] - 1) / split + 1 : 0u; }
  uint32_t tot_pairs, tot_ne;
  uint32_t pre = block_scan_excl<kInvSmallThreads>(lsum, scratch, tot_pairs);
  uint32_t pne = block_scan_excl<kInvSmallThreads>(lne, scratch, tot_ne);
  if (tid == 0) scratch[48] = atomicAdd(work_count, tot_ne * segs_per_block);
  __syncthreads();
  const uint32_t item_base = scratch[48];
  for (uint32_t b = b0; b < b1; ++b) {
    const uint32_t n = cnt[b];
    off[b] = pre;
    for (uint32_t done = 0; done < n; done += split) {
      for (uint32_t j = 0; j < segs_per_block; ++j) {
        WorkItem w;
        w.tile = b * segs_per_block + j;
        w.first = pre + done;
        w.count = min(split, n - done);
        w.reserved = 0;
        work[item_base + pne * segs_per_block + j] = w;
      }
      ++pne;
      if (split >= n) break;
    }
    pre += n;
  }
  __syncthreads();
  for (uint32_t i = tid; i < total; i += kInvSmallThreads) {
    const uint32_t q = i / sel_stride, sl = i - q * sel_stride;
    if (sl < sns[q]) {
      const uint32_t idx = atomicAdd(&off[ssel[i]], 1u);
      pairs[idx] = make_uint2(q, sl * block_size);
    }
  }
}

// Copies finished result rows to the peer replicas (variants that do not store to the peers themselves). One CTA per row.
__global__ void __launch_bounds__(256) replicate_rows_kernel(SelectArgs a) {
  const uint32_t row = blockIdx.x;
  const uint32_t orow_i = a.out_rows ? a.out_rows[row] : row;
  const int32_t* src = a.out_idx + uint64_t(orow_i) * a.out_stride;
  for (uint32_t r = 0; r < a.n_rep; ++r) {
    int32_t* dst = a.rep_out[r] + uint64_t(orow_i) * a.out_stride;
    if (a.vec_out) {
      for (uint32_t c = threadIdx.x; c < (a.out_width >> 2); c += blockDim.x)
        reinterpret_cast<int4*>(dst)[c] = reinterpret_cast<const int4*>(src)[c];
      for (uint32_t i = (a.out_width & ~3u) + threadIdx.x; i < a.out_width; i += blockDim.x) dst[i] = src[i];
    } else {
      for (uint32_t i = threadIdx.x; i < a.out_width; i += blockDim.x) dst[i] = src[i];
    }
    if (threadIdx.x == 0 && a.rep_count[r] && a.out_count) a.rep_count[r][orow_i] = a.out_count[orow_i];
  }
}

__global__ void zero_two_kernel(uint32_t* a, uint32_t* b) {
  *a = 0;
  *b = 0;
}

template <int KPL>
void launch_select_warp(const SelectArgs& args, uint32_t rows, cudaStream_t stream) {
  const uint32_t per_cta = kWarpSelThreads / 32;
  select_warp_kernel<KPL><<<(rows + per_cta - 1) / per_cta, kWarpSelThreads, 0, stream>>>(args, rows);
}

template <int THREADS, int PER4>
void launch_select_cta(const SelectArgs& args, uint32_t rows, cudaStream_t stream) {
  const size_t smem = (size_t(THREADS) * PER4 * 4 + kBins + kListCap + args.sel_stride + 96) * sizeof(uint32_t);
  auto kern = select_cta_kernel<THREADS, PER4>;
  smem_opt_in(reinterpret_cast<const void*>(kern), 200 * 1024);
  kern<<<rows, THREADS, smem, stream>>>(args);
}

template <int THREADS, int PER4>
void launch_select_tok(const SelectArgs& args, uint32_t rows, cudaStream_t stream) {
  const size_t smem = (size_t(THREADS) * PER4 * 4 + kBins + THREADS + args.sel_stride + 96) * sizeof(uint32_t);
  auto kern = select_tok_kernel<THREADS, PER4>;
  smem_opt_in(reinterpret_cast<const void*>(kern), 200 * 1024);
  kern<<<rows, THREADS, smem, stream>>>(args);
}

template <int THREADS, bool SMEM_KEYS>
void launch_select_variant(const SelectArgs& args, uint32_t rows, uint32_t n_cap, cudaStream_t stream) {
  const size_t smem = (size_t(kBins) + 64 + kListCap + args.sel_stride + (SMEM_KEYS ? n_cap : 0)) * sizeof(uint32_t);
  auto kern = select_rows_kernel<THREADS, SMEM_KEYS>;
  if (smem > 48 * 1024) smem_opt_in(reinterpret_cast<const void*>(kern), smem);
  kern<<<rows, THREADS, smem, stream>>>(args);
}

}  // namespace

int launch_select(const SelectArgs& args_in, uint32_t rows, uint32_t n_cap, cudaStream_t stream) {
  if (rows == 0) return 0;
  SelectArgs args = args_in;
  args.sel_row_stride = args_in.sel_stride;
  args.sel_stride = (args_in.mode == kSelCand) ? ((args_in.sel_stride + 3u) & ~3u) : 0u;  // smem words for the block list
  args.vec_ok = (args.stride % 4 == 0) && (reinterpret_cast<uintptr_t>(args.scores) % 16 == 0) ? 1u : 0u;
  const uint32_t B = args.block_size;
  args.block_shift = (B && (B & (B - 1)) == 0) ? uint32_t(__builtin_ctz(B)) : 32u;
  args.vec_out = (args.out_stride % 4 == 0) && (reinterpret_cast<uintptr_t>(args.out_idx) % 16 == 0) ? 1u : 0u;
  const bool legacy = getenv("HISA_SELECT_LEGACY") != nullptr;  // cross-check switches for the tests
  const bool cta_old = getenv("HISA_SELECT_CTA_SMEM") != nullptr;
  const bool block_mode = args.mode == kSelBlocks || args.mode == kSelBlocksGeneric;
  // bulk-copy path: 16-byte aligned rows whose stride covers the rounded-up chunk count
  const bool bulk_ok = args.vec_ok && args.scores != nullptr;
  bool fused_rep = false;  // the variant stores to the peer replicas itself
  if (!legacy && n_cap <= 128) launch_select_warp<4>(args, rows, stream);
  else if (!legacy && n_cap <= 512) launch_select_warp<16>(args, rows, stream);
  else if (!legacy && n_cap <= 1024) launch_select_warp<32>(args, rows, stream);
  else if (!legacy && bulk_ok && !block_mode && !cta_old && n_cap <= 256 * 9 * 4) { launch_select_tok<256, 9>(args, rows, stream); fused_rep = args.vec_out && args.keep <= uint32_t(kBins); }
  else if (!legacy && bulk_ok && !block_mode && !cta_old && n_cap <= 512 * 9 * 4) { launch_select_tok<512, 9>(args, rows, stream); fused_rep = args.vec_out && args.keep <= uint32_t(kBins); }
  else if (!legacy && bulk_ok && n_cap <= 256 * 9 * 4) launch_select_cta<256, 9>(args, rows, stream);
  else if (!legacy && bulk_ok && n_cap <= 512 * 9 * 4) launch_select_cta<512, 9>(args, rows, stream);
  else if (!legacy && bulk_ok && n_cap <= 1024 * 9 * 4) launch_select_cta<1024, 9>(args, rows, stream);
  else if (n_cap <= 2048) launch_select_variant<128, true>(args, rows, n_cap, stream);
  else if (n_cap <= 16384) launch_select_variant<256, true>(args, rows, n_cap, stream);
  else if (n_cap <= 49152) launch_select_variant<1024, true>(args, rows, n_cap, stream);
  else launch_select_variant<1024, false>(args, rows, n_cap, stream);
  if (args.n_rep == 0) return 1;
  if (fused_rep) return 1;
  replicate_rows_kernel<<<rows, 256, 0, stream>>>(args);
  return 2;
}

int launch_build_dense_work(const uint32_t* pos, uint32_t nq, uint32_t chunk, uint32_t seq_len, uint32_t unit_div,
                            uint32_t ntiles, WorkItem* work, uint32_t* work_count, uint32_t* work_cursor,
                            const uint32_t* dyn_len, uint32_t* zero_a, uint32_t* zero_b, cudaStream_t stream) {
  if (nq == 0) return 0;
  build_dense_work_kernel<<<1, kDenseThreads, 0, stream>>>(pos, nq, chunk, seq_len, unit_div, ntiles, work, work_count,
                                                           work_cursor, dyn_len, zero_a, zero_b);
  return 1;
}

int launch_invert_selection(const int32_t* sel, const uint32_t* nsel, uint32_t sel_stride, uint32_t nq, uint32_t chunk,
                            uint32_t num_blocks, uint32_t block_size, uint32_t segs_per_block, uint32_t split,
                            WorkItem* work, uint32_t* work_count, uint32_t* work_cursor, uint2* pairs,
                            uint32_t* global_counters, bool counters_zeroed, cudaStream_t stream) {
  if (nq == 0) return 0;
  int launched = 1;
  if (!counters_zeroed) {
    zero_two_kernel<<<1, 1, 0, stream>>>(work_count, work_cursor);
    launched = 2;
  }
  const uint32_t nchunks_all = (nq + chunk - 1) / chunk;
  const size_t smem_small = (size_t(num_blocks) * 2 + 64 + size_t(nq) * sel_stride + nq) * sizeof(uint32_t);
  if (nchunks_all == 1 && nq <= 1024 && smem_small <= invert_smem_limit() && !getenv("HISA_INVERT_BIG") &&
      (smem_small <= 48 * 1024 || smem_opt_in(reinterpret_cast<const void*>(invert_small_kernel), smem_small))) {
    invert_small_kernel<<<1, kInvSmallThreads, smem_small, stream>>>(sel, nsel, sel_stride, nq, num_blocks, block_size,
                                                                     segs_per_block, split ? split : 0xFFFFFFFFu, work,
                                                                     work_count, pairs);
    return launched;
  }
  size_t smem = (size_t(num_blocks) * 2 + 64) * sizeof(uint32_t);
  uint32_t* gcount = nullptr;
  if (smem > invert_smem_limit()) {
    if (!global_counters) return -1;  // the caller sizes the scratch with invert_global_words()
    gcount = global_counters;
    smem = 64 * sizeof(uint32_t);
  } else if (smem > 48 * 1024 && !smem_opt_in(reinterpret_cast<const void*>(invert_selection_kernel), smem)) {
    return -1;
  }
  const uint32_t nchunks = (nq + chunk - 1) / chunk;
  invert_selection_kernel<<<nchunks, kInvThreads, smem, stream>>>(sel, nsel, sel_stride, nq, chunk, num_blocks,
                                                                  block_size, segs_per_block, split ? split : 0xFFFFFFFFu, work,
                                                                  work_count, pairs, gcount);
  return launched;
}

size_t invert_smem_limit() { return 200 * 1024; }
size_t invert_global_words(uint32_t nq, uint32_t chunk, uint32_t num_blocks) {
  if ((size_t(num_blocks) * 2 + 64) * sizeof(uint32_t) <= invert_smem_limit()) return 0;
  return size_t((nq + chunk - 1) / chunk) * 2u * num_blocks;
}

int launch_expand_blocks(const int32_t* sel, const uint32_t* nsel, uint32_t sel_stride, const uint32_t* pos,
                         uint32_t nq, uint32_t seq_len, uint32_t block_size, int32_t* out_idx, uint64_t out_stride,
                         uint32_t out_width, uint32_t* out_count, cudaStream_t stream) {
  // block_sparse_select (hisa/block_sparse.hpp:12-19) = the dense-regime path of the candidate select:
  // keep >= every possible candidate count, so all causally valid tokens of the selected blocks are emitted.
  SelectArgs a{};
  a.scores = nullptr;
  a.stride = 0;
  a.pos = pos;
  a.seq_len = seq_len;
  a.block_size = block_size;
  a.keep = 0xFFFFFFFFu;
  a.mode = kSelCand;
  a.sel = sel;
  a.nsel = nsel;
  a.sel_stride = sel_stride;
  a.out_idx = out_idx;
  a.out_stride = out_stride;
  a.out_width = out_width;
  a.out_count = out_count;
  return launch_select(a, nq, 1, stream);
}

}  // namespace hisa_dev
