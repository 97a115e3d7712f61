// Fused tensor-core scorer for sm_100a (north-star kernels 2, 4 and 6: block scoring, token refinement
// and the flat DSA scorer are the same kernel over different work lists).
//
//   score[row, key] = sum_j gate[row, j] * relu( q[row, j, :] . key[:] )
//   reference: hisa::score_tokens (proj/core/include/hisa/dsa.hpp:13-20, Eq.1) and hisa::score_blocks
//   (hisa/hisa.hpp:16-21, Eq.5)
//
// Mapping onto Blackwell
//   * UMMA orientation: the 128 operand rows of a tile (keys / pooled keys) are the M axis = 128 TMEM
//     lanes; 4 queries x 64 heads are the N axis = 256 TMEM columns; K = 128 (x segments). After
//     tcgen05.ld each epilogue thread owns ONE key row and sees the 64 per-head dots of a query in its own
//     registers, so gate*ReLU and the head reduction are thread-local: the per-head score matrix exists
//     only in TMEM and never reaches shared memory or HBM.
//   * operands are staged by TMA (cp.async.bulk.tensor, 128B swizzle) straight into the UMMA canonical
//     K-major layout; one elected thread issues tcgen05.mma; accumulators are double-buffered in TMEM
//     (2 x 256 columns) so the MMA of group g+1 overlaps the epilogue of group g.
//   * work = (tile, list of queries). In list mode (stage 2) the queries of an item are the rows that
//     SELECTED that key block — the refinement is run block-major ("inverted"), because a key tile that is
//     loaded once and multiplied with N=256 query columns needs half the L2->SM bytes per scored pair of a
//     query-major gather (16 KB of q vs 32 KB of keys per pair) and keeps the full N=256 MMA shape.
//   * persistent CTAs (one per SM) pull items from a global cursor; a scheduler warp prefetches items so
//     the global atomic + item load are off the TMA producer's critical path.
//   * multi-term products: operands may be split into bf16 segments (pooled keys: hi|lo; fp32 inputs:
//     exact 3-way split); `terms[ib]` lists which A segments multiply B segment ib, all accumulated into
//     the same TMEM tile before the ReLU.
//
// Warp roles (352 threads): warps 0-7 epilogue (warp%4 = TMEM lane quarter, warp/4 = which 2 of the 4
// queries), warp 8 TMA producer, warp 9 MMA issuer + TMEM owner, warp 10 scheduler.
#include "kernels.cuh"
#include "ptx.cuh"

namespace hisa_dev {

namespace {

constexpr int kEpiWarps = 8;
constexpr int kProducerWarp = 8;
constexpr int kMmaWarp = 9;
constexpr int kSchedWarp = 10;
constexpr int kTcThreads = 11 * 32;
constexpr int kMetaSlots = 8;
constexpr int kUnitSlots = 4;
constexpr uint32_t kAHalfBytes = kTileRows * 128;      // one 64-element K-half of one A segment: 16 KB
constexpr uint32_t kASegBytes = 2 * kAHalfBytes;       // 32 KB
constexpr uint32_t kQBoxBytes = kHeads * 128;          // one query, one K-half: 8 KB
constexpr uint32_t kBChunkBytes = kGroupQ * kQBoxBytes;  // 32 KB
constexpr uint32_t kGateRowBytes = kHeads * 4;         // 256 B
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAccCols = kGroupQ * kHeads;        // 256

constexpr uint32_t kFlagFirst = 1u, kFlagLast = 2u, kFlagTerminate = 4u;

struct GroupMeta {
  uint32_t qrow[kGroupQ];
  uint32_t col[kGroupQ];
  uint32_t nvalid;
  uint32_t a_buf;
  uint32_t valid_rows;
  uint32_t flags;
};

template <int NSEG_A, int ABUF, int NST>
struct SmemLayout {
  static constexpr uint32_t a_off = 0;
  static constexpr uint32_t b_off = a_off + ABUF * NSEG_A * kASegBytes;
  static constexpr uint32_t w_off = b_off + NST * kBChunkBytes;
  static constexpr uint32_t meta_off = w_off + kMetaSlots * kGroupQ * kGateRowBytes;
  static constexpr uint32_t unit_off = meta_off + kMetaSlots * sizeof(GroupMeta);
  static constexpr uint32_t bar_off = unit_off + kUnitSlots * sizeof(WorkItem);
  // barriers: b_full[NST] b_empty[NST] a_full[ABUF] a_empty[ABUF] t_full[2] t_empty[2] w_full[8] u_full[4] u_empty[4]
  static constexpr uint32_t num_bars = 2 * NST + 2 * ABUF + 4 + kMetaSlots + 2 * kUnitSlots;
  static constexpr uint32_t tmem_off = bar_off + num_bars * 8;
  static constexpr uint32_t total = tmem_off + 16;
};

template <int NSEG_A, int ABUF, int NST>
__global__ void __launch_bounds__(kTcThreads, 1)
score_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, ScoreArgs a) {
  using L = SmemLayout<NSEG_A, ABUF, NST>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // dynamic smem is only guaranteed 16-byte aligned: round up to the 1024 B the 128B swizzle needs
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* s_a = smem + L::a_off;
  unsigned char* s_b = smem + L::b_off;
  float* s_w = reinterpret_cast<float*>(smem + L::w_off);
  GroupMeta* s_meta = reinterpret_cast<GroupMeta*>(smem + L::meta_off);
  WorkItem* s_unit = reinterpret_cast<WorkItem*>(smem + L::unit_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::bar_off);
  uint64_t* b_full = bars;
  uint64_t* b_empty = b_full + NST;
  uint64_t* a_full = b_empty + NST;
  uint64_t* a_empty = a_full + ABUF;
  uint64_t* t_full = a_empty + ABUF;
  uint64_t* t_empty = t_full + 2;
  uint64_t* w_full = t_empty + 2;
  uint64_t* u_full = w_full + kMetaSlots;
  uint64_t* u_empty = u_full + kUnitSlots;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::tmem_off);

  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < ABUF; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&t_full[i], 1); mbar_init(&t_empty[i], kEpiWarps); }
    for (int i = 0; i < kMetaSlots; ++i) mbar_init(&w_full[i], 1);
    for (int i = 0; i < kUnitSlots; ++i) { mbar_init(&u_full[i], 1); mbar_init(&u_empty[i], 1); }
    fence_barrier_init();
    fence_proxy_async();
  }
  if (warp == kMmaWarp) {
    tmem_alloc(s_tmem, kTmemCols);
    tmem_relinquish();
  }
  if (warp == kProducerWarp && lane == 0) {
    prefetch_tensormap(&map_a);
    prefetch_tensormap(&map_b);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *s_tmem;
  const uint32_t chunks_per_group = a.nseg_b * 2;

  if (warp == kSchedWarp) {
    // ================= scheduler: prefetch work items into the unit ring =================
    if (lane == 0) {
      const uint32_t nitems = *a.work_count;
      for (uint32_t useq = 0;; ++useq) {
        const uint32_t slot = useq % kUnitSlots;
        mbar_wait(&u_empty[slot], ((useq / kUnitSlots) & 1u) ^ 1u);
        const uint32_t id = atomicAdd(a.work_cursor, 1u);
        WorkItem w;
        if (id < nitems) {
          w = a.work[id];
        } else {
          w.tile = 0; w.first = 0; w.count = 0; w.reserved = 0;
        }
        s_unit[slot] = w;
        mbar_arrive(&u_full[slot]);
        if (w.count == 0) break;
      }
    }
  } else if (warp == kProducerWarp) {
    // ================= TMA producer =================
    uint32_t g = 0, cs = 0;
    for (uint32_t useq = 0;; ++useq) {
      const uint32_t slot = useq % kUnitSlots;
      mbar_wait(&u_full[slot], (useq / kUnitSlots) & 1u);
      const WorkItem item = s_unit[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&u_empty[slot]);
      if (item.count == 0) {
        if (lane == 0) {
          const uint32_t stage = cs % NST;
          mbar_wait(&b_empty[stage], ((cs / NST) & 1u) ^ 1u);
          const uint32_t ws = g % kMetaSlots;
          s_meta[ws].flags = kFlagTerminate;
          mbar_arrive(&w_full[ws]);
          mbar_arrive(&b_full[stage]);
        }
        break;
      }
      const uint32_t a_buf = useq % ABUF;
      const uint32_t row0 = tile_row0(a, item.tile);
      const uint32_t valid_rows = tile_valid_rows(a, item.tile);
      const uint32_t col_add = a.list_mode ? (item.tile % a.segs_per_block) * kTileRows : item.tile * kTileRows;
      if (lane == 0) {
        mbar_wait(&a_empty[a_buf], ((useq / ABUF) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&a_full[a_buf], NSEG_A * kASegBytes);
#pragma unroll
        for (int ia = 0; ia < NSEG_A; ++ia)
#pragma unroll
          for (int kh = 0; kh < 2; ++kh)
            tma_load_2d(s_a + a_buf * (NSEG_A * kASegBytes) + (ia * 2 + kh) * kAHalfBytes, &map_a, &a_full[a_buf],
                        ia * kDim + kh * 64, int32_t(row0));
      }
      const uint32_t ngroups = (item.count + kGroupQ - 1) / kGroupQ;
      for (uint32_t gb = 0; gb < ngroups; gb += 8) {
        // 32 lanes fetch the next 32 (row, col) entries in one coalesced load
        const uint32_t idx = gb * kGroupQ + lane;
        uint32_t prow = 0, pcol = 0;
        if (idx < item.count) {
          if (a.list_mode) {
            const uint2 p = a.pairs[item.first + idx];
            prow = p.x;
            pcol = p.y + col_add;
          } else {
            prow = item.first + idx;
            pcol = col_add;
          }
        }
        const uint32_t gend = min(8u, ngroups - gb);
        for (uint32_t gi = 0; gi < gend; ++gi) {
          uint32_t qrow[kGroupQ], qcol[kGroupQ];
#pragma unroll
          for (int qi = 0; qi < kGroupQ; ++qi) {
            qrow[qi] = __shfl_sync(0xffffffffu, prow, gi * kGroupQ + qi);
            qcol[qi] = __shfl_sync(0xffffffffu, pcol, gi * kGroupQ + qi);
          }
          const uint32_t gg = gb + gi;
          const uint32_t nvalid = min(uint32_t(kGroupQ), item.count - gg * kGroupQ);
          if (lane == 0) {
            uint32_t stage = cs % NST;
            mbar_wait(&b_empty[stage], ((cs / NST) & 1u) ^ 1u);
            const uint32_t ws = g % kMetaSlots;
            GroupMeta m;
#pragma unroll
            for (int qi = 0; qi < kGroupQ; ++qi) { m.qrow[qi] = qrow[qi]; m.col[qi] = qcol[qi]; }
            m.nvalid = nvalid;
            m.a_buf = a_buf;
            m.valid_rows = valid_rows;
            m.flags = (gg == 0 ? kFlagFirst : 0u) | (gg + 1 == ngroups ? kFlagLast : 0u);
            s_meta[ws] = m;
            mbar_arrive_expect_tx(&w_full[ws], nvalid * kGateRowBytes);
            for (uint32_t qi = 0; qi < nvalid; ++qi)
              bulk_load_1d(s_w + (ws * kGroupQ + qi) * kHeads, a.gates + uint64_t(qrow[qi]) * kHeads, kGateRowBytes,
                           &w_full[ws]);
            uint32_t c = cs;
            for (uint32_t ib = 0; ib < a.nseg_b; ++ib)
              for (uint32_t kh = 0; kh < 2; ++kh) {
                if (c != cs) {
                  stage = c % NST;
                  mbar_wait(&b_empty[stage], ((c / NST) & 1u) ^ 1u);
                }
                mbar_arrive_expect_tx(&b_full[stage], nvalid * kQBoxBytes);
                for (uint32_t qi = 0; qi < nvalid; ++qi)
                  tma_load_2d(s_b + stage * kBChunkBytes + qi * kQBoxBytes, &map_b, &b_full[stage],
                              int32_t(ib * kDim + kh * 64), int32_t(qrow[qi] * kHeads));
                ++c;
              }
          }
          cs += chunks_per_group;
          ++g;
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer (one thread) =================
    if (lane == 0) {
      uint32_t g = 0, cs = 0, units = 0;
      for (;;) {
        uint32_t stage = cs % NST;
        mbar_wait(&b_full[stage], (cs / NST) & 1u);
        const GroupMeta* mp = &s_meta[g % kMetaSlots];
        const uint32_t flags = mp->flags;
        if (flags & kFlagTerminate) break;
        const uint32_t nvalid = mp->nvalid;
        const uint32_t a_buf = mp->a_buf;
        if (flags & kFlagFirst) {
          mbar_wait(&a_full[a_buf], (units / ABUF) & 1u);
          ++units;
        }
        const uint32_t acc = g & 1u;
        mbar_wait(&t_empty[acc], ((g >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t idesc = umma_idesc_bf16(kTileRows, nvalid * kHeads);
        const uint32_t d_tmem = tmem_base + acc * kAccCols;
        const uint32_t a_base = smem_u32(s_a) + a_buf * (NSEG_A * kASegBytes);
        uint32_t accum = 0;
        uint32_t c = cs;
        for (uint32_t ib = 0; ib < a.nseg_b; ++ib)
          for (uint32_t kh = 0; kh < 2; ++kh) {
            if (c != cs) {
              stage = c % NST;
              mbar_wait(&b_full[stage], (c / NST) & 1u);
              tc_fence_after();
            }
            const uint32_t b_base = smem_u32(s_b) + stage * kBChunkBytes;
            const uint32_t mask = a.terms[ib];
#pragma unroll
            for (int ia = 0; ia < NSEG_A; ++ia) {
              if (mask & (1u << ia)) {
                const uint32_t a_tile = a_base + (ia * 2 + kh) * kAHalfBytes;
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4) {
                  umma_bf16(d_tmem, umma_smem_desc_sw128(a_tile + k4 * 32), umma_smem_desc_sw128(b_base + k4 * 32),
                            idesc, accum);
                  accum = 1;
                }
              }
            }
            umma_commit(&b_empty[stage]);  // stage reusable once these MMAs have read it
            ++c;
          }
        cs = c;
        umma_commit(&t_full[acc]);
        if (flags & kFlagLast) umma_commit(&a_empty[a_buf]);
        ++g;
      }
    }
  } else {
    // ================= epilogue: TMEM -> gate*ReLU head reduction -> HBM =================
    const uint32_t quarter = warp & 3u;
    const uint32_t half = warp >> 2;
    const uint32_t row_lane = quarter * 32 + lane;
    for (uint32_t g = 0;; ++g) {
      const uint32_t ws = g % kMetaSlots;
      mbar_wait(&w_full[ws], (g / kMetaSlots) & 1u);
      const GroupMeta* mp = &s_meta[ws];
      if (mp->flags & kFlagTerminate) break;
      const uint32_t nvalid = mp->nvalid;
      const uint32_t valid_rows = mp->valid_rows;
      const uint32_t acc = g & 1u;
      mbar_wait(&t_full[acc], (g >> 1) & 1u);
      __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the spin loops
      tc_fence_after();
#pragma unroll
      for (uint32_t qq = 0; qq < 2; ++qq) {
        const uint32_t qi = half * 2 + qq;
        if (qi < nvalid) {
          const uint32_t taddr = tmem_base + ((quarter * 32u) << 16) + acc * kAccCols + qi * kHeads;
          uint32_t v0[32], v1[32];
          tmem_ld_32x32b_x32(taddr, v0);
          tmem_ld_32x32b_x32(taddr + 32, v1);
          tmem_ld_wait();
          const float4* wv = reinterpret_cast<const float4*>(s_w + (ws * kGroupQ + qi) * kHeads);
          float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 w4 = wv[j4];
            s0 = fmaf(w4.x, fmaxf(__uint_as_float(v0[j4 * 4 + 0]), 0.f), s0);
            s1 = fmaf(w4.y, fmaxf(__uint_as_float(v0[j4 * 4 + 1]), 0.f), s1);
            s2 = fmaf(w4.z, fmaxf(__uint_as_float(v0[j4 * 4 + 2]), 0.f), s2);
            s3 = fmaf(w4.w, fmaxf(__uint_as_float(v0[j4 * 4 + 3]), 0.f), s3);
          }
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 w4 = wv[8 + j4];
            s0 = fmaf(w4.x, fmaxf(__uint_as_float(v1[j4 * 4 + 0]), 0.f), s0);
            s1 = fmaf(w4.y, fmaxf(__uint_as_float(v1[j4 * 4 + 1]), 0.f), s1);
            s2 = fmaf(w4.z, fmaxf(__uint_as_float(v1[j4 * 4 + 2]), 0.f), s2);
            s3 = fmaf(w4.w, fmaxf(__uint_as_float(v1[j4 * 4 + 3]), 0.f), s3);
          }
          const float score = (s0 + s1) + (s2 + s3);
          if (row_lane < valid_rows)
            a.out[uint64_t(mp->qrow[qi]) * a.out_stride + mp->col[qi] + row_lane] = score;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&t_empty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

template <int NSEG_A, int ABUF, int NST>
int launch_variant(const ScoreArgs& args, const CUtensorMap& map_a, const CUtensorMap& map_b, int num_sms,
                   cudaStream_t stream) {
  using L = SmemLayout<NSEG_A, ABUF, NST>;
  constexpr size_t smem = L::total + 1024;  // slack for the manual 1024 B alignment
  auto kern = score_tc_kernel<NSEG_A, ABUF, NST>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    configured = true;
  }
  kern<<<num_sms, kTcThreads, smem, stream>>>(map_a, map_b, args);
  return 1;
}

}  // namespace

size_t score_tc_smem_bytes(uint32_t nseg_a) {
  if (nseg_a == 1) return SmemLayout<1, 2, 4>::total + 1024;
  if (nseg_a == 2) return SmemLayout<2, 1, 4>::total + 1024;
  return SmemLayout<3, 1, 3>::total + 1024;
}

int launch_score_tc(const ScoreArgs& args, const CUtensorMap& map_a, const CUtensorMap& map_b, int num_sms,
                    cudaStream_t stream) {
  switch (args.nseg_a) {
    case 1: return launch_variant<1, 2, 4>(args, map_a, map_b, num_sms, stream);
    case 2: return launch_variant<2, 1, 4>(args, map_a, map_b, num_sms, stream);
    default: return launch_variant<3, 1, 3>(args, map_a, map_b, num_sms, stream);
  }
}

}  // namespace hisa_dev
