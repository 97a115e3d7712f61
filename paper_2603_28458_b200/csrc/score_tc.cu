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
//     exact 3-way split); TERMS lists which A segments multiply each B segment, all accumulated into the
//     same TMEM tile before the ReLU. Segment structure is a template parameter so the issue loop is
//     straight-line code.
//   * measured on B200 (tools/umma_bench.cu): a 128x256x16 tcgen05.mma retires every ~136 cycles when
//     the issuing thread keeps up, so the issue loop is written to be lean: warp-uniform control flow (all
//     lanes wait, one elected lane issues), descriptors built by adding constants to per-stage bases.
//
// Warp roles (608 threads): warps 0-15 epilogue (warp%4 = TMEM lane quarter, warp/4 = which of the 4 queries;
// four epilogue warps per SM sub-partition hide the TMEM-load and LDS latencies of each other), warp 16 TMA
// producer, warp 17 MMA issuer + TMEM owner, warp 18 scheduler.
#include "kernels.cuh"
#include "ptx.cuh"

namespace hisa_dev {

namespace {

constexpr int kEpiWarps = 16;
constexpr int kProducerWarp = 16;
constexpr int kMmaWarp = 17;
constexpr int kSchedWarp = 18;
constexpr int kTcThreads = 19 * 32;
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

// Per-group descriptor handed from the producer to the MMA and epilogue warps through shared memory.
struct GroupMeta {
  uint32_t qrow[kGroupQ];  // +0   output row of each query of the group
  uint32_t col[kGroupQ];   // +16  output column of lane 0
  uint32_t word;           // +32  nvalid | flags << 8 | valid_rows << 16
  uint32_t pad[3];
};
static_assert(sizeof(GroupMeta) == 48, "GroupMeta fields are read by byte offset");

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

__device__ __forceinline__ void sts_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t a) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(a) : "memory");
}
// packed fp32x2 FMA (sm_100): acc.{x,y} += a.{x,y} * b.{x,y}
__device__ __forceinline__ void ffma2(float2& acc, float a0, float a1, float b0, float b1) {
  uint64_t av, bv, cv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(av) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bv) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(cv) : "f"(acc.x), "f"(acc.y));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(cv) : "l"(av), "l"(bv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(acc.x), "=f"(acc.y) : "l"(cv));
}

// gate * relu head reduction over two tcgen05.ld.16x256b.x8 fragments (see ptx.cuh): this lane holds heads
// {8i + 2c, 8i + 2c + 1 : i = 0..7} of four key rows (two per fragment) and reads its 16 permuted gates with
// 4 x LDS.128; each gate pair feeds four packed FMAs, so only a few gate registers are live at a time.
__device__ __forceinline__ void reduce_fragments(const uint32_t (&va)[32], const uint32_t (&vb)[32], uint32_t waddr,
                                                 float2& a0, float2& a1, float2& a2, float2& a3) {
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const float4 w4 = waddr ? lds_f4(waddr + h * 16) : make_float4(1.f, 1.f, 1.f, 1.f);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int i = 2 * h + e;
      const float wx = e ? w4.z : w4.x, wy = e ? w4.w : w4.y;
      ffma2(a0, wx, wy, fmaxf(__uint_as_float(va[4 * i + 0]), 0.f), fmaxf(__uint_as_float(va[4 * i + 1]), 0.f));
      ffma2(a1, wx, wy, fmaxf(__uint_as_float(va[4 * i + 2]), 0.f), fmaxf(__uint_as_float(va[4 * i + 3]), 0.f));
      ffma2(a2, wx, wy, fmaxf(__uint_as_float(vb[4 * i + 0]), 0.f), fmaxf(__uint_as_float(vb[4 * i + 1]), 0.f));
      ffma2(a3, wx, wy, fmaxf(__uint_as_float(vb[4 * i + 2]), 0.f), fmaxf(__uint_as_float(vb[4 * i + 3]), 0.f));
    }
  }
}

// TERMS: bit (ib * 3 + ia) set <=> A segment ia is multiplied with B segment ib
template <int NSEG_A, int NSEG_B, uint32_t TERMS, int ABUF, int NST>
__global__ void __launch_bounds__(kTcThreads, 1)
score_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, ScoreArgs a) {
  using L = SmemLayout<NSEG_A, ABUF, NST>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // dynamic smem is only guaranteed 16-byte aligned: round up to the 1024 B the 128B swizzle needs
  // (pointer arithmetic on the __shared__ array keeps the address space known to the compiler: LDS/STS, not generic)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
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
  const long long cta_c0 = clock64();

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
  const uint32_t meta_base = smem_u32(s_meta);

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
    // ================= TMA producer (warp-uniform loop, one elected lane issues) =================
    uint32_t stage = 0, sph = 1;  // chunk ring position and the parity to wait for on b_empty
    uint32_t ws = 0;              // meta / gate slot = group index % 8
    uint64_t st_unit = 0, st_a = 0, st_b = 0;
    const uint32_t a_smem = smem_u32(s_a), b_smem = smem_u32(s_b), w_smem = smem_u32(s_w);
    for (uint32_t useq = 0;; ++useq) {
      const uint32_t slot = useq % kUnitSlots;
      mbar_wait_timed(&u_full[slot], (useq / kUnitSlots) & 1u, st_unit);
      const WorkItem item = s_unit[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&u_empty[slot]);
      if (item.count == 0) {
        if (lane == 0) {
          mbar_wait(&b_empty[stage], sph);
          sts_u32(meta_base + ws * uint32_t(sizeof(GroupMeta)) + 32, kFlagTerminate << 8);
          mbar_arrive(&w_full[ws]);
          mbar_arrive(&b_full[stage]);
          if (a.stats) {
            atomicAdd(a.stats + kStatProdUnit, st_unit);
            atomicAdd(a.stats + kStatProdAEmpty, st_a);
            atomicAdd(a.stats + kStatProdBEmpty, st_b);
          }
        }
        break;
      }
      const uint32_t a_buf = useq % ABUF;
      const uint32_t row0 = tile_row0(a, item.tile);
      const uint32_t valid_rows = tile_valid_rows(a, item.tile);
      const uint32_t col_add = a.list_mode ? (item.tile % a.segs_per_block) * kTileRows : item.tile * kTileRows;
      mbar_wait_timed(&a_empty[a_buf], ((useq / ABUF) & 1u) ^ 1u, st_a);
      __syncwarp();
      if (elect_one()) {
        mbar_arrive_expect_tx(&a_full[a_buf], NSEG_A * kASegBytes);
#pragma unroll
        for (int ia = 0; ia < NSEG_A; ++ia)
#pragma unroll
          for (int kh = 0; kh < 2; ++kh)
            tma_load_2d_addr(a_smem + a_buf * (NSEG_A * kASegBytes) + (ia * 2 + kh) * kAHalfBytes, &map_a,
                             smem_u32(&a_full[a_buf]), ia * kDim + kh * 64, int32_t(row0));
      }
      __syncwarp();
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
          const uint32_t flags = (gg == 0 ? kFlagFirst : 0u) | (gg + 1 == ngroups ? kFlagLast : 0u);
          mbar_wait_timed(&b_empty[stage], sph, st_b);  // first chunk of the group: also guards the meta/gate slot
          __syncwarp();
          if (elect_one()) {
            const uint32_t maddr = meta_base + ws * uint32_t(sizeof(GroupMeta));
            sts_v4(maddr, qrow[0], qrow[1], qrow[2], qrow[3]);
            sts_v4(maddr + 16, qcol[0], qcol[1], qcol[2], qcol[3]);
            sts_u32(maddr + 32, nvalid | (flags << 8) | (valid_rows << 16));
            const uint32_t wbar = smem_u32(&w_full[ws]);
            mbar_arrive_expect_tx(&w_full[ws], nvalid * kGateRowBytes);
#pragma unroll
            for (uint32_t qi = 0; qi < kGroupQ; ++qi)
              if (qi < nvalid)
                bulk_load_1d_addr(w_smem + (ws * kGroupQ + qi) * kGateRowBytes, a.gates + uint64_t(qrow[qi]) * kHeads,
                                  kGateRowBytes, wbar);
          }
          __syncwarp();
#pragma unroll
          for (int ib = 0; ib < NSEG_B; ++ib)
#pragma unroll
            for (int kh = 0; kh < 2; ++kh) {
              if (ib + kh > 0) {
                mbar_wait_timed(&b_empty[stage], sph, st_b);
                __syncwarp();
              }
              if (elect_one()) {
                const uint32_t fbar = smem_u32(&b_full[stage]);
                if (a.debug_flags & 2u) {
                  mbar_arrive(&b_full[stage]);
                } else {
                  mbar_arrive_expect_tx(&b_full[stage], nvalid * kQBoxBytes);
                  const uint32_t dst = b_smem + stage * kBChunkBytes;
#pragma unroll
                  for (uint32_t qi = 0; qi < kGroupQ; ++qi)
                    if (qi < nvalid)
                      tma_load_2d_addr(dst + qi * kQBoxBytes, &map_b, fbar, ib * kDim + kh * 64,
                                       int32_t(qrow[qi] * kHeads));
                }
              }
              __syncwarp();
              if (++stage == NST) { stage = 0; sph ^= 1u; }
            }
          ws = (ws + 1) % kMetaSlots;
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer =================
    // The whole warp runs the loop convergently (all lanes wait on the barriers and read the group meta);
    // one elected lane issues tcgen05.mma / tcgen05.commit. Warp-uniform control flow lets the compiler keep
    // descriptors in uniform registers instead of emitting per-instruction waterfall loops.
    uint32_t stage = 0, sph = 0;  // chunk ring position and the parity to wait for on b_full
    uint32_t ws = 0, g = 0, units = 0;
    uint64_t st_bf = 0, st_af = 0, st_te = 0;
    // descriptor bases in (addr >> 4) units; +2 per K=16 step (32 B) inside the 128-byte swizzle row
    const uint64_t a_desc0 = umma_smem_desc_sw128(smem_u32(s_a));
    const uint64_t b_desc0 = umma_smem_desc_sw128(smem_u32(s_b));
    for (;;) {
      mbar_wait_timed(&b_full[stage], sph, st_bf);
      const uint32_t word = lds_u32(meta_base + ws * uint32_t(sizeof(GroupMeta)) + 32);
      const uint32_t flags = (word >> 8) & 0xFFu;
      if (flags & kFlagTerminate) break;
      const uint32_t nvalid = word & 0xFFu;
      const uint32_t a_buf = units % ABUF;  // same sequence as the producer's useq % ABUF
      if (flags & kFlagFirst) mbar_wait_timed(&a_full[a_buf], (units / ABUF) & 1u, st_af);
      const uint32_t acc = g & 1u;
      mbar_wait_timed(&t_empty[acc], ((g >> 1) & 1u) ^ 1u, st_te);
      __syncwarp();
      tc_fence_after();
      const uint32_t idesc = umma_idesc_bf16(kTileRows, nvalid * kHeads);
      const uint32_t d_tmem = tmem_base + acc * kAccCols;
      const uint64_t a_desc = a_desc0 + uint64_t(a_buf * (NSEG_A * kASegBytes >> 4));
      bool first = true;
#pragma unroll
      for (int ib = 0; ib < NSEG_B; ++ib)
#pragma unroll
        for (int kh = 0; kh < 2; ++kh) {
          if (ib + kh > 0) {
            mbar_wait_timed(&b_full[stage], sph, st_bf);
            __syncwarp();
            tc_fence_after();
          }
          const uint64_t b_desc = b_desc0 + uint64_t(stage * (kBChunkBytes >> 4));
          if (elect_one()) {
#pragma unroll
            for (int ia = 0; ia < NSEG_A; ++ia) {
              if ((TERMS >> (ib * 3 + ia)) & 1u) {
                const uint64_t a_tile = a_desc + uint64_t((ia * 2 + kh) * (kAHalfBytes >> 4));
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4) {
                  umma_bf16(d_tmem, a_tile + 2 * k4, b_desc + 2 * k4, idesc, first ? 0u : 1u);
                  first = false;
                }
              }
            }
            umma_commit(&b_empty[stage]);  // stage reusable once these MMAs have read it
            if (ib == NSEG_B - 1 && kh == 1) {
              umma_commit(&t_full[acc]);
              if (flags & kFlagLast) umma_commit(&a_empty[a_buf]);
            }
          }
          first = false;
          __syncwarp();
          if (++stage == NST) { stage = 0; sph ^= 1u; }
        }
      if (flags & kFlagLast) ++units;
      ws = (ws + 1) % kMetaSlots;
      ++g;
    }
    if (a.stats && lane == 0) {
      atomicAdd(a.stats + kStatMmaBFull, st_bf);
      atomicAdd(a.stats + kStatMmaAFull, st_af);
      atomicAdd(a.stats + kStatMmaTEmpty, st_te);
      atomicAdd(a.stats + kStatGroups, (unsigned long long)g);
    }
  } else {
    // ================= epilogue: TMEM -> gate*ReLU head reduction -> HBM =================
    const uint32_t quarter = warp & 3u;
    const uint32_t qi = warp >> 2;  // which query of the group this warp reduces
    const uint32_t w_base = smem_u32(s_w);
    uint64_t st_w = 0, st_t = 0, st_busy = 0;
    for (uint32_t g = 0;; ++g) {
      const uint32_t ws = g % kMetaSlots;
      mbar_wait_timed(&w_full[ws], (g / kMetaSlots) & 1u, st_w);
      const uint32_t maddr = meta_base + ws * uint32_t(sizeof(GroupMeta));
      const uint32_t word = lds_u32(maddr + 32);
      if ((word >> 8) & kFlagTerminate) break;
      const uint32_t nvalid = word & 0xFFu;
      const uint32_t valid_rows = word >> 16;
      const uint32_t acc = g & 1u;
      mbar_wait_timed(&t_full[acc], (g >> 1) & 1u, st_t);
      const long long c0 = clock64();
      __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the spin loops
      tc_fence_after();
      const bool active = qi < nvalid && !(a.debug_flags & 1u);
      // Fragment layout (tcgen05.ld.16x256b): a lane owns 16 of the 64 heads for FOUR key rows, so it needs only
      // 16 gates (64 B) per query instead of all 64: the gate traffic through the 128 B/clk shared-memory port
      // is what bounded the 32x32b one-row-per-thread epilogue. The 4 lanes sharing a row are summed by shuffles.
      uint32_t v0[32], v1[32];
      if (active) {
        const uint32_t taddr = tmem_base + ((quarter * 32u) << 16) + acc * kAccCols + qi * kHeads;
        tmem_ld_16x256b_x8(taddr, v0);               // rows quarter*32 + {T/4, T/4 + 8}
        tmem_ld_16x256b_x8(taddr + (16u << 16), v1);  // rows quarter*32 + 16 + {T/4, T/4 + 8}
        tmem_ld_wait();
      }
      // the dots are in registers: hand the accumulator back before doing the math
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&t_empty[acc]);
      if (active && !(a.debug_flags & 8u)) {  // (debug 8: loads only, debug 16: no gate loads)
        const uint32_t waddr = (a.debug_flags & 16u) ? 0u : w_base + (ws * kGroupQ + qi) * kGateRowBytes + (lane & 3u) * 64u;
        float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
        reduce_fragments(v0, v1, waddr, a0, a1, a2, a3);
        const float s0 = a0.x + a0.y, s1 = a1.x + a1.y, s2 = a2.x + a2.y, s3 = a3.x + a3.y;
        // transposed butterfly over the 4 lanes of a row group: lane ends with the total of row slot (lane & 3)
        const bool b0 = lane & 1u, b1 = lane & 2u;
        float k0 = b0 ? s1 : s0, k1 = b0 ? s3 : s2;
        k0 += __shfl_xor_sync(0xffffffffu, b0 ? s0 : s1, 1);
        k1 += __shfl_xor_sync(0xffffffffu, b0 ? s2 : s3, 1);
        float z = b1 ? k1 : k0;
        z += __shfl_xor_sync(0xffffffffu, b1 ? k0 : k1, 2);
        const uint32_t row = quarter * 32 + (lane >> 2) + 8u * (lane & 3u);
        if (row < valid_rows)
          a.out[uint64_t(lds_u32(maddr + qi * 4)) * a.out_stride + lds_u32(maddr + 16 + qi * 4) + row] = z;
      }
      st_busy += uint64_t(clock64() - c0);
    }
    if (a.stats && warp == 0 && lane == 0) {
      atomicAdd(a.stats + kStatEpiWFull, st_w);
      atomicAdd(a.stats + kStatEpiTFull, st_t);
      atomicAdd(a.stats + kStatEpiBusy, st_busy);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
  if (a.stats && threadIdx.x == 0) atomicAdd(a.stats + kStatCta, (unsigned long long)(clock64() - cta_c0));
}

template <int NSEG_A, int NSEG_B, uint32_t TERMS, int ABUF, int NST>
int launch_variant(const ScoreArgs& args, const CUtensorMap& map_a, const CUtensorMap& map_b, int num_sms,
                   cudaStream_t stream) {
  using L = SmemLayout<NSEG_A, ABUF, NST>;
  constexpr size_t smem = L::total + 1024;  // slack for the manual 1024 B alignment
  auto kern = score_tc_kernel<NSEG_A, NSEG_B, TERMS, ABUF, NST>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    configured = true;
  }
  kern<<<num_sms, kTcThreads, smem, stream>>>(map_a, map_b, args);
  return 1;
}

constexpr uint32_t pack_terms(uint32_t t0, uint32_t t1, uint32_t t2) { return t0 | (t1 << 3) | (t2 << 6); }

}  // namespace

int launch_score_tc(const ScoreArgs& args, const CUtensorMap& map_a, const CUtensorMap& map_b, int num_sms,
                    cudaStream_t stream) {
  const uint32_t terms = pack_terms(args.terms[0], args.terms[1], args.terms[2]);
  // the segment structure is compiled in; these are the combinations the context produces
  if (args.nseg_a == 1 && args.nseg_b == 1 && terms == pack_terms(1, 0, 0))
    return launch_variant<1, 1, pack_terms(1, 0, 0), 2, 4>(args, map_a, map_b, num_sms, stream);
  if (args.nseg_a == 2 && args.nseg_b == 1 && terms == pack_terms(3, 0, 0))
    return launch_variant<2, 1, pack_terms(3, 0, 0), 1, 4>(args, map_a, map_b, num_sms, stream);
  if (args.nseg_a == 3 && args.nseg_b == 1 && terms == pack_terms(7, 0, 0))
    return launch_variant<3, 1, pack_terms(7, 0, 0), 1, 3>(args, map_a, map_b, num_sms, stream);
  if (args.nseg_a == 3 && args.nseg_b == 3 && terms == pack_terms(7, 3, 1))
    return launch_variant<3, 3, pack_terms(7, 3, 1), 1, 3>(args, map_a, map_b, num_sms, stream);
  return -1;  // unsupported segment structure (the context never builds one)
}

}  // namespace hisa_dev
