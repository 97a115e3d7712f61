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
//   * persistent CTAs (one per SM) pull items from a global cursor; the fetch of the next items is issued while the
//     current one is produced, so the global atomic + item load are off the TMA producers' critical path.
//   * multi-term products: operands may be split into bf16 segments (pooled keys: hi|lo; fp32 inputs:
//     exact 3-way split); TERMS lists which A segments multiply each B segment, all accumulated into the
//     same TMEM tile before the ReLU. Segment structure is a template parameter so the issue loop is
//     straight-line code.
//   * measured on B200 (tools/umma_bench.cu): a 128x256x16 tcgen05.mma retires every ~136 cycles when
//     the issuing thread keeps up, so the issue loop is written to be lean: warp-uniform control flow (all
//     lanes wait, one elected lane issues), descriptors built by adding constants to per-stage bases.
//
// Warp roles (640 threads): warps 0-15 epilogue in two sets of eight (set = warp / 8 takes the groups with
// g % 2 == set, i.e. it owns one of the two TMEM accumulators; inside a set warp % 4 = TMEM lane quarter and
// (warp / 4) % 2 = which PAIR of the group's 4 queries), warps 16-18 TMA producers (chunks dealt round-robin; producer 0
// also pulls work items from the global cursor), warp 19 MMA issuer + TMEM owner. With the sets half a period apart each SM sub-partition always has warps of both sets to issue
// from (tcgen05.ld / LDS / shuffle latencies of one set hide under the FMNMX/FFMA2 stream of the other), and every
// warp additionally keeps one 16-register tcgen05.ld in flight under its own math.
#include "kernels.cuh"
#include "ptx.cuh"

namespace hisa_dev {

namespace {

constexpr int kEpiWarps = 16;
constexpr int kEpiSetWarps = 8;  // epilogue warps per accumulator
constexpr int kProducerWarp = 16;  // first of kProducers TMA producer warps
constexpr int kMaxProducers = 3;   // warps reserved for producers; a variant uses NPROD <= 3 of them
constexpr int kMmaWarp = kProducerWarp + kMaxProducers;
constexpr int kEpiRegs = 104, kOtherRegs = 64;
constexpr int kTcThreads = (kMmaWarp + 1) * 32;  // 640: one more warp would drop the register budget from 96 to 80
constexpr int kMetaSlots = 8;
constexpr int kUnitSlots = 4;
constexpr uint32_t kAHalfBytes = kTileRows * 128;      // one 64-element K-half of one A segment: 16 KB
constexpr uint32_t kQBoxBytes = kHeads * 128;          // one query, one K-half: 8 KB
constexpr uint32_t kGateRowBytes = kHeads * 4;         // 256 B
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kATmemCols = 64;                    // one bf16 key tile in tensor memory: 128 lanes x 64 columns

constexpr uint32_t kFlagFirst = 1u, kFlagLast = 2u, kFlagTerminate = 4u;

// Per-group descriptor handed from the producer to the MMA and epilogue warps through shared memory.
struct GroupMeta {
  uint32_t qrow[4];        // +0   output row of each query of the group (3 or 4 in use)
  uint32_t col[4];         // +16  output column of lane 0
  uint32_t word;           // +32  nvalid | flags << 8 | valid_rows << 16
  uint32_t pad[3];
};
static_assert(sizeof(GroupMeta) == 48, "GroupMeta fields are read by byte offset");

template <int NSEG_A, int ABUF, int NST, int KH, int GQ>
struct SmemLayout {
  static constexpr uint32_t a_off = 0;
  static constexpr uint32_t b_off = a_off + ABUF * NSEG_A * KH * kAHalfBytes;
  static constexpr uint32_t w_off = b_off + NST * GQ * kQBoxBytes;
  static constexpr uint32_t meta_off = w_off + kMetaSlots * GQ * kGateRowBytes;
  static constexpr uint32_t unit_off = meta_off + kMetaSlots * sizeof(GroupMeta);
  static constexpr uint32_t bar_off = unit_off + kUnitSlots * sizeof(WorkItem);
  // barriers: b_full[NST] b_empty[NST] a_full[ABUF] a_empty[ABUF] t_full[2] t_empty[2] u_full[4] u_empty[4]
  static constexpr uint32_t num_bars = 2 * NST + 2 * ABUF + 4 + 2 * kUnitSlots;
  static constexpr uint32_t tmem_off = bar_off + num_bars * 8;
  static constexpr uint32_t total = tmem_off + 16;
};

// packed fp32x2 FMA (sm_100): acc.{x,y} += a.{x,y} * b.{x,y}
__device__ __forceinline__ void ffma2(float2& acc, float a0, float a1, float b0, float b1) {
  uint64_t av, bv, cv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(av) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bv) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(cv) : "f"(acc.x), "f"(acc.y));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(cv) : "l"(av), "l"(bv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(acc.x), "=f"(acc.y) : "l"(cv));
}

// gate * relu head reduction over ONE tcgen05.ld.16x128b.x8 fragment (16 lanes x 32 columns, see ptx.cuh): the lane
// holds heads {32 CH + 4i + c : i = 0..7} of two key rows; g0, g1 are the 8 permuted gates of those heads. Each gate
// pair feeds two packed FMAs, one per row.
__device__ __forceinline__ void reduce_frag(const uint32_t (&v)[16], const float4& g0, const float4& g1, float2& a0,
                                            float2& a1) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // heads 8i + c and 8i + 4 + c of this column half
    const float4& gq = i < 2 ? g0 : g1;
    const float wx = (i & 1) ? gq.z : gq.x, wy = (i & 1) ? gq.w : gq.y;
    ffma2(a0, wx, wy, fmaxf(__uint_as_float(v[4 * i + 0]), 0.f), fmaxf(__uint_as_float(v[4 * i + 2]), 0.f));
    ffma2(a1, wx, wy, fmaxf(__uint_as_float(v[4 * i + 1]), 0.f), fmaxf(__uint_as_float(v[4 * i + 3]), 0.f));
  }
}

// Transposed butterfly over the 4 lanes that share key rows: each lane enters with its partial sums of four rows and
// leaves with the full sum of row slot (lane & 3). Split into three steps so that the two shuffle latencies can be
// covered by the reduction of the next fragment.
struct RowSum {
  float keep0, keep1, got0, got1;
  __device__ __forceinline__ void step1(const float2& a0, const float2& a1, const float2& a2, const float2& a3, bool b0) {
    const float s0 = a0.x + a0.y, s1 = a1.x + a1.y, s2 = a2.x + a2.y, s3 = a3.x + a3.y;
    keep0 = b0 ? s1 : s0;
    keep1 = b0 ? s3 : s2;
    got0 = __shfl_xor_sync(0xffffffffu, b0 ? s0 : s1, 1);
    got1 = __shfl_xor_sync(0xffffffffu, b0 ? s2 : s3, 1);
  }
  __device__ __forceinline__ void step2(bool b1) {
    const float k0 = keep0 + got0, k1 = keep1 + got1;
    keep0 = b1 ? k1 : k0;
    got0 = __shfl_xor_sync(0xffffffffu, b1 ? k0 : k1, 2);
  }
  __device__ __forceinline__ float result() const { return keep0 + got0; }
};

// TERMS: bit (ib * 4 + ia) set <=> A segment ia is multiplied with B segment ib
// FP8: operands are e4m3 bytes (kind::f8f6f4, K = 32 per instruction): a 128-element row is ONE 128-byte swizzle
// row, so a segment is a single K slab (KH = 1) where bf16 needs two (KH = 2), and a group needs one 32 KB query
// chunk instead of two; the per-key dequantisation scale multiplies the finished row sum (scale > 0 commutes with
// the ReLU), the per-(query, head) scale is part of the gate.
// ATM: the key tile (A operand) is multiplied from TENSOR MEMORY. The tile still arrives by TMA in one shared-memory
// staging buffer; the MMA thread moves it with eight tcgen05.cp (128 rows x 32 bytes each) into 64 TMEM columns and every
// MMA of the item reads it there, so per K = 16 step the tensor core fetches only the query operand from shared memory
// (N x 32 bytes instead of (128 + N) x 32 bytes: the shared-memory port is this kernel's wall). 512 TMEM
// columns = 2 accumulators + 2 tile buffers, so the accumulators shrink to 192 columns: groups of THREE queries. The
// staging buffer is free again as soon as the copies have run, which leaves room for a deeper query ring (NST).
// tools/umma_ts_check.cu holds this operand path against the shared-memory form bit for bit.
// MEASURED (C3, same box, A/B): stage 2 7.22 ms against 6.92 ms for the shared-memory form, flat scorer 42 vs 40 ms: the
// N = 192 products issue at ~132 cycles each next to the epilogue's tcgen05.ld traffic (103 in isolation), which costs
// more than the lighter shared-memory port gives back. The variant is therefore OPT-IN (HISA_TC_ATMEM=1) and kept under
// test (tests/test_gpu_parity.py::test_tmem_tile_variant_matches) as the measured alternative.
template <int NSEG_A, int NSEG_B, uint32_t TERMS, int ABUF, int NST, bool FP8, bool ATM, bool STATS>
__global__ void __launch_bounds__(kTcThreads, 1)
score_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, ScoreArgs a) {
  // producer warps: three keep up with two 32 KB chunks per group (bf16); with one chunk per group (fp8) two are
  // enough and a third only takes issue slots from the epilogue warps of its sub-partition while it polls
  const uint32_t kProducers = a.producers;  // 1..kMaxProducers, chosen by the host per variant (HISA_TC_PRODUCERS overrides)
  constexpr int KH = FP8 ? 1 : 2;                     // 128-byte K slabs per operand segment
  constexpr int KBOX = FP8 ? 128 : 64;                // elements per slab
  constexpr uint32_t kASegBytes = KH * kAHalfBytes;   // one A segment: 16 KB (fp8) / 32 KB (bf16)
  constexpr int GQ = ATM ? 3 : kGroupQ;               // queries per group
  constexpr int GPB = 32 / GQ;                        // groups whose (row, col) pairs one warp-wide load fetches
  constexpr uint32_t kBChunkBytes = GQ * kQBoxBytes;  // one K slab of a group's queries: 32 KB (24 KB with ATM)
  constexpr uint32_t kAccCols = GQ * kHeads;          // TMEM columns of one accumulator
  static_assert(!ATM || (NSEG_A == 1 && !FP8 && ABUF == 1), "tile from tensor memory: one bf16 segment, one staging buffer");
  static_assert(2 * kAccCols + (ATM ? 2 * kATmemCols : 0) <= kTmemCols, "tensor memory budget");
  using L = SmemLayout<NSEG_A, ABUF, NST, KH, GQ>;
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
  uint64_t* u_full = t_empty + 2;
  uint64_t* u_empty = u_full + kUnitSlots;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + L::tmem_off);

  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const long long cta_c0 = STATS ? clock64() : 0;
  // role-level stall accounting only exists in the STATS instantiation (profiling on): the clock reads around every
  // wait cost the MMA warp tens of cycles per group, and tools/umma_queue_bench.cu shows the tensor pipe drains its
  // queue ~150-250 cycles after the issuing thread stops feeding it
  auto wait_timed = [&](uint64_t* bar, uint32_t parity, uint64_t& acc_cycles) {
    if (STATS) mbar_wait_timed(bar, parity, acc_cycles);
    else mbar_wait(bar, parity);
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < ABUF; ++i) { mbar_init(&a_full[i], 1); mbar_init(&a_empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&t_full[i], 1); mbar_init(&t_empty[i], kEpiSetWarps); }
    for (int i = 0; i < kUnitSlots; ++i) { mbar_init(&u_full[i], 1); mbar_init(&u_empty[i], kProducers); }
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

  // Register re-partitioning: the four non-epilogue warps (one warp group) give up a third of their registers, which
  // is exactly what lifts the sixteen epilogue warps from the 96-register launch budget to 104
  // (512 * 104 + 128 * 64 = 640 * 96). One textual setmaxnreg per warp group, as the instruction requires.
  if (warp >= kEpiWarps) setmaxnreg_dec<kOtherRegs>();
  if (warp >= kProducerWarp && warp < kProducerWarp + kProducers) {
    // ================= TMA producers (warp-uniform loops, one elected lane issues) =================
    // Issuing the copies of a group (4 query boxes per chunk + 4 gate rows) from ONE thread costs more cycles than
    // the tensor pipe needs for the group (measured: the lone producer was busy ~90 % of the time while the MMA
    // warp waited for data). All producer warps walk the same item / group / chunk sequence and chunk c is issued by
    // producer c % kProducers; whoever issues the first chunk of a group also writes its meta slot and gates.
    // Producer 0 alone loads the operand tiles and passes the terminate marker on. Its lane 0 is also the work
    // scheduler: items come from a global cursor (dynamic load balance over the persistent CTAs) and are published
    // to all producers through the unit ring; the atomic and the item load of item i+2 / i+1 are issued while item i
    // is being produced, so their latency never sits on the producer's critical path.
    const uint32_t pid = warp - kProducerWarp;
    uint32_t turn = 0;  // chunk counter modulo kProducers
    uint32_t pub = 0, fid = 0, nitems = 0;
    WorkItem fw;
    fw.tile = fw.first = fw.count = fw.reserved = 0;
    bool pub_done = false;
    auto fetch_item = [&](uint32_t id) {
      WorkItem w;
      if (id < nitems) w = a.work[id];
      else w.tile = w.first = w.count = w.reserved = 0;  // terminate marker
      return w;
    };
    auto publish = [&](const WorkItem& w) {
      const uint32_t slot = pub % kUnitSlots;
      mbar_wait(&u_empty[slot], ((pub / kUnitSlots) & 1u) ^ 1u);
      s_unit[slot] = w;
      mbar_arrive(&u_full[slot]);
      ++pub;
      if (w.count == 0) pub_done = true;
    };
    // Item ids: CTA c starts with item c (no round trip through the cursor), later ids are gridDim.x + cursor++. The item
    // count, the first item (read speculatively: the list has room for at least gridDim.x items) and the two cursor
    // increments for the next two ids are all in flight together, where the first item used to wait for the count, then
    // for an atomic, then for its own load (three dependent global round trips before a CTA's first TMA request).
    const uint32_t id_base = gridDim.x;
    if (pid == 0 && lane == 0) {
      const uint32_t id_a = atomicAdd(a.work_cursor, 1u);
      const uint32_t id_b = atomicAdd(a.work_cursor, 1u);
      WorkItem w0 = a.work[blockIdx.x];
      nitems = *a.work_count;
      if (blockIdx.x >= nitems) w0.tile = w0.first = w0.count = w0.reserved = 0;  // terminate marker
      publish(w0);
      if (!pub_done) {
        fw = fetch_item(id_base + id_a);
        fid = id_base + id_b;
      }
    }
    uint32_t stage = 0, sph = 1;  // chunk ring position and the parity to wait for on b_empty
    uint32_t ws = 0;              // meta / gate slot = group index % 8
    uint64_t st_unit = 0, st_a = 0, st_b = 0;
    const uint32_t a_smem = smem_u32(s_a), b_smem = smem_u32(s_b), w_smem = smem_u32(s_w);
    for (uint32_t useq = 0;; ++useq) {
      if (pid == 0 && lane == 0 && !pub_done) {  // publish item useq + 1, start fetching useq + 2 and the id after it
        publish(fw);
        if (!pub_done) {
          fw = fetch_item(fid);
          fid = id_base + atomicAdd(a.work_cursor, 1u);
        }
      }
      __syncwarp();
      const uint32_t slot = useq % kUnitSlots;
      wait_timed(&u_full[slot], (useq / kUnitSlots) & 1u, st_unit);
      const WorkItem item = s_unit[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&u_empty[slot]);
      if (item.count == 0) {
        if (lane == 0 && pid == 0) {
          mbar_wait(&b_empty[stage], sph);
          // both epilogue sets must see the marker: the set of group g reads slot ws, the other one slot ws + 1
          sts_u32(meta_base + ws * uint32_t(sizeof(GroupMeta)) + 32, kFlagTerminate << 8);
          sts_u32(meta_base + ((ws + 1) % kMetaSlots) * uint32_t(sizeof(GroupMeta)) + 32, kFlagTerminate << 8);
          mbar_arrive(&b_full[stage]);
          if (STATS && a.stats) {
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
      if (pid == 0) wait_timed(&a_empty[a_buf], ((useq / ABUF) & 1u) ^ 1u, st_a);
      __syncwarp();
      if (pid == 0 && elect_one()) {
        mbar_arrive_expect_tx(&a_full[a_buf], NSEG_A * kASegBytes);
#pragma unroll
        for (int ia = 0; ia < NSEG_A; ++ia)
#pragma unroll
          for (int kh = 0; kh < KH; ++kh)
            tma_load_2d_addr(a_smem + a_buf * (NSEG_A * kASegBytes) + (ia * KH + kh) * kAHalfBytes, &map_a,
                             smem_u32(&a_full[a_buf]), ia * kDim + kh * KBOX, int32_t(row0));
      }
      __syncwarp();
      const uint32_t ngroups = (item.count + GQ - 1) / GQ;
      for (uint32_t gb = 0; gb < ngroups; gb += GPB) {
        // the lanes fetch the (row, col) entries of the next GPB groups in one coalesced load
        const uint32_t idx = gb * GQ + lane;
        uint32_t prow = 0, pcol = 0;
        if (lane < GPB * GQ && idx < item.count) {
          if (a.list_mode) {
            const uint2 p = a.pairs[item.first + idx];
            prow = p.x;
            pcol = p.y + col_add;
          } else {
            prow = item.first + idx;
            pcol = col_add;
          }
        }
        const uint32_t gend = min(uint32_t(GPB), ngroups - gb);
        for (uint32_t gi = 0; gi < gend; ++gi) {
          uint32_t qrow[4], qcol[4];
          qrow[3] = qcol[3] = 0;
#pragma unroll
          for (int qi = 0; qi < GQ; ++qi) {
            qrow[qi] = __shfl_sync(0xffffffffu, prow, gi * GQ + qi);
            qcol[qi] = __shfl_sync(0xffffffffu, pcol, gi * GQ + qi);
          }
          const uint32_t gg = gb + gi;
          const uint32_t nvalid = min(uint32_t(GQ), item.count - gg * GQ);
          const uint32_t flags = (gg == 0 ? kFlagFirst : 0u) | (gg + 1 == ngroups ? kFlagLast : 0u);
          const bool mine0 = turn == pid;  // this producer issues the group's first chunk (and its meta + gates)
          if (mine0) wait_timed(&b_empty[stage], sph, st_b);  // also guards the meta/gate slot
          __syncwarp();
          if (mine0 && elect_one()) {
            const uint32_t maddr = meta_base + ws * uint32_t(sizeof(GroupMeta));
            sts_v4(maddr, qrow[0], qrow[1], qrow[2], qrow[3]);
            sts_v4(maddr + 16, qcol[0], qcol[1], qcol[2], qcol[3]);
            sts_u32(maddr + 32, nvalid | (flags << 8) | (valid_rows << 16));
            if (FP8) sts_u32(maddr + 36, row0);
            // the gates ride on the barrier of the group's first query chunk (one wait for the MMA warp; the epilogue
            // sees them through t_full)
            const uint32_t wbar = smem_u32(&b_full[stage]);
#pragma unroll
            for (uint32_t qi = 0; qi < uint32_t(GQ); ++qi)
              if (qi < nvalid)
                bulk_load_1d_addr(w_smem + (ws * GQ + qi) * kGateRowBytes, a.gates + uint64_t(qrow[qi]) * kHeads,
                                  kGateRowBytes, wbar);
          }
          __syncwarp();
#pragma unroll
          for (int ib = 0; ib < NSEG_B; ++ib)
#pragma unroll
            for (int kh = 0; kh < KH; ++kh) {
              const bool mine = turn == pid;
              if (mine && ib + kh > 0) wait_timed(&b_empty[stage], sph, st_b);
              __syncwarp();
              if (mine && elect_one()) {
                const uint32_t fbar = smem_u32(&b_full[stage]);
                const uint32_t gate_bytes = (ib + kh == 0) ? nvalid * kGateRowBytes : 0u;
                mbar_arrive_expect_tx(&b_full[stage], nvalid * kQBoxBytes + gate_bytes);
                const uint32_t dst = b_smem + stage * kBChunkBytes;
#pragma unroll
                for (uint32_t qi = 0; qi < uint32_t(GQ); ++qi)
                  if (qi < nvalid)
                    tma_load_2d_addr(dst + qi * kQBoxBytes, &map_b, fbar, ib * kDim + kh * KBOX,
                                     int32_t(qrow[qi] * kHeads));
              }
              __syncwarp();
              if (++stage == NST) { stage = 0; sph ^= 1u; }
              if (++turn == kProducers) turn = 0;
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
      wait_timed(&b_full[stage], sph, st_bf);
      const uint32_t word = lds_u32(meta_base + ws * uint32_t(sizeof(GroupMeta)) + 32);
      const uint32_t flags = (word >> 8) & 0xFFu;
      const uint32_t acc = g & 1u;
      if (flags & kFlagTerminate) {
        // the epilogue only watches t_full: pass the terminate marker on through it, to both sets
        mbar_wait(&t_empty[acc], ((g >> 1) & 1u) ^ 1u);
        mbar_wait(&t_empty[acc ^ 1u], (((g + 1) >> 1) & 1u) ^ 1u);
        if (lane == 0) {
          mbar_arrive(&t_full[acc]);
          mbar_arrive(&t_full[acc ^ 1u]);
        }
        break;
      }
      const uint32_t nvalid = word & 0xFFu;
      const uint32_t a_buf = units % ABUF;  // same sequence as the producer's useq % ABUF
      if (flags & kFlagFirst) wait_timed(&a_full[a_buf], (units / ABUF) & 1u, st_af);
      wait_timed(&t_empty[acc], ((g >> 1) & 1u) ^ 1u, st_te);
      __syncwarp();
      tc_fence_after();
      const uint32_t idesc = FP8 ? umma_idesc_e4m3(kTileRows, nvalid * kHeads) : umma_idesc_bf16(kTileRows, nvalid * kHeads);
      const uint32_t d_tmem = tmem_base + acc * kAccCols;
      const uint64_t a_desc = a_desc0 + uint64_t(a_buf * (NSEG_A * kASegBytes >> 4));
      // ATM: the item's tile lives in TMEM buffer (units & 1). That buffer was last read by the MMAs of item units - 2,
      // i.e. of groups <= g - 2, and the t_empty wait above has just proved those complete (the epilogue releases an
      // accumulator only after the commit of the group that filled it). tcgen05.cp and the tcgen05.mma that follow it
      // run in issue order, so no wait sits between the copies and the first product.
      const uint32_t a_tm = tmem_base + 2 * kAccCols + (units & 1u) * kATmemCols;
      if (ATM && (flags & kFlagFirst)) {
        if (elect_one()) {
#pragma unroll
          for (int kh = 0; kh < KH; ++kh)
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4)
              tmem_cp_128x256b(a_tm + (kh * 4 + k4) * 8, a_desc + uint64_t(kh * (kAHalfBytes >> 4) + 2 * k4));
          umma_commit(&a_empty[a_buf]);  // staging buffer reusable once the copies have read it
        }
        __syncwarp();
      }
      bool first = true;
#pragma unroll
      for (int ib = 0; ib < NSEG_B; ++ib)
#pragma unroll
        for (int kh = 0; kh < KH; ++kh) {
          if (ib + kh > 0) {
            wait_timed(&b_full[stage], sph, st_bf);
            __syncwarp();
            tc_fence_after();
          }
          const uint64_t b_desc = b_desc0 + uint64_t(stage * (kBChunkBytes >> 4));
          if (elect_one()) {
#pragma unroll
            for (int ia = 0; ia < NSEG_A; ++ia) {
              if ((TERMS >> (ib * 4 + ia)) & 1u) {
                const uint64_t a_tile = a_desc + uint64_t((ia * KH + kh) * (kAHalfBytes >> 4));
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4) {  // 32 bytes of K per instruction: 16 bf16 or 32 e4m3
                  if (FP8) umma_f8(d_tmem, a_tile + 2 * k4, b_desc + 2 * k4, idesc, first ? 0u : 1u);
                  else if (ATM) umma_bf16_ts(d_tmem, a_tm + (kh * 4 + k4) * 8, b_desc + 2 * k4, idesc, first ? 0u : 1u);
                  else umma_bf16(d_tmem, a_tile + 2 * k4, b_desc + 2 * k4, idesc, first ? 0u : 1u);
                  first = false;
                }
              }
            }
            umma_commit(&b_empty[stage]);  // stage reusable once these MMAs have read it
            if (ib == NSEG_B - 1 && kh == KH - 1) {
              umma_commit(&t_full[acc]);
              if (!ATM && (flags & kFlagLast)) umma_commit(&a_empty[a_buf]);
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
    if (STATS && a.stats && lane == 0) {
      atomicAdd(a.stats + kStatMmaBFull, st_bf);
      atomicAdd(a.stats + kStatMmaAFull, st_af);
      atomicAdd(a.stats + kStatMmaTEmpty, st_te);
      atomicAdd(a.stats + kStatGroups, (unsigned long long)g);
    }
  } else if (warp < kEpiWarps) {
    // ================= epilogue: TMEM -> gate*ReLU head reduction -> HBM =================
    // A warp reduces a 32-row quarter of the tile for TWO queries of every second group: eight fragments
    // F(query, row half, column half) of 16 registers (tcgen05.ld.16x128b.x8), streamed through two register buffers
    // so that the load of fragment i+1 is in flight while the FMNMX/FFMA2 work of fragment i issues. The accumulator
    // goes back to the MMA warp as soon as the eighth load has landed.
    // Fragment layout (tcgen05.ld.16x128b, twice the TMEM read rate of 16x256b): a lane owns 16 of the 64 heads for
    // two key rows per row half, so it needs only 16 gates (64 B) per query instead of all 64: the gate traffic
    // through the 128 B/clk shared-memory return path is what bounded a one-row-per-thread (32x32b) epilogue. The 4
    // lanes sharing a row are summed by shuffles.
    setmaxnreg_inc<kEpiRegs>();
    const uint32_t set = warp >> 3;        // accumulator / group parity this warp serves
    const uint32_t quarter = warp & 3u;
    const uint32_t qp = ((warp >> 2) & 1u) * 2u;  // first of the two queries this warp reduces
    const uint32_t w_lane = smem_u32(s_w) + qp * kGateRowBytes + (lane & 3u) * 16u;  // gate_slot: piece (h, c) at h*64 + c*16
    const uint32_t t_lane = tmem_base + ((quarter * 32u) << 16) + set * kAccCols + qp * kHeads;
    const uint32_t row = quarter * 32 + (lane >> 2) + 8u * (lane & 3u);
    const bool b0 = lane & 1u, b1 = lane & 2u;
    const uint32_t t_full_addr = smem_u32(&t_full[set]), t_empty_addr = smem_u32(&t_empty[set]);
    uint32_t vx[16], vy[16];
    if constexpr (ATM) {
      // Groups of three queries: the two warps of a (set, quarter) split the group's twelve fragments six and six. Warp
      // half 0 reduces query 0 and the first row half (TMEM lanes +0..15) of query 1, warp half 1 the second row half of
      // query 1 and query 2: row halves are different key rows, so nothing is combined across warps.
      const uint32_t half = (warp >> 2) & 1u;
      const uint32_t qf = half * 2u;                                  // the query this warp reduces completely
      const uint32_t t_base = tmem_base + ((quarter * 32u) << 16) + set * kAccCols;
      const uint32_t t_full_q = t_base + qf * kHeads;                 // its columns
      const uint32_t t_half_q = t_base + kHeads + ((half * 16u) << 16);  // query 1, this warp's row half
      const uint32_t w_base = smem_u32(s_w) + (lane & 3u) * 16u;
      const bool half_lane = ((lane >> 1) & 1u) == half;              // lanes that end up with a row of the half query
      for (uint32_t g = set;; g += 2) {
        const uint32_t ws = g % kMetaSlots;
        mbar_wait_addr_sleep(t_full_addr, (g >> 1) & 1u, a.epi_sleep_ns);
        const uint32_t maddr = meta_base + ws * uint32_t(sizeof(GroupMeta));
        const uint32_t word = lds_u32(maddr + 32);
        if ((word >> 8) & kFlagTerminate) break;
        const uint32_t nvalid = word & 0xFFu;
        const bool row_ok = row < (word >> 16);
        __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the spin loop
        tc_fence_after();
        const bool full_ok = qf < nvalid, half_ok = 1u < nvalid;
        const uint32_t waddr = w_base + ws * (GQ * kGateRowBytes);
        float4 gw[4];
        float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
        RowSum f;
        float* dst_full = nullptr;
        if (full_ok) {
          tmem_ld_16x128b_x8(t_full_q, vx);                               // F(qf, 0, 0)
#pragma unroll
          for (int h = 0; h < 4; ++h) gw[h] = lds_f4(waddr + qf * kGateRowBytes + h * 64);
          dst_full = a.out + uint64_t(lds_u32(maddr + qf * 4)) * a.out_stride + lds_u32(maddr + 16 + qf * 4) + row;
          tmem_ld_wait();
          tmem_ld_16x128b_x8(t_full_q + 32, vy);                          // F(qf, 0, 1)
          reduce_frag(vx, gw[0], gw[1], a0, a1);
          tmem_ld_wait();
          tmem_ld_16x128b_x8(t_full_q + (16u << 16), vx);                 // F(qf, 1, 0)
          reduce_frag(vy, gw[2], gw[3], a0, a1);
          tmem_ld_wait();
          tmem_ld_16x128b_x8(t_full_q + (16u << 16) + 32, vy);            // F(qf, 1, 1)
          reduce_frag(vx, gw[0], gw[1], a2, a3);
          tmem_ld_wait();
          if (half_ok) tmem_ld_16x128b_x8(t_half_q, vx);                  // F(1, half, 0)
          reduce_frag(vy, gw[2], gw[3], a2, a3);
          f.step1(a0, a1, a2, a3, b0);
        } else if (half_ok) {
          tmem_ld_16x128b_x8(t_half_q, vx);
        }
        if (half_ok) {
#pragma unroll
          for (int h = 0; h < 4; ++h) gw[h] = lds_f4(waddr + kGateRowBytes + h * 64);
          a0 = a1 = make_float2(0.f, 0.f);
          tmem_ld_wait();
          tmem_ld_16x128b_x8(t_half_q + 32, vy);                          // F(1, half, 1)
          if (full_ok) f.step2(b1);
          reduce_frag(vx, gw[0], gw[1], a0, a1);
          tmem_ld_wait();
        } else if (full_ok) {
          f.step2(b1);
        }
        // every dot this warp needs is in registers: hand the accumulator back to the MMA warp
        tc_fence_before();
        __syncwarp();
        if (elect_one()) mbar_arrive_addr(t_empty_addr);
        if (full_ok && row_ok) *dst_full = f.result();
        if (half_ok) {
          reduce_frag(vy, gw[2], gw[3], a0, a1);
          // two rows over four lanes: lane bit 0 picks the row, lane bit 1 only splits the heads
          const float s0 = a0.x + a0.y, s1 = a1.x + a1.y;
          float r = (b0 ? s1 : s0) + __shfl_xor_sync(0xffffffffu, b0 ? s0 : s1, 1);
          r += __shfl_xor_sync(0xffffffffu, r, 2);
          if (half_lane && row_ok)
            a.out[uint64_t(lds_u32(maddr + 4)) * a.out_stride + lds_u32(maddr + 16 + 4) + row] = r;
        }
      }
    } else
    for (uint32_t g = set;; g += 2) {
      const uint32_t ws = g % kMetaSlots;
      mbar_wait_addr_sleep(t_full_addr, (g >> 1) & 1u, a.epi_sleep_ns);
      const uint32_t maddr = meta_base + ws * uint32_t(sizeof(GroupMeta));
      const uint32_t word = lds_u32(maddr + 32);
      if ((word >> 8) & kFlagTerminate) break;
      const uint32_t nvalid = word & 0xFFu;
      const bool row_ok = row < (word >> 16);
      float kscale = 1.f;
      if (FP8 && row_ok && a.a_scale) kscale = __ldg(a.a_scale + lds_u32(maddr + 36) + row);
      __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the spin loop
      tc_fence_after();
      const bool act0 = qp < nvalid;
      const bool act1 = qp + 1 < nvalid;
      const uint32_t waddr = w_lane + ws * (GQ * kGateRowBytes);
      if (act0) {
        // fragment address: + 32 per column half, + 16 lanes per row half, + 64 columns for the second query
        tmem_ld_16x128b_x8(t_lane, vx);                                // F(0, 0, 0)
        float4 gw[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) gw[h] = lds_f4(waddr + h * 64);
        const uint2 qrows = lds_u2(maddr + qp * 4), qcols = lds_u2(maddr + 16 + qp * 4);
        float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
        RowSum f;
        tmem_ld_wait();
        tmem_ld_16x128b_x8(t_lane + 32, vy);                           // F(0, 0, 1)
        reduce_frag(vx, gw[0], gw[1], a0, a1);
        tmem_ld_wait();
        tmem_ld_16x128b_x8(t_lane + (16u << 16), vx);                  // F(0, 1, 0)
        reduce_frag(vy, gw[2], gw[3], a0, a1);
        tmem_ld_wait();
        tmem_ld_16x128b_x8(t_lane + (16u << 16) + 32, vy);             // F(0, 1, 1)
        reduce_frag(vx, gw[0], gw[1], a2, a3);
        tmem_ld_wait();
        if (act1) tmem_ld_16x128b_x8(t_lane + kHeads, vx);             // F(1, 0, 0)
        reduce_frag(vy, gw[2], gw[3], a2, a3);
        f.step1(a0, a1, a2, a3, b0);
        float* dst0 = a.out + uint64_t(qrows.x) * a.out_stride + qcols.x + row;
        if (act1) {
#pragma unroll
          for (int h = 0; h < 4; ++h) gw[h] = lds_f4(waddr + kGateRowBytes + h * 64);
          a0 = a1 = a2 = a3 = make_float2(0.f, 0.f);
          tmem_ld_wait();
          tmem_ld_16x128b_x8(t_lane + kHeads + 32, vy);                // F(1, 0, 1)
          f.step2(b1);
          reduce_frag(vx, gw[0], gw[1], a0, a1);
          tmem_ld_wait();
          tmem_ld_16x128b_x8(t_lane + kHeads + (16u << 16), vx);       // F(1, 1, 0)
          if (row_ok) *dst0 = f.result() * kscale;
          reduce_frag(vy, gw[2], gw[3], a0, a1);
          tmem_ld_wait();
          tmem_ld_16x128b_x8(t_lane + kHeads + (16u << 16) + 32, vy);  // F(1, 1, 1)
          reduce_frag(vx, gw[0], gw[1], a2, a3);
          tmem_ld_wait();
        } else {
          f.step2(b1);
          if (row_ok) *dst0 = f.result() * kscale;
        }
        // all dots of the group are in registers: hand the accumulator back to the MMA warp
        tc_fence_before();
        __syncwarp();
        if (elect_one()) mbar_arrive_addr(t_empty_addr);
        if (act1) {
          reduce_frag(vy, gw[2], gw[3], a2, a3);
          f.step1(a0, a1, a2, a3, b0);
          f.step2(b1);
          if (row_ok) a.out[uint64_t(qrows.y) * a.out_stride + qcols.y + row] = f.result() * kscale;
        }
      } else {
        tc_fence_before();
        __syncwarp();
        if (elect_one()) mbar_arrive_addr(t_empty_addr);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
  if (STATS && a.stats && threadIdx.x == 0) {
    const unsigned long long life = (unsigned long long)(clock64() - cta_c0);
    atomicAdd(a.stats + kStatCta, life);
    atomicMax(a.stats + kStatCtaMax, life);  // longest-lived CTA of any launch since the last read: tail imbalance
  }
}

template <int NSEG_A, int NSEG_B, uint32_t TERMS, int ABUF, int NST, bool FP8, bool ATM, bool STATS>
void launch_instance(const ScoreArgs& args, const CUtensorMap& map_a, const CUtensorMap& map_b, int num_sms,
                     cudaStream_t stream) {
  using L = SmemLayout<NSEG_A, ABUF, NST, FP8 ? 1 : 2, ATM ? 3 : kGroupQ>;
  constexpr size_t smem = L::total + 1024;  // slack for the manual 1024 B alignment
  static_assert(smem <= 232448, "more shared memory than an SM has");
  auto kern = score_tc_kernel<NSEG_A, NSEG_B, TERMS, ABUF, NST, FP8, ATM, STATS>;
  smem_opt_in(reinterpret_cast<const void*>(kern), smem);
  kern<<<num_sms, kTcThreads, smem, stream>>>(map_a, map_b, args);
}

template <int NSEG_A, int NSEG_B, uint32_t TERMS, int ABUF, int NST, bool FP8 = false, bool ATM = false>
int launch_variant(const ScoreArgs& args, const CUtensorMap& map_a, const CUtensorMap& map_b, int num_sms,
                   cudaStream_t stream) {
  if (args.stats) launch_instance<NSEG_A, NSEG_B, TERMS, ABUF, NST, FP8, ATM, true>(args, map_a, map_b, num_sms, stream);
  else launch_instance<NSEG_A, NSEG_B, TERMS, ABUF, NST, FP8, ATM, false>(args, map_a, map_b, num_sms, stream);
  return 1;
}

constexpr uint32_t pack_terms(uint32_t t0, uint32_t t1, uint32_t t2) { return t0 | (t1 << 4) | (t2 << 8); }

}  // namespace

int launch_score_tc(const ScoreArgs& args, const CUtensorMap& map_a, const CUtensorMap& map_b, int num_sms,
                    cudaStream_t stream) {
  const uint32_t terms = pack_terms(args.terms[0], args.terms[1], args.terms[2]);
  // the segment structure is compiled in; these are the combinations the context produces
  if (args.fp8) {
    if (args.nseg_a == 1 && args.nseg_b == 1 && terms == pack_terms(1, 0, 0))
      return launch_variant<1, 1, pack_terms(1, 0, 0), 2, 5, true>(args, map_a, map_b, num_sms, stream);
    // pooled keys as four e4m3 terms (block scores of e4m3 storage): 64 KB tile, one buffer, four query stages
    if (args.nseg_a == 4 && args.nseg_b == 1 && terms == pack_terms(15, 0, 0))
      return launch_variant<4, 1, pack_terms(15, 0, 0), 1, 4, true>(args, map_a, map_b, num_sms, stream);
    return -1;
  }
  if (args.nseg_a == 1 && args.nseg_b == 1 && terms == pack_terms(1, 0, 0)) {
    if (args.a_tmem) return launch_variant<1, 1, pack_terms(1, 0, 0), 1, 7, false, true>(args, map_a, map_b, num_sms, stream);
    return launch_variant<1, 1, pack_terms(1, 0, 0), 2, 4>(args, map_a, map_b, num_sms, stream);
  }
  if (args.nseg_a == 2 && args.nseg_b == 1 && terms == pack_terms(3, 0, 0))
    return launch_variant<2, 1, pack_terms(3, 0, 0), 1, 4>(args, map_a, map_b, num_sms, stream);
  if (args.nseg_a == 3 && args.nseg_b == 1 && terms == pack_terms(7, 0, 0))
    return launch_variant<3, 1, pack_terms(7, 0, 0), 1, 3>(args, map_a, map_b, num_sms, stream);
  if (args.nseg_a == 3 && args.nseg_b == 3 && terms == pack_terms(7, 3, 1))
    return launch_variant<3, 3, pack_terms(7, 3, 1), 1, 3>(args, map_a, map_b, num_sms, stream);
  return -1;  // unsupported segment structure (the context never builds one)
}

}  // namespace hisa_dev
