// Context + C ABI implementation (include/hisa_cuda.h). Host-side orchestration only: every arithmetic
// step of the indexer runs in the CUDA kernels of pool.cu / score_tc.cu / select.cu. There is no CPU
// fallback anywhere in this file: a missing device or a failed launch is an error.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/hisa_cuda.h"
#include "kernels.cuh"

using namespace hisa_dev;

namespace {

thread_local std::string g_global_error;

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <class T> T* as() const { return static_cast<T*>(p); }
};

enum Stage { kStPrepare = 0, kStScoreBlocks, kStSelectBlocks, kStInvert, kStScoreTokens, kStTopK, kStTotal, kNumStages };

struct StageSpan {
  int stage;
  cudaEvent_t beg, end;
};

}  // namespace

struct hisa_cuda_ctx {
  hisa_cuda_config cfg{};
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::string err;

  // operand geometry
  uint32_t nseg_k = 1, nseg_q = 1, nseg_p = 2;
  uint32_t terms_tok[kMaxSeg] = {1, 0, 0};
  uint32_t terms_blk[kMaxSeg] = {3, 0, 0};
  bool q_zero_copy = false;  // caller's q already is the operand (bf16, H=64, d=128)
  bool fp8 = false;          // e4m3 storage: byte operands + per-key scales; stage 1 uses a bf16 copy of q

  // sequence state
  uint64_t seq_len = 0, key_cap = 0;
  uint64_t pooled_tokens = 0;  // tokens folded into the summaries so far
  // summaries installed by hisa_cuda_pool_set (a BlockSummaryCache snapshot that may cover fewer tokens than the key
  // sequence, hisa/hisa.hpp:16-21): eligibility is clipped to pool_blocks and the keys are not re-pooled
  bool pool_external = false;
  uint64_t pool_blocks = 0;
  DevBuf key_op, key_raw, key_scale, sums, counts, pooled_op, pool_scale;
  bool pool8 = false;  // e4m3 storage + tensor-core scorer: pooled keys are four e4m3 terms + a power-of-two scale per block

  // per-call workspace
  DevBuf q_raw, q_op, gates_raw, gates_pad, pos, J, sel, nsel, work, pairs, scalars, cand, flat, out_idx, out_count,
      out_cand, generic_scores, generic_n, export_a, export_b, flag, stats, inv_scratch;

  // decode steps as one graph launch: the device word `dlen` always holds seq_len; a small hisa_select whose arguments
  // repeat (same device pointers, same Q) is captured once with every kernel reading the sequence length from `dlen`,
  // and replayed by later calls while the sequence grows underneath it (hisa_cuda_pool_append updates `dlen`)
  DevBuf dlen;
  struct GraphSig {
    const void *q, *g, *pos, *idx, *cnt, *blk, *nblk, *cand, *key_base, *pool_base;
    uint64_t Q, key_cap;
    uint32_t Mb;
    bool operator==(const GraphSig& o) const { return memcmp(this, &o, sizeof *this) == 0; }
  };
  GraphSig g_sig{}, g_pending{};
  cudaGraphExec_t g_exec = nullptr;
  uint32_t g_seen = 0, g_launches = 0;
  bool g_enabled = true;
  bool dyn = false;      // kernels of the current call read the sequence length from dlen
  uint32_t dyn_Mb = 0;   // upper bound of the number of summarised blocks while the captured graph stays valid

  // output placement for row-sharded multi-GPU runs (hisa_cuda_set_output_placement)
  const uint32_t* place_rows = nullptr;
  uint64_t place_q0 = 0;  // first row of the current host-pipeline slice inside the call (select_pipelined)
  uint32_t place_nrep = 0;
  int32_t* place_rep_idx[kMaxReplicas] = {};
  uint32_t* place_rep_count[kMaxReplicas] = {};

  // downstream consumer (attention.hpp): latent table + per-call staging
  DevBuf attn_lat, attn_q, attn_qraw, attn_pos, attn_idx, attn_cnt, attn_out, attn_w;
  uint64_t attn_len = 0;
  uint32_t attn_dm = 0, attn_dm_pad = 0;
  bool attn_bf16 = false;
  cudaEvent_t attn_beg = nullptr, attn_end = nullptr;
  bool attn_timed = false;

  // tuning
  uint32_t chunk_dense = 128, chunk_list = 512;
  uint64_t workspace_bytes = 4ull << 30;

  // instrumentation
  bool profiling = false;    // CUDA events around every stage
  bool stall_stats = false;  // additionally run the instrumented scorer instantiation (role-level stall cycles)
  std::vector<StageSpan> spans;
  std::vector<cudaEvent_t> event_pool;
  size_t events_used = 0;
  uint64_t launches = 0, call_launches = 0;
  uint64_t items1 = 0, items2 = 0;
  StageSpan call_span{};
  bool call_open = false;
  uint64_t calls = 0;

  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;

  // host-buffer pipeline (select_impl): slices of pipe_rows rows are staged through double-buffered device
  // arrays so that the H2D copy of slice i+1 and the D2H copy of slice i-1 overlap the kernels of slice i
  uint32_t pipe_rows = 4096;
  bool pipe_ready = false;
  cudaStream_t in_stream = nullptr, out_stream = nullptr;
  cudaEvent_t ev_in_ready[2]{}, ev_in_free[2]{}, ev_out_ready[2]{}, ev_out_free[2]{};
  DevBuf st_q[2], st_g[2], st_pos[2], st_idx[2], st_cnt[2], st_cand[2], st_blk[2], st_nblk[2];
};

namespace {

uint32_t env_u32(const char* name, uint32_t dflt);

int fail(hisa_cuda_ctx* ctx, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  else g_global_error = buf;
  return code;
}

#define CU_TRY(ctx, expr)                                                                                   \
  do {                                                                                                      \
    cudaError_t e__ = (expr);                                                                               \
    if (e__ != cudaSuccess)                                                                                 \
      return fail(ctx, e__ == cudaErrorMemoryAllocation ? HISA_ERR_OUT_OF_MEMORY : HISA_ERR_CUDA,           \
                  "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e__), __FILE__, __LINE__);             \
  } while (0)

#define HISA_TRY(expr)            \
  do {                            \
    int rc__ = (expr);            \
    if (rc__ != HISA_OK) return rc__; \
  } while (0)

void drop_graph(hisa_cuda_ctx* ctx);

int ensure(hisa_cuda_ctx* ctx, DevBuf& b, size_t bytes) {
  if (bytes <= b.cap) return HISA_OK;
  // a captured decode graph holds the addresses of the workspace buffers as kernel arguments: a buffer that moves (a larger
  // call between two decode steps) must take the graph with it, or the next replay reads and writes freed memory
  drop_graph(ctx);
  if (b.p) {
    CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    CU_TRY(ctx, cudaFree(b.p));
    b.p = nullptr;
    b.cap = 0;
  }
  const size_t want = (bytes + 255) & ~size_t(255);
  CU_TRY(ctx, cudaMalloc(&b.p, want));
  b.cap = want;
  return HISA_OK;
}

void release(DevBuf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

uint32_t elem_bytes(const hisa_cuda_ctx* ctx) {
  return ctx->cfg.dtype == HISA_DTYPE_BF16 ? 2u : ctx->cfg.dtype == HISA_DTYPE_FP8_E4M3 ? 1u : 4u;
}
// element type code of the operand-preparation kernels: 0 f32, 1 bf16, 2 e4m3
uint32_t src_type(const hisa_cuda_ctx* ctx) { return ctx->cfg.dtype == HISA_DTYPE_BF16 ? 1u : ctx->cfg.dtype == HISA_DTYPE_FP8_E4M3 ? 2u : 0u; }
uint32_t round_up(uint32_t v, uint32_t m) { return (v + m - 1) / m * m; }
uint64_t round_up64(uint64_t v, uint64_t m) { return (v + m - 1) / m * m; }

cudaEvent_t next_event(hisa_cuda_ctx* ctx) {
  if (ctx->events_used == ctx->event_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->event_pool.push_back(e);
  }
  return ctx->event_pool[ctx->events_used++];
}

struct StageTimer {
  hisa_cuda_ctx* ctx;
  StageSpan span{};
  bool on;
  StageTimer(hisa_cuda_ctx* c, int stage) : ctx(c), on(c->profiling) {
    if (on) {
      span.stage = stage;
      span.beg = next_event(ctx);
      span.end = next_event(ctx);
      cudaEventRecord(span.beg, ctx->stream);
    }
  }
  ~StageTimer() {
    if (on) {
      cudaEventRecord(span.end, ctx->stream);
      ctx->spans.push_back(span);
    }
  }
};

void count_launches(hisa_cuda_ctx* ctx, int n) {
  ctx->launches += uint64_t(n);
  ctx->call_launches += uint64_t(n);
}

int check_launch(hisa_cuda_ctx* ctx, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, HISA_ERR_CUDA, "launch of %s failed: %s", what, cudaGetErrorString(e));
  return HISA_OK;
}

// 2-D map over a row-major operand whose rows are `cols` elements; the box is one 128-byte swizzle row wide
// (64 bf16 or 128 e4m3 elements) and `box_rows` rows tall
int make_map(hisa_cuda_ctx* ctx, CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
             bool bytes = false) {
  cuuint64_t gdim[2] = {cols, rows ? rows : 1};
  cuuint64_t gstride[1] = {cols * (bytes ? 1 : sizeof(__nv_bfloat16))};
  cuuint32_t box[2] = {bytes ? 128u : 64u, box_rows};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = ctx->encode(map, bytes ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                           const_cast<void*>(base), gdim, gstride, box,
                           estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(ctx, HISA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu base=%p", int(r),
                (unsigned long long)rows, (unsigned long long)cols, base);
  return HISA_OK;
}

uint64_t num_blocks_of(const hisa_cuda_ctx* ctx) {
  return (ctx->seq_len + ctx->cfg.block_size - 1) / ctx->cfg.block_size;
}
// blocks the current summaries cover: eligible blocks of a query are [0, floor(t/B)] clipped to this (hisa.hpp:16-21)
uint64_t pool_blocks_of(const hisa_cuda_ctx* ctx) {
  return ctx->pool_external ? std::min<uint64_t>(ctx->pool_blocks, num_blocks_of(ctx)) : num_blocks_of(ctx);
}

// ------------------------------------------------------------------------------------------------
// prepared per-call inputs (device pointers valid until the next call on the context)
// ------------------------------------------------------------------------------------------------
struct Prepared {
  const __nv_bfloat16* q_op = nullptr;  // [Q*64, nseg_q*128]
  const uint8_t* q8 = nullptr;          // fp8 storage: the caller's e4m3 bytes [Q*64, 128] (stage 2 / flat operand)
  const float* gates = nullptr;         // [Q, 64]
  const uint32_t* pos = nullptr;        // [Q]
  uint64_t Q = 0;
};

int copy_in(hisa_cuda_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return HISA_OK;
  CU_TRY(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
  return HISA_OK;
}

int read_flag(hisa_cuda_ctx* ctx, uint32_t* value) {
  CU_TRY(ctx, cudaMemcpyAsync(value, ctx->flag.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return HISA_OK;
}

int prepare_inputs(hisa_cuda_ctx* ctx, const void* queries, const float* gates, const uint32_t* positions,
                   uint64_t Q, int check_finite, Prepared* out) {
  if (ctx->seq_len == 0) return fail(ctx, HISA_ERR_EMPTY_SEQUENCE, "selection over an empty key sequence");
  if (Q == 0) {
    out->Q = 0;
    return HISA_OK;
  }
  if (!queries || !gates || !positions)
    return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "queries, gates and positions must be non-null");
  if (Q > 0x7FFFFFFFull / kHeads) return fail(ctx, HISA_ERR_UNSUPPORTED, "too many query rows in one call");
  StageTimer timer(ctx, kStPrepare);
  const uint32_t H = ctx->cfg.num_heads, d = ctx->cfg.dim, eb = elem_bytes(ctx);
  const uint32_t st = src_type(ctx);

  // positions
  const uint32_t* pos_dev = positions;
  if (!is_device_ptr(positions)) {
    HISA_TRY(ensure(ctx, ctx->pos, Q * sizeof(uint32_t)));
    HISA_TRY(copy_in(ctx, ctx->pos.p, positions, Q * sizeof(uint32_t)));
    pos_dev = ctx->pos.as<uint32_t>();
  }
  // queries
  const size_t q_elems = size_t(Q) * H * d;
  const void* q_dev = queries;
  if (!is_device_ptr(queries)) {
    DevBuf& dst = ctx->q_zero_copy ? ctx->q_op : ctx->q_raw;
    HISA_TRY(ensure(ctx, dst, q_elems * eb));
    HISA_TRY(copy_in(ctx, dst.p, queries, q_elems * eb));
    q_dev = dst.p;
  }
  // gates
  const float* g_dev = gates;
  if (!is_device_ptr(gates)) {
    HISA_TRY(ensure(ctx, ctx->gates_raw, size_t(Q) * H * sizeof(float)));
    HISA_TRY(copy_in(ctx, ctx->gates_raw.p, gates, size_t(Q) * H * sizeof(float)));
    g_dev = ctx->gates_raw.as<float>();
  }
  if (check_finite) {
    HISA_TRY(ensure(ctx, ctx->flag, 16));
    CU_TRY(ctx, cudaMemsetAsync(ctx->flag.p, 0, 16, ctx->stream));
    uint32_t* f = ctx->flag.as<uint32_t>();
    count_launches(ctx, launch_check_finite(q_dev, st, q_elems, f, ctx->stream));
    count_launches(ctx, launch_check_finite(g_dev, 0, size_t(Q) * H, f + 1, ctx->stream));
    count_launches(ctx, launch_check_positions(pos_dev, Q, uint32_t(ctx->seq_len), f + 2, ctx->stream));
    uint32_t flags[3];
    CU_TRY(ctx, cudaMemcpyAsync(flags, f, sizeof flags, cudaMemcpyDeviceToHost, ctx->stream));
    CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (flags[0]) return fail(ctx, HISA_ERR_NON_FINITE, "inputs: non-finite value in queries");
    if (flags[1]) return fail(ctx, HISA_ERR_NON_FINITE, "inputs: non-finite value in gates");
    if (flags[2]) return fail(ctx, HISA_ERR_SHAPE_MISMATCH, "inputs: a query position exceeds the sequence length %llu",
                              (unsigned long long)ctx->seq_len);
  }
  // operands
  if (ctx->q_zero_copy) {
    out->q_op = static_cast<const __nv_bfloat16*>(q_dev);
  } else if (ctx->pool8) {
    out->q_op = nullptr;  // every scorer reads the e4m3 bytes
  } else {
    HISA_TRY(ensure(ctx, ctx->q_op, size_t(Q) * kHeads * ctx->nseg_q * kDim * sizeof(__nv_bfloat16)));
    count_launches(ctx, launch_convert_rows(q_dev, st, Q, H, d, ctx->nseg_q, ctx->q_op.as<__nv_bfloat16>(), kHeads,
                                            ctx->stream));
    out->q_op = ctx->q_op.as<__nv_bfloat16>();
  }
  if (ctx->fp8) out->q8 = static_cast<const uint8_t*>(q_dev);  // H = 64, d = 128 is required for fp8: zero-copy
  // gates are always re-laid out (padded to 64 heads, permuted to the epilogue's lane order): 256 B per query
  HISA_TRY(ensure(ctx, ctx->gates_pad, size_t(Q) * kHeads * sizeof(float)));
  count_launches(ctx, launch_permute_gates(g_dev, Q, H, ctx->gates_pad.as<float>(), ctx->stream));
  out->gates = ctx->gates_pad.as<float>();
  out->pos = pos_dev;
  out->Q = Q;
  return check_launch(ctx, "input preparation");
}

// ------------------------------------------------------------------------------------------------
// scorer dispatch
// ------------------------------------------------------------------------------------------------
struct ScoreJob {
  int stats_slot;  // 0: stage 1, 1: stage 2 / flat
  uint32_t counter_slot = 0;  // which pair of device scalars holds the work count / cursor (0: sc[0..1], 2: sc[2..3])
  const __nv_bfloat16* a_op;
  uint64_t a_rows;
  uint32_t nseg_a;
  const uint32_t* terms;
  const __nv_bfloat16* q_op;  // rows [0, nq*64)
  uint64_t nq;
  const float* gates;
  float* out;
  uint64_t out_stride;
  bool list_mode;
  const uint2* pairs;
  uint32_t max_items;
  // fp8 storage (stage 2 / flat only): byte operands and the per-key scale
  const uint8_t* a8 = nullptr;
  const uint8_t* q8 = nullptr;
  const float* a_scale = nullptr;
};

// HISA_TC_ATMEM=1 (bf16 keys and queries, one segment each): the token scorer multiplies the key tile from tensor memory,
// in groups of three queries. Measured slower than the shared-memory-operand form (score_tc.cu), hence opt-in.
bool token_scorer_uses_tmem_tile(const hisa_cuda_ctx* ctx) {
  return !ctx->fp8 && ctx->nseg_k == 1 && ctx->nseg_q == 1 && env_u32("HISA_TC_ATMEM", 0) != 0;
}

int run_scorer(hisa_cuda_ctx* ctx, const ScoreJob& j) {
  ScoreArgs a{};
  uint32_t* sc = ctx->scalars.as<uint32_t>();
  a.work = ctx->work.as<WorkItem>();
  a.work_count = sc + j.counter_slot;
  a.work_cursor = sc + j.counter_slot + 1;
  a.pairs = j.pairs;
  a.gates = j.gates;
  a.out = j.out;
  a.out_stride = j.out_stride;
  a.list_mode = j.list_mode ? 1u : 0u;
  const uint32_t B = ctx->cfg.block_size;
  a.segs_per_block = j.list_mode ? (B + kTileRows - 1) / kTileRows : 1u;
  a.block_rows = j.list_mode ? B : uint32_t(kTileRows);
  a.nseg_a = j.nseg_a;
  a.nseg_b = ctx->nseg_q;
  for (int i = 0; i < kMaxSeg; ++i) a.terms[i] = j.terms[i];
  a.a_rows = uint32_t(j.a_rows);
  a.fp8 = j.a8 ? 1u : 0u;
  a.a_scale = j.a_scale;
  a.epi_sleep_ns = env_u32("HISA_TC_EPI_SLEEP", 0);
  a.a_tmem = (!j.a8 && a.nseg_a == 1 && a.nseg_b == 1 && token_scorer_uses_tmem_tile(ctx)) ? 1u : 0u;
  a.producers = std::min<uint32_t>(std::max<uint32_t>(env_u32("HISA_TC_PRODUCERS", j.a8 ? 2 : 3), 1), 3);
  a.stats = nullptr;
  if (ctx->profiling && ctx->stall_stats) {
    if (!ctx->stats.p) {
      HISA_TRY(ensure(ctx, ctx->stats, 2 * 16 * sizeof(unsigned long long)));
      CU_TRY(ctx, cudaMemsetAsync(ctx->stats.p, 0, 2 * 16 * sizeof(unsigned long long), ctx->stream));
    }
    a.stats = ctx->stats.as<unsigned long long>() + 16 * j.stats_slot;
  }
  if (ctx->cfg.scorer == HISA_SCORER_SIMT) {
    count_launches(ctx, launch_score_simt(a, j.a_op, j.q_op, j.max_items, ctx->stream));
  } else {
    CUtensorMap map_a, map_b;
    if (j.a8) {
      a.nseg_b = 1;
      HISA_TRY(make_map(ctx, &map_a, j.a8, j.a_rows, uint64_t(a.nseg_a) * kDim, kTileRows, true));
      HISA_TRY(make_map(ctx, &map_b, j.q8, j.nq * kHeads, kDim, kHeads, true));
    } else {
      HISA_TRY(make_map(ctx, &map_a, j.a_op, j.a_rows, uint64_t(j.nseg_a) * kDim, kTileRows));
      HISA_TRY(make_map(ctx, &map_b, j.q_op, j.nq * kHeads, uint64_t(ctx->nseg_q) * kDim, kHeads));
    }
    const int n = launch_score_tc(a, map_a, map_b, ctx->num_sms, ctx->stream);
    if (n < 0) return fail(ctx, HISA_ERR_UNSUPPORTED, "no tensor-core scorer variant for this operand segment structure");
    count_launches(ctx, n);
  }
  return check_launch(ctx, "scorer");
}

// operands of a token-scoring job (stage 2, flat, score_tokens) for query rows [q0, ...)
void set_token_operands(hisa_cuda_ctx* ctx, const Prepared& p, uint64_t q0, ScoreJob& j) {
  // graph replay: the map covers the whole key allocation, rows beyond the live sequence are never selected
  j.a_rows = ctx->dyn ? ctx->key_cap : ctx->seq_len;
  j.terms = ctx->terms_tok;
  if (ctx->fp8) {
    j.a8 = ctx->key_op.as<uint8_t>();
    j.q8 = p.q8 + q0 * kHeads * kDim;
    j.a_scale = ctx->key_scale.as<float>();
    j.nseg_a = 1;
  } else {
    j.a_op = ctx->key_op.as<__nv_bfloat16>();
    j.nseg_a = ctx->nseg_k;
    j.q_op = p.q_op + q0 * kHeads * ctx->nseg_q * kDim;
  }
}

void drop_graph(hisa_cuda_ctx* ctx) {
  if (ctx->g_exec) cudaGraphExecDestroy(ctx->g_exec);
  ctx->g_exec = nullptr;
  ctx->g_seen = 0;
  memset(&ctx->g_sig, 0, sizeof ctx->g_sig);
  memset(&ctx->g_pending, 0, sizeof ctx->g_pending);
}

// Upper bound of the block count under which a captured decode graph stays valid: the next boundary at which
// launch_select would pick another kernel variant for the block scores, clipped to the rows the pooled operand has.
uint32_t block_bucket(const hisa_cuda_ctx* ctx, uint32_t M) {
  static const uint32_t bounds[] = {128u, 512u, 1024u, 9216u, 18432u, 36864u, 49152u};
  uint32_t b = 0xFFFFFFFFu;
  for (uint32_t x : bounds)
    if (M <= x) { b = x; break; }
  const uint64_t alloc = ctx->key_cap / ctx->cfg.block_size + 1;  // rows of pooled_op (grow_keys)
  return uint32_t(std::min<uint64_t>(b, alloc));
}

int ensure_pool(hisa_cuda_ctx* ctx) {
  if (ctx->pool_external || ctx->pooled_tokens == ctx->seq_len) return HISA_OK;
  return hisa_cuda_pool_build(ctx);
}

// Queries per dense work item. The configured chunk (128: stage 1 at 64K has 4 pooled-key tiles, and with 256-query
// chunks its 640 items were 4.3 per SM, i.e. a CTA balance of 0.86; 1280 items give 0.95 and 0.57 -> 0.51 ms) amortises
// a tile load over many queries; calls with few rows
// (decode batches, the paper's 1024-row tail) would then produce fewer items than there are SMs, so the chunk is
// halved until every SM has about two items (never below two MMA groups).
uint32_t dense_chunk_for(const hisa_cuda_ctx* ctx, uint64_t nq, uint32_t ntiles) {
  uint32_t chunk = ctx->chunk_dense;
  while (chunk > 8 && ((nq + chunk - 1) / chunk) * ntiles < 2ull * uint64_t(ctx->num_sms)) chunk /= 2;
  return chunk;
}

// Queries per chunk of the block-major refinement (one work item per chunk and selected key block). 512 queries
// amortise a key-tile load over ~16 groups at prefill sizes; a call with few rows (the paper's 1024-row tail, a
// pipeline slice) would then leave the 148 persistent CTAs with a handful of long items each (6.9 per SM at 1024
// rows: 0.205 ms for stage 2 against 0.163 ms with 128-query chunks), so the chunk is halved until a call has at
// least eight chunks (never below 64 queries).
uint32_t list_chunk_for(const hisa_cuda_ctx* ctx, uint64_t nq) {
  uint32_t chunk = ctx->chunk_list;
  while (chunk > 64 && (nq + chunk - 1) / chunk < 8) chunk /= 2;
  return chunk;
}

// stage 1: J[q, b] for rows [0, nq) -> ctx->J with stride Mpad
int run_score_blocks(hisa_cuda_ctx* ctx, const Prepared& p, uint64_t q0, uint64_t nq, uint32_t Mpad) {
  const uint32_t M = ctx->dyn ? ctx->dyn_Mb : uint32_t(pool_blocks_of(ctx));
  const uint32_t ntiles = Mpad / kTileRows;
  const uint32_t chunk = dense_chunk_for(ctx, nq, ntiles);
  const uint32_t nchunks = uint32_t((nq + chunk - 1) / chunk);
  HISA_TRY(ensure(ctx, ctx->work, std::max<size_t>(size_t(nchunks) * ntiles, size_t(ctx->num_sms)) * sizeof(WorkItem)));  // >= one slot per CTA
  HISA_TRY(ensure(ctx, ctx->J, size_t(nq) * Mpad * sizeof(float)));
  uint32_t* sc = ctx->scalars.as<uint32_t>();
  StageTimer timer(ctx, kStScoreBlocks);
  // sc[2], sc[3]: the counters of the stage-2 work list, cleared by this kernel (one launch less per call)
  count_launches(ctx, launch_build_dense_work(p.pos + q0, uint32_t(nq), chunk, uint32_t(ctx->seq_len),
                                              ctx->cfg.block_size, ntiles, ctx->work.as<WorkItem>(), sc, sc + 1,
                                              ctx->dyn ? ctx->dlen.as<uint32_t>() : nullptr, sc + 2, sc + 3, ctx->stream));
  ScoreJob j{};
  j.a_rows = M;
  static const uint32_t terms_pool8[kMaxSeg] = {(1u << kPool8Seg) - 1u, 0, 0};
  if (ctx->pool8) {
    // e4m3 storage: the queries stay e4m3 bytes and meet the pooled keys as four e4m3 terms in kind::f8f6f4 (no bf16 copy
    // of the queries); the block's power-of-two scale multiplies the finished row sum like a key's scale does in stage 2
    j.a8 = ctx->pooled_op.as<uint8_t>();
    j.q8 = p.q8 + q0 * kHeads * kDim;
    j.a_scale = ctx->pool_scale.as<float>();
    j.nseg_a = kPool8Seg;
    j.terms = terms_pool8;
  } else {
    j.a_op = ctx->pooled_op.as<__nv_bfloat16>();
    j.nseg_a = ctx->nseg_p;
    j.terms = ctx->terms_blk;
    j.q_op = p.q_op + q0 * kHeads * ctx->nseg_q * kDim;
  }
  j.nq = nq;
  j.gates = p.gates + q0 * kHeads;
  j.out = ctx->J.as<float>();
  j.out_stride = Mpad;
  j.list_mode = false;
  j.max_items = nchunks * ntiles;
  ctx->items1 += j.max_items;
  return run_scorer(ctx, j);
}

int run_select_blocks(hisa_cuda_ctx* ctx, const Prepared& p, uint64_t q0, uint64_t nq, uint32_t Mpad, int32_t* sel,
                      uint32_t* nsel) {
  StageTimer timer(ctx, kStSelectBlocks);
  SelectArgs s{};
  s.scores = ctx->J.as<float>();
  s.stride = Mpad;
  s.pos = p.pos + q0;
  s.seq_len = uint32_t(ctx->seq_len);
  s.num_blocks = ctx->dyn ? ctx->dyn_Mb : uint32_t(pool_blocks_of(ctx));
  s.dyn_len = ctx->dyn ? ctx->dlen.as<uint32_t>() : nullptr;
  s.block_size = ctx->cfg.block_size;
  s.keep = ctx->cfg.block_budget;
  s.mode = kSelBlocks;
  s.tie_break = ctx->cfg.tie_break;
  s.force_first_last = ctx->cfg.force_first_last;
  s.forced_in_budget = ctx->cfg.forced_in_budget;
  s.out_idx = sel;
  s.out_stride = ctx->cfg.block_budget + 2;
  s.out_width = ctx->cfg.block_budget + 2;
  s.out_count = nsel;
  count_launches(ctx, launch_select(s, uint32_t(nq), s.num_blocks, ctx->stream));
  return check_launch(ctx, "select_blocks");
}

// gives `dst` (host or device, may be null) the contents of a device staging array
int copy_out(hisa_cuda_ctx* ctx, void* dst, const void* src_dev, size_t bytes, bool* need_sync) {
  if (!dst || dst == src_dev || bytes == 0) return HISA_OK;
  CU_TRY(ctx, cudaMemcpyAsync(dst, src_dev, bytes, cudaMemcpyDefault, ctx->stream));
  if (!is_device_ptr(dst)) *need_sync = true;
  return HISA_OK;
}

// Profiling spans accumulate over every call since the last hisa_cuda_last_stage_times() read.
void begin_call(hisa_cuda_ctx* ctx) {
  ctx->calls += 1;
  ctx->call_open = false;
  if (ctx->profiling) {
    ctx->call_span.stage = kStTotal;
    ctx->call_span.beg = next_event(ctx);
    ctx->call_span.end = next_event(ctx);
    cudaEventRecord(ctx->call_span.beg, ctx->stream);
    ctx->call_open = true;
  }
}
void end_call(hisa_cuda_ctx* ctx) {
  if (ctx->call_open) {
    cudaEventRecord(ctx->call_span.end, ctx->stream);
    ctx->spans.push_back(ctx->call_span);
    ctx->call_open = false;
  }
}

enum Strategy { kDsa = 0, kHisa = 1, kBlockSparse = 2 };

// One selection over rows [0, Q): everything is enqueued on ctx->stream. Host pointers are accepted (copied on the
// same stream, then the stream is synchronised); with device pointers the call returns without synchronising.
int select_core(hisa_cuda_ctx* ctx, Strategy strat, const void* queries, const float* gates, const uint32_t* positions,
                uint64_t Q, int check_finite, int32_t* out_idx, uint32_t* out_count, int32_t* out_blocks,
                uint32_t* out_nblocks, uint32_t* out_cand) {
  Prepared p;
  HISA_TRY(prepare_inputs(ctx, queries, gates, positions, Q, check_finite, &p));
  if (Q == 0) return HISA_OK;

  const hisa_cuda_config& c = ctx->cfg;
  const uint32_t B = c.block_size, S = c.block_budget + 2, k = c.token_budget;
  const uint32_t L = uint32_t(ctx->seq_len);
  const uint32_t M = ctx->dyn ? ctx->dyn_Mb : uint32_t(strat == kDsa ? num_blocks_of(ctx) : pool_blocks_of(ctx));
  const uint32_t Mpad = round_up(M, kTileRows);
  const uint32_t Lpad = round_up(L, kTileRows);
  const uint32_t out_width = strat == kBlockSparse ? S * B : k;
  const uint64_t cand_cols = uint64_t(S) * B;

  HISA_TRY(ensure(ctx, ctx->scalars, 64));
  bool need_sync = false;
  const bool idx_dev = is_device_ptr(out_idx), cnt_dev = is_device_ptr(out_count);
  const bool blk_dev = is_device_ptr(out_blocks), nblk_dev = is_device_ptr(out_nblocks);
  const bool cand_dev = is_device_ptr(out_cand);

  // rows per pass, bounded by the workspace budget
  uint64_t per_row = 0;
  if (strat == kDsa) per_row = uint64_t(Lpad) * 4;
  else per_row = uint64_t(Mpad) * 4 + (strat == kHisa ? cand_cols * 4 : 0) + uint64_t(S) * 12;
  uint64_t pass_rows = std::max<uint64_t>(ctx->workspace_bytes / std::max<uint64_t>(per_row, 1), 1);
  const uint64_t chunk_lcm = uint64_t(ctx->chunk_dense) * ctx->chunk_list / std::min(ctx->chunk_dense, ctx->chunk_list);
  if (pass_rows >= chunk_lcm) pass_rows = pass_rows / chunk_lcm * chunk_lcm;
  pass_rows = std::min<uint64_t>(pass_rows, Q);
  pass_rows = std::min<uint64_t>(pass_rows, uint64_t(ctx->chunk_dense) * 4096);

  if (!idx_dev) HISA_TRY(ensure(ctx, ctx->out_idx, size_t(pass_rows) * out_width * 4));
  if (!cnt_dev) HISA_TRY(ensure(ctx, ctx->out_count, size_t(pass_rows) * 4));
  if (!cand_dev) HISA_TRY(ensure(ctx, ctx->out_cand, size_t(pass_rows) * 4));
  if (strat != kDsa) {
    if (!blk_dev) HISA_TRY(ensure(ctx, ctx->sel, size_t(pass_rows) * S * 4));
    if (!nblk_dev) HISA_TRY(ensure(ctx, ctx->nsel, size_t(pass_rows) * 4));
  }

  // placed output: row i of the call lands at row place_rows[i] of the caller's (full-size) device arrays
  const bool placed = (ctx->place_rows || ctx->place_nrep) && strat != kBlockSparse;
  if (placed && (!idx_dev || (out_count && !cnt_dev) || (out_cand && !cand_dev)))
    return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "output placement needs device output arrays");
  auto place = [&](SelectArgs& s, uint64_t q0) {
    if (!placed) return;
    const uint64_t first = ctx->place_q0 + q0;  // row of the API call this launch starts at
    s.out_rows = ctx->place_rows ? ctx->place_rows + first : nullptr;
    s.n_rep = ctx->place_nrep;
    for (uint32_t r = 0; r < ctx->place_nrep; ++r) {
      // without a row map the replicas are indexed like the local arrays: by the row of the call
      s.rep_out[r] = ctx->place_rep_idx[r] + (ctx->place_rows ? 0 : first * out_width);
      s.rep_count[r] = ctx->place_rep_count[r] ? ctx->place_rep_count[r] + (ctx->place_rows ? 0 : first) : nullptr;
    }
  };

  for (uint64_t q0 = 0; q0 < Q; q0 += pass_rows) {
    const uint64_t nq = std::min<uint64_t>(pass_rows, Q - q0);
    const bool mapped = placed && ctx->place_rows;  // the row map already addresses the full arrays
    int32_t* idx_dst = idx_dev ? out_idx + (mapped ? 0 : q0 * out_width) : ctx->out_idx.as<int32_t>();
    uint32_t* cnt_dst = cnt_dev ? out_count + (mapped ? 0 : q0) : (placed ? nullptr : ctx->out_count.as<uint32_t>());
    uint32_t* cand_dst = cand_dev ? out_cand + (mapped ? 0 : q0) : (placed ? nullptr : ctx->out_cand.as<uint32_t>());

    if (strat == kDsa) {
      // ---- flat indexer: score the whole causal prefix, then top-k (dsa.hpp:29-32) ----
      const uint32_t ntiles = Lpad / kTileRows;
      const uint32_t chunk = dense_chunk_for(ctx, nq, ntiles);
      const uint32_t nchunks = uint32_t((nq + chunk - 1) / chunk);
      HISA_TRY(ensure(ctx, ctx->work, std::max<size_t>(size_t(nchunks) * ntiles, size_t(ctx->num_sms)) * sizeof(WorkItem)));  // >= one slot per CTA
      HISA_TRY(ensure(ctx, ctx->flat, size_t(nq) * Lpad * 4));
      uint32_t* sc = ctx->scalars.as<uint32_t>();
      {
        StageTimer timer(ctx, kStScoreTokens);
        count_launches(ctx, launch_build_dense_work(p.pos + q0, uint32_t(nq), chunk, L, 1, ntiles,
                                                    ctx->work.as<WorkItem>(), sc, sc + 1, nullptr, nullptr, nullptr, ctx->stream));
        ScoreJob j{};
        j.stats_slot = 1;
        set_token_operands(ctx, p, q0, j);
        j.nq = nq;
        j.gates = p.gates + q0 * kHeads;
        j.out = ctx->flat.as<float>();
        j.out_stride = Lpad;
        j.list_mode = false;
        j.max_items = nchunks * ntiles;
        ctx->items2 += j.max_items;
        HISA_TRY(run_scorer(ctx, j));
      }
      {
        StageTimer timer(ctx, kStTopK);
        SelectArgs s{};
        s.scores = ctx->flat.as<float>();
        s.stride = Lpad;
        s.pos = p.pos + q0;
        s.seq_len = L;
        s.num_blocks = M;
        s.block_size = B;
        s.keep = k;
        s.mode = kSelFlat;
        s.tie_break = c.tie_break;
        s.out_idx = idx_dst;
        s.out_stride = out_width;
        s.out_width = out_width;
        s.out_count = cnt_dst;
        s.out_cand = cand_dst;
        place(s, q0);
        count_launches(ctx, launch_select(s, uint32_t(nq), L, ctx->stream));
        HISA_TRY(check_launch(ctx, "top-k"));
      }
    } else {
      int32_t* sel = blk_dev ? out_blocks + q0 * S : ctx->sel.as<int32_t>();
      uint32_t* nsel = nblk_dev ? out_nblocks + q0 : ctx->nsel.as<uint32_t>();
      // ---- stage 1: block scores + top-m with forced blocks (hisa.hpp:16-28) ----
      HISA_TRY(run_score_blocks(ctx, p, q0, nq, Mpad));
      HISA_TRY(run_select_blocks(ctx, p, q0, nq, Mpad, sel, nsel));
      if (strat == kBlockSparse) {
        StageTimer timer(ctx, kStTopK);
        count_launches(ctx, launch_expand_blocks(sel, nsel, S, p.pos + q0, uint32_t(nq), L, B, idx_dst, out_width,
                                                 out_width, cnt_dst, ctx->stream));
        HISA_TRY(check_launch(ctx, "expand blocks"));
      } else {
        // ---- stage 2: block-major refinement over the selected blocks, then top-k (hisa.hpp:30-45) ----
        const uint32_t spb = (B + kTileRows - 1) / kTileRows;
        const uint32_t chunk_list = list_chunk_for(ctx, nq);
        const uint32_t nchunks = uint32_t((nq + chunk_list - 1) / chunk_list);
        // Every query of a chunk selects the sink and the local block, so those two query lists are far longer than
        // the rest (512 queries = 128 MMA groups at prefill sizes, and the local block's item is the LAST one of the
        // work list: one CTA's tail). Long lists are cut into several items: at most 128 queries (32 groups) at
        // prefill sizes (stage 2 7.44 -> 7.22 ms, CTA balance 0.975 -> 0.988; 64 costs more in tile reloads than it
        // balances), at most 16 queries for calls of <= 2048 rows, where one forced-block list was a large share of an
        // SM's whole work (decode: longest CTA 61K cycles against a mean of 28K before the split).
        // (whole MMA groups per item: groups are 3 queries when the scorer multiplies the tile from tensor memory)
        const uint32_t gq = token_scorer_uses_tmem_tile(ctx) ? 3u : uint32_t(kGroupQ);
        const uint32_t split =
            nq <= 2048 ? env_u32("HISA_LIST_SPLIT", 4u * gq) : env_u32("HISA_LIST_SPLIT_BIG", gq == 3u ? 126u : 128u);
        const uint64_t pairs_chunk = uint64_t(chunk_list) * S;
        const uint64_t items_cap =
            uint64_t(nchunks) * (std::min<uint64_t>(M, pairs_chunk) + (split ? pairs_chunk / split : 0)) * spb;
        HISA_TRY(ensure(ctx, ctx->work, std::max<size_t>(size_t(items_cap), size_t(ctx->num_sms)) * sizeof(WorkItem)));
        HISA_TRY(ensure(ctx, ctx->pairs, size_t(nchunks) * chunk_list * S * sizeof(uint2)));
        HISA_TRY(ensure(ctx, ctx->cand, size_t(nq) * cand_cols * 4));
        // (graph replay: the variant must not depend on the current length)
        const uint32_t topk_cap = uint32_t(ctx->dyn ? cand_cols : std::min<uint64_t>(cand_cols, L));
        const size_t inv_words = invert_global_words(uint32_t(nq), chunk_list, M);
        if (inv_words) HISA_TRY(ensure(ctx, ctx->inv_scratch, inv_words * sizeof(uint32_t)));
        uint32_t* sc = ctx->scalars.as<uint32_t>();
        {
          StageTimer timer(ctx, kStInvert);
          const int n_inv = launch_invert_selection(sel, nsel, S, uint32_t(nq), chunk_list, M, B, spb, split,
                                                    ctx->work.as<WorkItem>(), sc + 2, sc + 3, ctx->pairs.as<uint2>(),
                                                    inv_words ? ctx->inv_scratch.as<uint32_t>() : nullptr,
                                                    /*counters_zeroed=*/true, ctx->stream);
          if (n_inv < 0)
            return fail(ctx, HISA_ERR_UNSUPPORTED, "invert selection: %u key blocks need more shared memory than an SM has", M);
          count_launches(ctx, n_inv);
          HISA_TRY(check_launch(ctx, "invert selection"));
        }
        {
          StageTimer timer(ctx, kStScoreTokens);
          ScoreJob j{};
          j.stats_slot = 1;
          set_token_operands(ctx, p, q0, j);
          j.nq = nq;
          j.gates = p.gates + q0 * kHeads;
          j.out = ctx->cand.as<float>();
          j.out_stride = cand_cols;
          j.list_mode = true;
          j.counter_slot = 2;
          j.pairs = ctx->pairs.as<uint2>();
          j.max_items = uint32_t(std::min<uint64_t>(items_cap, 0xFFFFFFFFull));
          ctx->items2 += j.max_items;
          HISA_TRY(run_scorer(ctx, j));
        }
        {
          StageTimer timer(ctx, kStTopK);
          SelectArgs s{};
          s.scores = ctx->cand.as<float>();
          s.stride = cand_cols;
          s.pos = p.pos + q0;
          s.seq_len = L;
          s.num_blocks = M;
          s.block_size = B;
          s.keep = k;
          s.mode = kSelCand;
          s.sel = sel;
          s.nsel = nsel;
          s.sel_stride = S;
          s.dyn_len = ctx->dyn ? ctx->dlen.as<uint32_t>() : nullptr;
          s.tie_break = c.tie_break;
          s.force_first_last = c.force_first_last;  // lets the kernel derive a row's last selected block from its position
          s.out_idx = idx_dst;
          s.out_stride = out_width;
          s.out_width = out_width;
          s.out_count = cnt_dst;
          s.out_cand = cand_dst;
          place(s, q0);
          count_launches(ctx, launch_select(s, uint32_t(nq), topk_cap, ctx->stream));
          HISA_TRY(check_launch(ctx, "top-k"));
        }
      }
      if (!blk_dev) HISA_TRY(copy_out(ctx, out_blocks ? out_blocks + q0 * S : nullptr, sel, size_t(nq) * S * 4, &need_sync));
      if (!nblk_dev) HISA_TRY(copy_out(ctx, out_nblocks ? out_nblocks + q0 : nullptr, nsel, size_t(nq) * 4, &need_sync));
    }
    if (!idx_dev) HISA_TRY(copy_out(ctx, out_idx + q0 * out_width, idx_dst, size_t(nq) * out_width * 4, &need_sync));
    if (!cnt_dev) HISA_TRY(copy_out(ctx, out_count ? out_count + q0 : nullptr, cnt_dst, size_t(nq) * 4, &need_sync));
    if (!cand_dev) HISA_TRY(copy_out(ctx, out_cand ? out_cand + q0 : nullptr, cand_dst, size_t(nq) * 4, &need_sync));
  }
  if (need_sync) CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return HISA_OK;
}

int pipe_init(hisa_cuda_ctx* ctx) {
  if (ctx->pipe_ready) return HISA_OK;
  CU_TRY(ctx, cudaStreamCreateWithFlags(&ctx->in_stream, cudaStreamNonBlocking));
  CU_TRY(ctx, cudaStreamCreateWithFlags(&ctx->out_stream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    CU_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_in_ready[i], cudaEventDisableTiming));
    CU_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_in_free[i], cudaEventDisableTiming));
    CU_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_out_ready[i], cudaEventDisableTiming));
    CU_TRY(ctx, cudaEventCreateWithFlags(&ctx->ev_out_free[i], cudaEventDisableTiming));
  }
  ctx->pipe_ready = true;
  return HISA_OK;
}

// Host-buffer path: the rows are cut into slices; slice i+1 is copied in (in_stream) and slice i-1 copied out
// (out_stream) while the kernels of slice i run on ctx->stream. Pointers that already are device memory are
// passed through untouched.
int select_pipelined(hisa_cuda_ctx* ctx, Strategy strat, const void* queries, const float* gates,
                     const uint32_t* positions, uint64_t Q, int check_finite, int32_t* out_idx, uint32_t* out_count,
                     int32_t* out_blocks, uint32_t* out_nblocks, uint32_t* out_cand) {
  HISA_TRY(pipe_init(ctx));
  const hisa_cuda_config& c = ctx->cfg;
  const uint32_t H = c.num_heads, d = c.dim, eb = elem_bytes(ctx);
  const uint32_t S = c.block_budget + 2;
  const uint32_t out_width = strat == kBlockSparse ? S * c.block_size : c.token_budget;
  const bool q_host = !is_device_ptr(queries), g_host = !is_device_ptr(gates), p_host = !is_device_ptr(positions);
  const bool idx_host = !is_device_ptr(out_idx), cnt_host = out_count && !is_device_ptr(out_count);
  const bool cand_host = out_cand && !is_device_ptr(out_cand);
  const bool blk_host = strat != kDsa && out_blocks && !is_device_ptr(out_blocks);
  const bool nblk_host = strat != kDsa && out_nblocks && !is_device_ptr(out_nblocks);
  const uint64_t P = ctx->pipe_rows;
  const size_t q_row = size_t(H) * d * eb;
  for (int i = 0; i < 2; ++i) {
    if (q_host) HISA_TRY(ensure(ctx, ctx->st_q[i], P * q_row));
    if (g_host) HISA_TRY(ensure(ctx, ctx->st_g[i], P * H * sizeof(float)));
    if (p_host) HISA_TRY(ensure(ctx, ctx->st_pos[i], P * 4));
    if (idx_host) HISA_TRY(ensure(ctx, ctx->st_idx[i], P * out_width * 4));
    if (cnt_host) HISA_TRY(ensure(ctx, ctx->st_cnt[i], P * 4));
    if (cand_host) HISA_TRY(ensure(ctx, ctx->st_cand[i], P * 4));
    if (blk_host) HISA_TRY(ensure(ctx, ctx->st_blk[i], P * S * 4));
    if (nblk_host) HISA_TRY(ensure(ctx, ctx->st_nblk[i], P * 4));
  }
  const uint64_t nslices = (Q + P - 1) / P;
  // HISA_PIPE_TRACE=1: timed events around every copy and kernel span, printed as a per-slice timeline (ms from the
  // start of the call) — a debugging aid for the overlap, never on in measurements
  const bool trace = env_u32("HISA_PIPE_TRACE", 0) != 0;
  std::vector<cudaEvent_t> tev;
  auto mark = [&](cudaStream_t st) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    tev.push_back(e);
  };
  mark(ctx->stream);
  auto copy_in_slice = [&](uint64_t s) -> int {
    const int b = int(s & 1);
    const uint64_t q0 = s * P, nq = std::min<uint64_t>(P, Q - q0);
    if (s >= 2) CU_TRY(ctx, cudaStreamWaitEvent(ctx->in_stream, ctx->ev_in_free[b], 0));
    mark(ctx->in_stream);
    if (q_host)
      CU_TRY(ctx, cudaMemcpyAsync(ctx->st_q[b].p, static_cast<const char*>(queries) + q0 * q_row, nq * q_row,
                                  cudaMemcpyHostToDevice, ctx->in_stream));
    if (g_host)
      CU_TRY(ctx, cudaMemcpyAsync(ctx->st_g[b].p, gates + q0 * H, nq * H * sizeof(float), cudaMemcpyHostToDevice,
                                  ctx->in_stream));
    if (p_host)
      CU_TRY(ctx, cudaMemcpyAsync(ctx->st_pos[b].p, positions + q0, nq * 4, cudaMemcpyHostToDevice, ctx->in_stream));
    CU_TRY(ctx, cudaEventRecord(ctx->ev_in_ready[b], ctx->in_stream));
    mark(ctx->in_stream);
    return HISA_OK;
  };
  HISA_TRY(copy_in_slice(0));
  for (uint64_t s = 0; s < nslices; ++s) {
    const int b = int(s & 1);
    const uint64_t q0 = s * P, nq = std::min<uint64_t>(P, Q - q0);
    if (s + 1 < nslices) HISA_TRY(copy_in_slice(s + 1));
    CU_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_in_ready[b], 0));
    if (s >= 2) CU_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_out_free[b], 0));
    const void* q_s = q_host ? ctx->st_q[b].p : static_cast<const void*>(static_cast<const char*>(queries) + q0 * q_row);
    const float* g_s = g_host ? ctx->st_g[b].as<float>() : gates + q0 * H;
    const uint32_t* p_s = p_host ? ctx->st_pos[b].as<uint32_t>() : positions + q0;
    // a row map addresses the caller's full device arrays: no per-slice offset on them, the map is offset instead
    const bool mapped = ctx->place_rows != nullptr && strat != kBlockSparse;
    int32_t* idx_s = idx_host ? ctx->st_idx[b].as<int32_t>() : out_idx + (mapped ? 0 : q0 * out_width);
    uint32_t* cnt_s = !out_count ? nullptr : cnt_host ? ctx->st_cnt[b].as<uint32_t>() : out_count + (mapped ? 0 : q0);
    uint32_t* cand_s = !out_cand ? nullptr : cand_host ? ctx->st_cand[b].as<uint32_t>() : out_cand + (mapped ? 0 : q0);
    ctx->place_q0 = q0;
    int32_t* blk_s = (strat == kDsa || !out_blocks) ? nullptr : blk_host ? ctx->st_blk[b].as<int32_t>() : out_blocks + q0 * S;
    uint32_t* nblk_s = (strat == kDsa || !out_nblocks) ? nullptr : nblk_host ? ctx->st_nblk[b].as<uint32_t>() : out_nblocks + q0;
    mark(ctx->stream);
    HISA_TRY(select_core(ctx, strat, q_s, g_s, p_s, nq, check_finite, idx_s, cnt_s, blk_s, nblk_s, cand_s));
    mark(ctx->stream);
    CU_TRY(ctx, cudaEventRecord(ctx->ev_in_free[b], ctx->stream));
    CU_TRY(ctx, cudaEventRecord(ctx->ev_out_ready[b], ctx->stream));
    CU_TRY(ctx, cudaStreamWaitEvent(ctx->out_stream, ctx->ev_out_ready[b], 0));
    mark(ctx->out_stream);
    if (idx_host)
      CU_TRY(ctx, cudaMemcpyAsync(out_idx + q0 * out_width, idx_s, nq * out_width * 4, cudaMemcpyDeviceToHost, ctx->out_stream));
    if (cnt_host) CU_TRY(ctx, cudaMemcpyAsync(out_count + q0, cnt_s, nq * 4, cudaMemcpyDeviceToHost, ctx->out_stream));
    if (cand_host) CU_TRY(ctx, cudaMemcpyAsync(out_cand + q0, cand_s, nq * 4, cudaMemcpyDeviceToHost, ctx->out_stream));
    if (blk_host) CU_TRY(ctx, cudaMemcpyAsync(out_blocks + q0 * S, blk_s, nq * S * 4, cudaMemcpyDeviceToHost, ctx->out_stream));
    if (nblk_host) CU_TRY(ctx, cudaMemcpyAsync(out_nblocks + q0, nblk_s, nq * 4, cudaMemcpyDeviceToHost, ctx->out_stream));
    CU_TRY(ctx, cudaEventRecord(ctx->ev_out_free[b], ctx->out_stream));
    mark(ctx->out_stream);
  }
  ctx->place_q0 = 0;
  CU_TRY(ctx, cudaStreamSynchronize(ctx->out_stream));
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (trace) {
    // event order: [0] call start, then per slice s: in-begin/in-end are pushed when slice s is copied (slice 0 first,
    // slice s+1 before the kernels of slice s), kernels-begin/end and out-begin/end in loop order
    std::vector<float> t(tev.size());
    for (size_t i = 0; i < tev.size(); ++i) cudaEventElapsedTime(&t[i], tev[0], tev[i]);
    std::vector<float> in_b(nslices), in_e(nslices), k_b(nslices), k_e(nslices), o_b(nslices), o_e(nslices);
    size_t i = 1;
    in_b[0] = t[i++]; in_e[0] = t[i++];
    for (uint64_t s = 0; s < nslices; ++s) {
      if (s + 1 < nslices) { in_b[s + 1] = t[i++]; in_e[s + 1] = t[i++]; }
      k_b[s] = t[i++]; k_e[s] = t[i++]; o_b[s] = t[i++]; o_e[s] = t[i++];
    }
    fprintf(stderr, "slice   h2d[beg end]     kernels[beg end]   d2h[beg end]  (ms)\n");
    for (uint64_t s = 0; s < nslices; ++s)
      fprintf(stderr, "%5llu  %7.3f %7.3f   %7.3f %7.3f   %7.3f %7.3f\n", (unsigned long long)s, in_b[s], in_e[s], k_b[s], k_e[s],
              o_b[s], o_e[s]);
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
  }
  return HISA_OK;
}

// Small hisa_select calls whose arguments repeat (a decode loop: same device buffers, same Q, the sequence one key
// longer each time) become ONE graph launch. Call 1 of a signature runs normally; call 2 runs with every kernel reading
// the sequence length from ctx->dlen and with operand maps / strides sized for the block-count bucket (this sizes all
// buffers); call 3 captures that same launch sequence into a graph; later calls replay it. Nothing is ever computed
// differently: the graph holds the same kernels with the same arguments.
constexpr uint64_t kGraphMaxRows = 2048;

int select_maybe_graph(hisa_cuda_ctx* ctx, Strategy strat, const void* queries, const float* gates, const uint32_t* positions,
                       uint64_t Q, int check_finite, int32_t* out_idx, uint32_t* out_count, int32_t* out_blocks,
                       uint32_t* out_nblocks, uint32_t* out_cand) {
  const bool eligible = ctx->g_enabled && strat == kHisa && Q > 0 && Q <= kGraphMaxRows && !check_finite && !ctx->profiling &&
                        !ctx->pool_external && !ctx->place_rows && !ctx->place_nrep && ctx->pooled_tokens == ctx->seq_len &&
                        ctx->dlen.p != nullptr;
  if (!eligible)
    return select_core(ctx, strat, queries, gates, positions, Q, check_finite, out_idx, out_count, out_blocks, out_nblocks, out_cand);
  hisa_cuda_ctx::GraphSig sig;
  memset(&sig, 0, sizeof sig);
  sig.q = queries; sig.g = gates; sig.pos = positions; sig.idx = out_idx; sig.cnt = out_count; sig.blk = out_blocks;
  sig.nblk = out_nblocks; sig.cand = out_cand; sig.key_base = ctx->key_op.p; sig.pool_base = ctx->pooled_op.p;
  sig.Q = Q; sig.key_cap = ctx->key_cap;
  sig.Mb = block_bucket(ctx, uint32_t(num_blocks_of(ctx)));
  if (ctx->g_exec && sig == ctx->g_sig) {
    CU_TRY(ctx, cudaGraphLaunch(ctx->g_exec, ctx->stream));
    count_launches(ctx, int(ctx->g_launches));
    return HISA_OK;
  }
  if (sig == ctx->g_pending) ++ctx->g_seen;
  else { ctx->g_pending = sig; ctx->g_seen = 1; }
  if (ctx->g_seen == 1)
    return select_core(ctx, strat, queries, gates, positions, Q, check_finite, out_idx, out_count, out_blocks, out_nblocks, out_cand);
  ctx->dyn = true;
  ctx->dyn_Mb = sig.Mb;
  if (ctx->g_seen == 2) {
    const int rc = select_core(ctx, strat, queries, gates, positions, Q, check_finite, out_idx, out_count, out_blocks, out_nblocks, out_cand);
    ctx->dyn = false;
    return rc;
  }
  // capture; any failure falls back to plain launches and switches the graph path off for this context
  const uint64_t before = ctx->call_launches, before_all = ctx->launches;
  cudaGraph_t graph = nullptr;
  int rc = HISA_OK;
  if (cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    cudaGetLastError();
    ctx->g_enabled = false;
    ctx->dyn = false;
    return select_core(ctx, strat, queries, gates, positions, Q, check_finite, out_idx, out_count, out_blocks, out_nblocks, out_cand);
  }
  rc = select_core(ctx, strat, queries, gates, positions, Q, check_finite, out_idx, out_count, out_blocks, out_nblocks, out_cand);
  const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
  ctx->dyn = false;
  const uint32_t captured = uint32_t(ctx->call_launches - before);
  ctx->call_launches = before;  // nothing ran yet
  ctx->launches = before_all;
  if (rc != HISA_OK || ce != cudaSuccess || !graph) {
    cudaGetLastError();
    if (graph) cudaGraphDestroy(graph);
    ctx->g_enabled = false;
    return select_core(ctx, strat, queries, gates, positions, Q, check_finite, out_idx, out_count, out_blocks, out_nblocks, out_cand);
  }
  drop_graph(ctx);
  const cudaError_t ie = cudaGraphInstantiate(&ctx->g_exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    cudaGetLastError();
    ctx->g_exec = nullptr;
    ctx->g_enabled = false;
    return select_core(ctx, strat, queries, gates, positions, Q, check_finite, out_idx, out_count, out_blocks, out_nblocks, out_cand);
  }
  ctx->g_sig = sig;
  ctx->g_launches = captured;
  CU_TRY(ctx, cudaGraphLaunch(ctx->g_exec, ctx->stream));
  count_launches(ctx, int(captured));
  return HISA_OK;
}

int select_impl(hisa_cuda_ctx* ctx, Strategy strat, const void* queries, const float* gates, const uint32_t* positions,
                uint64_t Q, int check_finite, int32_t* out_idx, uint32_t* out_count, int32_t* out_blocks,
                uint32_t* out_nblocks, uint32_t* out_cand) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  if (!out_idx && Q) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "out_idx must be non-null");
  CU_TRY(ctx, cudaSetDevice(ctx->device));
  begin_call(ctx);
  ctx->place_q0 = 0;
  if (ctx->seq_len == 0) return fail(ctx, HISA_ERR_EMPTY_SEQUENCE, "selection over an empty key sequence");
  if (strat != kDsa) HISA_TRY(ensure_pool(ctx));
  if (Q && (!queries || !gates || !positions))
    return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "queries, gates and positions must be non-null");
  const bool any_host = Q && (!is_device_ptr(queries) || !is_device_ptr(gates) || !is_device_ptr(positions) ||
                              !is_device_ptr(out_idx) || (out_count && !is_device_ptr(out_count)) ||
                              (out_cand && !is_device_ptr(out_cand)) || (out_blocks && !is_device_ptr(out_blocks)) ||
                              (out_nblocks && !is_device_ptr(out_nblocks)));
  int rc;
  if (any_host && ctx->pipe_rows && Q > ctx->pipe_rows)
    rc = select_pipelined(ctx, strat, queries, gates, positions, Q, check_finite, out_idx, out_count, out_blocks,
                          out_nblocks, out_cand);
  else if (any_host)
    rc = select_core(ctx, strat, queries, gates, positions, Q, check_finite, out_idx, out_count, out_blocks, out_nblocks,
                     out_cand);
  else
    rc = select_maybe_graph(ctx, strat, queries, gates, positions, Q, check_finite, out_idx, out_count, out_blocks,
                            out_nblocks, out_cand);
  HISA_TRY(rc);
  end_call(ctx);
  return HISA_OK;
}

uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  return uint32_t(strtoul(v, nullptr, 10));
}

}  // namespace

namespace hisa_dev {
bool smem_opt_in(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;  // (device, kernel) -> bytes already granted
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  std::lock_guard<std::mutex> g(mu);
  size_t& have = done[{dev, func}];
  if (have >= bytes) return true;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  have = bytes;
  return true;
}
}  // namespace hisa_dev

// ==================================================================================================
// C ABI
// ==================================================================================================
extern "C" {

void hisa_cuda_config_init(hisa_cuda_config* cfg, uint32_t block_size, uint32_t block_budget, uint32_t token_budget,
                           uint32_t num_heads, uint32_t dim, uint32_t dtype) {
  memset(cfg, 0, sizeof *cfg);
  cfg->block_size = block_size;
  cfg->block_budget = block_budget;
  cfg->token_budget = token_budget;
  cfg->num_heads = num_heads;
  cfg->dim = dim;
  cfg->force_first_last = 1;
  cfg->forced_in_budget = 0;
  cfg->tie_break = HISA_TIE_SMALLEST_INDEX;
  cfg->pool_mode = HISA_POOL_MEAN;
  cfg->dtype = dtype;
  cfg->scorer = HISA_SCORER_TENSOR;
}

int hisa_cuda_config_validate(const hisa_cuda_config* c) {
  if (!c) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null config");
  if (c->block_size == 0 || c->block_budget == 0 || c->token_budget == 0 || c->num_heads == 0 || c->dim == 0)
    return fail(nullptr, HISA_ERR_INFEASIBLE_CONFIG, "config: all integer fields must be strictly positive");
  const uint64_t cap = uint64_t(c->block_budget) * c->block_size;
  if (cap < c->token_budget)
    return fail(nullptr, HISA_ERR_INFEASIBLE_CONFIG,
                "infeasible config: block budget times block size must satisfy mB >= k (got %u*%u=%llu < %u)",
                c->block_budget, c->block_size, (unsigned long long)cap, c->token_budget);
  return HISA_OK;
}

int hisa_cuda_abi_version(void) { return HISA_CUDA_ABI_VERSION; }

const char* hisa_cuda_status_name(int s) {
  switch (s) {
    case HISA_OK: return "OK";
    case HISA_ERR_INFEASIBLE_CONFIG: return "InfeasibleConfig";
    case HISA_ERR_CAUSAL_VIOLATION: return "CausalViolation";
    case HISA_ERR_EMPTY_SEQUENCE: return "EmptySequence";
    case HISA_ERR_DIMENSION_MISMATCH: return "DimensionMismatch";
    case HISA_ERR_NON_FINITE: return "NonFiniteValue";
    case HISA_ERR_SHAPE_MISMATCH: return "ShapeMismatch";
    case HISA_ERR_EMPTY_SELECTION: return "EmptySelection";
    case HISA_ERR_INVALID_ARGUMENT: return "InvalidArgument";
    case HISA_ERR_UNSUPPORTED: return "Unsupported";
    case HISA_ERR_NO_DEVICE: return "NoDevice";
    case HISA_ERR_CUDA: return "CudaError";
    case HISA_ERR_OUT_OF_MEMORY: return "OutOfMemory";
    default: return "Unknown";
  }
}

const char* hisa_cuda_last_error(const hisa_cuda_ctx* ctx) { return ctx ? ctx->err.c_str() : g_global_error.c_str(); }

int hisa_cuda_device_count(int* count) {
  if (!count) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null count");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *count = 0;
    return fail(nullptr, HISA_ERR_NO_DEVICE, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *count = n;
  return HISA_OK;
}

int hisa_cuda_create(int device, const hisa_cuda_config* cfg, hisa_cuda_ctx** out) {
  if (!out) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  HISA_TRY(hisa_cuda_config_validate(cfg));
  if (cfg->num_heads > uint32_t(kHeads))
    return fail(nullptr, HISA_ERR_UNSUPPORTED, "num_heads %u > %d is not covered by the sm_100a kernels", cfg->num_heads, kHeads);
  if (cfg->dim > uint32_t(kDim))
    return fail(nullptr, HISA_ERR_UNSUPPORTED, "dim %u > %d is not covered by the sm_100a kernels", cfg->dim, kDim);
  if (cfg->dtype != HISA_DTYPE_F32 && cfg->dtype != HISA_DTYPE_BF16 && cfg->dtype != HISA_DTYPE_FP8_E4M3)
    return fail(nullptr, HISA_ERR_UNSUPPORTED, "unknown dtype %u", cfg->dtype);
  if (cfg->dtype == HISA_DTYPE_FP8_E4M3 && (cfg->num_heads != uint32_t(kHeads) || cfg->dim != uint32_t(kDim)))
    return fail(nullptr, HISA_ERR_UNSUPPORTED, "fp8 storage is built for num_heads = %d, dim = %d only", kHeads, kDim);
  if (cfg->dtype == HISA_DTYPE_FP8_E4M3 && cfg->scorer == HISA_SCORER_SIMT)
    return fail(nullptr, HISA_ERR_UNSUPPORTED, "the SIMT cross-check scorer does not read fp8 operands");
  if (cfg->tie_break > 1 || cfg->pool_mode > 1 || cfg->scorer > 1)
    return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "config enum field out of range");
  if (uint64_t(cfg->block_budget) + 2 > 0xFFFFFFull || uint64_t(cfg->block_budget + 2) * cfg->block_size > 0x7FFFFFFFull)
    return fail(nullptr, HISA_ERR_UNSUPPORTED, "candidate pool (m+2)*B too large");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(nullptr, HISA_ERR_NO_DEVICE, "no CUDA device available (this library has no CPU fallback)");
  }
  if (device < 0 || device >= n) return fail(nullptr, HISA_ERR_NO_DEVICE, "device %d out of range (%d devices)", device, n);
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess)
    return fail(nullptr, HISA_ERR_NO_DEVICE, "cudaGetDeviceProperties(%d) failed", device);
  if (prop.major != 10)
    return fail(nullptr, HISA_ERR_NO_DEVICE, "device %d is sm_%d%d; the kernels are built for sm_100a only", device,
                prop.major, prop.minor);
  hisa_cuda_ctx* ctx = new hisa_cuda_ctx();
  ctx->cfg = *cfg;
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return fail(nullptr, HISA_ERR_CUDA, "could not create a stream on device %d", device);
  }
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qres;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres) != cudaSuccess || !fn) {
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return fail(nullptr, HISA_ERR_CUDA, "cuTensorMapEncodeTiled entry point not available");
  }
  ctx->encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);

  const bool bf16 = cfg->dtype == HISA_DTYPE_BF16;
  ctx->fp8 = cfg->dtype == HISA_DTYPE_FP8_E4M3;
  if (bf16 || ctx->fp8) {
    // fp8: stage 2 and the flat scorer read the e4m3 bytes of q and k directly. Stage 1 reads the e4m3 queries too, against
    // pooled keys stored as four e4m3 terms + a power-of-two scale per block (pool8). HISA_FP8_BLOCKS=0 or the SIMT
    // cross-check scorer: stage 1 multiplies a bf16 copy of q (e4m3 values are exact in bf16) with bf16 hi|lo pooled keys
    ctx->nseg_k = ctx->nseg_q = 1;
    ctx->nseg_p = std::min<uint32_t>(std::max<uint32_t>(env_u32("HISA_POOL_SEGS", 2), 1), kMaxSeg);
    ctx->terms_tok[0] = 1; ctx->terms_tok[1] = ctx->terms_tok[2] = 0;
    ctx->terms_blk[0] = (1u << ctx->nseg_p) - 1; ctx->terms_blk[1] = ctx->terms_blk[2] = 0;
  } else {
    // exact 3-way bf16 split of fp32 operands; keep the six largest cross terms (error ~2^-24 relative)
    ctx->nseg_k = ctx->nseg_q = ctx->nseg_p = 3;
    ctx->terms_tok[0] = 0b111; ctx->terms_tok[1] = 0b011; ctx->terms_tok[2] = 0b001;
    for (int i = 0; i < kMaxSeg; ++i) ctx->terms_blk[i] = ctx->terms_tok[i];
  }
  ctx->pool8 = ctx->fp8 && cfg->scorer != HISA_SCORER_SIMT && env_u32("HISA_FP8_BLOCKS", 1) != 0;
  if (ctx->pool8) ctx->nseg_p = 2;  // four e4m3 terms take the bytes of two bf16 segments: one buffer layout for both forms
  ctx->q_zero_copy = bf16 && cfg->num_heads == uint32_t(kHeads) && cfg->dim == uint32_t(kDim);
  ctx->chunk_dense = std::max<uint32_t>(env_u32("HISA_CHUNK_DENSE", 128), 4);
  ctx->chunk_list = std::max<uint32_t>(env_u32("HISA_CHUNK_LIST", 512), 4);
  ctx->workspace_bytes = uint64_t(std::max<uint32_t>(env_u32("HISA_WORKSPACE_MB", 4096), 16)) << 20;
  ctx->pipe_rows = env_u32("HISA_PIPE_ROWS", 4096);  // 0 disables the host-buffer pipeline
  ctx->g_enabled = env_u32("HISA_DECODE_GRAPH", 1) != 0;
  *out = ctx;
  return HISA_OK;
}

int hisa_cuda_destroy(hisa_cuda_ctx* ctx) {
  if (!ctx) return HISA_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  drop_graph(ctx);
  release(ctx->dlen);
  for (DevBuf* b : {&ctx->key_op, &ctx->key_raw, &ctx->key_scale, &ctx->sums, &ctx->counts, &ctx->pooled_op, &ctx->pool_scale,
                    &ctx->q_raw, &ctx->q_op,
                    &ctx->gates_raw, &ctx->gates_pad, &ctx->pos, &ctx->J, &ctx->sel, &ctx->nsel, &ctx->work, &ctx->pairs,
                    &ctx->scalars, &ctx->cand, &ctx->flat, &ctx->out_idx, &ctx->out_count, &ctx->out_cand,
                    &ctx->generic_scores, &ctx->generic_n, &ctx->export_a, &ctx->export_b, &ctx->flag, &ctx->stats,
                    &ctx->inv_scratch,
                    &ctx->attn_lat, &ctx->attn_q, &ctx->attn_qraw, &ctx->attn_pos, &ctx->attn_idx, &ctx->attn_cnt,
                    &ctx->attn_out, &ctx->attn_w})
    release(*b);
  if (ctx->attn_beg) cudaEventDestroy(ctx->attn_beg);
  if (ctx->attn_end) cudaEventDestroy(ctx->attn_end);
  for (int i = 0; i < 2; ++i)
    for (DevBuf* b : {&ctx->st_q[i], &ctx->st_g[i], &ctx->st_pos[i], &ctx->st_idx[i], &ctx->st_cnt[i], &ctx->st_cand[i],
                      &ctx->st_blk[i], &ctx->st_nblk[i]})
      release(*b);
  if (ctx->pipe_ready) {
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(ctx->ev_in_ready[i]); cudaEventDestroy(ctx->ev_in_free[i]);
      cudaEventDestroy(ctx->ev_out_ready[i]); cudaEventDestroy(ctx->ev_out_free[i]);
    }
    cudaStreamDestroy(ctx->in_stream);
    cudaStreamDestroy(ctx->out_stream);
  }
  for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return HISA_OK;
}

int hisa_cuda_synchronize(hisa_cuda_ctx* ctx) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return HISA_OK;
}

void* hisa_cuda_stream(hisa_cuda_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

int hisa_cuda_host_alloc(void** ptr, size_t bytes) {
  if (!ptr) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null pointer");
  cudaError_t e = cudaHostAlloc(ptr, bytes ? bytes : 1, cudaHostAllocDefault);
  if (e != cudaSuccess) return fail(nullptr, HISA_ERR_OUT_OF_MEMORY, "cudaHostAlloc(%zu): %s", bytes, cudaGetErrorString(e));
  return HISA_OK;
}
int hisa_cuda_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
  return HISA_OK;
}
int hisa_cuda_device_alloc(hisa_cuda_ctx* ctx, void** ptr, size_t bytes) {
  if (!ctx || !ptr) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "null argument");
  CU_TRY(ctx, cudaSetDevice(ctx->device));
  CU_TRY(ctx, cudaMalloc(ptr, bytes ? bytes : 1));
  return HISA_OK;
}
int hisa_cuda_device_free(hisa_cuda_ctx* ctx, void* ptr) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  if (ptr) {
    CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    CU_TRY(ctx, cudaFree(ptr));
  }
  return HISA_OK;
}
int hisa_cuda_memcpy(hisa_cuda_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return HISA_OK;
}

// ---- keys and block summaries ---------------------------------------------------------------------

static int grow_keys(hisa_cuda_ctx* ctx, uint64_t need_tokens) {
  if (need_tokens <= ctx->key_cap) return HISA_OK;
  drop_graph(ctx);  // the captured kernels hold the old operand addresses
  uint64_t cap = std::max<uint64_t>(need_tokens, ctx->key_cap + ctx->key_cap / 2);
  cap = round_up64(cap, 1024);
  const size_t row_bytes = ctx->fp8 ? size_t(kDim) : size_t(ctx->nseg_k) * kDim * sizeof(__nv_bfloat16);
  const uint64_t mcap = (cap + ctx->cfg.block_size - 1) / ctx->cfg.block_size + 1;
  DevBuf nk, ns, nc, np, nsc, npsc;
  CU_TRY(ctx, cudaMalloc(&nk.p, cap * row_bytes));
  if (ctx->fp8) {
    CU_TRY(ctx, cudaMalloc(&nsc.p, cap * sizeof(float)));
    nsc.cap = cap * sizeof(float);
  }
  CU_TRY(ctx, cudaMalloc(&ns.p, mcap * kDim * sizeof(double)));
  CU_TRY(ctx, cudaMalloc(&nc.p, mcap * sizeof(uint32_t)));
  CU_TRY(ctx, cudaMalloc(&np.p, mcap * ctx->nseg_p * kDim * sizeof(__nv_bfloat16)));
  nk.cap = cap * row_bytes; ns.cap = mcap * kDim * sizeof(double); nc.cap = mcap * sizeof(uint32_t);
  np.cap = mcap * ctx->nseg_p * kDim * sizeof(__nv_bfloat16);
  CU_TRY(ctx, cudaMemsetAsync(np.p, 0, np.cap, ctx->stream));
  if (ctx->pool8) {  // one scale per pooled row, padded to whole 128-row tiles (the scorer's epilogue reads a tile's worth)
    npsc.cap = (mcap + kTileRows) * sizeof(float);
    CU_TRY(ctx, cudaMalloc(&npsc.p, npsc.cap));
    CU_TRY(ctx, cudaMemsetAsync(npsc.p, 0, npsc.cap, ctx->stream));
  }
  if (ctx->seq_len) {
    const uint64_t M = num_blocks_of(ctx);
    CU_TRY(ctx, cudaMemcpyAsync(nk.p, ctx->key_op.p, ctx->seq_len * row_bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    if (ctx->fp8)
      CU_TRY(ctx, cudaMemcpyAsync(nsc.p, ctx->key_scale.p, ctx->seq_len * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
    CU_TRY(ctx, cudaMemcpyAsync(ns.p, ctx->sums.p, M * kDim * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    CU_TRY(ctx, cudaMemcpyAsync(nc.p, ctx->counts.p, M * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    CU_TRY(ctx, cudaMemcpyAsync(np.p, ctx->pooled_op.p, M * ctx->nseg_p * kDim * sizeof(__nv_bfloat16),
                                cudaMemcpyDeviceToDevice, ctx->stream));
    if (ctx->pool8)
      CU_TRY(ctx, cudaMemcpyAsync(npsc.p, ctx->pool_scale.p, M * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  release(ctx->key_op); release(ctx->sums); release(ctx->counts); release(ctx->pooled_op); release(ctx->key_scale);
  release(ctx->pool_scale);
  ctx->key_op = nk; ctx->sums = ns; ctx->counts = nc; ctx->pooled_op = np; ctx->key_scale = nsc; ctx->pool_scale = npsc;
  ctx->key_cap = cap;
  return HISA_OK;
}

// converts n keys (host or device, ctx dtype, [n, dim]) into operand rows [first, first+n)
// fp8: `scales` (host or device, may be null = 1) are the per-key dequantisation scales
static int ingest_keys(hisa_cuda_ctx* ctx, const void* keys, const float* scales, uint64_t first, uint64_t n,
                       int check_finite) {
  const uint32_t d = ctx->cfg.dim, eb = elem_bytes(ctx);
  const uint32_t st = src_type(ctx);
  const void* src = keys;
  const bool direct = (st == 1 || st == 2) && d == uint32_t(kDim);
  void* dst = ctx->key_op.as<uint8_t>() + first * (ctx->fp8 ? size_t(kDim) : size_t(ctx->nseg_k) * kDim * sizeof(__nv_bfloat16));
  if (direct) {
    HISA_TRY(copy_in(ctx, dst, keys, n * d * eb));
    src = dst;
  } else if (!is_device_ptr(keys)) {
    HISA_TRY(ensure(ctx, ctx->key_raw, n * d * eb));
    HISA_TRY(copy_in(ctx, ctx->key_raw.p, keys, n * d * eb));
    src = ctx->key_raw.p;
  }
  if (ctx->fp8) {
    float* sdst = ctx->key_scale.as<float>() + first;
    if (scales) HISA_TRY(copy_in(ctx, sdst, scales, n * sizeof(float)));
    else count_launches(ctx, launch_fill_f32(sdst, n, 1.0f, ctx->stream));
  }
  if (check_finite) {
    HISA_TRY(ensure(ctx, ctx->flag, 16));
    CU_TRY(ctx, cudaMemsetAsync(ctx->flag.p, 0, 16, ctx->stream));
    count_launches(ctx, launch_check_finite(src, st, n * d, ctx->flag.as<uint32_t>(), ctx->stream));
    if (ctx->fp8) count_launches(ctx, launch_check_finite(ctx->key_scale.as<float>() + first, 0, n, ctx->flag.as<uint32_t>(), ctx->stream));
    uint32_t bad = 0;
    HISA_TRY(read_flag(ctx, &bad));
    if (bad) return fail(ctx, HISA_ERR_NON_FINITE, "inputs: non-finite value in keys");
  }
  if (!direct)
    count_launches(ctx, launch_convert_rows(src, st, n, 1, d, ctx->nseg_k, static_cast<__nv_bfloat16*>(dst), 1, ctx->stream));
  return check_launch(ctx, "key ingestion");
}

static int pool_update(hisa_cuda_ctx* ctx, uint64_t first, uint64_t n) {
  // the kernel also publishes the new sequence length (first + n) in the device word replayed graphs read
  HISA_TRY(ensure(ctx, ctx->dlen, 16));
  if (ctx->fp8)
    count_launches(ctx, launch_pool_update_fp8(ctx->key_op.as<uint8_t>(), ctx->key_scale.as<float>(), first, n,
                                               ctx->cfg.block_size, ctx->cfg.pool_mode, ctx->sums.as<double>(),
                                               ctx->counts.as<uint32_t>(), ctx->pooled_op.as<__nv_bfloat16>(), ctx->nseg_p,
                                               ctx->pool8 ? ctx->pool_scale.as<float>() : nullptr, ctx->dlen.as<uint32_t>(),
                                               ctx->stream));
  else
    count_launches(ctx, launch_pool_update(ctx->key_op.as<__nv_bfloat16>(), ctx->nseg_k, first, n, ctx->cfg.block_size,
                                           ctx->cfg.dim, ctx->cfg.pool_mode, ctx->sums.as<double>(), ctx->counts.as<uint32_t>(),
                                           ctx->pooled_op.as<__nv_bfloat16>(), ctx->nseg_p, ctx->dlen.as<uint32_t>(),
                                           ctx->stream));
  return HISA_OK;
}

static int upload_keys_impl(hisa_cuda_ctx* ctx, const void* keys, const float* scales, uint64_t seq_len, int check_finite) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaSetDevice(ctx->device));
  if (seq_len == 0) return fail(ctx, HISA_ERR_EMPTY_SEQUENCE, "upload_keys: key matrix has no rows");
  if (!keys) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "null keys");
  if (scales && !ctx->fp8) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "key scales are only meaningful for fp8 storage");
  if (seq_len > 0x7FFFFF00ull) return fail(ctx, HISA_ERR_UNSUPPORTED, "sequence too long");
  ctx->seq_len = 0;
  ctx->pooled_tokens = 0;
  ctx->pool_external = false;
  drop_graph(ctx);
  HISA_TRY(grow_keys(ctx, seq_len));
  HISA_TRY(ingest_keys(ctx, keys, scales, 0, seq_len, check_finite));
  ctx->seq_len = seq_len;
  HISA_TRY(ensure(ctx, ctx->dlen, 16));
  const uint32_t len32 = uint32_t(seq_len);
  CU_TRY(ctx, cudaMemcpyAsync(ctx->dlen.p, &len32, sizeof len32, cudaMemcpyHostToDevice, ctx->stream));
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));  // len32 lives on this stack frame
  return HISA_OK;
}

static int pool_append_impl(hisa_cuda_ctx* ctx, const void* keys, const float* scales, uint64_t n, uint32_t key_dim) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaSetDevice(ctx->device));
  if (key_dim != ctx->cfg.dim)
    return fail(ctx, HISA_ERR_DIMENSION_MISMATCH, "append: key has %u components, cache dimension is %u", key_dim, ctx->cfg.dim);
  if (n == 0) return HISA_OK;
  if (!keys) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "null keys");
  if (scales && !ctx->fp8) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "key scales are only meaningful for fp8 storage");
  // installed snapshots (hisa_cuda_pool_set) are replaced by summaries of the keys the context holds
  if (ctx->pool_external || ctx->pooled_tokens != ctx->seq_len) HISA_TRY(hisa_cuda_pool_build(ctx));
  HISA_TRY(grow_keys(ctx, ctx->seq_len + n));
  HISA_TRY(ingest_keys(ctx, keys, scales, ctx->seq_len, n, 0));
  HISA_TRY(pool_update(ctx, ctx->seq_len, n));
  ctx->seq_len += n;
  ctx->pooled_tokens = ctx->seq_len;
  return check_launch(ctx, "pool append");
}

int hisa_cuda_upload_keys(hisa_cuda_ctx* ctx, const void* keys, uint64_t seq_len, int check_finite) {
  return upload_keys_impl(ctx, keys, nullptr, seq_len, check_finite);
}

int hisa_cuda_upload_keys_scaled(hisa_cuda_ctx* ctx, const void* keys, const float* key_scales, uint64_t seq_len,
                                 int check_finite) {
  return upload_keys_impl(ctx, keys, key_scales, seq_len, check_finite);
}

int hisa_cuda_pool_build(hisa_cuda_ctx* ctx) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaSetDevice(ctx->device));
  if (ctx->seq_len == 0) return fail(ctx, HISA_ERR_EMPTY_SEQUENCE, "build_block_summaries: key matrix has no rows");
  HISA_TRY(pool_update(ctx, 0, ctx->seq_len));
  ctx->pooled_tokens = ctx->seq_len;
  ctx->pool_external = false;
  return check_launch(ctx, "pool build");
}

int hisa_cuda_pool_set(hisa_cuda_ctx* ctx, const double* sums, const uint32_t* counts, uint64_t num_blocks,
                       uint64_t num_tokens) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaSetDevice(ctx->device));
  if (ctx->seq_len == 0) return fail(ctx, HISA_ERR_EMPTY_SEQUENCE, "pool_set: upload the key sequence first");
  if (num_blocks == 0 || num_tokens == 0) return fail(ctx, HISA_ERR_EMPTY_SEQUENCE, "pool_set: empty block summary cache");
  if (!sums || !counts) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "pool_set: null summaries");
  const uint64_t B = ctx->cfg.block_size;
  if ((num_tokens + B - 1) / B != num_blocks)
    return fail(ctx, HISA_ERR_SHAPE_MISMATCH, "pool_set: %llu tokens in blocks of %llu do not make %llu blocks",
                (unsigned long long)num_tokens, (unsigned long long)B, (unsigned long long)num_blocks);
  // blocks beyond the key sequence can never be eligible (t <= L - 1 after clipping): they are dropped
  const uint32_t M = uint32_t(std::min<uint64_t>(num_blocks, num_blocks_of(ctx)));
  const uint32_t d = ctx->cfg.dim;
  const double* s_dev = sums;
  const uint32_t* c_dev = counts;
  if (!is_device_ptr(sums)) {
    HISA_TRY(ensure(ctx, ctx->export_a, size_t(M) * d * sizeof(double)));
    HISA_TRY(copy_in(ctx, ctx->export_a.p, sums, size_t(M) * d * sizeof(double)));
    s_dev = ctx->export_a.as<double>();
  }
  if (!is_device_ptr(counts)) {
    HISA_TRY(ensure(ctx, ctx->generic_n, size_t(M) * 4));
    HISA_TRY(copy_in(ctx, ctx->generic_n.p, counts, size_t(M) * 4));
    c_dev = ctx->generic_n.as<uint32_t>();
  }
  count_launches(ctx, launch_pool_import(s_dev, c_dev, M, d, ctx->cfg.pool_mode, ctx->sums.as<double>(),
                                         ctx->counts.as<uint32_t>(), ctx->pooled_op.as<__nv_bfloat16>(), ctx->nseg_p,
                                         ctx->pool8 ? ctx->pool_scale.as<float>() : nullptr, ctx->stream));
  HISA_TRY(check_launch(ctx, "pool import"));
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));  // the caller's host arrays may go away after the call
  ctx->pool_external = true;
  drop_graph(ctx);
  ctx->pool_blocks = M;
  ctx->pooled_tokens = std::min<uint64_t>(num_tokens, ctx->seq_len);
  return HISA_OK;
}

int hisa_cuda_pool_append(hisa_cuda_ctx* ctx, const void* keys, uint64_t n, uint32_t key_dim) {
  return pool_append_impl(ctx, keys, nullptr, n, key_dim);
}

int hisa_cuda_pool_append_scaled(hisa_cuda_ctx* ctx, const void* keys, const float* key_scales, uint64_t n,
                                 uint32_t key_dim) {
  return pool_append_impl(ctx, keys, key_scales, n, key_dim);
}

int hisa_cuda_pool_read(hisa_cuda_ctx* ctx, double* sums, uint32_t* counts, double* pooled) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaSetDevice(ctx->device));
  if (ctx->seq_len == 0) return fail(ctx, HISA_ERR_EMPTY_SEQUENCE, "no block summaries: empty sequence");
  HISA_TRY(ensure_pool(ctx));
  const uint32_t M = uint32_t(pool_blocks_of(ctx)), d = ctx->cfg.dim;
  const size_t bytes = size_t(M) * d * sizeof(double);
  HISA_TRY(ensure(ctx, ctx->export_a, bytes));
  HISA_TRY(ensure(ctx, ctx->export_b, bytes));
  count_launches(ctx, launch_pool_export(ctx->sums.as<double>(), ctx->counts.as<uint32_t>(), M, d, ctx->cfg.pool_mode,
                                         ctx->export_a.as<double>(), ctx->export_b.as<double>(), ctx->stream));
  HISA_TRY(check_launch(ctx, "pool export"));
  if (sums) CU_TRY(ctx, cudaMemcpyAsync(sums, ctx->export_a.p, bytes, cudaMemcpyDefault, ctx->stream));
  if (pooled) CU_TRY(ctx, cudaMemcpyAsync(pooled, ctx->export_b.p, bytes, cudaMemcpyDefault, ctx->stream));
  if (counts) CU_TRY(ctx, cudaMemcpyAsync(counts, ctx->counts.p, size_t(M) * 4, cudaMemcpyDefault, ctx->stream));
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return HISA_OK;
}

int hisa_cuda_seq_len(const hisa_cuda_ctx* ctx, uint64_t* seq_len, uint64_t* num_blocks) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  if (seq_len) *seq_len = ctx->seq_len;
  if (num_blocks) *num_blocks = num_blocks_of(ctx);
  return HISA_OK;
}

// ---- batched selection ------------------------------------------------------------------------------

int hisa_cuda_hisa_select(hisa_cuda_ctx* ctx, const void* queries, const float* gates, const uint32_t* positions,
                          uint64_t num_queries, int check_finite, int32_t* out_idx, uint32_t* out_count,
                          int32_t* out_blocks, uint32_t* out_nblocks, uint32_t* out_cand) {
  return select_impl(ctx, kHisa, queries, gates, positions, num_queries, check_finite, out_idx, out_count, out_blocks,
                     out_nblocks, out_cand);
}

int hisa_cuda_dsa_select(hisa_cuda_ctx* ctx, const void* queries, const float* gates, const uint32_t* positions,
                         uint64_t num_queries, int check_finite, int32_t* out_idx, uint32_t* out_count,
                         uint32_t* out_cand) {
  return select_impl(ctx, kDsa, queries, gates, positions, num_queries, check_finite, out_idx, out_count, nullptr,
                     nullptr, out_cand);
}

int hisa_cuda_block_sparse_select(hisa_cuda_ctx* ctx, const void* queries, const float* gates,
                                  const uint32_t* positions, uint64_t num_queries, int check_finite, int32_t* out_idx,
                                  uint32_t* out_count, int32_t* out_blocks, uint32_t* out_nblocks) {
  return select_impl(ctx, kBlockSparse, queries, gates, positions, num_queries, check_finite, out_idx, out_count,
                     out_blocks, out_nblocks, nullptr);
}

int hisa_cuda_set_output_placement(hisa_cuda_ctx* ctx, const uint32_t* out_rows, int num_replicas,
                                   int32_t* const* replica_idx, uint32_t* const* replica_count) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  if (num_replicas < 0 || num_replicas > kMaxReplicas)
    return fail(ctx, HISA_ERR_UNSUPPORTED, "at most %d output replicas", kMaxReplicas);
  if (num_replicas && !replica_idx) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "null replica list");
  if (out_rows && !is_device_ptr(out_rows)) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "out_rows must be device memory");
  ctx->place_rows = out_rows;
  ctx->place_nrep = uint32_t(num_replicas);
  for (int r = 0; r < kMaxReplicas; ++r) {
    ctx->place_rep_idx[r] = r < num_replicas ? replica_idx[r] : nullptr;
    ctx->place_rep_count[r] = (r < num_replicas && replica_count) ? replica_count[r] : nullptr;
    if (r < num_replicas && !ctx->place_rep_idx[r]) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "null replica pointer");
  }
  return HISA_OK;
}

// ---- single stages ------------------------------------------------------------------------------------

int hisa_cuda_score_blocks(hisa_cuda_ctx* ctx, const void* queries, const float* gates, const uint32_t* positions,
                           uint64_t Q, float* out_scores, uint32_t* out_neligible) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaSetDevice(ctx->device));
  begin_call(ctx);
  if (ctx->seq_len == 0) return fail(ctx, HISA_ERR_EMPTY_SEQUENCE, "score_blocks: empty block summary cache");
  HISA_TRY(ensure_pool(ctx));
  Prepared p;
  HISA_TRY(prepare_inputs(ctx, queries, gates, positions, Q, 0, &p));
  if (Q == 0) return HISA_OK;
  if (Q > uint64_t(ctx->chunk_dense) * 4096) return fail(ctx, HISA_ERR_UNSUPPORTED, "score_blocks: too many rows in one call");
  HISA_TRY(ensure(ctx, ctx->scalars, 64));
  const uint32_t M = uint32_t(pool_blocks_of(ctx)), Mpad = round_up(M, kTileRows);
  HISA_TRY(run_score_blocks(ctx, p, 0, Q, Mpad));
  if (out_scores)
    CU_TRY(ctx, cudaMemcpy2DAsync(out_scores, size_t(M) * 4, ctx->J.p, size_t(Mpad) * 4, size_t(M) * 4, Q,
                                  cudaMemcpyDefault, ctx->stream));
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (out_neligible) {
    // eligibility is pure index arithmetic on the positions (hisa.hpp:18-19)
    std::vector<uint32_t> pos(Q);
    CU_TRY(ctx, cudaMemcpy(pos.data(), p.pos, Q * 4, cudaMemcpyDefault));
    std::vector<uint32_t> ne(Q);
    for (uint64_t i = 0; i < Q; ++i)
      ne[i] = std::min<uint32_t>(std::min<uint32_t>(pos[i], uint32_t(ctx->seq_len) - 1) / ctx->cfg.block_size, M - 1) + 1;
    CU_TRY(ctx, cudaMemcpy(out_neligible, ne.data(), Q * 4, cudaMemcpyDefault));
  }
  end_call(ctx);
  return HISA_OK;
}

static int generic_select(hisa_cuda_ctx* ctx, bool blocks, const float* scores, uint64_t stride, const uint32_t* n,
                          uint64_t rows, uint32_t keep, uint32_t out_width, int32_t* out_idx, uint32_t* out_count) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaSetDevice(ctx->device));
  begin_call(ctx);
  if (rows == 0) return HISA_OK;
  if (!scores || !n || !out_idx) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "null argument");
  if (keep == 0) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "k must be at least 1");
  const float* s_dev = scores;
  if (!is_device_ptr(scores)) {
    HISA_TRY(ensure(ctx, ctx->generic_scores, rows * stride * 4));
    HISA_TRY(copy_in(ctx, ctx->generic_scores.p, scores, rows * stride * 4));
    s_dev = ctx->generic_scores.as<float>();
  }
  std::vector<uint32_t> n_host(rows);
  CU_TRY(ctx, cudaMemcpyAsync(n_host.data(), n, rows * 4, cudaMemcpyDefault, ctx->stream));
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  uint32_t n_cap = 1;
  for (uint64_t i = 0; i < rows; ++i) {
    if (n_host[i] > stride) return fail(ctx, HISA_ERR_SHAPE_MISMATCH, "row %llu has more candidates than the score stride", (unsigned long long)i);
    if (blocks && n_host[i] == 0) return fail(ctx, HISA_ERR_EMPTY_SELECTION, "select_blocks: no eligible block in row %llu", (unsigned long long)i);
    n_cap = std::max(n_cap, n_host[i]);
  }
  HISA_TRY(ensure(ctx, ctx->generic_n, rows * 4));
  HISA_TRY(copy_in(ctx, ctx->generic_n.p, n_host.data(), rows * 4));
  const bool idx_dev = is_device_ptr(out_idx), cnt_dev = is_device_ptr(out_count);
  if (!idx_dev) HISA_TRY(ensure(ctx, ctx->out_idx, rows * out_width * 4));
  if (!cnt_dev) HISA_TRY(ensure(ctx, ctx->out_count, rows * 4));
  SelectArgs s{};
  s.scores = s_dev;
  s.stride = stride;
  s.n_in = ctx->generic_n.as<uint32_t>();
  s.seq_len = 0xFFFFFFFFu;
  s.block_size = ctx->cfg.block_size;
  s.keep = keep;
  s.mode = blocks ? kSelBlocksGeneric : kSelGeneric;
  s.tie_break = ctx->cfg.tie_break;
  s.force_first_last = ctx->cfg.force_first_last;
  s.forced_in_budget = ctx->cfg.forced_in_budget;
  s.out_idx = idx_dev ? out_idx : ctx->out_idx.as<int32_t>();
  s.out_stride = out_width;
  s.out_width = out_width;
  s.out_count = cnt_dev ? out_count : ctx->out_count.as<uint32_t>();
  count_launches(ctx, launch_select(s, uint32_t(rows), n_cap, ctx->stream));
  HISA_TRY(check_launch(ctx, "select"));
  bool need_sync = true;
  if (!idx_dev) HISA_TRY(copy_out(ctx, out_idx, s.out_idx, rows * out_width * 4, &need_sync));
  if (!cnt_dev) HISA_TRY(copy_out(ctx, out_count, s.out_count, rows * 4, &need_sync));
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  end_call(ctx);
  return HISA_OK;
}

int hisa_cuda_select_blocks(hisa_cuda_ctx* ctx, const float* scores, uint64_t score_stride, const uint32_t* neligible,
                            uint64_t num_queries, int32_t* out_blocks, uint32_t* out_nblocks) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  return generic_select(ctx, true, scores, score_stride, neligible, num_queries, ctx->cfg.block_budget,
                        ctx->cfg.block_budget + 2, out_blocks, out_nblocks);
}

int hisa_cuda_top_k(hisa_cuda_ctx* ctx, const float* scores, uint64_t score_stride, const uint32_t* n, uint64_t num_rows,
                    uint32_t k, int32_t* out_idx, uint32_t* out_count) {
  return generic_select(ctx, false, scores, score_stride, n, num_rows, k, k, out_idx, out_count);
}

int hisa_cuda_score_tokens(hisa_cuda_ctx* ctx, const void* queries, const float* gates, const uint32_t* positions,
                           uint64_t Q, float* out_scores, uint64_t out_stride) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaSetDevice(ctx->device));
  begin_call(ctx);
  if (ctx->seq_len == 0) return fail(ctx, HISA_ERR_EMPTY_SEQUENCE, "score_tokens: empty key sequence");
  Prepared p;
  HISA_TRY(prepare_inputs(ctx, queries, gates, positions, Q, 0, &p));
  if (Q == 0) return HISA_OK;
  if (!out_scores) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "null out_scores");
  const uint32_t L = uint32_t(ctx->seq_len), Lpad = round_up(L, kTileRows);
  if (out_stride < Lpad) return fail(ctx, HISA_ERR_SHAPE_MISMATCH, "score_tokens: out_stride %llu < %u", (unsigned long long)out_stride, Lpad);
  if (Q > uint64_t(ctx->chunk_dense) * 4096) return fail(ctx, HISA_ERR_UNSUPPORTED, "score_tokens: too many rows in one call");
  HISA_TRY(ensure(ctx, ctx->scalars, 64));
  const uint32_t ntiles = Lpad / kTileRows;
  const uint32_t chunk = dense_chunk_for(ctx, Q, ntiles);
  const uint32_t nchunks = uint32_t((Q + chunk - 1) / chunk);
  HISA_TRY(ensure(ctx, ctx->work, std::max<size_t>(size_t(nchunks) * ntiles, size_t(ctx->num_sms)) * sizeof(WorkItem)));  // >= one slot per CTA
  const bool out_dev = is_device_ptr(out_scores);
  if (!out_dev) HISA_TRY(ensure(ctx, ctx->flat, size_t(Q) * Lpad * 4));
  uint32_t* sc = ctx->scalars.as<uint32_t>();
  StageTimer* timer = new StageTimer(ctx, kStScoreTokens);
  count_launches(ctx, launch_build_dense_work(p.pos, uint32_t(Q), chunk, L, 1, ntiles, ctx->work.as<WorkItem>(),
                                              sc, sc + 1, nullptr, nullptr, nullptr, ctx->stream));
  ScoreJob j{};
  set_token_operands(ctx, p, 0, j);
  j.nq = Q;
  j.gates = p.gates;
  j.out = out_dev ? out_scores : ctx->flat.as<float>();
  j.out_stride = out_dev ? out_stride : Lpad;
  j.list_mode = false;
  j.max_items = nchunks * ntiles;
  int rc = run_scorer(ctx, j);
  delete timer;
  HISA_TRY(rc);
  if (!out_dev)
    CU_TRY(ctx, cudaMemcpy2DAsync(out_scores, out_stride * 4, ctx->flat.p, size_t(Lpad) * 4, size_t(Lpad) * 4, Q,
                                  cudaMemcpyDefault, ctx->stream));
  end_call(ctx);
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return HISA_OK;
}

// ---- downstream consumer: attention over the selection (attention.hpp:13-59) -------------------------------

int hisa_cuda_attn_set_latents(hisa_cuda_ctx* ctx, const void* latents, uint64_t seq_len, uint32_t d_model, uint32_t dtype,
                               int check_finite) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaSetDevice(ctx->device));
  if (dtype != HISA_DTYPE_F32 && dtype != HISA_DTYPE_BF16)
    return fail(ctx, HISA_ERR_UNSUPPORTED, "attention: latent_states must be float32 or bfloat16");
  if (d_model == 0) return fail(ctx, HISA_ERR_DIMENSION_MISMATCH, "attention: d_model must be positive");
  if (seq_len == 0) return fail(ctx, HISA_ERR_EMPTY_SEQUENCE, "attention: empty latent sequence");
  if (seq_len > 0x7FFFFFFFull) return fail(ctx, HISA_ERR_UNSUPPORTED, "attention: seq_len beyond int32 indices");
  if (!latents) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "attention: null latent_states");
  const bool bf16 = dtype == HISA_DTYPE_BF16;
  const uint32_t dm_pad = attend_padded_dim(d_model, bf16);
  if (!dm_pad) return fail(ctx, HISA_ERR_UNSUPPORTED, "attention: d_model %u > 512", d_model);
  const size_t eb = bf16 ? 2 : 4;
  ctx->attn_len = 0;
  HISA_TRY(ensure(ctx, ctx->attn_lat, size_t(seq_len) * dm_pad * eb));
  const void* src = latents;
  const bool direct = dm_pad == d_model;  // already in the kernel's layout: one copy, no padding pass
  if (!is_device_ptr(latents)) {
    void* stage = ctx->attn_lat.p;
    if (!direct) {
      HISA_TRY(ensure(ctx, ctx->attn_qraw, size_t(seq_len) * d_model * eb));
      stage = ctx->attn_qraw.p;
    }
    HISA_TRY(copy_in(ctx, stage, latents, size_t(seq_len) * d_model * eb));
    src = stage;
  } else if (direct) {
    HISA_TRY(copy_in(ctx, ctx->attn_lat.p, latents, size_t(seq_len) * d_model * eb));
    src = ctx->attn_lat.p;
  }
  if (check_finite) {
    HISA_TRY(ensure(ctx, ctx->flag, 64));
    CU_TRY(ctx, cudaMemsetAsync(ctx->flag.p, 0, 64, ctx->stream));
    count_launches(ctx, launch_check_finite(src, bf16 ? 1u : 0u, seq_len * d_model, ctx->flag.as<uint32_t>(), ctx->stream));
    uint32_t bad = 0;
    HISA_TRY(read_flag(ctx, &bad));
    if (bad) return fail(ctx, HISA_ERR_NON_FINITE, "attention: non-finite value in latent_states");
  }
  if (!direct)
    count_launches(ctx, launch_pad_rows(src, bf16, seq_len, d_model, dm_pad, ctx->attn_lat.p, bf16, ctx->stream));
  HISA_TRY(check_launch(ctx, "latent ingestion"));
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->attn_len = seq_len;
  ctx->attn_dm = d_model;
  ctx->attn_dm_pad = dm_pad;
  ctx->attn_bf16 = bf16;
  return HISA_OK;
}

static int attend_impl(hisa_cuda_ctx* ctx, const void* query_states, uint32_t q_dtype, const uint32_t* positions, uint64_t Q,
                       const int32_t* selected, uint64_t sel_stride, const uint32_t* counts, bool dense, double scale,
                       float* out, float* weights) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaSetDevice(ctx->device));
  if (ctx->attn_len == 0) return fail(ctx, HISA_ERR_EMPTY_SEQUENCE, "attention: no latent_states (hisa_cuda_attn_set_latents)");
  if (q_dtype != HISA_DTYPE_F32 && q_dtype != HISA_DTYPE_BF16)
    return fail(ctx, HISA_ERR_UNSUPPORTED, "attention: query_states must be float32 or bfloat16");
  ctx->attn_timed = false;
  if (Q == 0) return HISA_OK;
  if (Q > 0xFFFFFFFFull) return fail(ctx, HISA_ERR_UNSUPPORTED, "attention: too many rows in one call");
  if (!query_states || !positions || !out) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "attention: null argument");
  if (!dense && !selected) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "sparse_attend: null selection");
  if (!dense && sel_stride == 0) return fail(ctx, HISA_ERR_EMPTY_SELECTION, "sparse_attend: empty selection");
  const uint32_t dm = ctx->attn_dm, dmp = ctx->attn_dm_pad;
  const bool qbf = q_dtype == HISA_DTYPE_BF16;
  const size_t qeb = qbf ? 2 : 4;
  // query states -> f32 [Q, dm_pad]
  const void* q_dev = query_states;
  if (!is_device_ptr(query_states)) {
    HISA_TRY(ensure(ctx, ctx->attn_qraw, size_t(Q) * dm * qeb));
    HISA_TRY(copy_in(ctx, ctx->attn_qraw.p, query_states, size_t(Q) * dm * qeb));
    q_dev = ctx->attn_qraw.p;
  }
  if (qbf || dm != dmp) {
    HISA_TRY(ensure(ctx, ctx->attn_q, size_t(Q) * dmp * 4));
    count_launches(ctx, launch_pad_rows(q_dev, qbf, Q, dm, dmp, ctx->attn_q.p, false, ctx->stream));
    q_dev = ctx->attn_q.p;
  }
  auto stage_in = [&](DevBuf& buf, const void* p, size_t bytes, const void** dev) -> int {
    *dev = p;
    if (p && !is_device_ptr(p)) {
      HISA_TRY(ensure(ctx, buf, bytes));
      HISA_TRY(copy_in(ctx, buf.p, p, bytes));
      *dev = buf.p;
    }
    return HISA_OK;
  };
  const void *pos_dev = nullptr, *idx_dev = nullptr, *cnt_dev = nullptr;
  HISA_TRY(stage_in(ctx->attn_pos, positions, Q * 4, &pos_dev));
  if (!dense) {
    HISA_TRY(stage_in(ctx->attn_idx, selected, Q * sel_stride * 4, &idx_dev));
    HISA_TRY(stage_in(ctx->attn_cnt, counts, Q * 4, &cnt_dev));
  }
  const bool out_dev = is_device_ptr(out), w_dev = weights && is_device_ptr(weights);
  if (!out_dev) HISA_TRY(ensure(ctx, ctx->attn_out, Q * dm * 4));
  if (weights && !w_dev) HISA_TRY(ensure(ctx, ctx->attn_w, Q * sel_stride * 4));
  HISA_TRY(ensure(ctx, ctx->flag, 64));
  CU_TRY(ctx, cudaMemsetAsync(ctx->flag.p, 0, 64, ctx->stream));
  AttendArgs a{};
  a.latents = ctx->attn_lat.p;
  a.queries = static_cast<const float*>(q_dev);
  a.pos = static_cast<const uint32_t*>(pos_dev);
  a.idx = static_cast<const int32_t*>(idx_dev);
  a.count = static_cast<const uint32_t*>(cnt_dev);
  a.idx_stride = dense ? 0 : sel_stride;
  a.num_rows = uint32_t(Q);
  a.seq_len = uint32_t(ctx->attn_len);
  a.d_model = dm;
  a.dm_pad = dmp;
  a.latents_bf16 = ctx->attn_bf16 ? 1u : 0u;
  a.scale = float(scale > 0.0 ? scale : 1.0 / std::sqrt(double(dm)));  // attention.hpp:20-21
  a.out = out_dev ? out : ctx->attn_out.as<float>();
  a.weights = !weights || dense ? nullptr : (w_dev ? weights : ctx->attn_w.as<float>());
  a.weights_stride = sel_stride;
  a.flag = ctx->flag.as<uint32_t>();
  a.force_simt = env_u32("HISA_ATTEND_SIMT", 0);
  if (!ctx->attn_beg) {
    CU_TRY(ctx, cudaEventCreate(&ctx->attn_beg));
    CU_TRY(ctx, cudaEventCreate(&ctx->attn_end));
  }
  CU_TRY(ctx, cudaEventRecord(ctx->attn_beg, ctx->stream));
  const int launched = launch_sparse_attend(a, ctx->stream);
  CU_TRY(ctx, cudaEventRecord(ctx->attn_end, ctx->stream));
  if (!launched) return fail(ctx, HISA_ERR_UNSUPPORTED, "attention: no kernel for d_model %u", dm);
  count_launches(ctx, launched);
  HISA_TRY(check_launch(ctx, "sparse_attend"));
  ctx->attn_timed = true;
  uint32_t flags = 0;
  HISA_TRY(read_flag(ctx, &flags));
  if (flags & 4u) return fail(ctx, HISA_ERR_SHAPE_MISMATCH, "attention: a query position is not below seq_len %llu",
                              (unsigned long long)ctx->attn_len);
  if (flags & 2u) return fail(ctx, HISA_ERR_CAUSAL_VIOLATION, "sparse_attend: a selected index exceeds its query position");
  if (flags & 1u) return fail(ctx, HISA_ERR_EMPTY_SELECTION, "sparse_attend: empty selection");
  bool need_sync = false;
  if (!out_dev) HISA_TRY(copy_out(ctx, out, a.out, Q * dm * 4, &need_sync));
  if (a.weights && !w_dev) HISA_TRY(copy_out(ctx, weights, a.weights, Q * sel_stride * 4, &need_sync));
  if (need_sync) CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return HISA_OK;
}

int hisa_cuda_sparse_attend(hisa_cuda_ctx* ctx, const void* query_states, uint32_t q_dtype, const uint32_t* positions,
                            uint64_t num_queries, const int32_t* selected, uint64_t sel_stride, const uint32_t* counts,
                            double scale, float* out, float* weights) {
  return attend_impl(ctx, query_states, q_dtype, positions, num_queries, selected, sel_stride, counts, false, scale, out,
                     weights);
}

int hisa_cuda_dense_attend(hisa_cuda_ctx* ctx, const void* query_states, uint32_t q_dtype, const uint32_t* positions,
                           uint64_t num_queries, double scale, float* out) {
  return attend_impl(ctx, query_states, q_dtype, positions, num_queries, nullptr, 0, nullptr, true, scale, out, nullptr);
}

int hisa_cuda_attn_last_ms(hisa_cuda_ctx* ctx, float* ms) {
  if (!ctx || !ms) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "null argument");
  *ms = 0.f;
  if (!ctx->attn_timed) return HISA_OK;
  CU_TRY(ctx, cudaEventSynchronize(ctx->attn_end));
  CU_TRY(ctx, cudaEventElapsedTime(ms, ctx->attn_beg, ctx->attn_end));
  return HISA_OK;
}

// ---- instrumentation -------------------------------------------------------------------------------------

int hisa_cuda_set_profiling(hisa_cuda_ctx* ctx, int enable) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  ctx->profiling = enable != 0;
  ctx->stall_stats = (enable & 2) != 0;
  return HISA_OK;
}

int hisa_cuda_last_stage_times(hisa_cuda_ctx* ctx, hisa_cuda_stage_times* out) {
  if (!ctx || !out) return fail(ctx, HISA_ERR_INVALID_ARGUMENT, "null argument");
  memset(out, 0, sizeof *out);
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  float* slot[kNumStages] = {&out->prepare_ms,  &out->score_blocks_ms, &out->select_blocks_ms, &out->invert_ms,
                             &out->score_tokens_ms, &out->top_k_ms,     &out->total_ms};
  for (const StageSpan& s : ctx->spans) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, s.beg, s.end) == cudaSuccess) *slot[s.stage] += ms;
  }
  cudaGetLastError();
  out->launches = ctx->call_launches;
  out->work_items_stage1 = ctx->items1;
  out->work_items_stage2 = ctx->items2;
  out->calls = ctx->calls;
  ctx->spans.clear();
  ctx->events_used = 0;
  ctx->call_launches = 0;
  ctx->items1 = ctx->items2 = 0;
  ctx->calls = 0;
  return HISA_OK;
}

int hisa_cuda_scorer_stall_cycles(hisa_cuda_ctx* ctx, uint64_t* stage1, uint64_t* stage2) {
  if (!ctx) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null context");
  CU_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  unsigned long long host[32] = {0};
  if (ctx->stats.p) {
    CU_TRY(ctx, cudaMemcpy(host, ctx->stats.p, sizeof host, cudaMemcpyDeviceToHost));
    CU_TRY(ctx, cudaMemset(ctx->stats.p, 0, sizeof host));
  }
  for (int i = 0; i < 16; ++i) {
    if (stage1) stage1[i] = host[i];
    if (stage2) stage2[i] = host[16 + i];
  }
  return HISA_OK;
}

int hisa_cuda_launch_count(const hisa_cuda_ctx* ctx, uint64_t* launches) {
  if (!ctx || !launches) return fail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null argument");
  *launches = ctx->launches;
  return HISA_OK;
}

}  // extern "C"
