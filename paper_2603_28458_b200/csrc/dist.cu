// Multi-GPU driver behind the C ABI (include/hisa_cuda.h, hisa_cuda_dist_*): query rows sharded over G B200s.
//
// Reference contract: every query row is independent ("callers may fan out queries across workers freely",
// SPEC.md:246 "parallel across queries"; hisa/parallel.hpp:15-19 is the reference's own fan-out over rows). The only
// shared state is the read-only key sequence and its block summaries; the only exchange is that every GPU ends up with
// the whole int32 [Q, k] index matrix.
//
//   * partition   rows are dealt in 512-row tiles, zig-zag over the ranks (0 1 .. G-1 G-1 .. 1 0 ...): causal work is
//                 triangular (flat) or ramps up to (m+2)B candidates (hierarchical), contiguous chunks would not balance;
//   * replicate   keys (16-32 MiB, 256 MiB at 1M tokens) by ncclBroadcast over NVLink from the rank that holds them; the
//                 block summaries are recomputed on every GPU (10 us) rather than broadcast;
//   * compute     one hisa_cuda_ctx + stream per GPU; a rank's rows run in `num_slices` slices of whole tiles;
//   * gather      two implementations of "every GPU holds every index row":
//        PEER  (default when every pair of ranks has peer access, i.e. an NVSwitch box driven from one process): the
//              top-k kernel itself stores each finished row to the row's place in EVERY GPU's result matrix
//              (hisa_cuda_set_output_placement: peer stores over NVLink). Compute and collective are one kernel; the
//              transfer overlaps the selection row by row, nothing is staged, permuted or launched afterwards.
//        NCCL  per-tile ncclBroadcast (root = the tile's owner, in place in the final matrix), grouped per slice and
//              issued on a second stream, so the gather of slice i runs under the kernels of slice i+1.
//     Both leave results in GLOBAL row order on every GPU; the G-GPU result equals the 1-GPU result bit for bit because
//     the same kernels run on the same rows.
//
// Process models: hisa_cuda_dist_create drives G GPUs from ONE process (ncclCommInitAll, one host thread per GPU);
// hisa_cuda_dist_create_rank is one rank of a multi-process job (ncclCommInitRank with an id from
// hisa_cuda_dist_unique_id; torchrun / MPI style launchers). NCCL is loaded with dlopen so that single-GPU users of
// libhisa_b200.so need no NCCL at all.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hisa_cuda.h"

namespace {

constexpr uint32_t kTile = HISA_DIST_TILE_ROWS;
constexpr int kMaxSlices = 16;

thread_local std::string g_dist_error;

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  bool load(std::string& err) {
    if (handle) return true;
    // a process that already loaded NCCL (e.g. through torch) gets that copy: same soname
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (handle) break;
    }
    if (!handle) {
      err = std::string("NCCL is not available: ") + (dlerror() ? dlerror() : "dlopen failed");
      return false;
    }
    auto sym = [&](const char* n) { return dlsym(handle, n); };
    GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(sym("ncclGetUniqueId"));
    CommInitRank = reinterpret_cast<decltype(CommInitRank)>(sym("ncclCommInitRank"));
    CommInitAll = reinterpret_cast<decltype(CommInitAll)>(sym("ncclCommInitAll"));
    CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
    Broadcast = reinterpret_cast<decltype(Broadcast)>(sym("ncclBroadcast"));
    AllGather = reinterpret_cast<decltype(AllGather)>(sym("ncclAllGather"));
    GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
    GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
    CommGetAsyncError = reinterpret_cast<decltype(CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
    if (!GetUniqueId || !CommInitRank || !CommInitAll || !CommDestroy || !Broadcast || !GroupStart || !GroupEnd ||
        !GetErrorString) {
      err = "libnccl.so.2 lacks a required entry point";
      return false;
    }
    return true;
  }
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

// zig-zag deal of tiles over ranks (the same arithmetic as paper_2603_28458_b200/sharding.py)
inline int tile_owner(uint64_t tile, int world) {
  const uint64_t phase = tile % (2ull * uint64_t(world));
  return int(phase < uint64_t(world) ? phase : 2ull * uint64_t(world) - 1 - phase);
}
inline uint64_t num_tiles(uint64_t rows) { return (rows + kTile - 1) / kTile; }
inline uint32_t tile_len(uint64_t tile, uint64_t rows) { return uint32_t(std::min<uint64_t>(kTile, rows - tile * kTile)); }

std::vector<uint32_t> tiles_of(uint64_t rows, int world, int rank) {
  std::vector<uint32_t> t;
  for (uint64_t i = 0; i < num_tiles(rows); ++i)
    if (tile_owner(i, world) == rank) t.push_back(uint32_t(i));
  return t;
}

// one worker thread per local GPU: jobs are closures executed in submission order
class Worker {
 public:
  Worker() : th_([this] { loop(); }) {}
  ~Worker() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    th_.join();
  }
  void submit(std::function<void()> fn) {
    {
      std::lock_guard<std::mutex> g(mu_);
      jobs_.push_back(std::move(fn));
      ++pending_;
    }
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [this] { return pending_ == 0; });
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> fn;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [this] { return stop_ || !jobs_.empty(); });
        if (jobs_.empty()) return;
        fn = std::move(jobs_.front());
        jobs_.erase(jobs_.begin());
      }
      fn();
      {
        std::lock_guard<std::mutex> g(mu_);
        --pending_;
      }
      done_cv_.notify_all();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::function<void()>> jobs_;
  int pending_ = 0;
  bool stop_ = false;
  std::thread th_;
};

struct Rank {
  int device = 0, rank = 0;
  hisa_cuda_ctx* ctx = nullptr;
  cudaStream_t stream = nullptr, comm_stream = nullptr;
  ncclComm_t comm = nullptr;
  cudaEvent_t slice_done[kMaxSlices] = {}, comm_done = nullptr, t_beg = nullptr, t_end = nullptr;
  unsigned char* key_stage = nullptr;
  size_t key_stage_cap = 0;
  float* scale_stage = nullptr;
  size_t scale_stage_cap = 0;
  int32_t* out_idx = nullptr;     // [rows_cap, k] the full result on this GPU
  uint32_t* out_count = nullptr;  // [rows_cap]
  uint64_t rows_cap = 0;
  uint32_t* row_map = nullptr;    // device [local rows]: global row of every local row
  uint64_t row_map_cap = 0, row_map_rows = 0;  // rows the map was built for (0 = none)
  std::unique_ptr<Worker> worker;
  int status = HISA_OK;
  std::string err;
};

}  // namespace

struct hisa_cuda_dist {
  hisa_cuda_config cfg{};
  int world = 1, first_rank = 0;
  bool single_process = true;
  int gather = HISA_DIST_GATHER_NCCL;
  bool have_nccl = false;
  std::vector<Rank> ranks;  // local ranks
  std::string err;
  bool timed = false;
  uint64_t last_rows = 0;
};

namespace {

int dfail(hisa_cuda_dist* d, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (d) d->err = buf;
  else g_dist_error = buf;
  return code;
}

#define DCU(r, expr)                                                                                            \
  do {                                                                                                          \
    cudaError_t e__ = (expr);                                                                                   \
    if (e__ != cudaSuccess) {                                                                                   \
      (r).status = e__ == cudaErrorMemoryAllocation ? HISA_ERR_OUT_OF_MEMORY : HISA_ERR_CUDA;                    \
      (r).err = std::string(#expr) + " failed: " + cudaGetErrorString(e__);                                     \
      return;                                                                                                   \
    }                                                                                                           \
  } while (0)
#define DNCCL(r, expr)                                                                                          \
  do {                                                                                                          \
    ncclResult_t n__ = (expr);                                                                                  \
    if (n__ != ncclSuccess) {                                                                                   \
      (r).status = HISA_ERR_CUDA;                                                                               \
      (r).err = std::string(#expr) + " failed: " + g_nccl.GetErrorString(n__);                                  \
      return;                                                                                                   \
    }                                                                                                           \
  } while (0)
#define DHISA(r, expr)                                                                                          \
  do {                                                                                                          \
    int s__ = (expr);                                                                                           \
    if (s__ != HISA_OK) {                                                                                       \
      (r).status = s__;                                                                                         \
      (r).err = hisa_cuda_last_error((r).ctx);                                                                  \
      return;                                                                                                   \
    }                                                                                                           \
  } while (0)

// runs fn on every local rank's worker thread and joins; returns the first failure
int run_all(hisa_cuda_dist* d, const std::function<void(Rank&)>& fn) {
  for (Rank& r : d->ranks) {
    r.status = HISA_OK;
    r.err.clear();
    Rank* rp = &r;
    r.worker->submit([rp, &fn] {
      cudaSetDevice(rp->device);
      fn(*rp);
    });
  }
  for (Rank& r : d->ranks) r.worker->wait();
  for (Rank& r : d->ranks)
    if (r.status != HISA_OK) return dfail(d, r.status, "rank %d (device %d): %s", r.rank, r.device, r.err.c_str());
  return HISA_OK;
}

void rank_release(Rank& r) {
  cudaSetDevice(r.device);
  if (r.stream) cudaStreamSynchronize(r.stream);
  if (r.comm_stream) cudaStreamSynchronize(r.comm_stream);
  if (r.comm) g_nccl.CommDestroy(r.comm);
  for (cudaEvent_t& e : r.slice_done)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {r.comm_done, r.t_beg, r.t_end})
    if (e) cudaEventDestroy(e);
  for (void* p : {static_cast<void*>(r.key_stage), static_cast<void*>(r.scale_stage), static_cast<void*>(r.out_idx),
                  static_cast<void*>(r.out_count), static_cast<void*>(r.row_map)})
    if (p) cudaFree(p);
  if (r.comm_stream) cudaStreamDestroy(r.comm_stream);
  if (r.ctx) hisa_cuda_destroy(r.ctx);
  r = Rank{};
}

int rank_setup(hisa_cuda_dist* d, Rank& r) {
  if (cudaSetDevice(r.device) != cudaSuccess) return dfail(d, HISA_ERR_NO_DEVICE, "cudaSetDevice(%d) failed", r.device);
  const int rc = hisa_cuda_create(r.device, &d->cfg, &r.ctx);
  if (rc != HISA_OK) return dfail(d, rc, "rank %d: %s", r.rank, hisa_cuda_last_error(nullptr));
  r.stream = static_cast<cudaStream_t>(hisa_cuda_stream(r.ctx));
  if (cudaStreamCreateWithFlags(&r.comm_stream, cudaStreamNonBlocking) != cudaSuccess)
    return dfail(d, HISA_ERR_CUDA, "rank %d: could not create the communication stream", r.rank);
  for (cudaEvent_t& e : r.slice_done)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return dfail(d, HISA_ERR_CUDA, "event creation failed");
  if (cudaEventCreateWithFlags(&r.comm_done, cudaEventDisableTiming) != cudaSuccess || cudaEventCreate(&r.t_beg) != cudaSuccess ||
      cudaEventCreate(&r.t_end) != cudaSuccess)
    return dfail(d, HISA_ERR_CUDA, "event creation failed");
  r.worker = std::make_unique<Worker>();
  return HISA_OK;
}

// grows a device buffer (contents are not kept)
template <class T>
bool grow(T*& p, size_t& cap, size_t need_elems) {
  if (need_elems <= cap) return true;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  if (cudaMalloc(reinterpret_cast<void**>(&p), std::max<size_t>(need_elems, 1) * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cap = need_elems;
  return true;
}

size_t elem_bytes(const hisa_cuda_config& c) { return c.dtype == HISA_DTYPE_BF16 ? 2 : c.dtype == HISA_DTYPE_FP8_E4M3 ? 1 : 4; }

// every pair of distinct local devices can map each other's memory
bool enable_peer_access(hisa_cuda_dist* d) {
  for (Rank& a : d->ranks)
    for (Rank& b : d->ranks) {
      if (a.device == b.device) continue;
      int ok = 0;
      if (cudaDeviceCanAccessPeer(&ok, a.device, b.device) != cudaSuccess || !ok) {
        cudaGetLastError();
        return false;
      }
    }
  for (Rank& a : d->ranks) {
    cudaSetDevice(a.device);
    for (Rank& b : d->ranks) {
      if (a.device == b.device) continue;
      const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return false;
      }
      cudaGetLastError();
    }
  }
  return true;
}

int finish_create(hisa_cuda_dist* d, uint32_t flags) {
  const int want = int(flags & 3u);
  // peer stores need every rank's result matrix mapped in this process: the single-process model on a P2P box
  const bool peer_ok = d->single_process && int(d->ranks.size()) == d->world && d->world - 1 <= 7 && enable_peer_access(d);
  if (want == HISA_DIST_GATHER_PEER && !peer_ok)
    return dfail(d, HISA_ERR_UNSUPPORTED, "peer-store gather needs all ranks in one process with peer access between every pair of GPUs");
  if (want == HISA_DIST_GATHER_NCCL && !d->have_nccl)
    return dfail(d, HISA_ERR_UNSUPPORTED, "NCCL gather requested but NCCL is not initialised");
  d->gather = want == HISA_DIST_GATHER_AUTO ? (peer_ok ? HISA_DIST_GATHER_PEER : HISA_DIST_GATHER_NCCL) : want;
  if (d->gather == HISA_DIST_GATHER_NCCL && !d->have_nccl && d->world > 1)
    return dfail(d, HISA_ERR_UNSUPPORTED, "no gather path: no peer access and no NCCL communicator");
  return HISA_OK;
}

}  // namespace

extern "C" {

const char* hisa_cuda_dist_last_error(const hisa_cuda_dist* d) { return d ? d->err.c_str() : g_dist_error.c_str(); }

int hisa_cuda_dist_plan(uint64_t num_rows, int world, int rank, uint64_t* count, uint32_t* rows_out) {
  if (world <= 0 || rank < 0 || rank >= world) return dfail(nullptr, HISA_ERR_INVALID_ARGUMENT, "rank %d outside world %d", rank, world);
  if (num_rows > 0xFFFFFFFFull) return dfail(nullptr, HISA_ERR_UNSUPPORTED, "more than 2^32 rows");
  uint64_t n = 0;
  for (uint64_t t = 0; t < num_tiles(num_rows); ++t) {
    if (tile_owner(t, world) != rank) continue;
    const uint32_t len = tile_len(t, num_rows);
    if (rows_out)
      for (uint32_t i = 0; i < len; ++i) rows_out[n + i] = uint32_t(t * kTile + i);
    n += len;
  }
  if (count) *count = n;
  return HISA_OK;
}

int hisa_cuda_dist_create(const int* devices, int num_devices, const hisa_cuda_config* cfg, uint32_t flags, hisa_cuda_dist** out) {
  if (!out) return dfail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  if (!devices || num_devices <= 0 || !cfg) return dfail(nullptr, HISA_ERR_INVALID_ARGUMENT, "need a device list and a config");
  if (num_devices > 64) return dfail(nullptr, HISA_ERR_UNSUPPORTED, "more than 64 devices");
  hisa_cuda_dist* d = new hisa_cuda_dist();
  d->cfg = *cfg;
  d->world = num_devices;
  d->single_process = true;
  d->ranks.resize(size_t(num_devices));
  auto bail = [&](int rc) {
    g_dist_error = d->err;
    for (Rank& r : d->ranks) {
      r.worker.reset();
      rank_release(r);
    }
    delete d;
    return rc;
  };
  for (int i = 0; i < num_devices; ++i) {
    d->ranks[size_t(i)].device = devices[i];
    d->ranks[size_t(i)].rank = i;
    const int rc = rank_setup(d, d->ranks[size_t(i)]);
    if (rc != HISA_OK) return bail(rc);
  }
  // NCCL communicators (one per GPU, one process): not possible when a device appears twice (the logical-rank mode
  // this library's tests use on a one-GPU box), and not needed for one rank unless the caller insists on it
  bool distinct = true;
  for (int i = 0; i < num_devices; ++i)
    for (int j = 0; j < i; ++j) distinct = distinct && devices[i] != devices[j];
  const int want = int(flags & 3u);
  if (distinct && (num_devices > 1 || want == HISA_DIST_GATHER_NCCL)) {
    std::lock_guard<std::mutex> g(g_nccl_mu);
    std::string err;
    if (g_nccl.load(err)) {
      std::vector<ncclComm_t> comms(size_t(num_devices), nullptr);
      const ncclResult_t nr = g_nccl.CommInitAll(comms.data(), num_devices, devices);
      if (nr == ncclSuccess) {
        for (int i = 0; i < num_devices; ++i) d->ranks[size_t(i)].comm = comms[size_t(i)];
        d->have_nccl = true;
      } else if (want == HISA_DIST_GATHER_NCCL) {
        d->err = std::string("ncclCommInitAll failed: ") + g_nccl.GetErrorString(nr);
        return bail(HISA_ERR_CUDA);
      }
    } else if (want == HISA_DIST_GATHER_NCCL) {
      d->err = err;
      return bail(HISA_ERR_UNSUPPORTED);
    }
  }
  const int rc = finish_create(d, flags);
  if (rc != HISA_OK) return bail(rc);
  *out = d;
  return HISA_OK;
}

int hisa_cuda_dist_unique_id(void* id, size_t bytes) {
  if (!id || bytes < sizeof(ncclUniqueId)) return dfail(nullptr, HISA_ERR_INVALID_ARGUMENT, "the id buffer must hold %zu bytes", sizeof(ncclUniqueId));
  std::lock_guard<std::mutex> g(g_nccl_mu);
  std::string err;
  if (!g_nccl.load(err)) return dfail(nullptr, HISA_ERR_UNSUPPORTED, "%s", err.c_str());
  ncclUniqueId uid;
  const ncclResult_t nr = g_nccl.GetUniqueId(&uid);
  if (nr != ncclSuccess) return dfail(nullptr, HISA_ERR_CUDA, "ncclGetUniqueId failed: %s", g_nccl.GetErrorString(nr));
  memset(id, 0, bytes);
  memcpy(id, &uid, sizeof uid);
  return HISA_OK;
}

int hisa_cuda_dist_create_rank(const void* id, int world, int rank, int device, const hisa_cuda_config* cfg, uint32_t flags,
                               hisa_cuda_dist** out) {
  if (!out) return dfail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  if (!id || !cfg || world <= 0 || rank < 0 || rank >= world) return dfail(nullptr, HISA_ERR_INVALID_ARGUMENT, "bad rank / world / id");
  if (int(flags & 3u) == HISA_DIST_GATHER_PEER)
    return dfail(nullptr, HISA_ERR_UNSUPPORTED, "peer-store gather needs all ranks in one process (hisa_cuda_dist_create)");
  hisa_cuda_dist* d = new hisa_cuda_dist();
  d->cfg = *cfg;
  d->world = world;
  d->first_rank = rank;
  d->single_process = false;
  d->ranks.resize(1);
  d->ranks[0].device = device;
  d->ranks[0].rank = rank;
  auto bail = [&](int rc) {
    g_dist_error = d->err;
    d->ranks[0].worker.reset();
    rank_release(d->ranks[0]);
    delete d;
    return rc;
  };
  int rc = rank_setup(d, d->ranks[0]);
  if (rc != HISA_OK) return bail(rc);
  {
    std::lock_guard<std::mutex> g(g_nccl_mu);
    std::string err;
    if (!g_nccl.load(err)) {
      d->err = err;
      return bail(HISA_ERR_UNSUPPORTED);
    }
  }
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  cudaSetDevice(device);
  const ncclResult_t nr = g_nccl.CommInitRank(&d->ranks[0].comm, world, uid, rank);
  if (nr != ncclSuccess) {
    d->err = std::string("ncclCommInitRank failed: ") + g_nccl.GetErrorString(nr);
    return bail(HISA_ERR_CUDA);
  }
  d->have_nccl = true;
  rc = finish_create(d, HISA_DIST_GATHER_NCCL);
  if (rc != HISA_OK) return bail(rc);
  *out = d;
  return HISA_OK;
}

int hisa_cuda_dist_destroy(hisa_cuda_dist* d) {
  if (!d) return HISA_OK;
  for (Rank& r : d->ranks) r.worker.reset();
  for (Rank& r : d->ranks) rank_release(r);
  delete d;
  return HISA_OK;
}

int hisa_cuda_dist_info(const hisa_cuda_dist* d, int* world, int* num_local, int* first_rank, int* gather) {
  if (!d) return dfail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null driver");
  if (world) *world = d->world;
  if (num_local) *num_local = int(d->ranks.size());
  if (first_rank) *first_rank = d->first_rank;
  if (gather) *gather = d->gather;
  return HISA_OK;
}

hisa_cuda_ctx* hisa_cuda_dist_ctx(hisa_cuda_dist* d, int local) {
  return d && local >= 0 && local < int(d->ranks.size()) ? d->ranks[size_t(local)].ctx : nullptr;
}

int hisa_cuda_dist_upload_keys(hisa_cuda_dist* d, const void* keys, const float* key_scales, uint64_t seq_len, int root) {
  if (!d) return dfail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null driver");
  if (root < 0 || root >= d->world) return dfail(d, HISA_ERR_INVALID_ARGUMENT, "root rank %d outside world %d", root, d->world);
  if (seq_len == 0) return dfail(d, HISA_ERR_EMPTY_SEQUENCE, "upload_keys: key matrix has no rows");
  const bool fp8 = d->cfg.dtype == HISA_DTYPE_FP8_E4M3;
  const size_t bytes = size_t(seq_len) * d->cfg.dim * elem_bytes(d->cfg);
  const bool root_here = root >= d->first_rank && root < d->first_rank + int(d->ranks.size());
  if (root_here && !keys) return dfail(d, HISA_ERR_INVALID_ARGUMENT, "the process that owns the root rank must pass the keys");
  const bool bcast = d->world > 1;
  if (bcast && !d->have_nccl) {
    // logical ranks on one device / no NCCL: every local rank reads the caller's array itself
    if (int(d->ranks.size()) != d->world) return dfail(d, HISA_ERR_UNSUPPORTED, "key replication across processes needs NCCL");
    return run_all(d, [&](Rank& r) {
      DHISA(r, fp8 ? hisa_cuda_upload_keys_scaled(r.ctx, keys, key_scales, seq_len, 0) : hisa_cuda_upload_keys(r.ctx, keys, seq_len, 0));
      DHISA(r, hisa_cuda_pool_build(r.ctx));
    });
  }
  return run_all(d, [&](Rank& r) {
    const void* src = keys;
    const float* ssrc = key_scales;
    if (bcast) {
      // stage on the root, ncclBroadcast over NVLink, then every rank ingests its device copy
      if (!grow(r.key_stage, r.key_stage_cap, bytes)) {
        r.status = HISA_ERR_OUT_OF_MEMORY;
        r.err = "key staging buffer";
        return;
      }
      if (fp8 && !grow(r.scale_stage, r.scale_stage_cap, size_t(seq_len))) {
        r.status = HISA_ERR_OUT_OF_MEMORY;
        r.err = "scale staging buffer";
        return;
      }
      if (r.rank == root) {
        DCU(r, cudaMemcpyAsync(r.key_stage, keys, bytes, cudaMemcpyDefault, r.stream));
        if (fp8) {
          if (key_scales) DCU(r, cudaMemcpyAsync(r.scale_stage, key_scales, seq_len * sizeof(float), cudaMemcpyDefault, r.stream));
          else {
            std::vector<float> ones(size_t(seq_len), 1.f);
            DCU(r, cudaMemcpyAsync(r.scale_stage, ones.data(), seq_len * sizeof(float), cudaMemcpyHostToDevice, r.stream));
            DCU(r, cudaStreamSynchronize(r.stream));
          }
        }
      }
      DNCCL(r, g_nccl.Broadcast(r.key_stage, r.key_stage, bytes, ncclUint8, root, r.comm, r.stream));
      if (fp8) DNCCL(r, g_nccl.Broadcast(r.scale_stage, r.scale_stage, size_t(seq_len), ncclFloat32, root, r.comm, r.stream));
      src = r.key_stage;
      ssrc = r.scale_stage;
    }
    DHISA(r, fp8 ? hisa_cuda_upload_keys_scaled(r.ctx, src, ssrc, seq_len, 0) : hisa_cuda_upload_keys(r.ctx, src, seq_len, 0));
    // block summaries are recomputed per GPU: 10 us of pooling beats a second broadcast
    DHISA(r, hisa_cuda_pool_build(r.ctx));
  });
}

int hisa_cuda_dist_select(hisa_cuda_dist* d, int strategy, const void* const* queries, const float* const* gates,
                          const uint32_t* const* positions, uint64_t total_rows, int num_slices) {
  if (!d) return dfail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null driver");
  if (strategy != HISA_DIST_DSA && strategy != HISA_DIST_HISA) return dfail(d, HISA_ERR_INVALID_ARGUMENT, "strategy must be HISA_DIST_DSA or HISA_DIST_HISA");
  if (total_rows == 0) return HISA_OK;
  if (total_rows > 0x7FFFFFFFull) return dfail(d, HISA_ERR_UNSUPPORTED, "too many rows");
  if (!queries || !gates || !positions) return dfail(d, HISA_ERR_INVALID_ARGUMENT, "null per-rank input lists");
  num_slices = std::max(1, std::min(num_slices, kMaxSlices));
  const uint32_t k = d->cfg.token_budget, H = d->cfg.num_heads;
  const size_t q_row = size_t(H) * d->cfg.dim * elem_bytes(d->cfg);
  const int world = d->world;
  const bool peer = d->gather == HISA_DIST_GATHER_PEER && world > 1;
  const bool nccl_gather = d->gather == HISA_DIST_GATHER_NCCL && world > 1;
  // the tile lists of ALL ranks: every rank issues the same sequence of broadcasts
  std::vector<std::vector<uint32_t>> tiles(static_cast<size_t>(world));
  for (int r = 0; r < world; ++r) tiles[size_t(r)] = tiles_of(total_rows, world, r);
  // result matrices first (the peer lists below need every rank's pointers)
  int rc = run_all(d, [&](Rank& r) {
    if (r.rows_cap < total_rows) {
      size_t cap_i = 0, cap_c = 0;
      if (r.out_idx) cudaFree(r.out_idx);
      if (r.out_count) cudaFree(r.out_count);
      r.out_idx = nullptr;
      r.out_count = nullptr;
      r.rows_cap = 0;
      if (!grow(r.out_idx, cap_i, size_t(total_rows) * k) || !grow(r.out_count, cap_c, size_t(total_rows))) {
        r.status = HISA_ERR_OUT_OF_MEMORY;
        r.err = "result matrix";
        return;
      }
      r.rows_cap = total_rows;
    }
    const std::vector<uint32_t>& mine = tiles[size_t(r.rank)];
    uint64_t n_local = 0;
    for (uint32_t t : mine) n_local += tile_len(t, total_rows);
    if (r.row_map_rows != total_rows) {
      std::vector<uint32_t> map;
      map.reserve(size_t(n_local));
      for (uint32_t t : mine)
        for (uint32_t i = 0; i < tile_len(t, total_rows); ++i) map.push_back(t * kTile + i);
      size_t cap = size_t(r.row_map_cap);
      if (!grow(r.row_map, cap, map.size())) {
        r.status = HISA_ERR_OUT_OF_MEMORY;
        r.err = "row map";
        return;
      }
      r.row_map_cap = cap;
      DCU(r, cudaMemcpyAsync(r.row_map, map.data(), map.size() * 4, cudaMemcpyHostToDevice, r.stream));
      DCU(r, cudaStreamSynchronize(r.stream));
      r.row_map_rows = total_rows;
    }
  });
  if (rc != HISA_OK) return rc;
  d->last_rows = total_rows;
  d->timed = true;
  rc = run_all(d, [&](Rank& r) {
    const int li = r.rank - d->first_rank;
    const std::vector<uint32_t>& mine = tiles[size_t(r.rank)];
    int32_t* rep_idx[7];
    uint32_t* rep_cnt[7];
    int nrep = 0;
    if (peer)
      for (Rank& o : d->ranks)
        if (o.rank != r.rank) {
          rep_idx[nrep] = o.out_idx;
          rep_cnt[nrep] = o.out_count;
          ++nrep;
        }
    DCU(r, cudaEventRecord(r.t_beg, r.stream));
    // slices of whole tiles; every rank uses the same tiles-per-slice so that slice s means the same tiles everywhere
    size_t max_tiles = 0;
    for (const auto& t : tiles) max_tiles = std::max(max_tiles, t.size());
    const size_t per = std::max<size_t>(1, (max_tiles + size_t(num_slices) - 1) / size_t(num_slices));
    uint64_t row0 = 0;  // first local row of the slice
    int issued = 0;
    for (size_t s0 = 0, s = 0; s0 < max_tiles; s0 += per, ++s) {
      uint64_t n = 0;
      for (size_t i = s0; i < std::min(mine.size(), s0 + per); ++i) n += tile_len(mine[i], total_rows);
      if (n) {
        DHISA(r, hisa_cuda_set_output_placement(r.ctx, r.row_map + row0, nrep, rep_idx, rep_cnt));
        const void* q = static_cast<const char*>(queries[li]) + row0 * q_row;
        const float* w = gates[li] + row0 * H;
        const uint32_t* p = positions[li] + row0;
        const int src = strategy == HISA_DIST_HISA
                            ? hisa_cuda_hisa_select(r.ctx, q, w, p, n, 0, r.out_idx, r.out_count, nullptr, nullptr, nullptr)
                            : hisa_cuda_dsa_select(r.ctx, q, w, p, n, 0, r.out_idx, r.out_count, nullptr);
        hisa_cuda_set_output_placement(r.ctx, nullptr, 0, nullptr, nullptr);
        DHISA(r, src);
        row0 += n;
      }
      if (nccl_gather) {
        // slice s of every rank is complete on its owner once that owner's slice event fires; the broadcasts of this
        // slice run on the communication stream under the kernels of the next slice
        DCU(r, cudaEventRecord(r.slice_done[s % kMaxSlices], r.stream));
        DCU(r, cudaStreamWaitEvent(r.comm_stream, r.slice_done[s % kMaxSlices], 0));
        DNCCL(r, g_nccl.GroupStart());
        for (int o = 0; o < world; ++o) {
          const std::vector<uint32_t>& ot = tiles[size_t(o)];
          for (size_t i = s0; i < std::min(ot.size(), s0 + per); ++i) {
            const uint64_t t = ot[i];
            const size_t rows = tile_len(t, total_rows);
            int32_t* ip = r.out_idx + t * kTile * k;
            uint32_t* cp = r.out_count + t * kTile;
            DNCCL(r, g_nccl.Broadcast(ip, ip, rows * k, ncclInt32, o, r.comm, r.comm_stream));
            DNCCL(r, g_nccl.Broadcast(cp, cp, rows, ncclUint32, o, r.comm, r.comm_stream));
          }
        }
        DNCCL(r, g_nccl.GroupEnd());
        ++issued;
      }
    }
    if (issued) {
      DCU(r, cudaEventRecord(r.comm_done, r.comm_stream));
      DCU(r, cudaStreamWaitEvent(r.stream, r.comm_done, 0));  // the step ends when this GPU holds every row
    }
    if (peer) DCU(r, cudaEventRecord(r.comm_done, r.stream));  // "my rows are stored everywhere"
    else DCU(r, cudaEventRecord(r.t_end, r.stream));
  });
  if (rc != HISA_OK || !peer) return rc;
  // peer stores: a GPU holds every row once EVERY rank's kernels have finished, so each stream waits for the others'
  // completion events (all recorded by now: the phase above has been joined) before its step counts as done
  return run_all(d, [&](Rank& r) {
    for (Rank& o : d->ranks)
      if (o.rank != r.rank) DCU(r, cudaStreamWaitEvent(r.stream, o.comm_done, 0));
    DCU(r, cudaEventRecord(r.t_end, r.stream));
  });
}

int hisa_cuda_dist_synchronize(hisa_cuda_dist* d) {
  if (!d) return dfail(nullptr, HISA_ERR_INVALID_ARGUMENT, "null driver");
  // peer stores of OTHER ranks land in this rank's matrix: "done" means every local stream has drained
  return run_all(d, [&](Rank& r) {
    DCU(r, cudaStreamSynchronize(r.stream));
    DCU(r, cudaStreamSynchronize(r.comm_stream));
    if (r.comm && g_nccl.CommGetAsyncError) {
      ncclResult_t async = ncclSuccess;
      DNCCL(r, g_nccl.CommGetAsyncError(r.comm, &async));
      if (async != ncclSuccess) {
        r.status = HISA_ERR_CUDA;
        r.err = std::string("NCCL asynchronous error: ") + g_nccl.GetErrorString(async);
      }
    }
  });
}

int hisa_cuda_dist_result(hisa_cuda_dist* d, int local, int32_t** idx, uint32_t** count) {
  if (!d || local < 0 || local >= int(d->ranks.size())) return dfail(d, HISA_ERR_INVALID_ARGUMENT, "bad local rank index");
  if (idx) *idx = d->ranks[size_t(local)].out_idx;
  if (count) *count = d->ranks[size_t(local)].out_count;
  return HISA_OK;
}

int hisa_cuda_dist_fetch(hisa_cuda_dist* d, int local, int32_t* host_idx, uint32_t* host_count) {
  if (!d || local < 0 || local >= int(d->ranks.size())) return dfail(d, HISA_ERR_INVALID_ARGUMENT, "bad local rank index");
  int rc = hisa_cuda_dist_synchronize(d);
  if (rc != HISA_OK) return rc;
  Rank& r = d->ranks[size_t(local)];
  if (!r.out_idx || d->last_rows == 0) return dfail(d, HISA_ERR_INVALID_ARGUMENT, "no result yet");
  cudaSetDevice(r.device);
  const uint32_t k = d->cfg.token_budget;
  if (host_idx && cudaMemcpy(host_idx, r.out_idx, size_t(d->last_rows) * k * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    return dfail(d, HISA_ERR_CUDA, "copy of the index matrix failed");
  if (host_count && cudaMemcpy(host_count, r.out_count, size_t(d->last_rows) * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    return dfail(d, HISA_ERR_CUDA, "copy of the counts failed");
  return HISA_OK;
}

int hisa_cuda_dist_last_ms(hisa_cuda_dist* d, float* ms) {
  if (!d || !ms) return dfail(d, HISA_ERR_INVALID_ARGUMENT, "null argument");
  *ms = 0.f;
  if (!d->timed) return HISA_OK;
  int rc = hisa_cuda_dist_synchronize(d);
  if (rc != HISA_OK) return rc;
  for (Rank& r : d->ranks) {
    cudaSetDevice(r.device);
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.t_beg, r.t_end) == cudaSuccess) *ms = std::max(*ms, t);
    else cudaGetLastError();
  }
  return HISA_OK;
}

}  // extern "C"
