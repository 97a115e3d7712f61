"""ctypes binding of the C ABI in include/hisa_cuda.h (libhisa_b200.so).

This is host-side plumbing for the Python callers in this repo (tests, bench.py): it binds exactly the
symbols a cgo/JNI/N-API stub would and adds no arithmetic. There is no CPU fallback:
if the library is missing, or no sm_100 device is present, everything here raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libhisa_b200.so")

DTYPE_F32, DTYPE_BF16, DTYPE_FP8 = 0, 1, 2
SCORER_TENSOR, SCORER_SIMT = 0, 1

# every symbol include/hisa_cuda.h declares
EXPORTED_SYMBOLS = [
    "hisa_cuda_upload_keys_scaled", "hisa_cuda_pool_append_scaled", "hisa_cuda_pool_set",
    "hisa_cuda_set_output_placement", "hisa_cuda_dist_plan", "hisa_cuda_dist_create", "hisa_cuda_dist_unique_id",
    "hisa_cuda_dist_create_rank", "hisa_cuda_dist_destroy", "hisa_cuda_dist_last_error", "hisa_cuda_dist_info",
    "hisa_cuda_dist_ctx", "hisa_cuda_dist_upload_keys", "hisa_cuda_dist_select", "hisa_cuda_dist_synchronize",
    "hisa_cuda_dist_result", "hisa_cuda_dist_fetch", "hisa_cuda_dist_last_ms",
    "hisa_cuda_config_init", "hisa_cuda_config_validate", "hisa_cuda_abi_version", "hisa_cuda_status_name",
    "hisa_cuda_last_error", "hisa_cuda_device_count", "hisa_cuda_create", "hisa_cuda_destroy",
    "hisa_cuda_synchronize", "hisa_cuda_stream", "hisa_cuda_host_alloc", "hisa_cuda_host_free",
    "hisa_cuda_device_alloc", "hisa_cuda_device_free", "hisa_cuda_memcpy", "hisa_cuda_upload_keys",
    "hisa_cuda_pool_build", "hisa_cuda_pool_append", "hisa_cuda_pool_read", "hisa_cuda_seq_len",
    "hisa_cuda_hisa_select", "hisa_cuda_dsa_select", "hisa_cuda_block_sparse_select", "hisa_cuda_score_blocks",
    "hisa_cuda_select_blocks", "hisa_cuda_score_tokens", "hisa_cuda_top_k", "hisa_cuda_set_profiling",
    "hisa_cuda_last_stage_times", "hisa_cuda_launch_count", "hisa_cuda_scorer_stall_cycles",
    "hisa_cuda_attn_set_latents", "hisa_cuda_sparse_attend", "hisa_cuda_dense_attend", "hisa_cuda_attn_last_ms",
]


class HisaError(RuntimeError):
    """Mirror of the reference's exception leaves (hisa/errors.hpp:10-28), keyed by the status name."""

    def __init__(self, code: int, name: str, msg: str):
        super().__init__(f"{name}: {msg}")
        self.code, self.name = code, name


class Config(C.Structure):
    _fields_ = [
        ("block_size", C.c_uint32), ("block_budget", C.c_uint32), ("token_budget", C.c_uint32),
        ("num_heads", C.c_uint32), ("dim", C.c_uint32),
        ("force_first_last", C.c_uint8), ("forced_in_budget", C.c_uint8), ("tie_break", C.c_uint8),
        ("pool_mode", C.c_uint8),
        ("dtype", C.c_uint32), ("scorer", C.c_uint32), ("reserved", C.c_uint32 * 4),
    ]


class StageTimes(C.Structure):
    _fields_ = [
        ("prepare_ms", C.c_float), ("score_blocks_ms", C.c_float), ("select_blocks_ms", C.c_float),
        ("invert_ms", C.c_float), ("score_tokens_ms", C.c_float), ("top_k_ms", C.c_float), ("total_ms", C.c_float),
        ("launches", C.c_uint64), ("work_items_stage1", C.c_uint64), ("work_items_stage2", C.c_uint64),
        ("calls", C.c_uint64),
    ]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def build(force: bool = False) -> str:
    """Compile the sm_100a library in-tree with nvcc (cross-compiles without a GPU)."""
    src_dir = os.path.join(_HERE, "csrc")
    srcs = [os.path.join(src_dir, f) for f in os.listdir(src_dir) if f.endswith((".cu", ".cuh", "Makefile"))]
    srcs.append(os.path.join(_HERE, "..", "include", "hisa_cuda.h"))
    stale = force or not os.path.exists(LIB_PATH) or any(os.path.getmtime(s) > os.path.getmtime(LIB_PATH) for s in srcs)
    if stale:
        r = subprocess.run(["make", "-C", src_dir, "-j8"], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("building libhisa_b200.so failed:\n" + r.stdout[-4000:] + r.stderr[-4000:])
    return LIB_PATH


_lib = None


def lib():
    """Loads libhisa_b200.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                               "(the product path has no CPU fallback)")
        _lib = C.CDLL(LIB_PATH)
        _lib.hisa_cuda_last_error.restype = C.c_char_p
        _lib.hisa_cuda_last_error.argtypes = [C.c_void_p]
        _lib.hisa_cuda_status_name.restype = C.c_char_p
        _lib.hisa_cuda_stream.restype = C.c_void_p
        _lib.hisa_cuda_stream.argtypes = [C.c_void_p]
        _lib.hisa_cuda_dist_last_error.restype = C.c_char_p
        _lib.hisa_cuda_dist_last_error.argtypes = [C.c_void_p]
        _lib.hisa_cuda_dist_ctx.restype = C.c_void_p
        _lib.hisa_cuda_dist_ctx.argtypes = [C.c_void_p, C.c_int]
    return _lib


def _check(rc: int, ctx=None):
    if rc != 0:
        L = lib()
        msg = L.hisa_cuda_last_error(ctx).decode(errors="replace")
        raise HisaError(rc, L.hisa_cuda_status_name(rc).decode(), msg)


def device_count() -> int:
    n = C.c_int(0)
    rc = lib().hisa_cuda_device_count(C.byref(n))
    return n.value if rc == 0 else 0


def make_config(block_size=128, block_budget=64, token_budget=2048, num_heads=64, dim=128, dtype=DTYPE_BF16,
                force_first_last=True, forced_in_budget=False, tie_break=0, pool_mode=0, scorer=SCORER_TENSOR) -> Config:
    cfg = Config()
    lib().hisa_cuda_config_init(C.byref(cfg), block_size, block_budget, token_budget, num_heads, dim, dtype)
    cfg.force_first_last, cfg.forced_in_budget = int(force_first_last), int(forced_in_budget)
    cfg.tie_break, cfg.pool_mode, cfg.scorer = tie_break, pool_mode, scorer
    return cfg


def config_validate(cfg: Config):
    _check(lib().hisa_cuda_config_validate(C.byref(cfg)))


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 bit patterns (uint16), round-to-nearest-even. Host-side data plumbing."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + r) >> 16).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


_E4M3_TABLE = None


def e4m3_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """e4m3 (fn: no infinities, S.1111.111 = NaN) bytes -> float32, exactly."""
    global _E4M3_TABLE
    if _E4M3_TABLE is None:
        t = np.zeros(256, np.float32)
        for v in range(256):
            s, e, m = v >> 7, (v >> 3) & 15, v & 7
            if e == 15 and m == 7:
                x = np.nan
            elif e == 0:
                x = m * 2.0 ** -9
            else:
                x = (1 + m / 8.0) * 2.0 ** (e - 7)
            t[v] = -x if s else x
        _E4M3_TABLE = t
    return _E4M3_TABLE[np.ascontiguousarray(b, dtype=np.uint8)]


def f32_to_e4m3_bits(a: np.ndarray) -> np.ndarray:
    """float32 -> e4m3 bytes, round-to-nearest-even, saturating at +-448. Host-side data plumbing."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    mag = np.minimum(np.abs(a).astype(np.float64), 448.0)
    e = np.floor(np.log2(np.maximum(mag, 2.0 ** -20)))
    e = np.clip(e, -6, 8)                     # exponent of the binade (subnormals share 2^-6)
    step = 2.0 ** (e - 3)                     # spacing of representable values in that binade
    q = np.rint(mag / step) * step            # np.rint rounds half to even; a carry lands on the next binade exactly
    q = np.minimum(q, 448.0)
    ee = np.floor(np.log2(np.maximum(q, 2.0 ** -20)))
    sub = q < 2.0 ** -6
    exp_field = np.where(sub, 0, ee + 7).astype(np.int64)
    man_field = np.where(sub, np.rint(q * 2.0 ** 9), np.rint((q / 2.0 ** ee - 1.0) * 8)).astype(np.int64)
    bits = (exp_field << 3) | man_field
    bits = np.where(q == 0, 0, bits)
    return (bits | (np.signbit(a).astype(np.int64) << 7)).astype(np.uint8)


def quantize_e4m3(a: np.ndarray, axis=-1):
    """Per-row symmetric quantisation: returns (e4m3 bytes, float32 scales) with a ~= float(bytes) * scale."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    amax = np.abs(a).max(axis=axis, keepdims=True)
    scale = np.where(amax > 0, amax / np.float32(448.0), np.float32(1.0)).astype(np.float32)
    return f32_to_e4m3_bits(a / scale), np.squeeze(scale, axis=axis)


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    return C.c_void_p(int(a))  # raw device/host address


class Indexer:
    """One context = one GPU + one stream. Thin wrapper over hisa_cuda_*; arrays are numpy (host) or raw
    integer device addresses."""

    def __init__(self, cfg: Config, device: int = 0):
        self.cfg = cfg
        self._owned = True
        self._ctx = C.c_void_p(None)
        _check(lib().hisa_cuda_create(C.c_int(device), C.byref(cfg), C.byref(self._ctx)))

    @classmethod
    def borrow(cls, ctx, cfg: Config):
        """Wraps a context somebody else owns (a rank of a Dist driver): same methods, close() leaves it alive."""
        self = cls.__new__(cls)
        self.cfg, self._ctx, self._owned = cfg, ctx, False
        return self

    def close(self):
        if self._ctx and self._owned:
            lib().hisa_cuda_destroy(self._ctx)
        self._ctx = C.c_void_p(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self): return self
    def __exit__(self, *a): self.close()

    # -- helpers
    @property
    def S(self): return self.cfg.block_budget + 2
    @property
    def k(self): return self.cfg.token_budget

    def _elems(self, a):
        """numpy array in the context dtype: f32 arrays stay f32 for DTYPE_F32, uint16 bf16 bits for DTYPE_BF16."""
        if not isinstance(a, np.ndarray):
            return a
        if self.cfg.dtype == DTYPE_BF16:
            return np.ascontiguousarray(a if a.dtype == np.uint16 else f32_to_bf16_bits(a))
        if self.cfg.dtype == DTYPE_FP8:
            if a.dtype != np.uint8:
                raise TypeError("fp8 storage takes e4m3 bytes (uint8); quantise with capi.quantize_e4m3")
            return np.ascontiguousarray(a)
        return np.ascontiguousarray(a, dtype=np.float32)

    def synchronize(self): _check(lib().hisa_cuda_synchronize(self._ctx), self._ctx)
    def set_profiling(self, on, stall_stats: bool = False):
        """on: CUDA events per stage; stall_stats: also run the instrumented scorer (slower by a few percent)."""
        _check(lib().hisa_cuda_set_profiling(self._ctx, C.c_int((1 if on else 0) | (2 if (on and stall_stats) else 0))), self._ctx)

    def stage_times(self) -> dict:
        st = StageTimes()
        _check(lib().hisa_cuda_last_stage_times(self._ctx, C.byref(st)), self._ctx)
        return st.as_dict()

    STALL_NAMES = ["cta", "prod_wait_sched", "prod_wait_tilebuf", "prod_wait_qstage", "mma_wait_qdata", "mma_wait_tile",
                   "mma_wait_epilogue", "mma_wait_gates", "cta_max", "epi_busy", "groups"]

    def scorer_stall_cycles(self) -> dict:
        a, b = (C.c_uint64 * 16)(), (C.c_uint64 * 16)()
        _check(lib().hisa_cuda_scorer_stall_cycles(self._ctx, a, b), self._ctx)
        return {"stage1": dict(zip(self.STALL_NAMES, list(a))), "stage2": dict(zip(self.STALL_NAMES, list(b)))}

    def launch_count(self) -> int:
        n = C.c_uint64(0)
        _check(lib().hisa_cuda_launch_count(self._ctx, C.byref(n)), self._ctx)
        return n.value

    def device_alloc(self, nbytes: int) -> int:
        p = C.c_void_p(None)
        _check(lib().hisa_cuda_device_alloc(self._ctx, C.byref(p), C.c_size_t(nbytes)), self._ctx)
        return p.value

    def device_free(self, addr: int): _check(lib().hisa_cuda_device_free(self._ctx, C.c_void_p(addr)), self._ctx)

    def memcpy(self, dst, src, nbytes: int):
        _check(lib().hisa_cuda_memcpy(self._ctx, _ptr(dst), _ptr(src), C.c_size_t(nbytes)), self._ctx)

    # -- keys / summaries
    def upload_keys(self, keys, seq_len=None, check_finite=False, scales=None):
        keys = self._elems(keys)
        L = keys.shape[0] if seq_len is None else seq_len
        if scales is not None:
            if isinstance(scales, np.ndarray):
                scales = np.ascontiguousarray(scales, dtype=np.float32)
            _check(lib().hisa_cuda_upload_keys_scaled(self._ctx, _ptr(keys), _ptr(scales), C.c_uint64(L),
                                                      C.c_int(int(check_finite))), self._ctx)
            return
        _check(lib().hisa_cuda_upload_keys(self._ctx, _ptr(keys), C.c_uint64(L), C.c_int(int(check_finite))), self._ctx)

    def pool_build(self): _check(lib().hisa_cuda_pool_build(self._ctx), self._ctx)

    def pool_set(self, sums, counts, num_tokens):
        """Installs caller-provided block summaries (BlockSummaryCache contents; may cover fewer tokens than the keys)."""
        sums = np.ascontiguousarray(sums, dtype=np.float64)
        counts = np.ascontiguousarray(counts, dtype=np.uint32)
        _check(lib().hisa_cuda_pool_set(self._ctx, _ptr(sums), _ptr(counts), C.c_uint64(counts.shape[0]),
                                        C.c_uint64(num_tokens)), self._ctx)

    def pool_append(self, keys, n=None, key_dim=None, scales=None):
        keys = self._elems(keys)
        if isinstance(keys, np.ndarray):
            keys2 = keys.reshape(-1, keys.shape[-1])
            n = keys2.shape[0] if n is None else n
            key_dim = keys2.shape[1] if key_dim is None else key_dim
        if scales is not None:
            if isinstance(scales, np.ndarray):
                scales = np.ascontiguousarray(scales, dtype=np.float32)
            _check(lib().hisa_cuda_pool_append_scaled(self._ctx, _ptr(keys), _ptr(scales), C.c_uint64(n),
                                                      C.c_uint32(key_dim)), self._ctx)
            return
        _check(lib().hisa_cuda_pool_append(self._ctx, _ptr(keys), C.c_uint64(n), C.c_uint32(key_dim)), self._ctx)

    def seq_len(self):
        L, M = C.c_uint64(0), C.c_uint64(0)
        _check(lib().hisa_cuda_seq_len(self._ctx, C.byref(L), C.byref(M)), self._ctx)
        return L.value, M.value

    def pool_read(self, num_blocks=None):
        """num_blocks: blocks the current summaries cover when they were installed with pool_set (default: all key blocks)"""
        L, M = self.seq_len()
        M = M if num_blocks is None else num_blocks
        d = self.cfg.dim
        sums, pooled, counts = np.empty((M, d)), np.empty((M, d)), np.empty(M, np.uint32)
        _check(lib().hisa_cuda_pool_read(self._ctx, _ptr(sums), _ptr(counts), _ptr(pooled)), self._ctx)
        return sums, counts, pooled

    # -- batched selection (host numpy in, host numpy out)
    def _select(self, which: str, queries, gates, positions, check_finite=False):
        q = self._elems(queries)
        w = np.ascontiguousarray(gates, dtype=np.float32)
        pos = np.ascontiguousarray(positions, dtype=np.uint32)
        Q = pos.shape[0]
        width = self.S * self.cfg.block_size if which == "block" else self.k
        idx = np.empty((Q, width), np.int32)
        count = np.empty(Q, np.uint32)
        blocks = np.full((Q, self.S), -1, np.int32)
        nblocks = np.zeros(Q, np.uint32)
        cand = np.zeros(Q, np.uint32)
        L = lib()
        if which == "hisa":
            rc = L.hisa_cuda_hisa_select(self._ctx, _ptr(q), _ptr(w), _ptr(pos), C.c_uint64(Q), C.c_int(int(check_finite)),
                                         _ptr(idx), _ptr(count), _ptr(blocks), _ptr(nblocks), _ptr(cand))
        elif which == "dsa":
            rc = L.hisa_cuda_dsa_select(self._ctx, _ptr(q), _ptr(w), _ptr(pos), C.c_uint64(Q), C.c_int(int(check_finite)),
                                        _ptr(idx), _ptr(count), _ptr(cand))
        else:
            rc = L.hisa_cuda_block_sparse_select(self._ctx, _ptr(q), _ptr(w), _ptr(pos), C.c_uint64(Q),
                                                 C.c_int(int(check_finite)), _ptr(idx), _ptr(count), _ptr(blocks), _ptr(nblocks))
        _check(rc, self._ctx)
        return {"idx": idx, "count": count, "blocks": blocks, "nblocks": nblocks, "cand": cand}

    def hisa_select(self, queries, gates, positions, **kw): return self._select("hisa", queries, gates, positions, **kw)
    def dsa_select(self, queries, gates, positions, **kw): return self._select("dsa", queries, gates, positions, **kw)
    def block_sparse_select(self, queries, gates, positions, **kw): return self._select("block", queries, gates, positions, **kw)

    # -- raw-pointer selection (device or pinned-host addresses; nothing is allocated or copied here)
    def hisa_select_raw(self, q, w, pos, Q, out_idx, out_count=None, out_blocks=None, out_nblocks=None, out_cand=None,
                        check_finite=False):
        _check(lib().hisa_cuda_hisa_select(self._ctx, _ptr(q), _ptr(w), _ptr(pos), C.c_uint64(Q), C.c_int(int(check_finite)),
                                           _ptr(out_idx), _ptr(out_count), _ptr(out_blocks), _ptr(out_nblocks),
                                           _ptr(out_cand)), self._ctx)

    def dsa_select_raw(self, q, w, pos, Q, out_idx, out_count=None, out_cand=None, check_finite=False):
        _check(lib().hisa_cuda_dsa_select(self._ctx, _ptr(q), _ptr(w), _ptr(pos), C.c_uint64(Q), C.c_int(int(check_finite)),
                                          _ptr(out_idx), _ptr(out_count), _ptr(out_cand)), self._ctx)

    # -- single stages
    def score_blocks(self, queries, gates, positions):
        q = self._elems(queries)
        w = np.ascontiguousarray(gates, dtype=np.float32)
        pos = np.ascontiguousarray(positions, dtype=np.uint32)
        Q = pos.shape[0]
        _, M = self.seq_len()
        out = np.zeros((Q, max(M, 1)), np.float32)
        ne = np.zeros(Q, np.uint32)
        _check(lib().hisa_cuda_score_blocks(self._ctx, _ptr(q), _ptr(w), _ptr(pos), C.c_uint64(Q), _ptr(out), _ptr(ne)), self._ctx)
        return out, ne

    def select_blocks(self, scores, neligible):
        scores = np.ascontiguousarray(scores, dtype=np.float32)
        ne = np.ascontiguousarray(neligible, dtype=np.uint32)
        Q = ne.shape[0]
        blocks = np.empty((Q, self.S), np.int32)
        nb = np.empty(Q, np.uint32)
        _check(lib().hisa_cuda_select_blocks(self._ctx, _ptr(scores), C.c_uint64(scores.shape[1]), _ptr(ne), C.c_uint64(Q),
                                             _ptr(blocks), _ptr(nb)), self._ctx)
        return blocks, nb

    def score_tokens(self, queries, gates, positions):
        q = self._elems(queries)
        w = np.ascontiguousarray(gates, dtype=np.float32)
        pos = np.ascontiguousarray(positions, dtype=np.uint32)
        Q = pos.shape[0]
        L, _ = self.seq_len()
        stride = (L + 127) // 128 * 128
        out = np.zeros((Q, stride), np.float32)
        _check(lib().hisa_cuda_score_tokens(self._ctx, _ptr(q), _ptr(w), _ptr(pos), C.c_uint64(Q), _ptr(out), C.c_uint64(stride)), self._ctx)
        return out

    def top_k(self, scores, n, k):
        scores = np.ascontiguousarray(scores, dtype=np.float32)
        n = np.ascontiguousarray(n, dtype=np.uint32)
        rows = n.shape[0]
        idx = np.empty((rows, k), np.int32)
        cnt = np.empty(rows, np.uint32)
        _check(lib().hisa_cuda_top_k(self._ctx, _ptr(scores), C.c_uint64(scores.shape[1]), _ptr(n), C.c_uint64(rows), C.c_uint32(k),
                                     _ptr(idx), _ptr(cnt)), self._ctx)
        return idx, cnt

    # -- downstream consumer (attention.hpp:13-59)
    @staticmethod
    def _attn_elems(a):
        """numpy -> (array, dtype code): uint16 arrays are bf16 bit patterns, everything else becomes float32."""
        if isinstance(a, np.ndarray) and a.dtype == np.uint16:
            return np.ascontiguousarray(a), DTYPE_BF16
        return np.ascontiguousarray(a, dtype=np.float32), DTYPE_F32

    def attn_set_latents(self, latent_states, check_finite=False):
        lat, dt = self._attn_elems(latent_states)
        L, dm = lat.shape
        _check(lib().hisa_cuda_attn_set_latents(self._ctx, _ptr(lat), C.c_uint64(L), C.c_uint32(dm), C.c_uint32(dt),
                                                C.c_int(int(check_finite))), self._ctx)
        self._attn_dm = dm

    def sparse_attend(self, query_states, positions, selected, counts=None, scale=0.0, want_weights=False):
        qs, dt = self._attn_elems(query_states)
        pos = np.ascontiguousarray(positions, dtype=np.uint32)
        sel = np.ascontiguousarray(selected, dtype=np.int32).reshape(pos.shape[0], -1)
        cnt = None if counts is None else np.ascontiguousarray(counts, dtype=np.uint32)
        Q = pos.shape[0]
        out = np.zeros((Q, self._attn_dm), np.float32)
        weights = np.zeros(sel.shape, np.float32) if want_weights else None
        _check(lib().hisa_cuda_sparse_attend(self._ctx, _ptr(qs), C.c_uint32(dt), _ptr(pos), C.c_uint64(Q), _ptr(sel),
                                             C.c_uint64(sel.shape[1]), _ptr(cnt), C.c_double(scale), _ptr(out),
                                             _ptr(weights)), self._ctx)
        return (out, weights) if want_weights else out

    def dense_attend(self, query_states, positions, scale=0.0):
        qs, dt = self._attn_elems(query_states)
        pos = np.ascontiguousarray(positions, dtype=np.uint32)
        Q = pos.shape[0]
        out = np.zeros((Q, self._attn_dm), np.float32)
        _check(lib().hisa_cuda_dense_attend(self._ctx, _ptr(qs), C.c_uint32(dt), _ptr(pos), C.c_uint64(Q), C.c_double(scale),
                                            _ptr(out)), self._ctx)
        return out

    def sparse_attend_raw(self, q, q_dtype, pos, Q, selected, sel_stride, counts, out, scale=0.0, weights=None):
        """device / pinned-host addresses only; nothing is allocated or copied here"""
        _check(lib().hisa_cuda_sparse_attend(self._ctx, _ptr(q), C.c_uint32(q_dtype), _ptr(pos), C.c_uint64(Q), _ptr(selected),
                                             C.c_uint64(sel_stride), _ptr(counts), C.c_double(scale), _ptr(out),
                                             _ptr(weights)), self._ctx)

    def attn_last_ms(self) -> float:
        ms = C.c_float(0.0)
        _check(lib().hisa_cuda_attn_last_ms(self._ctx, C.byref(ms)), self._ctx)
        return ms.value


# ---- multi-GPU driver (hisa_cuda_dist_*) ----------------------------------------------------------------------------
DIST_DSA, DIST_HISA = 0, 1
GATHER_AUTO, GATHER_NCCL, GATHER_PEER = 0, 1, 2
DIST_TILE_ROWS = 512


def _dist_check(rc: int, dist=None):
    if rc != 0:
        L = lib()
        msg = L.hisa_cuda_dist_last_error(dist).decode(errors="replace")
        raise HisaError(rc, L.hisa_cuda_status_name(rc).decode(), msg)


def dist_plan(num_rows: int, world: int, rank: int) -> np.ndarray:
    """Rows rank `rank` of `world` owns (ascending): the C library's own sharding arithmetic, no device needed."""
    n = C.c_uint64(0)
    _dist_check(lib().hisa_cuda_dist_plan(C.c_uint64(num_rows), C.c_int(world), C.c_int(rank), C.byref(n), None))
    rows = np.empty(n.value, np.uint32)
    _dist_check(lib().hisa_cuda_dist_plan(C.c_uint64(num_rows), C.c_int(world), C.c_int(rank), C.byref(n), _ptr(rows)))
    return rows


def dist_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _dist_check(lib().hisa_cuda_dist_unique_id(buf, C.c_size_t(128)))
    return bytes(buf)


class Dist:
    """hisa_cuda_dist: query rows sharded over GPUs. Dist(cfg, devices=[...]) drives all GPUs from this process;
    Dist(cfg, rank=r, world=w, device=d, unique_id=...) is one rank of a multi-process job."""

    def __init__(self, cfg: Config, devices=None, gather=GATHER_AUTO, rank=None, world=None, device=None, unique_id=None):
        self.cfg = cfg
        self._d = C.c_void_p(None)
        if devices is not None:
            arr = (C.c_int * len(devices))(*devices)
            _dist_check(lib().hisa_cuda_dist_create(arr, C.c_int(len(devices)), C.byref(cfg), C.c_uint32(gather), C.byref(self._d)))
        else:
            idbuf = (C.c_uint8 * 128)(*unique_id)
            _dist_check(lib().hisa_cuda_dist_create_rank(idbuf, C.c_int(world), C.c_int(rank), C.c_int(device), C.byref(cfg),
                                                         C.c_uint32(gather), C.byref(self._d)))
        w, nl, fr, g = C.c_int(0), C.c_int(0), C.c_int(0), C.c_int(0)
        _dist_check(lib().hisa_cuda_dist_info(self._d, C.byref(w), C.byref(nl), C.byref(fr), C.byref(g)), self._d)
        self.world, self.num_local, self.first_rank, self.gather = w.value, nl.value, fr.value, g.value

    def close(self):
        if self._d:
            lib().hisa_cuda_dist_destroy(self._d)
            self._d = C.c_void_p(None)

    def __enter__(self): return self
    def __exit__(self, *a): self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def ctx(self, local: int):
        return C.c_void_p(lib().hisa_cuda_dist_ctx(self._d, C.c_int(local)))

    def upload_keys(self, keys, seq_len, scales=None, root=0):
        _dist_check(lib().hisa_cuda_dist_upload_keys(self._d, _ptr(keys), _ptr(scales), C.c_uint64(seq_len), C.c_int(root)), self._d)

    def select(self, strategy, queries, gates, positions, total_rows, num_slices=4):
        """queries / gates / positions: one entry per LOCAL rank (numpy arrays = host memory, ints = device addresses)"""
        n = self.num_local
        qs = (C.c_void_p * n)(*[_ptr(q) for q in queries])
        ws = (C.c_void_p * n)(*[_ptr(w) for w in gates])
        ps = (C.c_void_p * n)(*[_ptr(p) for p in positions])
        _dist_check(lib().hisa_cuda_dist_select(self._d, C.c_int(strategy), qs, ws, ps, C.c_uint64(total_rows), C.c_int(num_slices)), self._d)

    def synchronize(self): _dist_check(lib().hisa_cuda_dist_synchronize(self._d), self._d)

    def result_ptrs(self, local=0):
        i, c = C.c_void_p(None), C.c_void_p(None)
        _dist_check(lib().hisa_cuda_dist_result(self._d, C.c_int(local), C.byref(i), C.byref(c)), self._d)
        return i.value, c.value

    def fetch(self, total_rows, local=0):
        idx = np.empty((total_rows, self.cfg.token_budget), np.int32)
        cnt = np.empty(total_rows, np.uint32)
        _dist_check(lib().hisa_cuda_dist_fetch(self._d, C.c_int(local), _ptr(idx), _ptr(cnt)), self._d)
        return idx, cnt

    def fetch_into(self, idx_addr, count_addr=None, local=0):
        """like fetch, into caller memory (pinned host addresses make the copy run at link speed)"""
        _dist_check(lib().hisa_cuda_dist_fetch(self._d, C.c_int(local), _ptr(idx_addr), _ptr(count_addr)), self._d)

    def last_ms(self) -> float:
        ms = C.c_float(0.0)
        _dist_check(lib().hisa_cuda_dist_last_ms(self._d, C.byref(ms)), self._d)
        return ms.value


def host_alloc(nbytes: int) -> int:
    p = C.c_void_p(None)
    _check(lib().hisa_cuda_host_alloc(C.byref(p), C.c_size_t(nbytes)))
    return p.value


def host_free(addr: int):
    lib().hisa_cuda_host_free(C.c_void_p(addr))


def host_array(addr: int, shape, dtype) -> np.ndarray:
    """numpy view over pinned host memory returned by host_alloc."""
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    buf = (C.c_uint8 * n).from_address(addr)
    return np.frombuffer(buf, dtype=dtype).reshape(shape)
