"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/_build/libhisa_oracle.so (the CPU restatement in oracle/hisa_oracle.cpp).
Importable only from tests/, bench.py's cpu_baseline / --impl reference legs and
__graft_entry__.smoke(); the product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libhisa_oracle.so")

ERR_NAMES = {
    0: "Ok", 1: "InfeasibleConfig", 2: "CausalViolation", 3: "EmptySequence", 4: "DimensionMismatch",
    5: "NonFiniteValue", 6: "ShapeMismatch", 7: "EmptySelection", 8: "InvalidArgument",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.name = ERR_NAMES.get(code, str(code))


def build(force: bool = False) -> str:
    """Compile the oracle library (and oracle/_ref when the reference tree is present)."""
    srcs = [os.path.join(_HERE, f) for f in ("hisa_oracle.cpp", "oracle_capi.cpp", "hisa_oracle.hpp")]
    stale = force or not os.path.exists(_LIB_PATH) or any(
        os.path.getmtime(s) > os.path.getmtime(_LIB_PATH) for s in srcs)
    if stale:
        subprocess.run(["make", "-C", _HERE, "all"], check=True, capture_output=True)
    return _LIB_PATH


class _Problem(C.Structure):
    _fields_ = [
        ("queries", C.c_void_p), ("gates", C.c_void_p), ("keys", C.c_void_p), ("positions", C.c_void_p),
        ("Q", C.c_uint32), ("L", C.c_uint32), ("H", C.c_uint32), ("d", C.c_uint32),
        ("block_size", C.c_uint32), ("block_budget", C.c_uint32), ("token_budget", C.c_uint32),
        ("force_first_last", C.c_uint8), ("forced_in_budget", C.c_uint8), ("tie_break", C.c_uint8),
        ("pool_mode", C.c_uint8), ("pool_tokens", C.c_uint32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.horacle_last_error.restype = C.c_char_p
        _lib.horacle_rng_new.restype = C.c_void_p
        _lib.horacle_rng_new.argtypes = [C.c_uint64]
        _lib.horacle_rng_free.argtypes = [C.c_void_p]
        for name, res in (("next_u64", C.c_uint64), ("uniform", C.c_double), ("normal", C.c_double)):
            f = getattr(_lib, "horacle_rng_" + name)
            f.restype = res
            f.argtypes = [C.c_void_p]
        _lib.horacle_rng_below.restype = C.c_uint64
        _lib.horacle_rng_below.argtypes = [C.c_void_p, C.c_uint64]
        _lib.horacle_splitmix64.restype = C.c_uint64
        _lib.horacle_splitmix64.argtypes = [C.c_uint64]
        _lib.horacle_mix_seed.restype = C.c_uint64
        _lib.horacle_mix_seed.argtypes = [C.c_uint64] * 4
        _lib.horacle_analytic_cost.restype = C.c_uint64
        _lib.horacle_analytic_cost.argtypes = [C.c_void_p, C.c_uint64, C.c_int]
        _lib.horacle_hardware_threads.restype = C.c_uint32
    return _lib


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().horacle_last_error().decode())


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Rng:
    """hisa-rng-v1 stream (reference: proj/core/include/hisa/rng.hpp:15-53)."""

    def __init__(self, seed: int):
        self._h = lib().horacle_rng_new(seed & 0xFFFFFFFFFFFFFFFF)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().horacle_rng_free(self._h)
            self._h = None

    def next_u64(self): return lib().horacle_rng_next_u64(self._h)
    def below(self, n): return lib().horacle_rng_below(self._h, n)
    def uniform(self): return lib().horacle_rng_uniform(self._h)
    def normal(self): return lib().horacle_rng_normal(self._h)


def splitmix64(x): return lib().horacle_splitmix64(x)
def mix_seed(a, b, c=0, d=0): return lib().horacle_mix_seed(a, b, c, d)
def hardware_threads(): return int(lib().horacle_hardware_threads())


def config_validate(B, m, k, H, d):
    _check(lib().horacle_config_validate(C.c_uint32(B), C.c_uint32(m), C.c_uint32(k), C.c_uint32(H), C.c_uint32(d)))


def make_positions(L, Q, placement="final"):
    out = np.empty(Q, dtype=np.uint32)
    _check(lib().horacle_make_positions(C.c_uint32(L), C.c_uint32(Q), C.c_int(0 if placement == "final" else 1), _p(out)))
    return out


@dataclass
class Problem:
    """Indexer inputs + config, all float32 row-major (inputs.hpp:20-56, config.hpp:26-67)."""
    queries: np.ndarray   # [Q, H, d]
    gates: np.ndarray     # [Q, H]
    keys: np.ndarray      # [L, d]
    positions: np.ndarray  # [Q] uint32
    block_size: int = 128
    block_budget: int = 64
    token_budget: int = 2048
    force_first_last: bool = True
    forced_in_budget: bool = False
    tie_break: int = 0   # 0 SmallestIndex, 1 LargestIndex
    pool_mode: int = 0   # 0 Mean, 1 Max
    pool_tokens: int = 0  # the block-summary cache covers the first pool_tokens keys (0 = all): decode snapshots

    def __post_init__(self):
        self.queries = np.ascontiguousarray(self.queries, dtype=np.float32)
        self.gates = np.ascontiguousarray(self.gates, dtype=np.float32)
        self.keys = np.ascontiguousarray(self.keys, dtype=np.float32)
        self.positions = np.ascontiguousarray(self.positions, dtype=np.uint32)
        assert self.queries.ndim == 3 and self.gates.ndim == 2 and self.keys.ndim == 2

    @property
    def Q(self): return int(self.positions.shape[0])
    @property
    def L(self): return int(self.keys.shape[0])
    @property
    def H(self): return int(self.queries.shape[1])
    @property
    def d(self): return int(self.queries.shape[2])

    def c_struct(self):
        s = _Problem()
        s.queries, s.gates = self.queries.ctypes.data, self.gates.ctypes.data
        s.keys, s.positions = self.keys.ctypes.data, self.positions.ctypes.data
        s.Q, s.L, s.H, s.d = self.Q, self.L, self.H, self.d
        s.block_size, s.block_budget, s.token_budget = self.block_size, self.block_budget, self.token_budget
        s.force_first_last, s.forced_in_budget = int(self.force_first_last), int(self.forced_in_budget)
        s.tie_break, s.pool_mode = self.tie_break, self.pool_mode
        s.pool_tokens = self.pool_tokens
        return s


def make_inputs(kind: str, seed: int, L: int, positions, H: int, d: int, **cfg) -> Problem:
    """kind: 'random' | 'lattice' | 'clustered' (synth.hpp:13-39). positions: uint32 array [Q]."""
    positions = np.ascontiguousarray(positions, dtype=np.uint32)
    Q = positions.shape[0]
    keys = np.empty((L, d), np.float32)
    queries = np.empty((Q, H, d), np.float32)
    gates = np.empty((Q, H), np.float32)
    pos_out = np.empty(Q, np.uint32)
    k = {"random": 0, "lattice": 1, "clustered": 2}[kind]
    _check(lib().horacle_make_inputs(C.c_int(k), C.c_uint64(seed), C.c_uint32(L), _p(positions), C.c_uint32(Q),
                                     C.c_uint32(H), C.c_uint32(d), _p(keys), _p(queries), _p(gates), _p(pos_out)))
    return Problem(queries, gates, keys, pos_out, **cfg)


def inputs_validate(p: Problem):
    s = p.c_struct()
    _check(lib().horacle_inputs_validate(C.byref(s)))


def analytic_cost(p: Problem, prefix_len: int, strategy: int) -> int:
    s = p.c_struct()
    return int(lib().horacle_analytic_cost(C.byref(s), C.c_uint64(prefix_len), C.c_int(strategy)))


def pool_build(keys: np.ndarray, B: int, mode: int = 0, incremental: bool = False):
    """-> (sums [M,d] f64, counts [M] u32, pooled [M,d] f64). block_summary.hpp:23-59."""
    keys = np.ascontiguousarray(keys, dtype=np.float32)
    L, d = keys.shape if keys.ndim == 2 else (0, 1)
    M = max(1, (L + B - 1) // B)
    sums = np.zeros((M, d), np.float64)
    counts = np.zeros(M, np.uint32)
    pooled = np.zeros((M, d), np.float64)
    nb = C.c_uint32(0)
    _check(lib().horacle_pool_build(_p(keys), C.c_uint64(L), C.c_uint32(d), C.c_uint32(B), C.c_int(mode),
                                    C.c_int(int(incremental)), _p(sums), _p(counts), _p(pooled), C.byref(nb)))
    return sums[:nb.value], counts[:nb.value], pooled[:nb.value]


def score_tokens(p: Problem, row: int, cand) -> tuple[np.ndarray, int]:
    cand = np.ascontiguousarray(cand, dtype=np.uint32)
    out = np.empty(cand.shape[0], np.float64)
    dots = C.c_uint64(0)
    s = p.c_struct()
    _check(lib().horacle_score_tokens(C.byref(s), C.c_uint32(row), _p(cand), C.c_uint64(cand.shape[0]), _p(out), C.byref(dots)))
    return out, dots.value


def top_k(scores, positions, k: int, tie_break: int = 0) -> np.ndarray:
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    positions = np.ascontiguousarray(positions, dtype=np.uint32)
    out = np.empty(max(1, min(k, scores.shape[0])), np.uint32)
    n = C.c_uint32(0)
    _check(lib().horacle_top_k(_p(scores), _p(positions), C.c_uint64(scores.shape[0]), C.c_uint32(k), C.c_int(tie_break),
                               _p(out), C.byref(n), None))
    return out[:n.value]


def score_blocks(p: Problem, row: int) -> np.ndarray:
    M = (p.L + p.block_size - 1) // p.block_size
    out = np.empty(max(M, 1), np.float64)
    n = C.c_uint32(0)
    s = p.c_struct()
    _check(lib().horacle_score_blocks(C.byref(s), C.c_uint32(row), _p(out), C.byref(n), None))
    return out[:n.value]


def score_pooled(p: Problem, row: int, pooled) -> np.ndarray:
    pooled = np.ascontiguousarray(pooled, dtype=np.float32)
    out = np.empty(pooled.shape[0], np.float64)
    n = C.c_uint32(0)
    s = p.c_struct()
    _check(lib().horacle_score_pooled(C.byref(s), C.c_uint32(row), _p(pooled), C.c_uint32(pooled.shape[0]), _p(out), C.byref(n)))
    return out[:n.value]


def select_blocks(scores, positions, p: Problem, t: int) -> np.ndarray:
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    positions = np.ascontiguousarray(positions, dtype=np.uint32)
    out = np.empty(scores.shape[0] + 2, np.uint32)
    n = C.c_uint32(0)
    s = p.c_struct()
    _check(lib().horacle_select_blocks(_p(scores), _p(positions), C.c_uint32(scores.shape[0]), C.byref(s), C.c_uint32(t), _p(out), C.byref(n)))
    return out[:n.value]


def candidate_union(blocks, B: int, t: int, L: int) -> np.ndarray:
    blocks = np.ascontiguousarray(blocks, dtype=np.uint32)
    out = np.empty(max(1, blocks.shape[0] * B), np.uint32)
    n = C.c_uint64(0)
    _check(lib().horacle_candidate_union(_p(blocks), C.c_uint32(blocks.shape[0]), C.c_uint32(B), C.c_uint32(t), C.c_uint32(L), _p(out), C.byref(n)))
    return out[:n.value]


STRATEGY = {"dsa": 0, "hisa": 1, "block": 2}


@dataclass
class BatchResult:
    idx: np.ndarray        # [n, stride] int32, -1 padded, ascending
    count: np.ndarray      # [n] uint32
    blocks: np.ndarray     # [n, m+2] int32, -1 padded
    nblocks: np.ndarray    # [n] uint32
    cand: np.ndarray       # [n] uint64 candidate_size
    dots: int


def select_batch(strategy: str, p: Problem, rows=None, threads: int = 0, idx_stride: int | None = None) -> BatchResult:
    """dsa_select / hisa_select / block_sparse_select over `rows` (default all), fanned out over threads."""
    if rows is None:
        rows = np.arange(p.Q, dtype=np.uint32)
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    n = rows.shape[0]
    if idx_stride is None:
        idx_stride = p.token_budget if strategy != "block" else (p.block_budget + 2) * p.block_size
    idx = np.empty((n, idx_stride), np.int32)
    count = np.empty(n, np.uint32)
    blocks = np.empty((n, p.block_budget + 2), np.int32)
    nblocks = np.empty(n, np.uint32)
    cand = np.empty(n, np.uint64)
    dots = C.c_uint64(0)
    s = p.c_struct()
    threads = threads or hardware_threads()
    _check(lib().horacle_select_batch(C.c_int(STRATEGY[strategy]), C.byref(s), _p(rows), C.c_uint32(n), C.c_uint32(threads),
                                      _p(idx), C.c_uint32(idx_stride), _p(count), _p(blocks), _p(nblocks), _p(cand),
                                      C.byref(dots)))
    return BatchResult(idx, count, blocks, nblocks, cand, dots.value)


def trace_row(strategy: str, p: Problem, row: int):
    """-> dict(J, blocks, omega, omega_scores) for one row (near-tie analysis in the parity tests)."""
    M = (p.L + p.block_size - 1) // p.block_size
    J = np.empty(max(M, 1), np.float64)
    blocks = np.empty(p.block_budget + 2, np.uint32)
    cap = p.L if strategy == "dsa" else min(p.L, (p.block_budget + 2) * p.block_size)
    omega = np.empty(max(cap, 1), np.uint32)
    scores = np.empty(max(cap, 1), np.float64)
    nJ, nb, no = C.c_uint32(0), C.c_uint32(0), C.c_uint64(0)
    s = p.c_struct()
    _check(lib().horacle_trace_row(C.c_int(STRATEGY[strategy]), C.byref(s), C.c_uint32(row), _p(J), C.byref(nJ), _p(blocks),
                                   C.byref(nb), _p(omega), _p(scores), C.byref(no)))
    return {"J": J[:nJ.value], "blocks": blocks[:nb.value], "omega": omega[:no.value], "omega_scores": scores[:no.value]}


def attend_batch(query_states, latent_states, positions, selected=None, counts=None, rows=None, scale: float = 0.0,
                 threads: int = 0, want_weights: bool = False):
    """sparse_attend (selected int32 [n, stride] -1 padded + counts [n]) or dense_attend (selected=None) for the
    query rows `rows` (default all). attention.hpp:48-59. -> out f32 [n, d_model] (, weights f64 [n, stride])."""
    qs = np.ascontiguousarray(query_states, dtype=np.float32)
    ls = np.ascontiguousarray(latent_states, dtype=np.float32)
    pos = np.ascontiguousarray(positions, dtype=np.uint32)
    Q, dm = qs.shape
    L = ls.shape[0]
    if rows is None:
        rows = np.arange(Q, dtype=np.uint32)
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    n = rows.shape[0]
    out = np.zeros((n, dm), np.float32)
    weights = None
    stride = 0
    if selected is not None:
        selected = np.ascontiguousarray(selected, dtype=np.int32)
        counts = np.ascontiguousarray(counts, dtype=np.uint32)
        assert selected.shape[0] == n and counts.shape[0] == n
        stride = selected.shape[1]
        if want_weights:
            weights = np.zeros((n, stride), np.float64)
    _check(lib().horacle_attend_batch(_p(qs), _p(ls), _p(pos), C.c_uint32(Q), C.c_uint32(L), C.c_uint32(dm),
                                      C.c_double(scale), _p(rows), C.c_uint32(n), _p(selected), C.c_uint32(stride),
                                      _p(counts), C.c_uint32(threads), _p(out), _p(weights)))
    return (out, weights) if want_weights else out
