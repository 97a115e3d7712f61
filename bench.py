#!/usr/bin/env python
"""bench.py — HISA hierarchical indexer throughput on B200 (metric of BASELINE.json).

    python bench.py --gpus N --steps K --warmup W            # this repo's CUDA path
    python bench.py --impl reference --gpus N --steps K ...  # the reference's CPU path (the oracle port)

A "step" is one pass of the hot path over one batch of synthetic input: hisa_select for ALL query rows of
the headline workload (C3: L=Q=65536, H=64, d=128, B=128, m=64, k=2048, bf16 q/k), inputs resident in HBM.
Prints ONE JSON line (rank 0). See DESIGN.md §7 for how each field is measured.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "indexer queries/sec (HISA hierarchical top-k, full causal prefill)"
UNIT = "queries/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--seq-len", type=int, default=65536)
    ap.add_argument("--block-size", type=int, default=128)
    ap.add_argument("--block-budget", type=int, default=64)
    ap.add_argument("--token-budget", type=int, default=2048)
    ap.add_argument("--flat-steps", type=int, default=2, help="timed steps of the flat DSA comparison (0 = skip)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--attend-steps", type=int, default=2,
                    help="timed runs of the downstream consumer (sparse_attend over the selected indices; 0 = skip)")
    ap.add_argument("--d-model", type=int, default=128, help="latent width of the downstream consumer")
    ap.add_argument("--cpu-rows", type=int, default=768, help="rows of the workload the CPU baseline is timed on")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--force-dist", action="store_true",
                    help="use the multi-GPU driver (hisa_cuda_dist_*, NCCL communicator) even with one rank")
    ap.add_argument("--no-configs", action="store_true", help="skip the array of the other BASELINE configurations")
    ap.add_argument("--configs-only", default="", help="comma list of configuration ids to time (default: all)")
    ap.add_argument("--slices", type=int, default=0, help="slices per rank of the sharded step (0 = 4, or 2 for short ranks)")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp8"],
                    help="storage of q/k: bf16 (headline) or e4m3 with per-token key scales (query scales folded into the gates)")
    return ap.parse_args()


def workload_name(a):
    store = "bf16 q/k" if a.dtype == "bf16" else "e4m3 q/k + f32 per-key scales"
    return (f"C3 prefill L=Q={a.seq_len} H=64 d=128 B={a.block_size} m={a.block_budget} k={a.token_budget} "
            f"{store}, fp32 gates, hisa_select")


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        p = json.load(open(path))
        return {"tflops": float(p.get("bf16_tflops_sustained", p.get("bf16_tflops", 1400.0))),
                "tflops_burst": float(p.get("bf16_tflops", 0.0)) or None,
                "hbm_gbs": float(p.get("hbm_gbs", 6650.0)), "source": "measured (MEASURED_PEAKS.json, sustained bf16)"}
    return {"tflops": 1400.0, "tflops_burst": None, "hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ------------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML while the timed region runs."""

    def __init__(self, index):
        self.index, self.samples, self.reasons, self._stop = index, [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "sw_power_cap": 0x4, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "hw_power_brake_slowdown": 0x80, "sync_boost": 0x10}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for n, bit in names.items():
                    if mask & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------- sharding
TILE_ROWS = 512  # hisa_cuda.h: HISA_DIST_TILE_ROWS (the plan itself comes from the C library: capi.dist_plan)


# ------------------------------------------------------------------------------------------- reference arm
def run_reference(a, rank, world):
    """The reference's own CPU implementation of the path. The reference tree ships headers only for this
    path (no .cpp, link fails), so the arm times the oracle port on all host cores, on a bounded sample of
    the same workload; value = rows processed / time."""
    if rank != 0:
        return
    from oracle import pyoracle
    L = a.seq_len
    rows_per_step = max(8, a.cpu_rows // 4)
    rng = np.random.default_rng(a.seed)
    keys = bf16_round(rng.standard_normal((L, 128), dtype=np.float32))
    threads = pyoracle.hardware_threads()
    times = []
    for it in range(a.warmup + a.steps):
        rows = np.sort(rng.choice(L, rows_per_step, replace=False)).astype(np.uint32)
        q = bf16_round(rng.standard_normal((rows_per_step, 64, 128), dtype=np.float32))
        w = rng.uniform(0.5, 1.5, (rows_per_step, 64)).astype(np.float32)
        prob = pyoracle.Problem(q, w, keys, rows, block_size=a.block_size, block_budget=a.block_budget,
                                token_budget=a.token_budget)
        t0 = time.perf_counter()
        pyoracle.select_batch("hisa", prob, threads=threads)
        dt = time.perf_counter() - t0
        if it >= a.warmup:
            times.append(dt)
    total = sum(times)
    value = rows_per_step * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64 accumulate over bf16-rounded f32", "data": "synthetic",
        "config": {"workload": workload_name(a), "sample": f"{rows_per_step} uniformly sampled query rows per step"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{rows_per_step} uniformly sampled rows of the workload per step, "
                                   f"{len(times)} steps, all host threads (pool build excluded)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def bf16_round(x):
    from paper_2603_28458_b200 import capi
    return capi.bf16_bits_to_f32(capi.f32_to_bf16_bits(x)).reshape(x.shape)


def run_consumer_leg(a, capi, ix, torch, dev, g, step_hisa, L, nq, k, pos, out_idx, out_count, peaks):
    """The step after the path: sparse_attend over the [Q, k] indices just selected.
    Shared-KV latents [L, d_model] bf16 (16 MiB at 64K x 128: L2-resident), one state vector per query."""
    step_hisa()
    ix.synchronize()
    dm = a.d_model
    g.manual_seed(a.seed + 5000)
    lat = torch.randn((L, dm), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    hs = torch.randn((nq, dm), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    u = torch.empty((nq, dm), device=dev, dtype=torch.float32)
    _check = capi._check
    _check(capi.lib().hisa_cuda_attn_set_latents(ix._ctx, capi._ptr(lat.data_ptr()), L, dm, capi.DTYPE_BF16, 0), ix._ctx)
    att_ms = []
    for it in range(a.attend_steps + 1):
        ix.sparse_attend_raw(hs.data_ptr(), capi.DTYPE_BF16, pos.data_ptr(), nq, out_idx.data_ptr(), k, out_count.data_ptr(),
                             u.data_ptr())
        if it:
            att_ms.append(ix.attn_last_ms())
    a_ms = float(np.median(att_ms))
    picked = int(out_count.to(torch.int64).sum().item())
    gather_bytes = picked * dm * 2
    hbm_bytes = picked * 4 + nq * (dm * 2 + dm * 4 + 8) + L * dm * 2
    consumer = {"op": "sparse_attend (hisa/attention.hpp:48-56) over the selected indices", "d_model": dm, "ms": a_ms,
                "queries_per_s": nq / (a_ms * 1e-3), "selected_tokens": picked,
                "gather_gbs_l2_to_sm": gather_bytes / (a_ms * 1e-3) / 1e9,
                # ceiling of this access pattern measured with tools/l2_gather_bench.cu (random 256-byte rows, XOR only)
                "gather_ceiling_gbs": 20600.0, "gather_frac": gather_bytes / (a_ms * 1e-3) / 1e9 / 20600.0,
                "hbm": {"bound": "hbm", "achieved": hbm_bytes / (a_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": hbm_bytes / (a_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                        "work": "indices + query states read, outputs written, latent table once (the gather itself is "
                                "served by L2: see gather_gbs_l2_to_sm)"},
                "finite": bool(torch.isfinite(u).all().item())}

    return consumer



# ------------------------------------------------------------------------------------------- the other BASELINE configs
def measure_config(torch, capi, dev, peaks, cid, name, L, rows, B, m, k, dtype="bf16", steps=3, warmup=1, flat_steps=1,
                   decode=False):
    """One BASELINE.json configuration through the C ABI on one GPU: device-resident synthetic inputs, CUDA events on the
    context's stream, per-stage events. decode=True: every step first appends ONE key (BlockSummaryCache::append,
    block_summary.hpp:27-30) and all queries sit at the newest position. Returns a dict for the `configs` array."""
    H, d = 64, 128
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    rows = np.asarray(rows, dtype=np.int64)
    nq = len(rows)
    cap = L + (steps + warmup + 16 if decode else 0)
    keys_f = torch.randn((cap, d), generator=g, device=dev, dtype=torch.float32)
    scales = None
    if dtype == "fp8":
        scales = (keys_f.abs().amax(dim=1) / 448.0).clamp_min(1e-12).contiguous()
        keys = (keys_f / scales[:, None]).to(torch.float8_e4m3fn)
        code = capi.DTYPE_FP8
    elif dtype == "f32":
        keys, code = keys_f, capi.DTYPE_F32
    else:
        keys, code = keys_f.to(torch.bfloat16), capi.DTYPE_BF16
    del keys_f
    w = torch.rand((nq, H), generator=g, device=dev, dtype=torch.float32) + 0.5
    if dtype == "fp8":
        q = torch.empty((nq, H, d), device=dev, dtype=torch.float8_e4m3fn)
        for r0 in range(0, nq, 8192):
            qf = torch.randn((min(8192, nq - r0), H, d), generator=g, device=dev, dtype=torch.float32)
            qs = (qf.abs().amax(dim=2) / 448.0).clamp_min(1e-12)
            q[r0:r0 + qf.shape[0]] = (qf / qs[:, :, None]).to(torch.float8_e4m3fn)
            w[r0:r0 + qf.shape[0]] *= qs
    else:
        q = torch.empty((nq, H, d), device=dev, dtype=torch.float32 if dtype == "f32" else torch.bfloat16)
        for r0 in range(0, nq, 16384):
            q[r0:r0 + 16384] = torch.randn((min(16384, nq - r0), H, d), generator=g, device=dev, dtype=torch.float32).to(q.dtype)
    pos = torch.from_numpy(rows).to(dev).to(torch.int32)
    out_idx = torch.empty((nq, k), device=dev, dtype=torch.int32)
    out_count = torch.empty((nq,), device=dev, dtype=torch.int32)
    out_cand = torch.empty((nq,), device=dev, dtype=torch.int32)
    torch.cuda.synchronize()
    eb = q.element_size()
    cfg = capi.make_config(B, m, k, H, d, code)
    with capi.Indexer(cfg, dev.index or 0) as ix, ClockSampler(dev.index or 0) as clocks:
        ix.upload_keys(keys.data_ptr(), seq_len=L, scales=scales.data_ptr() if scales is not None else None)
        ix.pool_build()
        ix.synchronize()
        stream = torch.cuda.ExternalStream(capi.lib().hisa_cuda_stream(ix._ctx), device=dev)
        state = {"L": L}

        if decode:
            # every query sits at the newest position: position >= seq_len is the streaming query (inputs.hpp:18-19), so the
            # position array never changes while keys are appended and the step is two C-ABI calls with constant arguments
            # (from the third step on hisa_cuda_hisa_select replays one captured CUDA graph)
            pos.fill_(2 ** 31 - 1)
            torch.cuda.synchronize()

        def step_hisa():
            if decode:
                at = state["L"]
                ix.pool_append(keys.data_ptr() + at * d * eb, n=1, key_dim=d,
                               scales=(scales.data_ptr() + at * 4) if scales is not None else None)
                state["L"] += 1
            ix.hisa_select_raw(q.data_ptr(), w.data_ptr(), pos.data_ptr(), nq, out_idx.data_ptr(), out_count.data_ptr(),
                               None, None, out_cand.data_ptr())

        def step_flat():
            ix.dsa_select_raw(q.data_ptr(), w.data_ptr(), pos.data_ptr(), nq, out_idx.data_ptr(), out_count.data_ptr(), None)

        def run(fn, n, wu, profile):
            for _ in range(wu):
                fn()
            ix.synchronize()
            if profile:
                ix.set_profiling(True)
                ix.stage_times()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record()
            t0 = time.perf_counter()
            for _ in range(n):
                fn()
            host_s = time.perf_counter() - t0
            with torch.cuda.stream(stream):
                e1.record()
            ix.synchronize()
            st = ix.stage_times() if profile else None
            if profile:
                ix.set_profiling(False)
            return e0.elapsed_time(e1) / n, st, host_s / n

        # decode steps are a handful of short kernels: stage events would be a large part of what they measure, so the
        # step is timed without them first and the per-stage split comes from a second, separately profiled pass
        ms, _, host_s = run(step_hisa, steps, warmup, profile=False)
        _, st, _ = run(step_hisa, max(1, min(steps, 5)), 0, profile=True)
        calls = max(st["calls"], 1)
        stages = {kk: vv / calls for kk, vv in st.items() if kk.endswith("_ms")}
        cand = int(out_cand.to(torch.int64).sum().item())
        pos64 = pos.to(torch.int64).clamp(max=state["L"] - 1)
        elig = int((pos64 // B + 1).sum().item())
        prefix = int((pos64 + 1).sum().item())
        flat_ms = flat_st = None
        if flat_steps:
            flat_ms, flat_st, _ = run(step_flat, flat_steps, 1, profile=True)
        tpeak = peaks["tflops"]
        if dtype == "fp8":
            fpath = os.path.join(ROOT, "profiles", "fp8_peak.json")
            tpeak = float(json.load(open(fpath))["fp8_tflops_sustained"]) if os.path.exists(fpath) else 2.0 * tpeak

        def frac(work, ms_, peak, scale):
            return round(work / (ms_ * 1e-3) / scale / peak, 4) if ms_ and ms_ > 0 else None
        out = {
            "id": cid, "workload": name, "dtype": dtype, "L": L, "Q": nq, "B": B, "m": m, "k": k,
            "ms_per_step": round(ms, 4), "queries_per_s": round(nq / (ms * 1e-3), 1),
            "stages_ms": {kk: round(vv, 4) for kk, vv in stages.items()},
            "launches_per_step": st["launches"] // calls,
            "host_enqueue_us_per_step": round(host_s * 1e6, 1),
            "roofline_frac": {
                "score_blocks (tensor, algorithmic)": frac(2.0 * d * H * elig, stages["score_blocks_ms"], peaks["tflops"], 1e12),
                "score_tokens (tensor)": frac(2.0 * d * H * cand, stages["score_tokens_ms"], tpeak, 1e12),
                "top_k (hbm)": frac(4.0 * cand + 4.0 * nq * k, stages["top_k_ms"], peaks["hbm_gbs"], 1e9),
                "select_blocks (hbm)": frac(4.0 * elig + 4.0 * nq * (m + 2), stages["select_blocks_ms"], peaks["hbm_gbs"], 1e9),
            },
            "stage2_tflops": round(2.0 * d * H * cand / (stages["score_tokens_ms"] * 1e-3) / 1e12, 1) if stages["score_tokens_ms"] > 0 else None,
            "flat_dsa": None,
            "clocks": clocks.summary(),
        }
        if flat_ms:
            fcalls = max(flat_st["calls"], 1)
            fk = flat_st["score_tokens_ms"] / fcalls
            out["flat_dsa"] = {"ms_per_step": round(flat_ms, 4), "scorer_ms": round(fk, 4),
                               "top_k_ms": round(flat_st["top_k_ms"] / fcalls, 4),
                               "scorer_tflops": round(2.0 * d * H * prefix / (fk * 1e-3) / 1e12, 1) if fk > 0 else None,
                               "hisa_speedup": round(flat_ms / ms, 3),
                               "hisa_speedup_scorers_only": round(fk / stages["score_tokens_ms"], 3) if stages["score_tokens_ms"] > 0 else None,
                               "flop_ratio_flat_over_hisa": round(prefix / max(cand + elig, 1), 3)}
    del q, w, keys, out_idx
    torch.cuda.empty_cache()
    return out


def run_configs(a, torch, capi, dev, peaks):
    """Every BASELINE.json configuration other than the headline one (which is the line itself), bounded to about a minute
    in total. Parity of these shapes is the job of tests/ (-m gpu); here they are timed."""
    table = [
        # id, name, L, rows, B, m, k, dtype, steps, warmup, flat_steps, decode
        ("C1", "CPU-reference shape: prefill L=Q=8192, m=32, f32 storage (3x3 bf16 split, 6 MMA terms)", 8192,
         np.arange(8192), 128, 32, 2048, "f32", 5, 2, 2, False),
        ("C2", "DeepSeek-V3.2 indexer shape: prefill L=Q=32768, bf16", 32768, np.arange(32768), 128, 64, 2048, "bf16", 5, 2, 2, False),
        ("C3-fp8", "headline shape with e4m3 q/k + per-key f32 scales", 65536, np.arange(65536), 128, 64, 2048, "fp8", 5, 2, 1, False),
        ("C3-paper", "the paper's measurement shape (PAPER.md:257): last 1024 query rows of a 64K context", 65536,
         np.arange(65536 - 1024, 65536), 128, 64, 2048, "bf16", 20, 3, 5, False),
        ("C3-4to1", "Fig. 2 panel b (PAPER.md:192,261): M:m = 4:1 at 64K, m=128 (16.6K candidates)", 65536, np.arange(65536),
         128, 128, 2048, "bf16", 3, 1, 0, False),
        ("C3-4to1-paper", "same, the paper's 1024-row tail", 65536, np.arange(65536 - 1024, 65536), 128, 128, 2048, "bf16", 20, 3, 5, False),
        ("C4", "prefill L=Q=131072 on ONE GPU (the sharded configuration's single-GPU leg)", 131072, np.arange(131072),
         128, 64, 2048, "bf16", 2, 1, 1, False),
        ("C5-128K", "decode: 64 queries at the newest position of a 128K prefix, +1 key appended per step", 131072,
         np.full(64, 131071), 128, 64, 2048, "bf16", 100, 10, 10, True),
        ("C5-1M", "decode: 64 queries at the newest position of a 1M prefix, +1 key appended per step", 1048576,
         np.full(64, 1048575), 128, 64, 2048, "bf16", 100, 10, 5, True),
    ]
    only = [c for c in a.configs_only.split(",") if c]
    out = []
    t_start = time.perf_counter()
    for cid, name, L, rows, B, m, k, dt, steps, wu, fsteps, dec in table:
        if only and cid not in only:
            continue
        if not only and time.perf_counter() - t_start > 75.0:
            out.append({"id": cid, "skipped": "time budget of the configs array spent"})
            continue
        try:
            out.append(measure_config(torch, capi, dev, peaks, cid, name, L, rows, B, m, k, dt, steps, wu, fsteps, dec))
        except Exception as exc:  # an extra: never lose the headline line over it
            out.append({"id": cid, "error": f"{type(exc).__name__}: {exc}"})
    return out


# ------------------------------------------------------------------------------------------- B200 arm
def run_b200(a, rank, world, local_rank):
    import torch
    from paper_2603_28458_b200 import capi

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device — the product path has no CPU fallback")
    if world > torch.cuda.device_count() and "LOCAL_RANK" in os.environ:
        raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} CUDA device(s) on this node")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # torch.distributed is launcher plumbing only (rendezvous, barrier, max over ranks of the timings, and carrying the
    # 128-byte NCCL id to the ranks); every byte of the data path — key replication, selection, the gather of the index
    # rows — goes through the C ABI's multi-GPU driver (hisa_cuda_dist_*: its own NCCL communicator, its own streams)
    dist = None
    use_driver = world > 1 or a.force_dist
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)

    L = Q = a.seq_len
    H, d, B, m, k = 64, 128, a.block_size, a.block_budget, a.token_budget
    g = torch.Generator(device=dev)
    g.manual_seed(a.seed)
    fp8 = a.dtype == "fp8"
    # keys exist on rank 0 only (the other ranks receive them by ncclBroadcast inside the driver); queries: each rank
    # generates only the rows it owns (synthetic, so nothing has to be scattered)
    keys = key_scales = None
    if rank == 0:
        keys = torch.randn((L, d), generator=g, device=dev, dtype=torch.float32)
        if fp8:  # per-token symmetric quantisation (synthetic-input plumbing; the product consumes bytes + scales)
            key_scales = (keys.abs().amax(dim=1) / 448.0).clamp_min(1e-12).contiguous()
            keys = (keys / key_scales[:, None]).to(torch.float8_e4m3fn)
        else:
            keys = keys.to(torch.bfloat16)
    rows = capi.dist_plan(Q, world, rank)  # the C library's own sharding plan: 512-row tiles, zig-zag over the ranks
    nq = len(rows)
    g.manual_seed(a.seed + 1000 + rank)
    w = torch.rand((nq, H), generator=g, device=dev, dtype=torch.float32) + 0.5
    if fp8:
        q = torch.empty((nq, H, d), device=dev, dtype=torch.float8_e4m3fn)
        for r0 in range(0, nq, 8192):  # quantise in slices: the f32 staging of all of q would be 2 GiB
            qf = torch.randn((min(8192, nq - r0), H, d), generator=g, device=dev, dtype=torch.float32)
            qs = (qf.abs().amax(dim=2) / 448.0).clamp_min(1e-12)
            q[r0:r0 + qf.shape[0]] = (qf / qs[:, :, None]).to(torch.float8_e4m3fn)
            w[r0:r0 + qf.shape[0]] *= qs      # the per-(query, head) scale is folded into the gate
        del qf, qs
    else:
        q = torch.randn((nq, H, d), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    pos = torch.from_numpy(rows.astype(np.int64)).to(dev).to(torch.int32)  # bit pattern == uint32 (values < 2^31)
    out_idx = torch.empty((nq, k), device=dev, dtype=torch.int32)
    out_count = torch.empty((nq,), device=dev, dtype=torch.int32)
    out_cand = torch.empty((nq,), device=dev, dtype=torch.int32)
    torch.cuda.synchronize()

    cfg = capi.make_config(B, m, k, H, d, capi.DTYPE_FP8 if fp8 else capi.DTYPE_BF16)
    driver = None
    n_slices = 1
    if use_driver:
        # one rank per process (the launcher's model): rank 0 makes the NCCL id, torch carries it to the others
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(capi.dist_unique_id()), dtype=torch.uint8))
        if dist:
            dist.broadcast(uid, src=0)
        driver = capi.Dist(cfg, rank=rank, world=world, device=local_rank, unique_id=bytes(uid.cpu().numpy().tobytes()))
        driver.upload_keys(keys.data_ptr() if rank == 0 else None, L,
                           scales=key_scales.data_ptr() if (fp8 and rank == 0) else None, root=0)
        ix = capi.Indexer.borrow(driver.ctx(0), cfg)
        # the rank's rows run in slices; the NCCL gather of slice i (second stream) runs under the kernels of slice i+1:
        # at 8 GPUs the gather of the indices costs about half of the per-rank compute
        n_slices = a.slices or (4 if nq > 8192 else 2)
    else:
        ix = capi.Indexer(cfg, local_rank)
        ix.upload_keys(keys.data_ptr(), seq_len=L, scales=key_scales.data_ptr() if fp8 else None)
    ix.pool_build()
    ix.synchronize()
    stream = torch.cuda.ExternalStream(capi.lib().hisa_cuda_stream(ix._ctx), device=dev)
    # K1 (block mean pooling) runs once per key sequence, outside the per-query step like in the reference's protocol
    # (hisa/bench.hpp:51-52); it is timed here on its own: full rebuild of all block summaries, CUDA events
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pool_reps = 10
    with torch.cuda.stream(stream):
        pe0.record()
    for _ in range(pool_reps):
        ix.pool_build()
    with torch.cuda.stream(stream):
        pe1.record()
    ix.synchronize()
    pool_ms = pe0.elapsed_time(pe1) / pool_reps

    def step_hisa():
        if driver is None:
            ix.hisa_select_raw(q.data_ptr(), w.data_ptr(), pos.data_ptr(), nq, out_idx.data_ptr(), out_count.data_ptr(),
                               None, None, out_cand.data_ptr())
        else:  # sharded step: select this rank's rows, every rank ends up with all Q index rows
            driver.select(capi.DIST_HISA, [q.data_ptr()], [w.data_ptr()], [pos.data_ptr()], Q, num_slices=n_slices)

    def step_flat():
        ix.dsa_select_raw(q.data_ptr(), w.data_ptr(), pos.data_ptr(), nq, out_idx.data_ptr(), out_count.data_ptr(), None)

    def timed(fn, steps, warmup, profile=False, stall_stats=False):
        for _ in range(warmup):
            fn()
        ix.synchronize()
        if driver is not None:
            driver.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        if profile:
            ix.set_profiling(True, stall_stats=stall_stats)
            ix.stage_times()  # reset accumulators
            if stall_stats:
                ix.scorer_stall_cycles()
        l0 = ix.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record()
        for _ in range(steps):
            fn()
        with torch.cuda.stream(stream):
            e1.record()  # the driver makes the context's stream wait for the gather: e1 = "this GPU holds every row"
        ix.synchronize()
        if driver is not None:
            driver.synchronize()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        stages = ix.stage_times() if profile else None
        if profile:
            stages["stalls"] = ix.scorer_stall_cycles() if stall_stats else None
            ix.set_profiling(False)
        launches = ix.launch_count() - l0
        if dist:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, stages, launches

    with ClockSampler(local_rank) as clocks:
        ms_total, stages, launches = timed(step_hisa, a.steps, a.warmup, profile=True)
    ms_step = ms_total / a.steps
    value = Q * a.steps / (ms_total * 1e-3)
    if driver is not None:
        # this rank's own rows out of its copy of the gathered matrix (+ the candidate sizes, which the sharded step
        # does not exchange: one plain call for them)
        ridx, _ = driver.result_ptrs(0)
        full = torch.empty((Q, k), device=dev, dtype=torch.int32)
        ix.memcpy(full.data_ptr(), ridx, Q * k * 4)
        hisa_idx = full[torch.from_numpy(rows.astype(np.int64)).to(dev)].clone()
        del full
        ix.hisa_select_raw(q.data_ptr(), w.data_ptr(), pos.data_ptr(), nq, out_idx.data_ptr(), out_count.data_ptr(),
                           None, None, out_cand.data_ptr())
        ix.synchronize()
        sharded_equals_plain = bool(torch.equal(hisa_idx, out_idx))
    else:
        sharded_equals_plain = None
        hisa_idx = out_idx.clone()  # the device-path result: the host-buffer (e2e) path must reproduce it bit for bit

    # ---- roofline of the dominant kernel (stage-2 fused scorer): algorithmic flops / live CUDA-event time
    cand_sum = int(out_cand.to(torch.int64).sum().item())
    if dist:
        t = torch.tensor([cand_sum], device=dev, dtype=torch.int64)
        dist.all_reduce(t)
        cand_sum_all = int(t.item())
    else:
        cand_sum_all = cand_sum
    peaks = load_peaks()
    flops_s2 = 2.0 * d * H * cand_sum          # this rank, one launch
    k_ms = stages["score_tokens_ms"] / a.steps   # per step (a step is several calls when the rows go in slices)
    achieved = flops_s2 / (k_ms * 1e-3) / 1e12 if k_ms > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic_score_tc_stage2_fp8.json" if a.dtype == "fp8" else "traffic_score_tc_stage2.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    if fp8:
        # dense e4m3 peak measured with the protocol of MEASURED_PEAKS.json (scripts/measure_fp8_peak.py); else 2x bf16
        fpath = os.path.join(ROOT, "profiles", "fp8_peak.json")
        if os.path.exists(fpath):
            peaks = dict(peaks, tflops=float(json.load(open(fpath))["fp8_tflops_sustained"]),
                         source="measured (profiles/fp8_peak.json: torch._scaled_mm e4m3 8192^3, sustained)")
        else:
            peaks = dict(peaks, tflops=2.0 * peaks["tflops"], source=peaks["source"] + " x2 for e4m3 (nominal fp8 : bf16 ratio)")
    roofline = {"bound": "tensor", "kernel": "score_tc_kernel (stage-2 block-major refinement)",
                "achieved": achieved, "peak": peaks["tflops"], "unit": "TFLOP/s",
                "frac": achieved / peaks["tflops"], "traffic": traffic, "peak_source": peaks["source"],
                "flops_per_launch": flops_s2, "kernel_ms": k_ms}
    # the kernel runs inside a long step under sw_power_cap, so the sustained peak is the denominator of `frac`; the burst
    # figure (a kernel timed alone, cold chip) is quoted beside it
    if not fp8 and peaks.get("tflops_burst"):
        roofline["peak_burst"] = peaks["tflops_burst"]
        roofline["frac_of_burst_peak"] = achieved / peaks["tflops_burst"]
    per_call = {kk: (vv / a.steps if kk.endswith("_ms") else vv) for kk, vv in stages.items()
                if kk != "stalls"}
    # ---- every stage against the roofline that bounds it (algorithmic work / CUDA-event time)
    pos64 = pos.to(torch.int64).clamp(max=L - 1)
    elig_sum = int((pos64 // B + 1).sum().item())                       # Σ_t eligible blocks
    nsel_max = nq * (m + 2)
    eb = q.element_size()

    def stage_roof(ms, bound, work, note, tensor_peak=None):
        peak = (tensor_peak or peaks["tflops"]) if bound == "tensor" else peaks["hbm_gbs"]
        ach = work / (ms * 1e-3) / (1e12 if bound == "tensor" else 1e9) if ms > 0 else 0.0
        return {"bound": bound, "ms": round(ms, 4), "achieved": round(ach, 1), "peak": peak,
                "unit": "TFLOP/s" if bound == "tensor" else "GB/s", "frac": round(ach / peak, 4), "work": note}
    stage_rooflines = {
        "score_blocks": stage_roof(per_call["score_blocks_ms"], "tensor", 2.0 * d * H * elig_sum,
                                   "2*d*H*sum_t(eligible blocks); the kernel spends 2 bf16 MMA terms per dot (hi|lo pooled keys)",
                                   tensor_peak=load_peaks()["tflops"]),
        "select_blocks": stage_roof(per_call["select_blocks_ms"], "hbm", 4.0 * elig_sum + 4.0 * nsel_max,
                                    "block scores read + block lists written (J is mostly L2-resident: 128 MiB)"),
        "score_tokens": stage_roof(per_call["score_tokens_ms"], "tensor", flops_s2, "2*d*H*sum_t|Omega_t|"),
        "top_k": stage_roof(per_call["top_k_ms"], "hbm", 4.0 * cand_sum + 4.0 * nq * k,
                            "candidate scores read + [Q,k] int32 indices written"),
    }
    # the whole step (every stage, launch gaps included) against the same tensor peak: algorithmic FLOPs of both scorers
    stage_rooflines["whole_step"] = stage_roof(ms_step, "tensor", flops_s2 + 2.0 * d * H * elig_sum,
                                               "(2*d*H*sum_t|Omega_t| + 2*d*H*sum_t eligible blocks) / ms_per_step")
    pool_bytes = float(L) * d * eb + (4.0 * L if fp8 else 0.0) + ((L + B - 1) // B) * d * (8.0 + 4.0)
    stage_rooflines["pool_build"] = stage_roof(pool_ms, "hbm", pool_bytes,
                                               "keys read once (+ per-key scales for e4m3), f64 sums + bf16 hi|lo pooled keys "
                                               "written; once per key sequence, not part of the per-query step; 16 MiB is "
                                               "launch-latency sized: 2.6 us at the HBM peak")
    # stage 1 issues more MMA work than the algorithmic count: whole 128-row tiles of pooled keys and two bf16 terms
    # (hi | lo split of the f32 means) per dot
    tiles_sum = int(((pos64 // B) // 128 + 1).sum().item())
    issued_s1 = 2.0 * d * H * 128 * tiles_sum * 2
    s1_ms = per_call["score_blocks_ms"]
    stage_rooflines["score_blocks"]["issued_mma_tflops"] = round(issued_s1 / (s1_ms * 1e-3) / 1e12, 1) if s1_ms > 0 else None
    stage_rooflines["score_blocks"]["issued_over_algorithmic"] = round(issued_s1 / max(2.0 * d * H * elig_sum, 1.0), 2)
    # role-level stall accounting: a short separate pass with the instrumented scorer instantiation (not timed)
    _, st_stages, _ = timed(step_hisa, min(a.steps, 3), 0, profile=True, stall_stats=True)
    stalls = {}
    for st_name, st in st_stages["stalls"].items():
        cta = max(st["cta"], 1)
        stalls[st_name] = {kk: (round(vv / cta, 4) if kk != "groups" else vv) for kk, vv in st.items()
                           if kk not in ("cta", "cta_max") and not kk.startswith("epi_")}
        # SM clock the kernel really ran at: CTA lifetime cycles (one persistent CTA per SM) / its CUDA-event time
        st_ms = st_stages["score_blocks_ms" if st_name == "stage1" else "score_tokens_ms"]
        if st_ms > 0:
            n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
            calls_st = max(st_stages["calls"], 1)
            # mean CTA lifetime / longest CTA lifetime: 1.0 = perfectly balanced persistent CTAs
            stalls[st_name]["cta_balance"] = round(st["cta"] / n_sm / calls_st / max(st["cta_max"], 1), 4)
            # SM clock the kernel really ran at: longest CTA lifetime (cycles) / the kernel's CUDA-event time
            stalls[st_name]["sm_mhz_in_kernel"] = round(st["cta_max"] / (st_ms / calls_st * 1e-3) / 1e6, 1)

    # ---- in-run comparison: the flat DSA indexer built from the same kernels
    flat = None
    if a.flat_steps > 0:
        fms, fstages, _ = timed(step_flat, a.flat_steps, 1, profile=True)
        flat_step = fms / a.flat_steps
        prefix = int((pos.to(torch.int64) + 1).sum().item())
        fk_ms = fstages["score_tokens_ms"] / max(fstages["calls"], 1)
        flat = {"ms_per_step": flat_step, "queries_per_s": Q / (flat_step * 1e-3), "hisa_speedup": flat_step / ms_step,
                "scorer_ms": fk_ms, "top_k_ms": fstages["top_k_ms"] / max(fstages["calls"], 1),
                "scorer_tflops": 2.0 * d * H * prefix / (fk_ms * 1e-3) / 1e12 if fk_ms > 0 else None,
                # the flat arm's top-k over whole prefixes is a weaker kernel than its scorer: the scorer-only ratio is the
                # speed-up that does not lean on it (it tracks the FLOP ratio of the two indexers)
                "hisa_speedup_scorers_only": fk_ms / per_call["score_tokens_ms"] if per_call["score_tokens_ms"] > 0 else None,
                "flop_ratio_flat_over_hisa": 2.0 * d * H * prefix / (flops_s2 + 2.0 * d * H * elig_sum)}

    # ---- the step after the path: sparse_attend over the [Q, k] indices just selected.
    # Shared-KV latents [L, d_model] bf16 (16 MiB at 64K x 128: L2-resident), one state vector per query.
    consumer = None
    if a.attend_steps > 0:
        try:
            consumer = run_consumer_leg(a, capi, ix, torch, dev, g, step_hisa, L, nq, k, pos, out_idx, out_count, peaks)
        except Exception as exc:  # an extra, not part of the driver contract: never lose the headline line over it
            consumer = {"error": f"{type(exc).__name__}: {exc}"}
    # ---- end to end through the C ABI with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if a.e2e_steps > 0:
        hq = torch.empty((nq, H, d), dtype=q.dtype, pin_memory=True)
        hw = torch.empty((nq, H), dtype=torch.float32, pin_memory=True)
        hpos = torch.empty((nq,), dtype=torch.int32, pin_memory=True)
        hidx = torch.empty((nq, k), dtype=torch.int32, pin_memory=True)
        hcnt = torch.empty((nq,), dtype=torch.int32, pin_memory=True)
        hq.copy_(q), hw.copy_(w), hpos.copy_(pos)
        torch.cuda.synchronize()

        def step_e2e():
            ix.hisa_select_raw(hq.data_ptr(), hw.data_ptr(), hpos.data_ptr(), nq, hidx.data_ptr(), hcnt.data_ptr())

        step_e2e()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(a.e2e_steps):
            step_e2e()
        ix.synchronize()
        dt = time.perf_counter() - t0
        if dist:
            t = torch.tensor([dt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        same = bool(torch.equal(hidx.to(dev), hisa_idx))
        e2e = {"value": Q * a.e2e_steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(hq.numel() * hq.element_size() + hw.numel() * 4 + hpos.numel() * 4) * world,
               "d2h_bytes_per_step": int(hidx.numel() * 4 + hcnt.numel() * 4) * world,
               "ms_per_step": 1e3 * dt / a.e2e_steps, "matches_device_path": same}

    # ---- CPU baseline: the oracle port on the host cores, bounded sample of the same workload (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        from oracle import pyoracle
        nrows = a.cpu_rows
        sel = np.sort(np.random.default_rng(0).choice(nq, nrows, replace=False))
        sel_t = torch.from_numpy(sel).to(dev)
        pq = q[sel_t].to(torch.float32).cpu().numpy()
        pw = w[sel_t].cpu().numpy()
        pk = keys.to(torch.float32).cpu().numpy()
        if fp8:  # the oracle is given the dequantised keys: float(k8) * scale (one f32 rounding, as on the GPU)
            pk = (pk * key_scales.cpu().numpy()[:, None]).astype(np.float32)
        prob = pyoracle.Problem(pq, pw, pk, rows[sel].astype(np.uint32), block_size=B, block_budget=m, token_budget=k)
        threads = pyoracle.hardware_threads()
        t0 = time.perf_counter()
        ref = pyoracle.select_batch("hisa", prob, threads=threads)
        dt = time.perf_counter() - t0
        # the same rows double as a parity spot-check of the timed configuration
        step_hisa()
        ix.synchronize()
        got = out_idx[sel_t].cpu().numpy()
        inter = sum(len(set(got[i][got[i] >= 0].tolist()) & set(ref.idx[i, :ref.count[i]].tolist())) for i in range(nrows))
        recall = inter / max(int(ref.count.sum()), 1)
        cpu = {"value": nrows / dt, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{nrows} uniformly sampled query rows of the timed workload, all host threads, "
                         f"pool build excluded; recall of the GPU result on these rows = {recall:.5f}"}

    q_gib = q.numel() * q.element_size() / 2**30
    # ---- N > 1: the sharded configuration of BASELINE.json (C4: L = Q = 131072) on the same ranks, a few steps
    c4 = None
    if driver is not None and world > 1 and a.seq_len != 131072:
        try:
            L4 = 131072
            rows4 = capi.dist_plan(L4, world, rank)
            n4 = len(rows4)
            g.manual_seed(a.seed + 77)
            k4 = torch.randn((L4, d), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16) if rank == 0 else None
            del q
            torch.cuda.empty_cache()
            q4 = torch.randn((n4, H, d), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
            w4 = torch.rand((n4, H), generator=g, device=dev, dtype=torch.float32) + 0.5
            p4 = torch.from_numpy(rows4.astype(np.int64)).to(dev).to(torch.int32)
            cfg4 = capi.make_config(B, m, k, H, d, capi.DTYPE_BF16)
            uid = torch.zeros(128, dtype=torch.uint8, device=dev)
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(capi.dist_unique_id()), dtype=torch.uint8))
            dist.broadcast(uid, src=0)
            with capi.Dist(cfg4, rank=rank, world=world, device=local_rank, unique_id=bytes(uid.cpu().numpy().tobytes())) as d4:
                d4.upload_keys(k4.data_ptr() if rank == 0 else None, L4, root=0)
                times = []
                for it in range(4):
                    dist.barrier()
                    d4.select(capi.DIST_HISA, [q4.data_ptr()], [w4.data_ptr()], [p4.data_ptr()], L4, num_slices=4)
                    t = torch.tensor([d4.last_ms()], device=dev, dtype=torch.float64)  # synchronises
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    if it:
                        times.append(float(t.item()))
            c4 = {"workload": "C4 prefill L=Q=131072 bf16, rows sharded over the ranks, keys NCCL-broadcast, index rows gathered",
                  "ms_per_step": float(np.median(times)), "queries_per_s": L4 / (float(np.median(times)) * 1e-3), "n_gpus": world}
        except Exception as exc:
            c4 = {"error": f"{type(exc).__name__}: {exc}"}

    # ---- the other BASELINE configurations (one GPU each; rank 0 only)
    configs = None
    if rank == 0 and world == 1 and not a.no_configs:
        del out_idx, hisa_idx
        if "q" in dir():
            del q
        torch.cuda.empty_cache()
        configs = run_configs(a, torch, capi, dev, load_peaks())

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16" if not fp8 else "e4m3 (fp32 accumulate; block scores in bf16 hi|lo)", "data": "synthetic",
            "config": {"workload": workload_name(a),
                       "l2": f"inputs larger than L2 (q is {q_gib:.1f} GiB per step)",
                       "sharding": f"query tiles of {TILE_ROWS} rows round-robin over ranks; keys NCCL-broadcast; "
                                   "indices all-gathered inside the step" if world > 1 else "single GPU"},
            # NVML is sampled every 20 ms and lags a timed region of ~90 ms; the clock the scorer kernels really ran at
            # (longest CTA lifetime in cycles / kernel time, from the instrumented pass) is reported beside it
            "clocks": dict(clocks.summary(), sm_mhz_in_scorer_kernels={kk: vv.get("sm_mhz_in_kernel") for kk, vv in stalls.items()}),
            "e2e": e2e, "gpu_launches": launches,
            "roofline": roofline, "stage_rooflines": stage_rooflines, "cpu_baseline": cpu, "flat_dsa": flat,
            "stages_ms_per_step": per_call, "consumer_sparse_attend": consumer,
            "scorer_stall_fraction_of_cta_time": stalls,
            "candidate_pairs_per_step": cand_sum_all,
            "configs": configs,
            "multi_gpu": None if driver is None else {
                "driver": "hisa_cuda_dist_* (C ABI): one rank per process, ncclCommInitRank, keys by ncclBroadcast, rows in "
                          f"{TILE_ROWS}-row zig-zag tiles, per-tile ncclBroadcast gather on a second stream under the next slice",
                "slices_per_rank": n_slices, "rows_this_rank": nq, "sharded_result_equals_plain_call": sharded_equals_plain,
                "c4_128k": c4},
        }
        print(json.dumps(line), flush=True)
    ix.close()
    if driver is not None:
        driver.close()
    if dist:
        dist.destroy_process_group()


def main():
    a = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # plain `python bench.py --gpus N`: launch the N ranks ourselves, exactly as the driver would
        import socket
        import subprocess
        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")          # communicator lines (nranks, NVLS, rings) go to stderr
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.run(cmd, env=env).returncode)
    if world != a.gpus and not (world == 1 and a.gpus == 1):
        print(f"bench.py: launched with WORLD_SIZE={world} but --gpus {a.gpus}; using the launcher's world size", file=sys.stderr)
    run_b200(a, rank, world, local_rank)


if __name__ == "__main__":
    main()
