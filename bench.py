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
                    help="initialise NCCL even with one rank (exercises the multi-GPU code path on a single GPU)")
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
                "hbm_gbs": float(p.get("hbm_gbs", 6650.0)), "source": "measured (MEASURED_PEAKS.json, sustained bf16)"}
    return {"tflops": 1400.0, "hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


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
from paper_2603_28458_b200.sharding import TILE_ROWS, rank_rows  # noqa: E402  (query tiles dealt zig-zag over ranks)


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


# ------------------------------------------------------------------------------------------- B200 arm
def run_b200(a, rank, world, local_rank):
    import torch
    from paper_2603_28458_b200 import capi

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device — the product path has no CPU fallback")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1 or a.force_dist:
        import torch.distributed as dist_mod
        dist = dist_mod
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)

    L = Q = a.seq_len
    H, d, B, m, k = 64, 128, a.block_size, a.block_budget, a.token_budget
    g = torch.Generator(device=dev)
    g.manual_seed(a.seed)
    # keys: generated on rank 0 and replicated (NCCL broadcast over NVLink); queries: each rank generates only
    # the rows it owns (synthetic, so nothing has to be scattered)
    fp8 = a.dtype == "fp8"
    keys = torch.randn((L, d), generator=g, device=dev, dtype=torch.float32)
    key_scales = None
    if fp8:  # per-token symmetric quantisation (synthetic-input plumbing; the product consumes bytes + scales)
        key_scales = (keys.abs().amax(dim=1) / 448.0).clamp_min(1e-12).contiguous()
        keys = (keys / key_scales[:, None]).to(torch.float8_e4m3fn)
    else:
        keys = keys.to(torch.bfloat16)
    if dist:
        dist.broadcast(keys.view(torch.uint8) if fp8 else keys, src=0)
        if fp8:
            dist.broadcast(key_scales, src=0)
    rows = rank_rows(Q, world, rank)
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
    # multi-GPU: the rank's rows are selected in slices, and the all-gather of slice i (NCCL, its own stream) runs
    # under the kernels of slice i+1 — at 8 GPUs the gather of the indices costs about half of the per-rank compute
    # (SURVEY.md §8e), so it must not be serialised behind it
    n_slices = 1 if not dist else (4 if nq > 8192 else 2)
    step_rows = -(-nq // (n_slices * TILE_ROWS)) * TILE_ROWS
    bounds = [min(i * step_rows, nq) for i in range(n_slices + 1)]
    gathered = [torch.empty((world * (bounds[i + 1] - bounds[i]), k), device=dev, dtype=torch.int32)
                for i in range(n_slices)] if dist else None
    comm_stream = torch.cuda.Stream(device=dev) if dist else None
    slice_done = [torch.cuda.Event() for _ in range(n_slices)] if dist else None
    torch.cuda.synchronize()

    cfg = capi.make_config(B, m, k, H, d, capi.DTYPE_FP8 if fp8 else capi.DTYPE_BF16)
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
        if not dist:
            ix.hisa_select_raw(q.data_ptr(), w.data_ptr(), pos.data_ptr(), nq, out_idx.data_ptr(), out_count.data_ptr(),
                               None, None, out_cand.data_ptr())
            return
        for i in range(n_slices):
            r0, r1 = bounds[i], bounds[i + 1]
            if r1 <= r0:
                continue
            ix.hisa_select_raw(q[r0:r1].data_ptr(), w[r0:r1].data_ptr(), pos[r0:r1].data_ptr(), r1 - r0,
                               out_idx[r0:r1].data_ptr(), out_count[r0:r1].data_ptr(), None, None,
                               out_cand[r0:r1].data_ptr())
            slice_done[i].record(stream)
            with torch.cuda.stream(comm_stream):
                comm_stream.wait_event(slice_done[i])
                dist.all_gather_into_tensor(gathered[i], out_idx[r0:r1])
        stream.wait_stream(comm_stream)  # the step ends when every rank holds every index row

    def step_flat():
        ix.dsa_select_raw(q.data_ptr(), w.data_ptr(), pos.data_ptr(), nq, out_idx.data_ptr(), out_count.data_ptr(), None)

    def timed(fn, steps, warmup, profile=False, stall_stats=False):
        for _ in range(warmup):
            fn()
        ix.synchronize()
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
            e1.record()
        ix.synchronize()
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
                "scorer_tflops": 2.0 * d * H * prefix / (fk_ms * 1e-3) / 1e12 if fk_ms > 0 else None}

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

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16" if not fp8 else "e4m3 (fp32 accumulate; block scores in bf16 hi|lo)", "data": "synthetic",
            "config": {"workload": workload_name(a),
                       "l2": f"inputs larger than L2 (q is {q.numel() * q.element_size() / 2**30:.1f} GiB per step)",
                       "sharding": f"query tiles of {TILE_ROWS} rows round-robin over ranks; keys NCCL-broadcast; "
                                   "indices all-gathered inside the step" if world > 1 else "single GPU"},
            "clocks": clocks.summary(), "e2e": e2e, "gpu_launches": launches,
            "roofline": roofline, "stage_rooflines": stage_rooflines, "cpu_baseline": cpu, "flat_dsa": flat,
            "stages_ms_per_step": per_call, "consumer_sparse_attend": consumer,
            "scorer_stall_fraction_of_cta_time": stalls,
            "candidate_pairs_per_step": cand_sum_all,
        }
        print(json.dumps(line), flush=True)
    ix.close()
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
    if world != a.gpus and world == 1 and a.gpus > 1:
        raise SystemExit("bench.py: --gpus N>1 must be launched with torch.distributed.run (one rank per GPU)")
    run_b200(a, rank, world, local_rank)


if __name__ == "__main__":
    main()
