#!/usr/bin/env python
"""Times the BASELINE.json configurations other than the headline one through the C ABI, on one GPU, with
device-resident inputs and CUDA events on the context's stream. One JSON line per configuration.

    C2      prefill L=Q=32768
    C3tail  the paper's measurement shape: the last 1024 query rows against L=65536 keys
    C4      prefill L=Q=131072 (single-GPU leg of the query-sharded configuration)
    C5      decode: 64 queries at the newest position of a 128K / 1M-token prefix; every step first appends ONE key
            (incremental tail-block update, BlockSummaryCache::append) and then selects

bench.py keeps the driver contract for the headline configuration (C3); this script only feeds DESIGN.md /
profiles/ with the rest. Usage: python scripts/bench_configs.py [C2 C3tail C4 C5a C5b]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_28458_b200 import capi  # noqa: E402

H, D, B, M_BUDGET, K = 64, 128, 128, 64, 2048


def timed(ix, stream, fn, steps, warmup):
    for _ in range(warmup):
        fn()
    ix.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record()
    for _ in range(steps):
        fn()
    with torch.cuda.stream(stream):
        e1.record()
    ix.synchronize()
    return e0.elapsed_time(e1) / steps


def run(name, L, rows, steps, warmup, flat_steps, decode=False):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    cap = L + (steps + warmup + 8 if decode else 0)
    keys = torch.randn((cap, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    nq = len(rows)
    q = torch.randn((nq, H, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    w = torch.rand((nq, H), generator=g, device=dev, dtype=torch.float32) + 0.5
    pos = torch.from_numpy(np.asarray(rows, dtype=np.int64)).to(dev).to(torch.int32)
    out_idx = torch.empty((nq, K), device=dev, dtype=torch.int32)
    out_count = torch.empty((nq,), device=dev, dtype=torch.int32)
    out_cand = torch.empty((nq,), device=dev, dtype=torch.int32)
    torch.cuda.synchronize()
    cfg = capi.make_config(B, M_BUDGET, K, H, D, capi.DTYPE_BF16)
    with capi.Indexer(cfg, 0) as ix:
        ix.upload_keys(keys.data_ptr(), seq_len=L)
        ix.pool_build()
        ix.synchronize()
        stream = torch.cuda.ExternalStream(capi.lib().hisa_cuda_stream(ix._ctx), device=dev)
        state = {"L": L}

        def step_hisa():
            if decode:  # one new token: tail-block update, then every query sits at the newest position
                ix.pool_append(keys.data_ptr() + state["L"] * D * 2, n=1, key_dim=D)
                state["L"] += 1
                with torch.cuda.stream(stream):
                    pos.fill_(state["L"] - 1)
            ix.hisa_select_raw(q.data_ptr(), w.data_ptr(), pos.data_ptr(), nq, out_idx.data_ptr(), out_count.data_ptr(),
                               None, None, out_cand.data_ptr())

        def step_flat():
            ix.dsa_select_raw(q.data_ptr(), w.data_ptr(), pos.data_ptr(), nq, out_idx.data_ptr(), out_count.data_ptr(), None)

        ix.set_profiling(True)
        ix.stage_times()
        ms = timed(ix, stream, step_hisa, steps, warmup)
        st = ix.stage_times()
        calls = max(st["calls"], 1)
        stages = {kk: round(vv / calls, 4) for kk, vv in st.items() if kk.endswith("_ms")}
        ix.set_profiling(False)
        cand = int(out_cand.to(torch.int64).sum().item())
        flat_ms = timed(ix, stream, step_flat, flat_steps, 1) if flat_steps else None
        prefix = int((pos.to(torch.int64) + 1).sum().item())
        line = {"config": name, "L": L, "Q": nq, "ms_per_step": round(ms, 4), "queries_per_s": round(nq / (ms * 1e-3), 1),
                "stages_ms": stages, "launches_per_step": st["launches"] // calls,
                "stage2_tflops": round(2.0 * D * H * cand / (stages["score_tokens_ms"] * 1e-3) / 1e12, 1)
                if stages["score_tokens_ms"] > 0 else None,
                "flat_ms_per_step": round(flat_ms, 4) if flat_ms else None,
                "flat_tflops": round(2.0 * D * H * prefix / (flat_ms * 1e-3) / 1e12, 1) if flat_ms else None,
                "hisa_speedup_vs_flat": round(flat_ms / ms, 3) if flat_ms else None}
        print(json.dumps(line), flush=True)


def main():
    want = sys.argv[1:] or ["C2", "C3tail", "C4", "C5a", "C5b"]
    for name in want:
        if name == "C2":
            run("C2 prefill L=Q=32768", 32768, np.arange(32768), 10, 3, 2)
        elif name == "C3tail":
            run("C3 paper shape: last 1024 rows of L=65536", 65536, np.arange(65536 - 1024, 65536), 20, 3, 5)
        elif name == "C4":
            run("C4 prefill L=Q=131072 (one GPU)", 131072, np.arange(131072), 3, 1, 1)
        elif name == "C5a":
            run("C5 decode Q=64 at L=131072 (+1 key appended per step)", 131072, np.full(64, 131071), 50, 5, 10, decode=True)
        elif name == "C5b":
            run("C5 decode Q=64 at L=1048576 (+1 key appended per step)", 1048576, np.full(64, 1048575), 50, 5, 10, decode=True)


if __name__ == "__main__":
    main()
