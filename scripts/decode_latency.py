#!/usr/bin/env python
"""Decode step (C5: 64 queries at the newest position, one key appended per step): device time per step with stage
profiling OFF, and the host time one step costs to enqueue. If the host time is the larger one the step is launch-bound
on the CPU side, not on the GPU."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_28458_b200 import capi  # noqa: E402

H, D, B, M, K = 64, 128, 128, 64, 2048
dev = torch.device("cuda", 0)
for L0 in (131072, 1048576):
    steps = 300
    g = torch.Generator(device=dev); g.manual_seed(1)
    keys = torch.randn((L0 + steps + 64, D), generator=g, device=dev).to(torch.bfloat16)
    q = torch.randn((64, H, D), generator=g, device=dev).to(torch.bfloat16)
    w = torch.rand((64, H), generator=g, device=dev) + 0.5
    pos = torch.full((64,), L0 - 1, device=dev, dtype=torch.int32)
    idx = torch.empty((64, K), device=dev, dtype=torch.int32)
    cnt = torch.empty((64,), device=dev, dtype=torch.int32)
    torch.cuda.synchronize()
    with capi.Indexer(capi.make_config(B, M, K, H, D, capi.DTYPE_BF16), 0) as ix:
        ix.upload_keys(keys.data_ptr(), seq_len=L0); ix.pool_build(); ix.synchronize()
        stream = torch.cuda.ExternalStream(capi.lib().hisa_cuda_stream(ix._ctx), device=dev)
        state = {"L": L0}
        # every query sits at the newest position: position == seq_len is the streaming query (inputs.hpp:18-19)
        big = torch.full((64,), 2**31 - 1, device=dev, dtype=torch.int32)

        def step():
            ix.pool_append(keys.data_ptr() + state["L"] * D * 2, n=1, key_dim=D)
            state["L"] += 1
            ix.hisa_select_raw(q.data_ptr(), w.data_ptr(), big.data_ptr(), 64, idx.data_ptr(), cnt.data_ptr())

        for _ in range(20):
            step()
        ix.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record()
        t0 = time.perf_counter()
        for _ in range(steps):
            step()
        host = time.perf_counter() - t0
        with torch.cuda.stream(stream):
            e1.record()
        ix.synchronize()
        print(f"L={L0}: device {e0.elapsed_time(e1) / steps * 1e3:.1f} us/step, host enqueue {host / steps * 1e6:.1f} us/step", flush=True)
