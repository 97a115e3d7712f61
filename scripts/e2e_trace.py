#!/usr/bin/env python
"""Where the end-to-end (host-buffer) step spends its time: all-host, host inputs only, host outputs only, all-device."""
import os
import sys
import time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_28458_b200 import capi  # noqa: E402

dev = torch.device("cuda", 0)
L = Q = 65536
H, d, B, m, k = 64, 128, 128, 64, 2048
g = torch.Generator(device=dev); g.manual_seed(1)
keys = torch.randn((L, d), generator=g, device=dev).to(torch.bfloat16)
q = torch.randn((Q, H, d), generator=g, device=dev).to(torch.bfloat16)
w = torch.rand((Q, H), generator=g, device=dev) + 0.5
pos = torch.arange(Q, device=dev, dtype=torch.int32)
idx = torch.empty((Q, k), device=dev, dtype=torch.int32)
cnt = torch.empty((Q,), device=dev, dtype=torch.int32)
hq = torch.empty((Q, H, d), dtype=torch.bfloat16, pin_memory=True); hq.copy_(q)
hw = torch.empty((Q, H), dtype=torch.float32, pin_memory=True); hw.copy_(w)
hpos = torch.empty((Q,), dtype=torch.int32, pin_memory=True); hpos.copy_(pos)
hidx = torch.empty((Q, k), dtype=torch.int32, pin_memory=True)
hcnt = torch.empty((Q,), dtype=torch.int32, pin_memory=True)
torch.cuda.synchronize()
ix = capi.Indexer(capi.make_config(B, m, k, H, d, capi.DTYPE_BF16), 0)
ix.upload_keys(keys.data_ptr(), seq_len=L); ix.pool_build(); ix.synchronize()


def run(name, a, b, c, o, oc, n=4):
    f = lambda: ix.hisa_select_raw(a.data_ptr(), b.data_ptr(), c.data_ptr(), Q, o.data_ptr(), oc.data_ptr())
    f(); ix.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    ix.synchronize()
    print(f"{name:28s} {(time.perf_counter() - t0) / n * 1e3:7.2f} ms/step", flush=True)


import os
run("all host", hq, hw, hpos, hidx, hcnt, n=1)
