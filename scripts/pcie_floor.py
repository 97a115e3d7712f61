#!/usr/bin/env python
"""PCIe floor of the end-to-end (host-buffer) step: pinned H2D of the step's inputs and D2H of its indices, alone and
concurrently, in pipeline-sized pieces. Explains bench.py's e2e number."""
import torch

dev = torch.device("cuda", 0)
Q, H, d, k = 65536, 64, 128, 2048
hq = torch.empty((Q, H, d), dtype=torch.bfloat16, pin_memory=True)
hidx = torch.empty((Q, k), dtype=torch.int32, pin_memory=True)
dq = torch.empty((Q, H, d), dtype=torch.bfloat16, device=dev)
didx = torch.zeros((Q, k), dtype=torch.int32, device=dev)
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, rows):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s_in.wait_stream(torch.cuda.current_stream())
    s_out.wait_stream(torch.cuda.current_stream())
    for r0 in range(0, Q, rows):
        if h2d:
            with torch.cuda.stream(s_in):
                dq[r0:r0 + rows].copy_(hq[r0:r0 + rows], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s_out):
                hidx[r0:r0 + rows].copy_(didx[r0:r0 + rows], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s_in)
    torch.cuda.current_stream().wait_stream(s_out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for rows in (4096, 16384, 65536):
    for name, a, b in (("h2d", True, False), ("d2h", False, True), ("both", True, True)):
        run(a, b, rows)
        ms = min(run(a, b, rows) for _ in range(3))
        gb = (hq.numel() * 2 if a else 0) / 1e9, (hidx.numel() * 4 if b else 0) / 1e9
        print(f"rows/piece={rows:6d} {name:5s} {ms:7.2f} ms  h2d {gb[0] / ms * 1e3:5.1f} GB/s  d2h {gb[1] / ms * 1e3:5.1f} GB/s")
