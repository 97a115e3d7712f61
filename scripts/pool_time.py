import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2603_28458_b200 import capi
dev = torch.device('cuda', 0)
for L in (65536, 1048576):
    keys = torch.randn((L, 128), device=dev).to(torch.bfloat16)
    cfg = capi.make_config(128, 64, 2048, 64, 128, capi.DTYPE_BF16)
    with capi.Indexer(cfg, 0) as ix:
        ix.upload_keys(keys.data_ptr(), seq_len=L)
        stream = torch.cuda.ExternalStream(capi.lib().hisa_cuda_stream(ix._ctx), device=dev)
        ix.pool_build(); ix.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream): e0.record()
        for _ in range(20): ix.pool_build()
        with torch.cuda.stream(stream): e1.record()
        ix.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"pool_build L={L}: {ms*1e3:.1f} us, {L*128*2/ms/1e6:.0f} GB/s")
