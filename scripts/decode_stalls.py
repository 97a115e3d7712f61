import os, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2603_28458_b200 import capi
H, D, B, M, K = 64, 128, 128, 64, 2048
dev = torch.device("cuda", 0)
L0 = 131072
g = torch.Generator(device=dev); g.manual_seed(1)
keys = torch.randn((L0 + 64, D), generator=g, device=dev).to(torch.bfloat16)
q = torch.randn((64, H, D), generator=g, device=dev).to(torch.bfloat16)
w = torch.rand((64, H), generator=g, device=dev) + 0.5
pos = torch.full((64,), L0 - 1, device=dev, dtype=torch.int32)
idx = torch.empty((64, K), device=dev, dtype=torch.int32)
cnt = torch.empty((64,), device=dev, dtype=torch.int32)
blk = torch.empty((64, M + 2), device=dev, dtype=torch.int32)
nblk = torch.empty((64,), device=dev, dtype=torch.int32)
torch.cuda.synchronize()
with capi.Indexer(capi.make_config(B, M, K, H, D, capi.DTYPE_BF16), 0) as ix:
    ix.upload_keys(keys.data_ptr(), seq_len=L0); ix.pool_build(); ix.synchronize()
    for _ in range(5):
        ix.hisa_select_raw(q.data_ptr(), w.data_ptr(), pos.data_ptr(), 64, idx.data_ptr(), cnt.data_ptr(), blk.data_ptr(), nblk.data_ptr())
    ix.synchronize()
    b = blk.cpu().numpy(); nb = nblk.cpu().numpy()
    flat = np.concatenate([b[i, :nb[i]] for i in range(64)])
    u, c = np.unique(flat, return_counts=True)
    print("distinct blocks", len(u), "pairs", len(flat), "groups", int(np.ceil(c / 4).sum()), "max list", c.max())
    ix.set_profiling(True, stall_stats=True); ix.stage_times(); ix.scorer_stall_cycles()
    n = 20
    for _ in range(n):
        ix.hisa_select_raw(q.data_ptr(), w.data_ptr(), pos.data_ptr(), 64, idx.data_ptr(), cnt.data_ptr())
    st = ix.stage_times(); sc = ix.scorer_stall_cycles()
    print({k: round(v / n * 1e3, 1) for k, v in st.items() if k.endswith("_ms")})
    for name in ("stage1", "stage2"):
        s = sc[name]; cta = max(s["cta"], 1)
        print(name, {k: round(v / cta, 3) for k, v in s.items() if k not in ("cta", "cta_max", "groups")}, "groups/call", s["groups"] / n,
              "cta cycles/call/SM", s["cta"] / n / 148, "cta_max", s["cta_max"])
