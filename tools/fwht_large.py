"""Time the FWHT at 2^15 .. 2^20 on 1 GiB (c1 sizes); MCK_LIB_PATH selects a build."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
buf = torch.randn(1 << 28, device="cuda")
res = []
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 15, 21):
    n = 1 << k
    mat = buf.view(-1, n)
    P.wht_fast_batch(mat)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(5):
        P.wht_fast_batch(mat)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    res.append(f"2^{k}: {2**31 / (ms / 1e3) / 1e9 / 6553:.3f}")
print(os.path.basename(os.environ.get("MCK_LIB_PATH", "default")), " ".join(res))
