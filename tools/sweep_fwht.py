"""Quick config-1 FWHT sweep (GB/s on algorithmic bytes, 1 GiB per length)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
buf = torch.randn(1 << 28, device="cuda")
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10, 21):
    mat = buf.view(-1, 1 << k)
    P.wht_fast_batch(mat)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(5):
        P.wht_fast_batch(mat)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"2^{k}: {ms:.3f} ms  {2**31/ms/1e6:.0f} GB/s  {2**31/ms/1e6/6459.6:.3f}")
