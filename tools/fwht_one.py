"""Run wht_fast_batch on one 1 GiB batch of 2^k rows a few times (ncu target)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
k = int(sys.argv[1]) if len(sys.argv) > 1 else 16
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
buf = torch.randn(1 << 28, device="cuda")
mat = buf.view(-1, 1 << k)
for _ in range(reps):
    P.wht_fast_batch(mat)
torch.cuda.synchronize()
