"""One large-n FWHT call (1 GiB) for an ncu launch list of its phases: python tools/fwht_phases.py K"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
k = int(sys.argv[1])
mat = torch.randn(1 << 28, device="cuda").view(-1, 1 << k)
P.wht_fast_batch(mat)
torch.cuda.synchronize()
P.wht_fast_batch(mat)
torch.cuda.synchronize()
print("done")
