"""FWHT timing at 2^k (k from argv): 7 trials of 10 calls on a 1 GiB batch; best and median fraction of HBM."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
buf = torch.randn(1 << 28, device="cuda")
for k in [int(a) for a in sys.argv[1:]]:
    mat = buf.view(-1, 1 << k)
    for _ in range(3):
        P.wht_fast_batch(mat)
    torch.cuda.synchronize()
    fr = []
    for _ in range(7):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(10):
            P.wht_fast_batch(mat)
        e.record(); torch.cuda.synchronize()
        fr.append(2**31 / (s.elapsed_time(e) / 10) / 1e6 / 6549.8)
    fr.sort()
    print(f"2^{k}: best {fr[-1]:.3f} median {fr[3]:.3f} worst {fr[0]:.3f}")
    buf.normal_()
