"""Device time of small (L2-resident) FWHT batches, 20 calls captured in one CUDA graph."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
for k in (14, 10):
    for mb in (6, 12, 24, 48, 96):
        mat = torch.randn((mb << 20) // (4 << k), 1 << k, device="cuda")
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            P.wht_fast_batch(mat)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=st):
                for _ in range(20):
                    P.wht_fast_batch(mat)
        torch.cuda.synchronize()
        g.replay(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        for _ in range(5):
            g.replay()
        e.record(); torch.cuda.synchronize()
        us = s.elapsed_time(e) / 100 * 1e3
        print(f"2^{k} {mb:3d} MiB: {us:7.2f} us per call  {2 * (mb << 20) / us / 1e3:.0f} GB/s (r+w)")
