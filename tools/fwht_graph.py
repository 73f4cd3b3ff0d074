"""Large-n FWHT: eager calls vs one CUDA-graph replay of the same call (host launch cost check)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
buf = torch.randn(1 << 28, device="cuda")
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 15, 21):
    mat = buf.view(-1, 1 << k)
    P.wht_fast_batch(mat)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(5):
        P.wht_fast_batch(mat)
    e.record(); torch.cuda.synchronize()
    eager = s.elapsed_time(e) / 5
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        P.wht_fast_batch(mat)  # warm outside capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            P.wht_fast_batch(mat)
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    s.record()
    for _ in range(5):
        g.replay()
    e.record(); torch.cuda.synchronize()
    gr = s.elapsed_time(e) / 5
    print(f"2^{k}: eager {eager:.3f} ms ({2**31/eager/1e6/6551.4:.3f})  graph {gr:.3f} ms ({2**31/gr/1e6/6551.4:.3f})")
