import sys
from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
from paper_1702_08159_b200 import synthetic
dev = torch.device("cuda")
spec0 = P.FeatureMapSpec(784, 8, P.RBF(1.0), 1234)
b0 = P.build_blocks(spec0)
x0 = torch.from_numpy(synthetic.image_rows(1000, 784, 1234)).to(dev)
o0 = [torch.empty((1000, 16384), device=dev) for _ in range(4)]
P.feature_map_batch(spec0, b0, x0, out=o0[0])
side = torch.cuda.Stream(dev)
side.wait_stream(torch.cuda.current_stream(dev))
def timed(fn, n):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
res = {}
for ns in (1, 2, 3):
    ss = [torch.cuda.Stream(dev) for _ in range(ns)]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for q in ss: q.wait_stream(side)
        for k in range(24):
            with torch.cuda.stream(ss[k % ns]):
                P.feature_map_batch(spec0, b0, x0, out=o0[k % 4])
        for q in ss: side.wait_stream(q)
    g.replay()
    res[ns] = timed(g.replay, 20) / 24 * 1e3
print({k: round(v, 2) for k, v in res.items()}, "us per batch; frac", round(1000 * (784 * 4 + 16384 * 4) / (min(res.values()) * 1e-6) / 1e9 / 6549.8, 3))
