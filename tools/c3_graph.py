"""c3: one training epoch (60 steps) as eager launches vs one CUDA graph replay."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
from paper_1702_08159_b200 import synthetic as S
x, y = S.class_images(60000, 784, 10, seed=1234)
xt, yt = S.class_images(10000, 784, 10, seed=1234, sample_seed=99)
spec = P.FeatureMapSpec(784, 8, P.RBF(1.0), 1234)
tr = P.Trainer(spec, P.Dataset(x, y, 10), P.Dataset(xt, yt, 10), P.TrainConfig(0.01, 1000, 2))
for s in range(tr.steps):
    tr.step(0, s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for s in range(tr.steps):
    tr.step(0, s)
torch.cuda.synchronize()
eager = (time.perf_counter() - t0) / tr.steps * 1e6
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    with torch.cuda.graph(g, stream=st):
        for s in range(tr.steps):
            tr.step(0, s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
graph = (time.perf_counter() - t0) / (5 * tr.steps) * 1e6
print(f"c3 step eager {eager:.1f} us, graph {graph:.1f} us")
