"""Time the config-3 training step (1000-row batch, float64 head)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
from paper_1702_08159_b200 import synthetic as S
x, y = S.class_images(60000, 784, 10, seed=1234)
xt, yt = S.class_images(10000, 784, 10, seed=1234, sample_seed=99)
spec = P.FeatureMapSpec(784, 8, P.RBF(1.0), 1234)
tr = P.Trainer(spec, P.Dataset(x, y, 10), P.Dataset(xt, yt, 10), P.TrainConfig(0.01, 1000, 1))
for s in range(5):
    tr.step(0, s)
torch.cuda.synchronize()
a, b = torch.cuda.Event(True), torch.cuda.Event(True)
a.record()
for s in range(60):
    tr.step(0, s)
b.record(); torch.cuda.synchronize()
print(f"c3 step {a.elapsed_time(b) / 60 * 1e3:.1f} us")
