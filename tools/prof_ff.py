"""Small driver for ncu captures: c2 expansion (4096-row batch) and the FWHT at a given length."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1702_08159_b200 as P
from paper_1702_08159_b200 import synthetic

what = sys.argv[1] if len(sys.argv) > 1 else "ff"
if what == "ff":
    spec = P.FeatureMapSpec(784, 16, P.RBFMatern(2.0, 40), 42)
    blocks = P.build_blocks(spec)
    x = torch.from_numpy(synthetic.image_rows(4096, 784, 42)).cuda()
    out = torch.empty((4096, 32768), device="cuda")
    for _ in range(4):
        P.feature_map_batch(spec, blocks, x, out=out)
elif what == "fwht":
    n = int(sys.argv[2])
    buf = torch.randn(1 << 28, device="cuda").view(-1, n)
    for _ in range(3):
        P.wht_fast_batch(buf)
torch.cuda.synchronize()
print("done")

if what == "c3":
    from paper_1702_08159_b200 import synthetic as S
    x, y = S.class_images(60000, 784, 10, seed=1234)
    xt, yt = S.class_images(10000, 784, 10, seed=1234, sample_seed=99)
    spec = P.FeatureMapSpec(784, 8, P.RBF(1.0), 1234)
    tr = P.Trainer(spec, P.Dataset(x, y, 10), P.Dataset(xt, yt, 10), P.TrainConfig(0.01, 1000, 1))
    for s in range(5):
        tr.step(0, s)
    tr.evaluate()
    torch.cuda.synchronize()
    print("c3 done")

if what == "c4":
    from paper_1702_08159_b200.large_scale import FusedClassifier
    spec = P.FeatureMapSpec(16384, 32, P.RBF(4.0), 4)
    fc = FusedClassifier(spec, 10, 1024)
    x = torch.randn((1024, 16384), device="cuda")
    y = torch.randint(0, 10, (1024,), device="cuda", dtype=torch.int32)
    fc.step(x, y, m_total=8192, lr=0.01)
    fc.step(x, y, m_total=8192, lr=0.01)
    torch.cuda.synchronize()
    print("c4 done")
