"""Small invocations of every hot kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Cases: fwht (rows 2^10, cluster 2^15 and 2^16, two-phase 2^18), pair (n=1024
expansion, fused gather), ff16k (n=16384 expansion), fused-ffma2, fused-tcgen05
(forward + backward + bucket update), head (c3 softmax head), factors.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1702_08159_b200 as P
from paper_1702_08159_b200 import synthetic

cases = sys.argv[1:] or ["factors", "fwht", "pair", "ff16k", "fused-ffma2", "fused-tcgen05", "head"]
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)

for c in cases:
    if c == "factors":
        P.build_blocks(P.FeatureMapSpec(784, 2, P.RBFMatern(2.0, 3), 5))
        P.build_blocks(P.FeatureMapSpec(300, 2, P.RBF(1.0), 6))
    elif c == "fwht":
        for n, rows in ((1024, 64), (1 << 15, 4), (1 << 16, 4), (1 << 18, 2)):
            P.wht_fast_batch(torch.randn((rows, n), generator=g, device=dev))
        P.wht_fast_batch(torch.randn((8, 1024), generator=g, device=dev), variant="parity")
    elif c == "pair":
        spec = P.FeatureMapSpec(784, 2, P.RBF(1.0), 7)
        bs = P.build_blocks(spec)
        x = torch.from_numpy(synthetic.image_rows(40, 784, 1)).to(dev)
        P.feature_map_batch(spec, bs, x)
        rows = torch.arange(0, 40, 3, dtype=torch.int32, device=dev)
        P.feature_map_batch(spec, bs, x, rows=rows)
    elif c == "ff16k":
        spec = P.FeatureMapSpec(16384, 1, P.RBF(4.0), 4)
        bs = P.build_blocks(spec)
        P.apply_zhat_batch(spec, bs, torch.randn((3, 16384), generator=g, device=dev))
    elif c.startswith("fused"):
        from paper_1702_08159_b200 import _native as nat
        from paper_1702_08159_b200.large_scale import FusedClassifier
        eng = c.split("-")[1]
        spec = P.FeatureMapSpec(1000, 3, P.RBF(2.0), 17)
        fc = FusedClassifier(spec, 10, 40, engine=eng, bucket_blocks=2)
        x = torch.randn((40, 1000), generator=g, device=dev)
        y = torch.randint(0, 10, (40,), generator=g, device=dev, dtype=torch.int32)
        fc.step(x, y, lr=0.1)
        fc.forward(x, y)
        fc._alloc_buckets()
        for (e0, cnt), buf in zip(fc.bucket_ranges(), fc._buckets):
            nat.call("mck_fused_backward_bucket", *fc._bwd_args(), e0, cnt, nat.ptr(buf),
                     nat.ptr(fc.scratch), fc.variant, nat.stream_handle(dev))
    elif c == "head":
        xs, ys = synthetic.class_images(300, 64, 10, seed=3)
        cfg = P.TrainConfig(0.05, 100, 1)
        P.train(P.FeatureMapSpec(64, 2, P.RBF(1.0), 2), P.Dataset(xs, ys, 10),
                P.Dataset(xs[:50], ys[:50], 10), cfg)
    torch.cuda.synchronize()
    print("case ok:", c, flush=True)
