"""c2 step (60000 rows, 4096-row batches) under several stream / output-buffer schedules."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
from paper_1702_08159_b200 import synthetic
spec = P.FeatureMapSpec(784, 16, P.RBFMatern(2.0, 40), 42)
bs = P.build_blocks(spec)
x = torch.from_numpy(synthetic.image_rows(60000, 784, 42)).cuda()
W = P.feature_dim(spec)
outs = [torch.empty((4096, W), device="cuda") for _ in range(4)]
spans = [(r0, min(60000, r0 + 4096)) for r0 in range(0, 60000, 4096)]
main = torch.cuda.current_stream()
streams = [torch.cuda.Stream() for _ in range(4)]
def sched(ns, nout):
    def fn():
        for q in streams[:ns]: q.wait_stream(main)
        for k, (r0, r1) in enumerate(spans):
            with torch.cuda.stream(streams[k % ns]):
                P.feature_map_batch(spec, bs, x[r0:r1], out=outs[k % nout])
        for q in streams[:ns]: main.wait_stream(q)
    return fn
def timed(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
alg = sum((r1 - r0) for r0, r1 in spans) * (784 * 4 + W * 4)
for ns, nout in ((1, 1), (2, 2), (2, 4), (3, 3), (4, 4)):
    ms = timed(sched(ns, nout))
    print(f"{ns} streams / {nout} outputs: {ms:.3f} ms  frac {alg / (ms / 1e3) / 1e9 / 6553:.4f}")
