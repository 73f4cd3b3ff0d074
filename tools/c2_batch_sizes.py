import sys
sys.path.insert(0, '.')
import torch
import paper_1702_08159_b200 as P
from paper_1702_08159_b200 import synthetic
spec = P.FeatureMapSpec(784, 16, P.RBFMatern(2.0, 40), 42)
blocks = P.build_blocks(spec)
x = torch.from_numpy(synthetic.image_rows(60000, 784, 42)).cuda()
out = torch.empty((4096, 32768), device="cuda")
for rows in (4096, 2656, 1000):
    for _ in range(5):
        P.feature_map_batch(spec, blocks, x[:rows], out=out)
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); a.record()
    for i in range(20):
        r0 = (i * 4096) % 50000
        P.feature_map_batch(spec, blocks, x[r0:r0 + rows], out=out)
    b.record(); torch.cuda.synchronize()
    print(rows, "rows:", round(a.elapsed_time(b) / 20 * 1e3, 1), "us")
