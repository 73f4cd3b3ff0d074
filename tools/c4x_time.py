"""c4 expansion (256 rows, materialised) and fused step timing for A/B of library builds."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
spec4 = P.FeatureMapSpec(16384, 32, P.RBF(4.0), 4)
b4 = P.build_blocks(spec4)
x4 = torch.randn((256, 16384), device="cuda")
o4 = torch.empty((256, 1 << 20), device="cuda")
for _ in range(2):
    P.feature_map_batch(spec4, b4, x4, normalize=False, out=o4)
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
torch.cuda.synchronize(); s.record()
for _ in range(5):
    P.feature_map_batch(spec4, b4, x4, normalize=False, out=o4)
e.record(); torch.cuda.synchronize()
print(f"c4 expansion 256 rows: {s.elapsed_time(e)/5:.3f} ms")
