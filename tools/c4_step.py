"""Time the config-4 fused training step (1024 rows of one rank) and the c3 step."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
from paper_1702_08159_b200.large_scale import FusedClassifier

spec = P.FeatureMapSpec(16384, 32, P.RBF(4.0), 4)
eng = next((a.split("=")[1] for a in sys.argv if a.startswith("--engine=")), "ffma2")
M = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--rows=")), 1024))
fc = FusedClassifier(spec, 10, M, engine=eng)
x = torch.randn((M, 16384), device="cuda")
y = torch.randint(0, 10, (M,), device="cuda", dtype=torch.int32)
for _ in range(2):
    fc.step(x, y, m_total=8192, lr=0.01)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(5):
    fc.step(x, y, m_total=8192, lr=0.01)
e.record()
torch.cuda.synchronize()
print(f"c4 step {s.elapsed_time(e) / 5:.3f} ms  (engine={eng})")
