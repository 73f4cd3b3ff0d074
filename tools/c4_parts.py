"""Time the config-4 fused forward and backward separately (1024 rows of one rank).

    MCK_LIB_PATH=... python tools/c4_parts.py [--engine=ffma2|tcgen05|reference]
"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P
from paper_1702_08159_b200.large_scale import FusedClassifier

eng = next((a.split("=")[1] for a in sys.argv if a.startswith("--engine=")), "ffma2")
spec = P.FeatureMapSpec(16384, 32, P.RBF(4.0), 4)
fc = FusedClassifier(spec, 10, 1024, engine=eng)
x = torch.randn((1024, 16384), device="cuda")
y = torch.randint(0, 10, (1024,), device="cuda", dtype=torch.int32)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


f = timed(lambda: fc.forward(x, y, m_total=8192))
b = timed(lambda: fc.backward(lr=0.01))
print(f"{os.path.basename(os.environ.get('MCK_LIB_PATH', 'default'))} engine={eng}: "
      f"forward {f:.3f} ms  backward {b:.3f} ms")
