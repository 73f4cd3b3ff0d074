"""A/B timing of the c2 expansion batch (4096 rows) for several builds of the
library: python tools/ab_ff.py lib1.so lib2.so ...  (each in a subprocess)."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def child():
    sys.path.insert(0, str(ROOT))
    import torch
    import paper_1702_08159_b200 as P
    from paper_1702_08159_b200 import synthetic
    spec = P.FeatureMapSpec(784, 16, P.RBFMatern(2.0, 40), 42)
    blocks = P.build_blocks(spec)
    xs = [torch.from_numpy(synthetic.image_rows(4096, 784, 42 + i)).cuda() for i in range(4)]
    out = torch.empty((4096, 32768), device="cuda")
    for i in range(10):
        P.feature_map_batch(spec, blocks, xs[i % 4], out=out)
    torch.cuda.synchronize()
    ts = []
    for r in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(40):
            P.feature_map_batch(spec, blocks, xs[i % 4], out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 40 * 1e3)
    ts.sort()
    us = ts[len(ts) // 2]
    gbs = 4096 * (784 * 4 + 32768 * 4) / us / 1e3
    print(json.dumps({"us": round(us, 2), "GBps": round(gbs, 1), "all": [round(t, 2) for t in ts]}))


if __name__ == "__main__":
    if sys.argv[1:2] == ["--child"]:
        child()
    else:
        for lib in sys.argv[1:]:
            env = dict(os.environ, MCK_LIB_PATH=str(Path(lib).resolve()))
            r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
            print(lib, r.stdout.strip() or r.stderr[-2000:], flush=True)
