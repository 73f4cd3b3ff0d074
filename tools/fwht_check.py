"""Correctness + speed of wht_fast_batch at 2^k (k from argv) against a float64 torch butterfly."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1702_08159_b200 as P


def ref(x):
    y = x.double()
    m, n = y.shape
    h = 1
    while h < n:
        y = y.view(m, n // (2 * h), 2, h)
        y = torch.stack((y[:, :, 0] + y[:, :, 1], y[:, :, 0] - y[:, :, 1]), 2).reshape(m, n)
        h *= 2
    return y


ks = [int(a) for a in sys.argv[1:]] or [16]
for k in ks:
    for rows in (1, 3, 149, 300):
        g = torch.Generator(device="cuda").manual_seed(k * 1000 + rows)
        x = torch.randn(rows, 1 << k, device="cuda", generator=g)
        want = ref(x)
        got = P.wht_fast_batch(x.clone())
        err = ((got.double() - want).abs().max() / want.abs().max()).item()
        print(f"2^{k} rows={rows}: scale-relative err {err:.2e}", "OK" if err < 1e-6 else "FAIL")
    buf = torch.randn(1 << 28, device="cuda")
    mat = buf.view(-1, 1 << k)
    for _ in range(2):
        P.wht_fast_batch(mat)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(10):
        P.wht_fast_batch(mat)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"2^{k}: {ms:.3f} ms  {2**31/ms/1e6:.0f} GB/s  {2**31/ms/1e6/6554.2:.3f}")
