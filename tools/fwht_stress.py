"""Stress the persistent / cluster FWHT kernels: many calls with varying row counts, two streams, checked against a float64 butterfly."""
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


torch.manual_seed(0)
bad = 0
for k in (14, 15, 16, 17, 18, 19, 20):
    n = 1 << k
    for rows in (1, 2, 3, 5, 7, 33, 34, 73, 74, 75, 147, 148, 149, 150, 295, 296, 297, 301, 450, 593):
        if rows * n > (1 << 27):
            continue
        x = torch.randn(rows, n, device="cuda")
        want = ref(x)
        for rep in range(3):
            got = P.wht_fast_batch(x.clone())
            err = ((got.double() - want).abs().max() / want.abs().max()).item()
            if not err < 1e-6:
                bad += 1
                print(f"FAIL 2^{k} rows={rows} rep={rep} err={err:.3e}")
    # two streams at once, many back-to-back calls
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    rows = max(1, min(300, (1 << 26) // n))
    a = torch.randn(rows, n, device="cuda"); b = torch.randn(rows, n, device="cuda")
    wa, wb = ref(a), ref(b)
    torch.cuda.synchronize()
    outs = []
    for i in range(10):
        ca, cb = a.clone(), b.clone()
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            P.wht_fast_batch(ca)
        with torch.cuda.stream(s2):
            P.wht_fast_batch(cb)
        torch.cuda.synchronize()
        ea = ((ca.double() - wa).abs().max() / wa.abs().max()).item()
        eb = ((cb.double() - wb).abs().max() / wb.abs().max()).item()
        if not (ea < 1e-6 and eb < 1e-6):
            bad += 1
            print(f"FAIL two streams 2^{k} it={i} {ea:.3e} {eb:.3e}")
    print(f"2^{k} done")
print("FAILURES", bad)
