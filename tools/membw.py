"""HBM write-only / read-only / copy bandwidth probe (torch kernels), for roofline context."""
import torch
n = 1 << 30  # 4 GiB fp32
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3
tw = t(lambda: a.fill_(1.0)); print(f"write-only fill: {4*n/tw/1e9:.0f} GB/s")
tc = t(lambda: b.copy_(a)); print(f"copy (r+w): {8*n/tc/1e9:.0f} GB/s")
tr = t(lambda: a.sum()); print(f"read-only sum: {4*n/tr/1e9:.0f} GB/s")
x = torch.empty(60000 * 784, device="cuda")
o = torch.empty(4096 * 32768, device="cuda")
tw2 = t(lambda: o.fill_(0.5), 50); print(f"write 537MB: {o.numel()*4/tw2/1e9:.0f} GB/s  {tw2*1e6:.1f} us")
