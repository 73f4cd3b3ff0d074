"""Pinned device-to-host copy bandwidth (the ceiling of bench.py's e2e leg)."""
import torch, time
dev = torch.device("cuda")
n = 537 * 1024 * 1024 // 4
src = [torch.empty(n, device=dev) for _ in range(2)]
dst = [torch.empty(n, pin_memory=True) for _ in range(4)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for k in range(2):
    dst[k].copy_(src[k], non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(8):
    dst[k % 4].copy_(src[k % 2], non_blocking=True)
torch.cuda.synchronize()
print("1 stream D2H GB/s", 8 * n * 4 / (time.perf_counter() - t0) / 1e9)
t0 = time.perf_counter()
for k in range(8):
    with torch.cuda.stream(s1 if k % 2 == 0 else s2):
        dst[k % 4].copy_(src[k % 2], non_blocking=True)
torch.cuda.synchronize()
print("2 streams D2H GB/s", 8 * n * 4 / (time.perf_counter() - t0) / 1e9)
