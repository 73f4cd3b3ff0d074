#!/usr/bin/env python
"""Benchmark of the B200 Fastfood hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (config 2 of BASELINE.json, the largest single-GPU expansion):
Matern kernel (sigma=2, t=40), d=784 padded to n=1024, E=16 -> 32,768 features
per row, over N=60,000 image-shaped rows (~80% exact zeros, rest U(0,1]),
streamed in batches of 4,096 rows.  One step = one pass over the 60,000 rows
(15 fused-expansion launches alternating between two streams and two reused
4,096-row output buffers; inputs 188 MB and each batch's output 537 MB exceed
the 126 MB L2, so no flush is needed).  Multi-GPU: every rank expands its own 60,000-row shard (weak
scaling, no collective on the data path); value = all ranks' features / max
rank time.

`--gpus N` without torchrun re-launches itself under
`torch.distributed.run` with N local ranks (NCCL, 127.0.0.1).

Extras (every rank, barrier + max-over-ranks device time; each with its
roofline and, at N = 1 on rank 0, the reference CPU path on the host cores):
c0 steady state (graph replay of back-to-back 1,000-row batches), the c1
FWHT sweep (rows of each length split over the ranks), c3 training (step
time, 20 epochs to the final accuracy; batches sharded + NCCL all-reduce at
N > 1) and the c4 fused training step (1,024 rows per rank of the 8,192-row
batch; bucketed all-reduce at N > 1) with its FP32 lane-op and MUFU
fractions.  --impl reference times the reference algorithm (the numpy oracle
port of mckernel, tests-pinned bit-exact to the reference) on this host's
cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

C2 = dict(d=784, E=16, sigma=2.0, t=40, seed=42, rows=60000, batch=4096, xseed=42)
METRIC = "Fastfood expanded features/s; batched FWHT GB/s vs HBM peak, 1/2/4/8 B200"


def env_int(k, d):
    return int(os.environ.get(k, d))


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return float(j["hbm_gbs"]), "measured", j
    return 6650.0, "fallback", {}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons during the timed region with a
    separate `nvidia-smi -lms` process (no GIL contention with the launches)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, interval_ms: int = 20):
        self.index, self.interval = index, interval_ms
        self.proc, self.lines = None, []

    def __enter__(self):
        import subprocess
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.interval)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # first sample before the timed region starts
        except OSError as exc:
            self.error = str(exc)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------ distributed
def dist_setup(backend):
    ws = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if ws > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # communicator log on stderr (ranks, channels, NVLS) for the driver
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, local, ws


def comm_info(ws):
    if ws == 1:
        return None
    import torch
    import torch.distributed as dist
    v = torch.cuda.nccl.version() if hasattr(torch.cuda, "nccl") else None
    return {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
            "nccl_version": ".".join(map(str, v)) if isinstance(v, tuple) else v}


def relaunch(args) -> int:
    """`bench.py --gpus N` outside torchrun: start N local ranks under torch.distributed.run."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "1")
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, ws, device):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ ours
def c2_spec(P):
    return P.FeatureMapSpec(C2["d"], C2["E"], P.RBFMatern(C2["sigma"], C2["t"]), C2["seed"])


def bench_ours(args):
    import numpy as np
    import torch

    import paper_1702_08159_b200 as P
    from paper_1702_08159_b200 import synthetic
    from paper_1702_08159_b200.streaming import HostStreamer

    # MCK_BENCH_BACKEND=gloo MCK_BENCH_SAME_DEVICE=1: code-path check of the
    # multi-rank legs on a one-GPU box (every rank on cuda:0, host-mediated
    # collectives; the numbers are not a scaling measurement)
    backend = os.environ.get("MCK_BENCH_BACKEND", "nccl")
    rank, local, ws = dist_setup(backend)
    if os.environ.get("MCK_BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    if rank == 0 and ws > 1:
        print(f"[bench] world_size={ws} backend={backend}", file=sys.stderr, flush=True)
    dev = torch.device("cuda", local)
    hbm, peak_kind, peak_json = peaks()

    spec = c2_spec(P)
    t0 = time.perf_counter()
    blocks = P.build_blocks(spec)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0

    rows, batch = C2["rows"], C2["batch"]
    width = P.feature_dim(spec)
    x_host = synthetic.image_rows(rows, C2["d"], C2["xseed"] + rank)
    x = torch.from_numpy(x_host).to(dev)
    # two batch output buffers and two streams: consecutive batches are
    # independent, so batch k+1's ramp-up overlaps batch k's tail
    outs = [torch.empty((batch, width), dtype=torch.float32, device=dev) for _ in range(2)]
    spans = [(r0, min(rows, r0 + batch)) for r0 in range(0, rows, batch)]
    stream = torch.cuda.current_stream(dev)
    bstreams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]

    def step(evs=None):
        if evs is not None:  # per-launch events: one stream, launches serialised
            for k, (r0, r1) in enumerate(spans):
                evs[k][0].record(stream)
                P.feature_map_batch(spec, blocks, x[r0:r1], out=outs[0])
                evs[k][1].record(stream)
            return
        for q in bstreams:
            q.wait_stream(stream)
        for k, (r0, r1) in enumerate(spans):
            with torch.cuda.stream(bstreams[k % 2]):
                P.feature_map_batch(spec, blocks, x[r0:r1], out=outs[k % 2])
        for q in bstreams:
            stream.wait_stream(q)

    for _ in range(args.warmup):
        step()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(ws)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start.record(stream)
        for s in range(args.steps):
            step()
        end.record(stream)
        torch.cuda.synchronize()
    barrier(ws)
    ms = start.elapsed_time(end) / args.steps
    ms = max_over_ranks(ms, ws, dev)
    feats_per_step = rows * width
    value = ws * feats_per_step / (ms / 1e3)

    # roofline of the dominant kernel (k_fastfood_pair, the only kernel in the
    # step): algorithmic bytes = input row read once + feature row written
    # once, over the timed region (CUDA events on the
    # stream that forks and joins the two batch streams; gaps included).  A
    # second pass with events around every launch on one stream (launches
    # serialised, kept out of `value`) gives the per-launch rate.
    bytes_per_row = C2["d"] * 4 + width * 4
    step_bytes = sum((r1 - r0) * bytes_per_row for r0, r1 in spans)
    achieved = step_bytes / (ms / 1e3) / 1e9
    rsteps = max(1, min(args.steps, 20))
    launch_evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in spans] for _ in range(rsteps)]
    for s in range(rsteps):
        step(launch_evs[s])
    torch.cuda.synchronize()
    tot_ms = tot_bytes = 0.0
    for s in range(rsteps):
        for k, (r0, r1) in enumerate(spans):
            tot_ms += launch_evs[s][k][0].elapsed_time(launch_evs[s][k][1])
            tot_bytes += (r1 - r0) * bytes_per_row
    achieved_evented = tot_bytes / (tot_ms / 1e3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("k_fastfood_c2", {}).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "kernel": "k_fastfood_pair<FEAT=1,FOLD=1,VEC=1> (n=1024, two rows per thread; scale 1/64 folded into C)",
                "alg_bytes_per_launch": int(batch * bytes_per_row),
                "avg_launch_us": round(ms / len(spans) * 1e3, 2),
                "achieved_source": "step bytes / timed region (15 launches on two streams, gaps included)",
                "evented": {"achieved": round(achieved_evented, 1),
                            "frac": round(achieved_evented / hbm, 4),
                            "avg_launch_us": round(tot_ms / (rsteps * len(spans)) * 1e3, 2),
                            "launches": rsteps * len(spans)}}

    # end-to-end through the host-buffer API (pinned host in/out, copies timed)
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(x_host).pin_memory()
        oh = torch.empty((rows, width), dtype=torch.float32, pin_memory=True)
        hs = HostStreamer(spec, blocks, batch)
        hs.run(xh, oh)                              # warm-up
        n_e2e = max(1, min(args.steps, 3))
        barrier(ws)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            hs.run(xh, oh)
        torch.cuda.synchronize()
        e2e_s = max_over_ranks((time.perf_counter() - t0) / n_e2e, ws, dev)
        e2e = {"value": ws * feats_per_step / e2e_s, "unit": "features/s",
               "h2d_bytes_per_step": int(xh.numel() * 4), "d2h_bytes_per_step": int(oh.numel() * 4),
               "ms_per_step": round(e2e_s * 1e3, 3),
               "bound": "PCIe device->host copy of the float32 features",
               "d2h_GBps": round(oh.numel() * 4 / e2e_s / 1e9, 1),
               "path": "paper_1702_08159_b200.streaming.HostStreamer.run (feature_map_batch per "
                       "4096-row batch; pinned host x and features; H2D/compute/D2H overlapped)"}
        del oh, xh

    line = {
        "metric": METRIC, "value": value, "unit": "features/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded MNIST-shaped rows: ~80% exact zeros, rest U(0,1]; MNIST absent)",
        "config": {"workload": "c2: Fastfood Matern expansion (sigma=2, t=40), 60000x784 -> "
                               "32768 features/row, E=16, n=1024, batches of 4096",
                   "rows_per_rank": rows, "batch_rows": batch, "expansions": C2["E"],
                   "padded_dim": 1024, "features_per_row": width,
                   "l2_policy": "inputs (188 MB) and per-batch outputs (537 MB) exceed L2",
                   "schedule": "15 batch launches alternating over 2 streams / 2 output buffers",
                   "parallelism": f"row shards x{ws} (no collective)"},
        "roofline": roofline, "e2e": e2e, "gpu_launches": args.steps * len(spans),
        "clocks": clk.summary(), "setup_s": {"build_blocks_c2": round(setup_s, 4)},
        "comm": comm_info(ws),
    }
    cpu = rank == 0 and ws == 1 and not args.no_cpu
    if not args.no_extras:
        del outs
        torch.cuda.empty_cache()
        line["extras"] = extras(args, P, torch, dev, hbm, rank, ws, cpu)
    if cpu:
        line["cpu_baseline"] = cpu_baseline_c2(sample_rows=args.cpu_rows, reps=2)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def timed(fn, reps, torch, ws, dev, stream=None):
    """ms per call: barrier + synchronize on both sides, CUDA events on the
    launching stream, max over ranks."""
    stream = stream or torch.cuda.current_stream(dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(ws)
    torch.cuda.synchronize()
    s.record(stream)
    for _ in range(reps):
        fn()
    e.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    return max_over_ranks(s.elapsed_time(e) / reps, ws, dev)


def sm_clock_hz():
    _, _, pj = peaks()
    return float(pj.get("sm_max_mhz", 1965.0)) * 1e6


def extras(args, P, torch, dev, hbm, rank, ws, cpu):
    """Per-config legs, each with a roofline and (N=1,
    rank 0) the reference CPU path.  Every rank runs every leg; times are the
    max over ranks; values are whole-job aggregates."""
    from paper_1702_08159_b200 import synthetic
    from paper_1702_08159_b200.distributed import shard_range
    out = {}
    cores = os.cpu_count() or 1

    # ---- config 0: RBF E=8, 1000 x 784 -> 16384 features/row.  Steady state:
    # 20 back-to-back batches replayed from one CUDA graph; 4 rotating output
    # buffers (262 MB > L2) so no write is absorbed by L2.
    spec0 = P.FeatureMapSpec(784, 8, P.RBF(1.0), 1234)
    b0 = P.build_blocks(spec0)
    x0 = torch.from_numpy(synthetic.image_rows(1000, 784, 1234 + rank)).to(dev)
    o0 = [torch.empty((1000, 16384), device=dev) for _ in range(4)]
    P.feature_map_batch(spec0, b0, x0, out=o0[0])
    one_ms = timed(lambda: P.feature_map_batch(spec0, b0, x0, out=o0[0]), 50, torch, ws, dev)
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        for k in range(20):
            P.feature_map_batch(spec0, b0, x0, out=o0[k % 4])
    graph.replay()
    g_ms = timed(graph.replay, 10, torch, ws, dev) / 20
    # the same 20 independent batches on two streams (fork/join inside one
    # graph), so one batch's ramp-up overlaps the other's tail
    s2 = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    graph2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph2, stream=side):
        for q in s2:
            q.wait_stream(side)
        for k in range(20):
            with torch.cuda.stream(s2[k % 2]):
                P.feature_map_batch(spec0, b0, x0, out=o0[k % 4])
        for q in s2:
            side.wait_stream(q)
    graph2.replay()
    g2_ms = timed(graph2.replay, 10, torch, ws, dev) / 20
    bpr0 = 784 * 4 + 16384 * 4
    gbs0 = 1000 * bpr0 / (min(g_ms, g2_ms) / 1e3) / 1e9
    out["c0"] = {"workload": "RBF sigma=1, E=8, 1000x784 -> 16384 features/row per rank",
                 "ms_per_batch_single_launch": round(one_ms, 4),
                 "ms_per_batch_steady_one_stream": round(g_ms, 4),
                 "ms_per_batch_steady": round(min(g_ms, g2_ms), 4),
                 "features_per_s": ws * 1000 * 16384 / (min(g_ms, g2_ms) / 1e3),
                 "roofline": {"bound": "hbm", "kernel": "k_fastfood_pair (n=1024)",
                              "achieved": round(gbs0, 1), "peak": hbm, "unit": "GB/s",
                              "frac": round(gbs0 / hbm, 4),
                              "alg_bytes_per_batch": 1000 * bpr0,
                              "method": "graph of 20 independent back-to-back batches, 4 rotating "
                                        "outputs; best of one stream and two streams"}}
    del o0, graph, graph2
    if cpu:
        out["c0"]["cpu_baseline"] = cpu_features(spec0, synthetic.image_rows(1000, 784, 1234), cores)

    # ---- config 1: FWHT sweep, 2^28 floats (1 GiB) per length in place, rows
    # split over the ranks; GB/s on algorithmic bytes (read + write once).
    sweep = {}
    total = 1 << 28
    g = torch.Generator(device=dev).manual_seed(7 + rank)
    buf = torch.randn(total // ws + (1 << 20), generator=g, device=dev)
    for k in range(10, 21):
        n = 1 << k
        rows = total // n
        lo, hi = shard_range(rows, rank, ws)
        mat = buf[:(hi - lo) * n].view(-1, n) if hi > lo else None
        fn = (lambda: P.wht_fast_batch(mat)) if mat is not None else (lambda: None)
        fn()
        ms = timed(fn, 5, torch, ws, dev)
        gbs = 2 ** 31 / (ms / 1e3) / 1e9
        kern = ("fwht_rows_kernel" if k <= 13 else "fwht_persistent14_kernel" if k == 14
                else "fwht_tmem_first_kernel (row on one SM)" if k <= 16
                else "fwht_tmem_virtual_kernel (two virtual rows per row)" if k == 17
                else "fwht_tmem_cluster_kernel" if k == 18 else "two-phase (columns + rows)")
        sweep[str(n)] = {"ms": round(ms, 4), "GBps": round(gbs, 1), "frac": round(gbs / hbm, 4),
                         "rows_per_rank": hi - lo, "kernel": kern}
    del buf
    if cpu:
        cpu_sweep = cpu_wht_sweep(cores)
        for n, v in cpu_sweep.items():
            sweep[n]["cpu_baseline"] = v
    out["c1_fwht_sweep"] = sweep

    # ---- config 4: fused expansion -> classifier training step, 1024 rows per
    # rank of the 8192-row global batch (features never in HBM).
    from paper_1702_08159_b200.large_scale import FusedClassifier
    spec4 = P.FeatureMapSpec(16384, 32, P.RBF(4.0), 4)
    t0 = time.perf_counter()
    fc = FusedClassifier(spec4, 10, 1024)
    torch.cuda.synchronize()
    setup4 = time.perf_counter() - t0
    x4 = torch.randn((1024, 16384), generator=torch.Generator(device=dev).manual_seed(7 + rank),
                     device=dev)
    y4 = torch.randint(0, 10, (1024,), device=dev, dtype=torch.int32,
                       generator=torch.Generator(device=dev).manual_seed(8 + rank))
    mt = 8192 if ws <= 8 else 1024 * ws          # global batch; this rank's shard is 1024 rows
    for _ in range(2):
        fc.step(x4, y4, m_total=mt, lr=0.01)
    ms4 = timed(lambda: fc.step(x4, y4, m_total=mt, lr=0.01), 5, torch, ws, dev)
    n4, E4, rows4 = 16384, 32, 1024
    # algorithmic lane work per step: one expansion of every (row, block):
    # 2 FWHTs x (n/2 log2 n butterflies x 2 add/sub) + G and C multiplies
    # (the backward reuses the forward's z); MUFU: cos and sin of every z in
    # the forward and again in the backward (features are never stored).
    lane_ops = rows4 * E4 * (2 * (n4 // 2) * 14 * 2 + 2 * n4)
    mufu = 2 * rows4 * E4 * 2 * n4
    f_sm = sm_clock_hz()
    lane_peak = 148 * 128 * f_sm
    mufu_peak = 148 * 16 * f_sm
    ach_l = lane_ops / (ms4 / 1e3)
    ach_m = mufu / (ms4 / 1e3)
    out["c4_fused_step"] = {
        "workload": "RBF sigma=4, n=d=16384, E=32 -> 2^20 features/row, 10 classes; "
                    "1024 rows per rank of the 8192-row global batch; fwd + bwd (recomputed "
                    "expansion) + SGD, features never written to HBM",
        "rows_per_rank": rows4, "ms_per_step": round(ms4, 3),
        "features_per_s": ws * rows4 * (1 << 20) / (ms4 / 1e3),
        "epoch_s": round((1 << 20) / (rows4 * ws) * ms4 / 1e3, 3),   # 2^20 rows at 1024 rows/rank/step
        "build_blocks_s": round(setup4, 3),
        "allreduce": (f"{len(fc.bucket_ranges())} float32 buckets of {fc.bucket_blocks} blocks "
                      f"(+ float64 [db|loss|hits]), overlapped with the backward" if ws > 1 else None),
        "roofline": {"bound": "fp32 lanes / MUFU", "unit": "op/s",
                     "lane_ops_per_step": lane_ops, "achieved": ach_l, "peak": lane_peak,
                     "frac": round(ach_l / lane_peak, 4),
                     "mufu_per_step": mufu, "mufu_achieved": ach_m, "mufu_peak": mufu_peak,
                     "mufu_frac": round(ach_m / mufu_peak, 4),
                     "peak_source": "148 SMs x 128 FP32 lanes (16 MUFU/clk) x sm_max_mhz; "
                                    "packed f32x2 ops counted as 2"}}
    if cpu:
        out["c4_fused_step"]["cpu_baseline"] = cpu_c4(spec4, fc, x4, y4, cores)
    del fc, x4, y4
    torch.cuda.empty_cache()

    # ---- config 3: end-to-end SGD, 60000 x 784, RBF E=8, batch 1000, lr 0.01,
    # 20 epochs; every global batch sharded over the ranks.
    x, y = synthetic.class_images(60000, 784, 10, seed=1234)
    xt, yt = synthetic.class_images(10000, 784, 10, seed=1234, sample_seed=99)
    cfg = P.TrainConfig(0.01, 1000, 20)
    tr = P.Trainer(spec0, P.Dataset(x, y, 10), P.Dataset(xt, yt, 10), cfg)
    tr.run_epoch(0)
    ms_epoch = timed(lambda: tr.run_epoch(1), 1, torch, ws, dev)
    tr.evaluate()
    barrier(ws)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    model, metrics = P.train(spec0, P.Dataset(x, y, 10), P.Dataset(xt, yt, 10), cfg)
    t20 = max_over_ranks(time.perf_counter() - t0, ws, dev)
    step_ms = ms_epoch / tr.steps
    c3_bytes = 1000 * (784 * 4 + 3 * 16384 * 4)   # x once; phi written, read by fwd and bwd
    gbs3 = c3_bytes / (step_ms / 1e3) / 1e9
    out["c3_train"] = {
        "workload": "60000x784 10-class synthetic, RBF sigma=1 E=8 (16384 features), softmax "
                    "head, batch 1000, lr 0.01, 20 epochs; eval on 10000 rows each epoch",
        "ms_per_step": round(step_ms, 4), "ms_per_epoch_steps": round(ms_epoch, 3),
        "features_per_s": 60000 * 16384 / (ms_epoch / 1e3),
        "time_to_20_epochs_s": round(t20, 3),
        "final_test_acc": metrics.records[-1].test_acc,
        "final_train_loss": metrics.records[-1].train_loss,
        "loss_history": [round(r.train_loss, 6) for r in metrics.records],
        "roofline": {"bound": "hbm", "achieved": round(gbs3, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(gbs3 / hbm, 4), "alg_bytes_per_step": c3_bytes,
                     "note": "x rows once + phi (65.5 MB) written and read by the forward and "
                             "backward (SURVEY 8d, ~200 MB/step); the step is latency-bound"}}
    if cpu:
        out["c3_train"]["cpu_baseline"] = cpu_c3(spec0, x, y, cores)
    return out


def cpu_features(spec, x, cores, reps=2):
    """Reference feature_map_batch (oracle port) over a thread pool, BLAS 1 thread."""
    import concurrent.futures as cf
    import numpy as np
    from threadpoolctl import threadpool_limits
    from oracle import fastfood as off
    ospec = off.OSpec.of(spec)
    with threadpool_limits(1):
        blocks = off.build_blocks(ospec)
        chunks = [c for c in np.array_split(x, 4 * cores) if len(c)]
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            with cf.ThreadPoolExecutor(cores) as ex:
                list(ex.map(lambda c: off.feature_map_batch(ospec, blocks, c), chunks))
            times.append(time.perf_counter() - t0)
    return {"value": len(x) * 2 * ospec.n * ospec.expansions / min(times), "unit": "features/s",
            "cores": cores, "kind": "port",
            "sample": f"all {len(x)} rows, ThreadPool x{cores}, 1 BLAS thread, best of {reps}"}


def cpu_wht_sweep(cores, floats=1 << 22):
    """Reference wht_fast_batch (oracle port) per length on `floats` floats."""
    import concurrent.futures as cf
    import numpy as np
    from threadpoolctl import threadpool_limits
    from oracle import wht as ow
    res = {}
    rng = np.random.default_rng(7)
    base = rng.standard_normal(floats).astype(np.float32)
    with threadpool_limits(1):
        for k in range(10, 21):
            n = 1 << k
            mat = base.copy().reshape(-1, n)
            chunks = [c for c in np.array_split(mat, min(cores, mat.shape[0])) if len(c)]
            best = None
            for _ in range(2):
                parts = [np.ascontiguousarray(c) for c in chunks]
                t0 = time.perf_counter()
                with cf.ThreadPoolExecutor(len(parts)) as ex:
                    list(ex.map(ow.wht_fast_batch, parts))
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
            res[str(n)] = {"GBps": round(floats * 8 / best / 1e9, 3), "cores": len(chunks),
                           "kind": "port", "sample": f"{floats} floats ({mat.shape[0]} rows)"}
    return res


def cpu_c3(spec, x, y, cores, steps=3):
    """Reference train step (oracle port: featurize, loss, sgd_step -- the
    forward runs twice, linear_model.py:218-219) with BLAS on all cores;
    extrapolated to s/epoch (60 steps) and 20 epochs."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    from oracle import fastfood as off
    from oracle import linear_model as olm
    ospec = off.OSpec.of(spec)
    blocks = off.build_blocks(ospec)
    w, b = np.zeros((10, 16384)), np.zeros(10)
    order = olm.epoch_order(0, 0, len(y))
    times = []
    with threadpool_limits(cores):
        for s in range(steps):
            idx = order[s * 1000:(s + 1) * 1000]
            t0 = time.perf_counter()
            xb = off.feature_map_batch(ospec, blocks, x[idx], normalize=False)
            olm.loss(w, b, xb, y[idx])
            olm.sgd_step(w, b, xb, y[idx], 0.01)
            times.append(time.perf_counter() - t0)
    st = float(np.median(times))
    return {"value": 1000 * 16384 / st, "unit": "features/s", "cores": cores, "kind": "port",
            "s_per_step": round(st, 4), "s_per_epoch": round(60 * st, 2),
            "time_to_20_epochs_s": round(1200 * st, 1),
            "sample": f"{steps} steps of 1000 rows (median), BLAS threads = {cores}; "
                      "evaluation excluded"}


def cpu_c4(spec, fc, x4, y4, cores, rows=4):
    """Reference path for config 4 on a sample: featurize `rows` rows through
    all 32 blocks (materialised, as the reference must), loss + sgd_step on
    them; extrapolated to one rank's 1024-row step.  The factor tables are the
    product's (identical to the reference's; building C-RBF on the CPU takes
    ~30 s per block), which does not change the timed work."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    from oracle import fastfood as off
    from oracle import linear_model as olm
    ospec = off.OSpec.of(spec)
    blocks = [off.OBlock(*fc.blocks[e].numpy(), e) for e in range(spec.expansions)]
    x = x4[:rows].cpu().numpy()
    y = y4[:rows].cpu().numpy().astype(np.int64)
    w, b = np.zeros((10, 1 << 20)), np.zeros(10)
    with threadpool_limits(cores):
        t0 = time.perf_counter()
        xb = off.feature_map_batch(ospec, blocks, x, normalize=False)
        olm.loss(w, b, xb, y)
        olm.sgd_step(w, b, xb, y, 0.01)
        dt = time.perf_counter() - t0
    per_row = dt / rows
    return {"value": rows * (1 << 20) / dt, "unit": "features/s", "cores": cores, "kind": "port",
            "s_per_rank_step_extrapolated": round(per_row * 1024, 2),
            "epoch_h_extrapolated": round(per_row * (1 << 20) / 3600, 2),
            "sample": f"{rows} rows x 32 blocks (n=16384), featurize + loss + sgd_step, "
                      f"extrapolated x{1024 // rows} to a 1024-row rank step"}


# ------------------------------------------------------------------ CPU / reference
def cpu_baseline_c2(sample_rows=4096, reps=2, warmup=0, steps=None):
    """Reference algorithm (numpy oracle port, bit-exact to mckernel) on the host cores.

    Mirrors the reference CLI's `features --workers` harness (cli.py:233-241):
    a thread pool of one worker per core over row chunks, BLAS pinned to one
    thread.  Returns the cpu_baseline object; value in features/s.
    """
    import concurrent.futures as cf
    import multiprocessing as mp

    import numpy as np
    from threadpoolctl import threadpool_limits

    from oracle import fastfood as off
    from paper_1702_08159_b200 import synthetic

    cores = os.cpu_count() or 1
    ospec = off.OSpec(C2["d"], C2["E"], "matern", C2["sigma"], C2["t"], C2["seed"])
    t0 = time.perf_counter()
    with threadpool_limits(1):
        ctx = mp.get_context("fork")
        with ctx.Pool(min(cores, ospec.expansions)) as pool:
            blocks = pool.starmap(off.build_block, [(ospec, e) for e in range(ospec.expansions)])
    build_s = time.perf_counter() - t0
    x = synthetic.image_rows(C2["rows"], C2["d"], C2["xseed"])[:sample_rows]
    chunks = [c for c in np.array_split(x, 4 * cores) if len(c)]

    def run():
        with cf.ThreadPoolExecutor(cores) as ex:
            parts = list(ex.map(lambda c: off.feature_map_batch(ospec, blocks, c), chunks))
        return parts

    times = []
    with threadpool_limits(1):
        for _ in range(warmup):
            run()
        for _ in range(reps if steps is None else steps):
            t0 = time.perf_counter()
            run()
            times.append(time.perf_counter() - t0)
    width = 2 * ospec.n * ospec.expansions
    best = min(times)
    return {"value": sample_rows * width / best, "unit": "features/s", "cores": cores,
            "kind": "port",
            "sample": f"c2 rows 0..{sample_rows - 1} of 60000 (one {sample_rows}-row batch), "
                      f"feature_map_batch of the numpy oracle port, ThreadPool x{cores} with "
                      f"1 BLAS thread, best of {len(times)}",
            "times_s": [round(t, 4) for t in times], "build_blocks_s": round(build_s, 2)}


def bench_reference(args):
    rank = env_int("RANK", 0)
    ws = env_int("WORLD_SIZE", 1)
    if rank != 0:
        return
    cb = cpu_baseline_c2(sample_rows=args.cpu_rows, warmup=args.warmup, steps=args.steps)
    line = {
        "metric": METRIC, "impl": "reference", "value": cb["value"], "unit": "features/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(min(cb["times_s"]) * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded MNIST-shaped rows; MNIST absent)",
        "config": {"workload": "c2: Fastfood Matern expansion (sigma=2, t=40), 60000x784 -> "
                               "32768 features/row, E=16, n=1024, batches of 4096",
                   "sample_rows_per_step": args.cpu_rows},
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "features/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "reference = numpy restatement of mckernel's CPU path (oracle/, pinned bit-exact "
                "to the reference by tests/test_oracle_golden.py); runs on rank 0 only",
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-rows", type=int, default=4096)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
