#!/usr/bin/env python
"""Benchmark of the B200 Fastfood hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (config 2 of BASELINE.json, the largest single-GPU expansion):
Matern kernel (sigma=2, t=40), d=784 padded to n=1024, E=16 -> 32,768 features
per row, over N=60,000 image-shaped rows (~80% exact zeros, rest U(0,1]),
streamed in batches of 4,096 rows.  One step = one pass over the 60,000 rows
(15 fused-expansion launches into a reused 4,096-row output buffer; inputs
188 MB and each batch's output 537 MB exceed the 126 MB L2, so no flush is
needed).  Multi-GPU: every rank expands its own 60,000-row shard (weak
scaling, no collective on the data path); value = all ranks' features / max
rank time.

Extras on the single-GPU run: the config-1 FWHT sweep (GB/s per length),
config 0 (1000-row batch) and one config-3 training epoch.
--impl reference times the reference algorithm (the numpy oracle port of
mckernel, tests-pinned bit-exact to the reference) on this host's cores.
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
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend)
    return rank, local, ws


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

    rank, local, ws = dist_setup("nccl")
    torch.cuda.set_device(local)
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
    out = torch.empty((batch, width), dtype=torch.float32, device=dev)
    spans = [(r0, min(rows, r0 + batch)) for r0 in range(0, rows, batch)]
    stream = torch.cuda.current_stream(dev)

    def step(evs=None):
        for k, (r0, r1) in enumerate(spans):
            if evs is not None:
                evs[k][0].record(stream)
            P.feature_map_batch(spec, blocks, x[r0:r1], out=out)
            if evs is not None:
                evs[k][1].record(stream)

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
    # once.  Its average launch duration is the timed
    # region (CUDA events on the launching stream) over the launches in it --
    # gaps between launches included, so this is a lower bound on the
    # kernel's own rate.  A second pass with events around every launch
    # (which stop a launch from overlapping its predecessor's tail, so it is
    # kept out of `value`) gives the per-launch spread.
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
                "achieved_source": "timed region / launches (inter-launch gaps included)",
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
                   "parallelism": f"row shards x{ws} (no collective)"},
        "roofline": roofline, "e2e": e2e, "gpu_launches": args.steps * len(spans),
        "clocks": clk.summary(), "setup_s": {"build_blocks_c2": round(setup_s, 4)},
    }
    if ws == 1 and rank == 0 and not args.no_extras:
        line["extras"] = extras(args, P, torch, dev, hbm)
    if rank == 0 and ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_c2(sample_rows=args.cpu_rows, reps=2)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def time_cuda(fn, reps, torch, stream=None):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def extras(args, P, torch, dev, hbm):
    import numpy as np
    from paper_1702_08159_b200 import synthetic
    out = {}
    # config 1: FWHT sweep, 2^28 floats (1 GiB) per length, in place; GB/s on
    # algorithmic bytes (read + write once = 2^31 B)
    sweep = {}
    g = torch.Generator(device=dev).manual_seed(7)
    buf = torch.randn(1 << 28, generator=g, device=dev)
    for k in range(10, 21):
        n = 1 << k
        mat = buf.view(-1, n)
        P.wht_fast_batch(mat)
        ms = time_cuda(lambda: P.wht_fast_batch(mat), 5, torch)
        sweep[str(n)] = {"ms": round(ms, 4), "GBps": round(2 ** 31 / (ms / 1e3) / 1e9, 1),
                         "frac": round(2 ** 31 / (ms / 1e3) / 1e9 / hbm, 4)}
    del buf
    out["c1_fwht_sweep"] = sweep
    # config 0: 1000 x 784, RBF E=8 -> 16384 features/row (launch-latency sized)
    spec0 = P.FeatureMapSpec(784, 8, P.RBF(1.0), 1234)
    b0 = P.build_blocks(spec0)
    x0 = torch.from_numpy(synthetic.image_rows(1000, 784, 1234)).to(dev)
    o0 = torch.empty((1000, 16384), device=dev)
    P.feature_map_batch(spec0, b0, x0, out=o0)
    ms0 = time_cuda(lambda: P.feature_map_batch(spec0, b0, x0, out=o0), 50, torch)
    out["c0_features"] = {"ms_per_batch": round(ms0, 4),
                          "features_per_s": 1000 * 16384 / (ms0 / 1e3),
                          "GBps": round(1000 * (3136 + 65536) / (ms0 / 1e3) / 1e9, 1)}
    # config 4 expansion alone (n = 16384, E = 32, sigma = 4): 256 rows ->
    # 2^20 features/row materialised (the fused classifier path is K6)
    spec4 = P.FeatureMapSpec(16384, 32, P.RBF(4.0), 4)
    t0 = time.perf_counter()
    b4 = P.build_blocks(spec4)
    torch.cuda.synchronize()
    setup4 = time.perf_counter() - t0
    x4 = torch.randn((256, 16384), generator=torch.Generator(device=dev).manual_seed(7),
                     device=dev)
    o4 = torch.empty((256, 1 << 20), device=dev)
    P.feature_map_batch(spec4, b4, x4, normalize=False, out=o4)
    ms4 = time_cuda(lambda: P.feature_map_batch(spec4, b4, x4, normalize=False, out=o4), 5, torch)
    out["c4_expansion"] = {"rows": 256, "ms": round(ms4, 4),
                           "features_per_s": 256 * (1 << 20) / (ms4 / 1e3),
                           "GBps": round(256 * (65536 + 4 * (1 << 20)) / (ms4 / 1e3) / 1e9, 1),
                           "build_blocks_s": round(setup4, 3)}
    del o4, x4
    # config 4 fused training step (K6): one rank's 1024-row shard of the
    # 8192-row global batch; forward + backward (expansion recomputed) + SGD,
    # features never written to HBM
    from paper_1702_08159_b200.large_scale import FusedClassifier
    fc = FusedClassifier(spec4, 10, 1024)
    x4 = torch.randn((1024, 16384), generator=torch.Generator(device=dev).manual_seed(7),
                     device=dev)
    y4 = torch.randint(0, 10, (1024,), device=dev, dtype=torch.int32)
    fc.step(x4, y4, m_total=8192, lr=0.01)
    ms_step = time_cuda(lambda: fc.step(x4, y4, m_total=8192, lr=0.01), 3, torch)
    out["c4_fused_step"] = {"rows_per_rank": 1024, "global_batch": 8192, "ms_per_step": round(ms_step, 3),
                            "features_per_s": 1024 * (1 << 20) / (ms_step / 1e3),
                            "note": "forward+backward+update; features_per_s counts each row's 2^20 "
                                    "features once per step"}
    del fc, x4
    # config 3: one training epoch (60 steps of 1000 rows + 10k-row evaluation)
    x, y = synthetic.class_images(60000, 784, 10, seed=1234)
    xt, yt = synthetic.class_images(10000, 784, 10, seed=1234, sample_seed=99)
    cfg = P.TrainConfig(0.01, 1000, 2)
    tr = P.Trainer(spec0, P.Dataset(x, y, 10), P.Dataset(xt, yt, 10), cfg)
    for s in range(tr.steps):
        tr.step(0, s)
    torch.cuda.synchronize()
    t_steps = time_cuda(lambda: [tr.step(1, s) for s in range(tr.steps)], 1, torch)
    tr.evaluate()  # first call allocates the evaluation buffers
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr.evaluate()  # returns host scalars (synchronises)
    t_eval = (time.perf_counter() - t0) * 1e3
    out["c3_train"] = {"ms_per_epoch_steps": round(t_steps, 3), "ms_eval": round(t_eval, 3),
                       "ms_per_step": round(t_steps / tr.steps, 4),
                       "features_per_s": 60000 * 16384 / (t_steps / 1e3),
                       "epoch_loss": tr.epoch_loss()}
    return out


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
    chunks = np.array_split(x, 4 * cores)

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
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-rows", type=int, default=4096)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
