"""bench.py's JSON contract on the CPU side.

The reference arm (`--impl reference`) runs the numpy oracle port of the
reference's CPU path and needs no GPU: its line must carry the driver's keys.
Our arm must fail loudly without a GPU (no CPU fallback).
"""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _run(*args, timeout=600):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)


def test_reference_arm_line():
    r = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-rows", "32")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference"
    assert line["metric"].startswith("Fastfood") or "features" in line["unit"]
    assert line["unit"] == "features/s" and line["value"] > 0
    assert line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"],
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("c2")


def test_our_arm_fails_without_gpu():
    r = _run("--steps", "1", "--warmup", "3", "--no-extras", timeout=300)
    assert r.returncode != 0
    assert not r.stdout.strip(), "no bench line may be printed without a GPU"


def test_gpus_flag_launches_ranks():
    # `bench.py --gpus 2` outside torchrun starts 2 ranks itself; rank 0 prints the line
    r = _run("--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "0",
             "--cpu-rows", "16")
    assert r.returncode == 0, r.stderr[-2000:]
    assert "launching 2 ranks" in r.stderr
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert json.loads(lines[0])["n_gpus"] == 2
