"""Summarise ncu captures into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py REPORT.ncu-rep NAME [--alg-bytes B] [--key KEY]
    python tools/ncu_summary.py --launches LAUNCHES.csv NAME

Writes profiles/NAME.md (metrics + top stall reasons + hottest source lines)
and merges {KEY: {...}} into profiles/ncu_summary.json.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/shared throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__clock_frequency.avg", "SM clock"),
]


def ncu_csv(rep: str, *args) -> list[list[str]]:
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise(rep: str, name: str, alg_bytes: float | None, key: str | None):
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
    kname = m.get("Kernel Name", ("", "?"))[1]
    lines = [f"# {name}", "", f"Report: `{Path(rep).name}`; kernel `{kname}`", "",
             "| metric | value | unit |", "|---|---|---|"]
    res = {"kernel": kname}
    for k, label in METRICS:
        if k in m:
            u, v = m[k]
            lines.append(f"| {label} (`{k}`) | {v} | {u} |")
            try:
                res[k] = float(v.replace(",", ""))
                res[k + ".unit"] = u
            except ValueError:
                pass
    # DRAM bytes (normalise to bytes)
    def to_bytes(k):
        u, v = m.get(k, ("byte", "0"))
        f = float(v.replace(",", ""))
        return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    traffic = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
    res["dram_bytes_per_launch"] = traffic
    lines += ["", f"DRAM traffic per launch: {traffic / 1e6:.1f} MB"]
    if alg_bytes:
        res["alg_bytes_per_launch"] = alg_bytes
        lines.append(f"Algorithmic bytes per launch: {alg_bytes / 1e6:.1f} MB "
                     f"(traffic / algorithmic = {traffic / alg_bytes:.3f}; writes still in L2 at "
                     "kernel end are not counted by ncu)")
    stalls = sorted(((h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "")))
                     for h, (u, v) in m.items()
                     if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
                     and v.replace(",", "").replace(".", "").isdigit()), key=lambda t: -t[1])
    tot = sum(v for _, v in stalls) or 1
    lines += ["", "Warp-state samples (top):", ""]
    lines += [f"- {n}: {100 * v / tot:.1f}%" for n, v in stalls[:8] if v > 0]
    res["stalls"] = {n: v for n, v in stalls if v > 0}
    # hottest source lines
    src = ncu_csv(rep, "--page", "source", "--print-source=cuda,sass")
    hot = []
    for r in src[3:]:
        if len(r) > 5 and r[0].isdigit():
            try:
                hot.append((int(r[4]), r[0], r[1].strip()[:100]))
            except ValueError:
                pass
    if hot:
        t = sum(h[0] for h in hot) or 1
        lines += ["", "Hottest source lines (warp-stall samples):", ""]
        lines += [f"- {100 * s / t:.1f}% line {ln}: `{txt}`" for s, ln, txt in sorted(hot, reverse=True)[:10]]
    PROF.mkdir(exist_ok=True)
    (PROF / f"{name}.md").write_text("\n".join(lines) + "\n")
    if key:
        js = PROF / "ncu_summary.json"
        data = json.loads(js.read_text()) if js.exists() else {}
        data[key] = res
        js.write_text(json.dumps(data, indent=1))
    print("\n".join(lines))


def launches(path: str, name: str):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, start = r, i + 1
            break
    ix = {h: j for j, h in enumerate(hdr)}
    agg: dict[tuple[str, str], list[float]] = {}
    for r in rows[start:]:
        if len(r) < len(hdr):
            continue
        k = r[ix["Kernel Name"]]
        k = k.split("(")[0] if "(" in k else k
        agg.setdefault((k, r[ix["Metric Name"]] + " [" + r[ix["Metric Unit"]] + "]"), []).append(
            float(r[ix["Metric Value"]].replace(",", "")))
    tot_t = sum(sum(v) for (k, mname), v in agg.items() if mname.startswith("gpu__time_duration"))
    lines = [f"# {name}", "", f"Source: `{Path(path).name}` (ncu launch list, cold-cache, serialised: "
             "compare shares, not absolutes)", "",
             "| kernel | metric | launches | sum | mean | share of time |", "|---|---|---|---|---|---|"]
    for (k, mname), v in sorted(agg.items()):
        share = f"{100 * sum(v) / tot_t:.1f}%" if mname.startswith("gpu__time_duration") else ""
        lines.append(f"| `{k[:70]}` | {mname} | {len(v)} | {sum(v):.4g} | {sum(v) / len(v):.4g} | {share} |")
    (PROF / f"{name}.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("name")
    ap.add_argument("--alg-bytes", type=float)
    ap.add_argument("--key")
    ap.add_argument("--launches", action="store_true")
    a = ap.parse_args()
    if a.launches:
        launches(a.report, a.name)
    else:
        summarise(a.report, a.name, a.alg_bytes, a.key)
