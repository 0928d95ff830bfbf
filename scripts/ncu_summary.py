"""Summarise an ncu capture (and optionally a launch list) into profiles/.

  python scripts/ncu_summary.py gpurun_out/prof.ncu-rep --name r01_sweep_div_tma \
      [--launches gpurun_out/launches.csv] [--json profiles/ncu_sweep_div.json] \
      [--algo-bytes 10737418240]

Writes profiles/<name>.md with the metrics the roofline story needs (duration,
DRAM bytes read+write per launch vs algorithmic, DRAM throughput, occupancy,
registers, issue activity, top stall reasons, pipe utilisation) and, with
--json, the per-launch DRAM traffic bench.py reports as roofline.traffic.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (occupancy)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block", "smem/block"),
    ("launch__occupancy_limit_registers", "CTA/SM limit (registers)"),
    ("launch__occupancy_limit_shared_mem", "CTA/SM limit (smem)"),
    ("launch__grid_size", "grid (CTAs)"),
    ("launch__block_size", "block (threads)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__cycles_elapsed.avg.per_second", "DRAM clock"),
]


def kernel_source_sha() -> str:
    """sha256 (16 hex) over the CUDA sources of the library (same as bench.py)."""
    import hashlib
    h = hashlib.sha256()
    src = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1201_2118_b200", "csrc")
    for n in sorted(os.listdir(src)):
        if n.endswith((".cu", ".cuh", ".hpp")):
            with open(os.path.join(src, n), "rb") as f:
                h.update(n.encode() + f.read())
    return h.hexdigest()[:16]


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    launches = []
    for v in rows[2:]:
        launches.append({h[i]: (v[i], u[i]) for i in range(min(len(h), len(v)))})
    return launches


def to_bytes(val: str, unit: str) -> float:
    x = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return x * scale


def to_ms(val: str, unit: str) -> float:
    x = float(val.replace(",", ""))
    return x * {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3, "nsecond": 1e-6}.get(unit, 1.0)


def launch_table(path: str):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    t, n = defaultdict(float), defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        t[name] += to_ms(r[vi], r[ui])
        n[name] += 1
    tot = sum(t.values()) or 1.0
    lines = ["| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k in sorted(t, key=lambda k: -t[k]):
        lines.append(f"| `{k}` | {n[k]} | {t[k]:.3f} | {100 * t[k] / tot:.1f}% |")
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--name", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--json")
    ap.add_argument("--algo-bytes", type=float, default=None)
    ap.add_argument("--note", default="")
    ap.add_argument("--sum-launches", action="store_true",
                    help="the captured launches together form one unit (e.g. the launches of one pass): "
                         "the JSON traffic is their sum")
    a = ap.parse_args()
    L = raw(a.rep)
    md = [f"# ncu summary: {a.name}", "", f"source: `{os.path.basename(a.rep)}` (`ncu --set full --clock-control none`), {len(L)} profiled launch(es)", ""]
    if a.note:
        md += [a.note, ""]
    js = {"name": a.name, "launches": []}
    for q, m in enumerate(L):
        kname = m.get("Kernel Name", ("?", ""))[0]
        md += [f"## launch {q}: `{kname[:120]}`", "", "| metric | value |", "|---|---|"]
        rec = {"kernel": kname}
        for key, label in KEYS:
            if key in m:
                v, u = m[key]
                md.append(f"| {label} (`{key}`) | {v} {u} |")
                rec[key] = [v, u]
        rd = to_bytes(*m["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in m else None
        wr = to_bytes(*m["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in m else None
        dur = to_ms(*m["gpu__time_duration.sum"]) if "gpu__time_duration.sum" in m else None
        if rd is not None and wr is not None:
            tr = rd + wr
            rec["dram_bytes_per_launch"] = tr
            md.append(f"| DRAM read+write per launch | {tr / 1e9:.3f} GB |")
            if dur:
                md.append(f"| DRAM GB/s (ncu, cold, serialised) | {tr / (dur / 1e3) / 1e9:.1f} |")
            if a.algo_bytes:
                md.append(f"| algorithmic bytes per launch | {a.algo_bytes / 1e9:.3f} GB |")
                md.append(f"| traffic / algorithmic | {tr / a.algo_bytes:.3f} |")
        stalls = []
        for k, (v, u) in m.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        md += ["", "top stall reasons (warps stalled per issue):", ""]
        md += [f"- {n}: {x:.3f}" for x, n in stalls[:8]]
        md.append("")
        js["launches"].append(rec)
    if a.launches:
        md += ["## launch list (`--metrics gpu__time_duration.sum`; cold-cache, serialised: compare shares)", "", launch_table(a.launches), ""]
    os.makedirs("profiles", exist_ok=True)
    with open(os.path.join("profiles", a.name + ".md"), "w") as f:
        f.write("\n".join(md))
    if a.json:
        first = js["launches"][0] if js["launches"] else {}
        if a.sum_launches:
            js["dram_bytes_per_launch"] = sum(r.get("dram_bytes_per_launch") or 0.0 for r in js["launches"])
            js["note"] = a.note or "traffic = the sum over the captured launches (one unit)"
        else:
            js["dram_bytes_per_launch"] = first.get("dram_bytes_per_launch")
        js["algo_bytes_per_launch"] = a.algo_bytes
        # provenance: bench.py flags the traffic as stale once the kernel source changes
        js["kernel_source_sha"] = kernel_source_sha()
        js["captured_from"] = os.path.basename(a.rep)
        with open(a.json, "w") as f:
            json.dump(js, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
