#!/usr/bin/env python3
"""Summarise an ncu launch list (+ optional --set full report) into profiles/.

    python tools/profile_summary.py TAG gpurun_out/launches_TAG.csv [gpurun_out/k1_TAG.ncu-rep] \
        [--alg-bytes N] [--kernel SUBSTR (default splitkv)] [--traffic-out k1_traffic.json]

Writes profiles/TAG_launches.csv (our kernels + per-kernel totals) and
profiles/TAG_ncu_summary.md (speed-of-light, DRAM bytes per launch vs the
algorithmic bytes, occupancy, stall summary).
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    out = []
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            out.append((r[ki], float(r[vi])))
    return out


def ncu_raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    return [{h[i]: (r[i], u[i]) for i in range(len(h))} for r in rows[2:]]


def main():
    tag, launches = sys.argv[1], sys.argv[2]
    rep = sys.argv[3] if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else None
    alg = None
    if "--alg-bytes" in sys.argv:
        alg = int(sys.argv[sys.argv.index("--alg-bytes") + 1])
    kern = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else "splitkv"
    tout = sys.argv[sys.argv.index("--traffic-out") + 1] if "--traffic-out" in sys.argv else "k1_traffic.json"
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    L = read_launches(launches)
    tot = {}
    for name, ns in L:
        k = name.split("(")[0]
        c, t = tot.get(k, (0, 0.0))
        tot[k] = (c + 1, t + ns)
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.csv"), "w") as f:
        f.write("kernel,launches,total_us,mean_us\n")
        for k, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1]):
            f.write(f"\"{k}\",{c},{t / 1e3:.1f},{t / c / 1e3:.1f}\n")
    md = [f"# {tag}: ncu summary", "", "## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised)", "",
          "| kernel | launches | total µs | mean µs |", "|---|---|---|---|"]
    for k, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1])[:12]:
        md.append(f"| `{k[:90]}` | {c} | {t / 1e3:.1f} | {t / c / 1e3:.1f} |")
    summary = {}
    if rep:
        for rec in ncu_raw(rep):
            name = rec.get("Kernel Name", ("?", ""))[0]
            if kern not in name:
                continue
            def g(m):
                v = rec.get(m)
                return float(v[0].replace(",", "")) if v and v[0] not in ("", "n/a") else None
            dur_ns = g("gpu__time_duration.sum")
            rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
            unit_r = rec.get("dram__bytes_read.sum", ("", ""))[1]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd_b = rd * scale.get(unit_r, 1) if rd is not None else None
            wr_b = wr * scale.get(rec.get("dram__bytes_write.sum", ("", ""))[1], 1) if wr is not None else None
            dur_unit = rec.get("gpu__time_duration.sum", ("", ""))[1]
            dur_s = dur_ns * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(dur_unit, 1e-9)
            summary = {
                "kernel": name, "duration_s": dur_s, "dram_read_bytes": rd_b, "dram_write_bytes": wr_b,
                "dram_bytes_per_launch": (rd_b or 0) + (wr_b or 0),
                "dram_gbs": ((rd_b or 0) + (wr_b or 0)) / dur_s / 1e9 if dur_s else None,
                "dram_pct_peak": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                "sm_pct": g("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                "tensor_pct": g("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                "regs": g("launch__registers_per_thread"),
                "sm_ghz": g("sm__cycles_elapsed.avg.per_second"),
                "smem_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
                "algorithmic_bytes": alg,
            }
            break
        if summary:
            md += ["", "## Top kernel (`ncu --set full --clock-control none`)", "",
                   f"- kernel: `{summary['kernel']}`",
                   f"- duration: {summary['duration_s'] * 1e6:.1f} µs at {summary['sm_ghz']} GHz SM clock",
                   f"- DRAM read {summary['dram_read_bytes'] / 1e9:.4f} GB, write {summary['dram_write_bytes'] / 1e6:.2f} MB"
                   f" -> {summary['dram_gbs']:.0f} GB/s ({summary['dram_pct_peak']}% of ncu's DRAM peak)",
                   f"- SM throughput {summary['sm_pct']}%, tensor pipe {summary['tensor_pct']}%, "
                   f"{summary['regs']:.0f} regs/thread, shared bank conflicts {summary['smem_bank_conflicts']}"]
            if alg:
                md.append(f"- algorithmic bytes/launch {alg / 1e9:.4f} GB; traffic/algorithmic = "
                          f"{summary['dram_bytes_per_launch'] / alg:.4f}")
            with open(os.path.join(ROOT, "profiles", tout), "w") as f:
                json.dump(summary, f, indent=1)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
