#!/usr/bin/env python3
"""Print the key raw metrics and the top stalled SASS lines of an ncu report.
    python tools/ncu_top.py REPORT.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2] if len(r) > 2 else r[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg", "launch__registers_per_thread",
        "smsp__cycles_active.avg.pct_of_peak_sustained_elapsed"]
for i, name in enumerate(h):
    if any(name.endswith(k) for k in keys):
        print(f"{name} = {v[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
ai, si, wi, ei = (hh.index("Address"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"),
                  hh.index("Instructions Executed"))
data = []
for row in rows[2:]:
    try:
        data.append((int(row[wi] or 0), row[ai], row[si], row[ei]))
    except Exception:
        pass
tot = sum(d[0] for d in data)
print("total stall samples", tot)
idx = {d[1]: i for i, d in enumerate(data)}
for d in sorted(data, reverse=True)[:n]:
    i = idx[d[1]]
    prev = " | ".join(x[2].strip()[:40] for x in data[max(0, i - 2):i])
    print(f"{d[0]:6d} {d[1][-5:]} {d[2].strip()[:70]:70s} x{d[3]}  << {prev}")
