"""Summarise an ncu report: headline metrics, stall reasons and the hottest SASS lines.

usage: python tools/ncu_hot.py REPORT.ncu-rep [TOP]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
keys = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum", "dram__bytes_read.sum"]
for k in keys:
    print(f"{k:60s} {d.get(k, '')}")
for k in rows[0]:
    if k.startswith("smsp__average_warps_issue_stalled") and float(d[k] or 0) > 0.05:
        print(f"{k:60s} {d[k]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ia, isrc, iss = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = [(r[0], r[isrc].strip(), int(r[ia] or 0), int(r[iss] or 0)) for r in rows[2:] if len(r) > ia]
tot, ts = sum(x[2] for x in data), sum(x[3] for x in data)
print("instructions", tot, "stall samples", ts)
brx = [i for i, x in enumerate(data) if x[1].startswith("BRX")]
if brx:
    b = brx[0]
    print("dispatches", data[b][2], "inst/dispatch", round(tot / max(1, data[b][2]), 2))
ops = collections.Counter()
for a, s_, n, sm in data:
    op = s_.split()[1] if s_.startswith("@") else s_.split()[0]
    ops[op] += n
print("by opcode:", ", ".join(f"{k} {v / tot:.1%}" for k, v in ops.most_common(14)))
for i, (a, s_, n, sm) in enumerate(data):
    if sm >= sorted((x[3] for x in data), reverse=True)[min(top_n, len(data)) - 1]:
        print(f"{i:5d} {n:>11} {sm:>6}  {s_[:80]}")
