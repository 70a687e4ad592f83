"""Summarise an ncu report (.ncu-rep) into a small JSON for profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json [label]
Extracts duration, throughput, occupancy, DRAM bytes, pipe utilisation, smem
wavefronts and the warp-stall breakdown (from the source page samples).
"""
import csv
import io
import json
import subprocess
import sys


def page(rep, name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    label = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = page(rep, "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    m = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
             "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}
    want = {
        "kernel": "Kernel Name",
        "duration_s": "gpu__time_duration.sum",
        "sm_clock_hz": "smsp__cycles_elapsed.avg.per_second",
        "dram_read_bytes": "dram__bytes_read.sum",
        "dram_write_bytes": "dram__bytes_write.sum",
        "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "fp32_ffma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "warps_active_avg": "sm__warps_active.avg.per_cycle_active",
        "registers_per_thread": "launch__registers_per_thread",
        "grid_size": "launch__grid_size",
        "block_size": "launch__block_size",
        "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    }
    out = {"label": label, "report": rep}
    for k, v in want.items():
        if v in m:
            try:
                out[k] = float(m[v].replace(",", "")) * scale.get(u.get(v, ""), 1.0)
            except ValueError:
                out[k] = m[v]
    src = page(rep, "source", ("--print-source", "sass"))
    if len(src) > 2:
        h = src[1]
        rows = [dict(zip(h, r)) for r in src[2:] if len(r) == len(h)]
        reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
        tot = {r: sum(float(d[r] or 0) for d in rows) for r in reasons}
        s = sum(tot.values()) or 1.0
        out["stall_pct"] = {k[6:]: round(v / s * 100, 1) for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v}
        wf = sum(float(d.get("L1 Wavefronts Shared", 0) or 0) for d in rows)
        ex = sum(float(d.get("L1 Wavefronts Shared Excessive", 0) or 0) for d in rows)
        out["smem_wavefronts_excessive_pct"] = round(100 * ex / wf, 1) if wf else None
    with open(dst, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
