"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*) of
bench.py into profiles/: per-kernel launch counts, the timed step's sf3x3 launches
(13 per step, one per VGG16 conv) with duration and DRAM bytes, and time shares.

usage: python tools/launch_summary.py launches.csv OUT.json
"""
import csv
import json
import sys


def main():
    src, dst = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(src)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    launches = {}
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        L = launches.setdefault(int(d["ID"]), {"kernel": d["Kernel Name"], "grid": d["Grid Size"], "block": d["Block Size"]})
        unit, val = d["Metric Unit"], float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9,
                 "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        L[d["Metric Name"]] = val * scale
    ids = sorted(launches)
    per_kernel = {}
    for k in ids:
        name = launches[k]["kernel"].split("(")[0]
        pk = per_kernel.setdefault(name, {"launches": 0, "time_s": 0.0})
        pk["launches"] += 1
        pk["time_s"] += launches[k].get("gpu__time_duration.sum", 0.0)
    sf = [launches[k] for k in ids if "sf3x3_kernel" in launches[k]["kernel"]]
    # bench order: 3 warm-up steps, `steps` timed steps, then per-layer timing.  A step
    # runs the 13 convs on two half-batch streams (26 launches): take the first timed
    # step; per-launch figures below are per full-batch layer (the two halves summed),
    # the unit bench.py's roofline uses.
    per_step = 26
    step = sf[3 * per_step:4 * per_step] if len(sf) >= 4 * per_step else sf[:per_step]
    tot_t = sum(s.get("gpu__time_duration.sum", 0) for s in step)
    tot_b = sum(s.get("dram__bytes_read.sum", 0) + s.get("dram__bytes_write.sum", 0) for s in step)
    out = {
        "source": src,
        "note": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                "--clock-control none; cold-cache serialised launches: compare shares, not absolutes",
        "per_kernel": per_kernel,
        "step_sf3x3": [
            {"grid": s["grid"], "time_s": s.get("gpu__time_duration.sum"),
             "dram_bytes": s.get("dram__bytes_read.sum", 0) + s.get("dram__bytes_write.sum", 0)}
            for s in step
        ],
        "step_sf3x3_time_s": tot_t,
        "step_sf3x3_dram_bytes": tot_b,
        "sf3x3_dram_bytes_per_launch": tot_b / 13.0,
        "note_per_launch": "per full-batch conv layer (step total / 13)",
    }
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "step_sf3x3"}, indent=1))


if __name__ == "__main__":
    main()
