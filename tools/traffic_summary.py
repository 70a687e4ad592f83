"""Summarise the ncu launch list of tools/prof_forward.py (one eager VGG16 forward, one
batch part, cold caches) into profiles/: sfjit launches grouped per layer (the engine
launches a layer's ceil(K / KT) groups in order; KT = 64 on the C <= 64 layers, else 48), kernel time and DRAM bytes per layer.
bench.py reads dram_bytes_per_layer from the result as the roofline's `traffic`.

usage: python tools/traffic_summary.py launches.csv OUT.json
"""
import csv
import json
import sys

KS = [64, 64, 128, 128, 256, 256, 256, 512, 512, 512, 512, 512, 512]
CS = [3] + KS[:-1]
# filters per group as the engine picks them: 64 on the shallow (C <= 64) layers, else 48
KT = [64 if c <= 64 else 48 for c in CS]


def main():
    src, dst = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(src)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    launches = {}
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        L = launches.setdefault(int(d["ID"]), {"kernel": d["Kernel Name"]})
        L[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    order = [launches[k] for k in sorted(launches)]
    jit = [L for L in order if L["kernel"].startswith("sfjit")]
    other = [L for L in order if not L["kernel"].startswith("sfjit")]
    dur = lambda L: L["gpu__time_duration.sum"] * 1e-6  # ns -> ms
    per_layer, pos = [], 0
    for li, k in enumerate(KS):
        g = (k + KT[li] - 1) // KT[li]
        grp = jit[pos:pos + g]
        pos += g
        per_layer.append({"layer": li, "groups": g, "kernel_ns_sum": sum(L["gpu__time_duration.sum"] for L in grp),
                          "dram_read": sum(L["dram__bytes_read.sum"] for L in grp),
                          "dram_write": sum(L["dram__bytes_write.sum"] for L in grp)})
    assert pos == len(jit), (pos, len(jit))
    tot = sum(p["dram_read"] + p["dram_write"] for p in per_layer)
    ms_jit, ms_other = sum(dur(L) for L in jit), sum(dur(L) for L in other)
    out = {"what": "ncu launch list of one VGG16 forward (config 3, batch 32, eager, 1 part): tools/prof_forward.py "
                   "under ncu --nvtx --nvtx-include profiled/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                   "dram__bytes_write.sum --clock-control none (cold caches, kernels serialised; a layer's group "
                   "launches run one after another here, concurrently in the bench)",
           "sfjit_launches": len(jit), "sfjit_kernel_ms_sum": ms_jit,
           "other_kernels": sorted({L["kernel"] for L in other}), "other_kernel_ms": ms_other,
           "sfjit_share_of_kernel_time": ms_jit / (ms_jit + ms_other) if ms_jit + ms_other else None,
           "dram_bytes_per_layer": tot / len(KS), "dram_bytes_total": tot, "per_layer": per_layer}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "per_layer"}, indent=1))


if __name__ == "__main__":
    main()
