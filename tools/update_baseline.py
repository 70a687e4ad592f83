"""Regenerate BASELINE.md §3 (GPU results) from the committed profiles/ files."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(name):
    with open(os.path.join(ROOT, "profiles", name)) as fh:
        return json.load(fh)


def c4_ranges(rows, mode, zf):
    v = [r["tflops"] for r in rows if r["mode"] == mode and r["zero_frac"] == zf and r["layer"] > 0]
    return f"{min(v):.1f}–{max(v):.1f}"


def main():
    c3, c5 = load("r01_bench_c3.json"), load("r01_bench_c5_1gpu.json")
    ref, ref5 = load("r01_bench_reference.json"), load("r01_bench_reference_c5.json")
    c12, c4 = load("r01_configs_12.json"), load("r01_c4_sweep.json")
    step_tf = c3["nnz_gflops"] / 1e3 if "nnz_gflops" in c3 else None
    sweep = {}
    with open(os.path.join(ROOT, "profiles", "r01_batch_sweep.txt")) as fh:
        for line in fh:
            if line.startswith("batch "):
                f = line.split()
                sweep[int(f[1])] = (float(f[6]), float(f[8]))  # ms/step, img/s
    sf = {z: c4_ranges(c4, "sf", z) for z in (0.5, 0.75, 0.9, 0.95, 0.99)}
    si = {z: c4_ranges(c4, "si", z) for z in (0.5, 0.9)}
    sif = {z: c4_ranges(c4, "si_fast", z) for z in (0.5, 0.9)}
    text = f'''## 3. GPU results

Measured on one B200 (148 SMs, SM clock {c3["clocks"]["sm_mhz"]:.0f} MHz under load, no throttle
reasons), CUDA 12.9, round 1.  FP32 roofline denominator = the measured FFMA probe
({c3["roofline"]["peak"]:.1f} TF/s); HBM = 6534.5 GB/s.  CPU rows are the oracle port of the
reference path (`oracle/`, OpenMP) on the same box's {c3["cpu_baseline"]["cores"]} host threads.

| Config | Metric | Value | Source |
|---|---|---|---|
| C1: SF 64→64 @56², 95% zeros, N=1 | time per layer call (device, graph-launched) | {c12["c1_exact"]["us_per_call_graph"]:.1f} µs = {c12["c1_exact"]["nnz_gflops"]:.0f} nnz-GFLOP/s (reference-order kernel, bit-exact, what the layer API runs; the tiled fast kernel fills only 16 CTAs here: {c12["c1_fast"]["us_per_call_graph"]:.1f} µs, {c12["c1_fast_small_grid"]["us_per_call_graph"]:.1f} µs with its small-grid plan of 1 filter per warp) | `profiles/r01_configs_12.json` |
| C1 | vs the reference on CPU (1 thread, §2.2) | 26.5 ms → ×{26500 / c12["c1_exact"]["us_per_call_graph"]:.0f} | §2.2 |
| C2: SI 128→128 @28², 90% input zeros, N=1 | strip kernel (shared-memory weights) on device nodes | {c12["c2_kernel"]["us_per_call_graph"]:.1f} µs = {c12["c2_kernel"]["nnz_gflops"]:.0f} nnz-GFLOP/s (bit-exact) | `profiles/r01_configs_12.json` |
| C2 | GPU encoder + kernel (incl. the node-count sync) | {c12["c2_encode_plus_kernel"]["us_per_call"]:.0f} µs; vs the reference on CPU (1 thread, §2.2): 78.8 ms | same |
| C3: VGG16 @224², 90% zeros, batch 32 | images/s, inputs in HBM (`value`) | {c3["value"]:.0f} img/s ({c3["ms_per_step"]:.2f} ms/step = {c3["nnz_gflops"] / 1e3:.1f} nnz-TFLOP/s over the step); the kernel's launches average {c3["roofline"]["achieved"]:.2f} nnz-TFLOP/s = {100 * c3["roofline"]["frac"]:.1f} % of FP32 peak; DRAM {c3["roofline"]["traffic"] / 1e6:.0f} MB per layer vs {c3["roofline"]["algorithmic_bytes_per_launch"] / 1e6:.0f} MB algorithmic | `profiles/r01_bench_c3.json`, `profiles/r01_bench_launches_summary.json` |
| C3, batch 1 (latency) | device time per image, input in HBM | {sweep[1][0]:.2f} ms ({sweep[1][1]:.0f} img/s); batch 4: {sweep[4][1]:.0f} img/s, 8: {sweep[8][1]:.0f}, 16: {sweep[16][1]:.0f}, 64: {sweep[64][1]:.0f} | `profiles/r01_batch_sweep.txt` |
| C3 | images/s through `network.forward` with host buffers (`e2e`) | {c3["e2e"]["value"]:.0f} img/s (inputs in pinned memory); {c3["e2e"]["pageable"]["value"]:.0f} with pageable numpy inputs | same |
| C3 | reference CPU path (oracle port, {c3["cpu_baseline"]["cores"]} threads, {c3["cpu_baseline"]["sample"].split(",")[0]}) | {c3["cpu_baseline"]["value"]:.2f} img/s → GPU e2e ×{c3["e2e"]["value"] / c3["cpu_baseline"]["value"]:.0f} | same, `profiles/r01_bench_reference.json` ({ref["value"]:.2f} img/s) |
| C4: 13 layers × SF {{50,75,90,95,99}} % / SI {{50,75,90,95}} %, batch 32 | nnz-TFLOP/s per layer (L1–L12; L0 has 3 input channels) | SF 50 %: {sf[0.5]}, 75 %: {sf[0.75]}, 90 %: {sf[0.9]}, 95 %: {sf[0.95]}, 99 %: {sf[0.99]}; SI channel-major kernel 50 %: {sif[0.5]}, 90 %: {sif[0.9]} (the bit-exact strip kernel: {si[0.5]} / {si[0.9]}); normwise error of the channel-major kernel vs the exact one ≤ {max(r.get("normwise_err_vs_exact", 0) for r in c4):.1e} | `profiles/r01_c4_sweep.json` |
| C5: VGG16, batch 256, 95 % zeros, 1 GPU | images/s | {c5["value"]:.0f} img/s ({c5["roofline"]["achieved"]:.2f} nnz-TFLOP/s per launch = {100 * c5["roofline"]["frac"]:.1f} %); e2e {c5["e2e"]["value"]:.0f} img/s; reference CPU path {ref5["value"]:.2f} img/s | `profiles/r01_bench_c5_1gpu.json`, `profiles/r01_bench_reference_c5.json` |
| C5, 2/4/8 GPUs | images/s | not measurable here (gpurun gives one GPU); the batch-sharded driver's host logic is tested with gloo at world size 2 | — |

Against the north star's target (≥ 50 % of the per-layer roofline) the sparse-filter
kernel reaches {100 * c3["roofline"]["frac"]:.0f} % at 90 % zeros and ~34 % at 50 %; DESIGN.md §5 gives the measured
bounds (jump-table dispatch latency and per-channel patch reloads through shared memory).
'''
    p = os.path.join(ROOT, "BASELINE.md")
    s = open(p).read()
    s = s[: s.index("## 3. GPU results")] + text
    open(p, "w").write(s)


if __name__ == "__main__":
    main()
