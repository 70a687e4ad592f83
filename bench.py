"""Benchmark: VGG16 conv-stack inference with fine-grained sparse filters on B200.

Workload (BASELINE.json config 3, the flagship): VGG16's 13 3x3 convs (+ReLU, 5x
2x2 max-pools) at 224x224, 90% i.i.d. filter zeros, batch 32 per GPU, fp32, seeded
synthetic inputs/weights (workloads.py).  One step = one forward pass of the rank's
batch through the stack (+ the NCCL gather of the outputs when N > 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c5] [--impl reference]

Prints ONE JSON line (rank 0).  `value` is images/s over all ranks with inputs
resident in HBM (device-timed, CUDA events, max over ranks); `e2e` is the same
metric through the public reference-compatible API (network.forward on host
DenseTensor3 lists: pinned H2D + device layout conversion + stack + D2H inside the
timed region); `roofline` reports the sparse-filter conv kernel's nnz-FLOP rate
against the measured FP32 CUDA-core peak; `cpu_baseline` is the oracle port of the
reference's CPU path on this host's cores.  `--impl reference` times only that CPU
path (rank 0) and prints its line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (per-GPU batch, filter zero fraction, description)
    "c3": (32, 0.90, "VGG16 conv stack, 224x224, batch 32/GPU, 90% i.i.d. filter zeros (BASELINE config 3)"),
    "c5": (256, 0.95, "VGG16 conv stack, 224x224, batch 256 total, 95% i.i.d. filter zeros (BASELINE config 5)"),
}
METRIC = "VGG16 conv-stack images/s (sparse-filter, fp32)"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks/throttle sampler running during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [v for v in sm if mx and v > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def fp32_peak_tflops(torch, lib):
    """Measured FFMA throughput (TFLOP/s) with the library's probe kernel."""
    from paper_2212_08815_b200._lib import call, ptr, stream

    props = torch.cuda.get_device_properties(0)
    blocks, iters = props.multi_processor_count * 8, 4096
    out = torch.zeros(blocks, device="cuda")
    for _ in range(2):
        call("fscnn_fp32_probe", ptr(out), blocks, iters, stream())
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call("fscnn_fp32_probe", ptr(out), blocks, iters, stream())
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b)
        best = max(best, blocks * 256 * iters * 256 / (ms * 1e-3) / 1e12)
    nominal = props.multi_processor_count * 128 * 2 * 1.965e9 / 1e12
    return best, nominal


def host_threads(oracle) -> int:
    """Threads for the CPU arm: every core this process may run on.  torchrun exports
    OMP_NUM_THREADS=1 to its ranks when the variable is unset, which would silently make
    the N>1 reference arm single-threaded -- the count is passed to the oracle explicitly
    (omp_set_num_threads) unless the caller chose one with FSCNN_CPU_THREADS."""
    if not oracle.max_threads() or oracle.lib().oracle_has_openmp() == 0:
        return 1
    env = os.environ.get("FSCNN_CPU_THREADS")
    if env:
        return max(1, int(env))
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def cpu_baseline(layers, hw, sample_images, budget_s=12.0, seed=2024):
    """Oracle port of the reference CPU path on this host, all cores; images/s."""
    from oracle import oracle
    from paper_2212_08815_b200 import workloads as wl

    banks = []
    for wt, b in layers:
        nodes, seg = oracle.encode_bank(wt)
        banks.append((nodes, seg, wt.shape[0], b))
    threads = host_threads(oracle)
    x = wl.vgg16_input(1, seed=seed, hw=hw)
    oracle.vgg_forward(x, banks, threads)  # warm (page-in)
    done, t0 = 0, time.perf_counter()
    while done < sample_images and (done == 0 or time.perf_counter() - t0 < budget_s):
        oracle.vgg_forward(x, banks, threads)
        done += 1
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": "images/s", "cores": threads, "kind": "port",
            "sample": f"{done} image(s) of the same workload (batch-1 forwards), {dt:.1f} s, oracle/ C port "
                      "of the reference numba kernels (strategy-II arithmetic), OpenMP over output pixels"}


def bench_config(desc, n_total, world, backend, zf):
    """The line's ``config`` object -- the same for both arms (the reference arm times a
    bounded sample of this workload, described in its ``cpu_baseline.sample``)."""
    return {"workload": desc, "global_batch": n_total, "seq_len": None,
            "parallelism": f"dp{world} (batch-sharded, filters broadcast once)",
            "collectives": backend if world > 1 else None,
            "filter_zero_fraction": zf,
            "l2": "working set > L2 (activations 0.4 GB per layer at batch 32)"}


def run_reference(args):
    """--impl reference: the reference CPU path (oracle port), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle
    from paper_2212_08815_b200 import workloads as wl

    batch, zf, desc = WORKLOADS[args.workload]
    layers = wl.vgg16_weights(seed=103, zero_frac=zf)
    banks = []
    for wt, b in layers:
        nodes, seg = oracle.encode_bank(wt)
        banks.append((nodes, seg, wt.shape[0], b))
    x = wl.vgg16_input(1, seed=104)
    threads = host_threads(oracle)
    for _ in range(args.warmup):
        oracle.vgg_forward(x, banks, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.vgg_forward(x, banks, threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.workload == "c3" else "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded numpy, workloads.py): x~N(0,1), W~N(0,sqrt(2/fan_in)) i.i.d. masked",
        "config": bench_config(desc, batch * args.gpus if args.workload == "c3" else batch, args.gpus,
                               os.environ.get("FSCNN_DIST_BACKEND", "nccl"), zf),
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": "port",
                         "sample": "1 image of the workload per step (the reference forwards images one by one: "
                                   "batch-1 forwards, OpenMP over output pixels) through the oracle/ C port of "
                                   "the reference kernels, on rank 0's host cores"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def _relaunch(args) -> int:
    """--gpus N > 1 without a torchrun environment: re-run this command under
    torch.distributed.run with N local ranks (one process per GPU, 127.0.0.1 rendezvous)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _relaunch(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2212_08815_b200 import _lib, distributed as pdist, network, workloads as wl
    from paper_2212_08815_b200.engine import VGGEngine
    from paper_2212_08815_b200.sparse_core import DenseTensor3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FSCNN_DIST_BACKEND=gloo: functional check of the N-rank path on a box with fewer
    # GPUs than ranks (ranks share GPUs, collectives through host memory) -- not a
    # performance configuration; the default is NCCL with one GPU per rank
    backend = os.environ.get("FSCNN_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    per_gpu, zf, desc = WORKLOADS[args.workload]
    if args.workload == "c5":
        lo, hi = pdist.shard_range(per_gpu, rank, world)
        n_local = hi - lo
    else:
        n_local = per_gpu
    hw = 224
    layers = wl.vgg16_weights(seed=103, zero_frac=zf) if rank == 0 else None

    # filters: rank 0 encodes (reference node format), NCCL broadcast, every rank packs
    # (distributed.ShardedVGG); one GPU: the engine directly
    sharded = None
    if world > 1:
        sharded = pdist.ShardedVGG(layers, hw=hw, device=dev)
        eng = sharded.engine
    else:
        eng = VGGEngine(layers, batch=n_local, hw=hw)
    t_jit = time.perf_counter()
    eng.wait_compiled()  # the specialised kernels' compile jobs (cached on disk by content hash)
    t_jit = time.perf_counter() - t_jit
    jit_on = all(st.jit is not None for st in eng.steps)
    n_total = n_local * world if args.workload == "c3" else per_gpu

    # inputs resident in HBM (per rank seeded shard)
    def shard_input(r):
        if args.workload == "c3":
            return wl.vgg16_input(n_local, seed=104 + r)
        a, b = pdist.shard_range(per_gpu, r, world)
        return wl.vgg16_input(per_gpu, seed=104)[a:b]

    x_np = shard_input(rank)
    x = torch.from_numpy(x_np).to(dev)
    flops_img = eng.flops_per_image()

    def step():
        if sharded is not None:
            return sharded.forward_device(x, total=n_total)
        return eng.forward_device(x)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    _lib.reset_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    launches = _lib.launch_count()
    if world > 1:
        dist.barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    sampler.stop()
    if world > 1:
        elapsed_ms = pdist.max_over_ranks(elapsed_ms, dev)
    images = n_total * args.steps
    value = images / (elapsed_ms * 1e-3)

    # per-layer kernel times on the launching stream (roofline of the dominant kernel)
    layer_ms = [0.0] * len(eng.steps)
    reps = 3
    bufs = eng._buffers(n_local)
    from paper_2212_08815_b200 import device as pdev

    xh = eng.stage_input(x)
    for _ in range(reps):
        cur, w = xh, hw
        for i, (st, out) in enumerate(zip(eng.steps, bufs)):
            st.conv(cur, out, w, n_local)  # the layer's code into L2 (as the step's later parts find it)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            st.conv(cur, out, w, n_local)
            b.record()
            b.synchronize()
            layer_ms[i] += a.elapsed_time(b) / reps
            cur = out
            w = w // 2 if st.pool else w
    peak_meas, peak_nom = fp32_peak_tflops(torch, _lib)
    # DRAM traffic per layer of the dominant kernel from the committed ncu summaries of this
    # step: the whole CUDA graph profiled as one workload (profiles/r02_graph_traffic.json:
    # kernels concurrent, L2 shared, as timed here) and, beside it, the serialised
    # cold-cache launch list (profiles/r02_bench_traffic.json: every group kernel of a
    # layer re-reads the layer's input from DRAM there)
    traffic, traffic_src, traffic_serial = None, None, None

    def _prof(name):
        path = os.path.join(ROOT, "profiles", name)
        if not (os.path.exists(path) and args.workload == "c3"):
            return None
        with open(path) as fh:
            return json.load(fh)

    if jit_on:
        d = _prof("r02_bench_traffic.json")
        if d:
            traffic_serial = d.get("dram_bytes_per_layer")
            traffic, traffic_src = traffic_serial, "profiles/r02_bench_traffic.json (ncu launch list, serialised, cold cache)"
        d = _prof("r02_graph_traffic.json")
        if d:
            traffic = d["dram_bytes_per_layer"]
            traffic_src = ("profiles/r02_graph_traffic.json (ncu --graph-profiling graph --cache-control none: "
                           "the step's CUDA graph as one workload, total DRAM bytes / 13 layers)")
    else:
        d = _prof("r01_bench_launches_summary.json")
        if d:
            traffic = d.get("sf3x3_dram_bytes_per_launch")
            traffic_src = "profiles/r01_bench_launches_summary.json (ncu, cold cache)"
    kern_ms = sum(layer_ms)
    per_launch_tf = flops_img * n_local / (kern_ms * 1e-3) / 1e12
    # the dominant kernel family is ~100 % of the step's kernel time (ncu launch list,
    # profiles/r02_bench_traffic.json), so the step's own rate is its achieved rate
    achieved_tf = flops_img * n_total / (elapsed_ms / args.steps * 1e-3) / 1e12 / world

    # e2e through the public API (host DenseTensor3 in, host DenseTensor3 out)
    e2e = None
    if world > 1:
        # every rank runs ShardedVGG.forward on the full host batch concurrently (its shard
        # H2D, its stack, NCCL all-gather of the device outputs, D2H of the full batch on
        # rank 0); the time is the max over ranks of each rank's wall clock
        full_np = np.concatenate([shard_input(r) for r in range(world)]) if args.workload == "c3" \
            else wl.vgg16_input(per_gpu, seed=104)
        batch = network.pinned_batch(n_total, (3, hw, hw))
        lo, hi = sharded.shard(n_total)
        for i in range(lo, hi):
            batch[i].data[:] = DenseTensor3.from_array(full_np[i]).data
        e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
        for _ in range(3):
            sharded.forward(batch, dst=0)
        torch.cuda.synchronize()
        passes = sorted(sharded.timed_forward(batch, dst=0, reps=e2e_steps)[1] for _ in range(3))
        dt = passes[1]
        e2e = {"value": n_total * e2e_steps / dt, "unit": "images/s",
               "h2d_bytes_per_step": int(n_total * 3 * hw * hw * 4),
               "d2h_bytes_per_step": int(n_total * eng.out_c * eng.out_hw * eng.out_hw * 4),
               "path": f"distributed.ShardedVGG.forward(list[DenseTensor3]) on {world} ranks concurrently: "
                       "each rank's shard H2D from pinned host memory, its stack, NCCL all-gather of the "
                       "device outputs, D2H of the full batch on rank 0; max over ranks of the wall clock, "
                       "median of 3 timed passes"}
    elif rank == 0:
        prepared = network.prepared_from_engine(eng)
        # the step's inputs sit in pinned host memory (network.pinned_batch: one DMA, no
        # host packing); pageable DenseTensor3 lists are packed first (e2e["pageable"])
        batch = network.pinned_batch(n_local, (3, hw, hw))
        for i in range(n_local):
            batch[i].data[:] = DenseTensor3.from_array(x_np[i]).data
        pageable = [DenseTensor3.from_array(x_np[i]) for i in range(n_local)]
        e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
        # untimed warm-up of the public-API path (pinned-buffer caches, copy streams,
        # both input kinds) so the timed passes see steady state
        for _ in range(max(3, e2e_steps)):
            network.forward(prepared, batch)
        for _ in range(2):
            network.forward(prepared, pageable)
        torch.cuda.synchronize()

        def timed_pass(inputs):
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                network.forward(prepared, inputs)
            return time.perf_counter() - t0

        # median of three timed passes: a pass is ~0.1 s of wall clock, short enough for
        # one host-side hiccup (page faults, a pinned-allocator refill) to skew it
        dt = sorted(timed_pass(batch) for _ in range(3))[1]
        dt_pageable = sorted(timed_pass(pageable) for _ in range(3))[1]
        e2e = {"value": n_local * e2e_steps / dt, "unit": "images/s",
               "h2d_bytes_per_step": int(n_local * 3 * hw * hw * 4),
               "d2h_bytes_per_step": int(n_local * eng.out_c * eng.out_hw * eng.out_hw * 4),
               "path": "network.forward(prepared, list[DenseTensor3]) with the inputs in pinned host "
                       "memory (network.pinned_batch); host WHC in, host DenseTensor3 out; median of "
                       "3 timed passes",
               "pageable": {"value": n_local * e2e_steps / dt_pageable,
                            "note": "same call with pageable numpy inputs (threaded pack into pinned staging)"}}

    # config 3 also names batch 1: one image through the same prepared stack (device-timed,
    # graph-replayed forwards; below 12 images the jump-table kernel's small-grid plans run)
    batch1 = None
    if world == 1 and args.workload == "c3":
        x1 = x[:1].contiguous()
        for _ in range(5):
            eng.forward_device(x1)
        torch.cuda.synchronize()
        reps1 = 50
        a1, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a1.record()
        for _ in range(reps1):
            eng.forward_device(x1)
        b1.record()
        b1.synchronize()
        ms1 = a1.elapsed_time(b1) / reps1
        batch1 = {"ms_per_forward": ms1, "images_per_s": 1e3 / ms1,
                  "nnz_tflops": flops_img / (ms1 * 1e-3) / 1e12,
                  "note": "batch 1 (config 3's other batch size), inputs in HBM, CUDA events over 50 "
                          "graph-replayed forwards; jump-table kernel small-grid plans below 12 images"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl.vgg16_weights(seed=103, zero_frac=zf), hw, sample_images=64)

    if rank == 0:
        peaks = _peaks()
        clocks = sampler.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.workload == "c3" else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded numpy, workloads.py): x~N(0,1), W~N(0,sqrt(2/fan_in)) i.i.d. masked",
            "config": bench_config(desc, n_total, world, backend, zf),
            "nnz_gflops": flops_img * n_total * args.steps / (elapsed_ms * 1e-3) / 1e9,
            "nnz_gflop_per_image": flops_img / 1e9,
            "roofline": {"bound": "fp32",
                         "kernel": ("sfjit: per-layer specialised sparse-filter kernels (one per 48-filter group, "
                                    "weights as FFMA2 immediates); achieved = the timed step's nnz-FLOP rate per "
                                    "GPU (CUDA events over the timed region; the step is these kernels, replayed "
                                    "as a CUDA graph)" if jit_on else
                                    "sf3x3_kernel: achieved = the timed step's nnz-FLOP rate per GPU"),
                         "achieved": achieved_tf, "peak": peak_meas, "unit": "TFLOP/s",
                         "frac": achieved_tf / peak_meas,
                         "per_launch_achieved": per_launch_tf,
                         "per_launch_note": "each layer alone, full batch, one part, second launch timed "
                                            "(code L2-resident) with CUDA events on its stream",
                         "peak_source": "measured FFMA probe (fscnn_fp32_probe) on this GPU; "
                                        f"nominal 148x128x2x1.965GHz = {peak_nom:.1f}",
                         "frac_of_nominal": achieved_tf / peak_nom,
                         "step_frac": achieved_tf / peak_meas,
                         "hbm_gbs_peak": peaks.get("hbm_gbs"),
                         "achieved_hbm_gbs": eng.bytes_per_image() * n_local / (kern_ms * 1e-3) / 1e9,
                         "traffic": traffic, "traffic_unit": "bytes/launch", "traffic_source": traffic_src,
                         "traffic_serialised_cold": traffic_serial,
                         "algorithmic_bytes_per_launch": eng.bytes_per_image() * n_local / len(eng.steps),
                         "per_layer_ms": [round(v, 4) for v in layer_ms]},
            "gpu_launches": launches,
            "prepare": {"sfjit": jit_on, "compile_wait_s": round(t_jit, 2),
                        "note": "bank compile (nvJitLink on host threads, overlapped with encoding) joined "
                                "before the timed region; cached on disk by content hash"},
            "clocks": clocks,
            "e2e": e2e,
            "batch1": batch1,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
