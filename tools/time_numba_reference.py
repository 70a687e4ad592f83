"""Context line: the reference's own CPU path (sparse_infer, numba) timed on the VGG16
config-3 workload (224x224, 90 % i.i.d. filter zeros), workers = 1 and all cores.

The reference cannot travel to the GPU box (it is read-only outside the repo and its
sources must not be copied in), so this runs in the build container; the result is
recorded in profiles/r02_numba_reference.json as context next to the oracle port that
bench.py's reference arm times on the GPU host.

  NUMBA_CACHE_DIR=/tmp/nc PYTHONPATH=/root/reference/pkg/src python tools/time_numba_reference.py
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sparse_infer as si  # noqa: E402  (the reference package, from PYTHONPATH)

from paper_2212_08815_b200 import workloads as wl  # noqa: E402

n_img = int(os.environ.get("N_IMG", "4"))
layers = wl.vgg16_weights(seed=103, zero_frac=0.9)
net = si.build_benchmark_net("vgg16_desk", 1.0, input_hw=224, variant="sparse_filter")
weights = si.NetworkWeights(entries=[si.ConvParams(filters=f, bias=b) for f, b in layers])
t0 = time.perf_counter()
prepared = si.prepare(net, weights)
prep_s = time.perf_counter() - t0
x = wl.vgg16_input(n_img, seed=104)
batch = [si.DenseTensor3.from_array(a) for a in x]
si.forward(prepared, batch[:1], workers=1)  # numba JIT warm-up
out = {"prepare_s": prep_s, "images": n_img, "host_cores": os.cpu_count()}
for workers, strat in ((1, "strategy_ii"), (os.cpu_count(), "strategy_ii"), (os.cpu_count(), "strategy_i")):
    st = si.ForwardStrategy(si.StrategyKind[strat.upper()])
    res = si.forward(prepared, batch, workers=workers, strategy=st)
    out[f"workers{workers}_{strat}_images_per_s"] = n_img / res.report.seconds
    print(workers, strat, n_img / res.report.seconds, flush=True)
print(json.dumps(out))
