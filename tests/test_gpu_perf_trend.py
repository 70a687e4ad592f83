"""Performance trend (the reference's acceptance check, test_acceptance.py:219-251, SURVEY.md
§4): no absolute numbers, only that sparsity pays -- the sparse-filter conv at 1 % density
beats the every-weight baseline conv on the same layer, and its time does not fall as the
density rises (5 % slack for timing noise).  Device time from CUDA events, median of 7."""
import statistics

import numpy as np
import pytest
import torch

from paper_2212_08815_b200 import device

pytestmark = pytest.mark.gpu


def _time(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def test_sparse_filter_time_trend():
    rng = np.random.default_rng(17)
    n, c, k, h = 8, 128, 128, 56
    x = torch.from_numpy(rng.standard_normal((n, c, h, h)).astype(np.float32)).cuda()
    xh = device.to_halo(x)
    dense_w = rng.normal(0, np.sqrt(2 / (c * 9)), (k, c, 3, 3)).astype(np.float32)
    bias = torch.zeros(k, dtype=torch.float32, device="cuda")
    times = []
    for density in (0.01, 0.05, 0.1, 0.5, 1.0):
        w = dense_w * (rng.random(dense_w.shape) < density)
        bank = device.sf_pack(torch.from_numpy(w.astype(np.float32)).cuda())
        times.append(_time(lambda: device.sf_conv3x3(xh, bank, bias, relu=True, pool=False, w=h)))
    t_dense = _time(lambda: device.dense_conv_exact(x, torch.from_numpy(dense_w).cuda(), 1, 1, bias))
    assert times[0] < t_dense, (times, t_dense)
    for a, b in zip(times, times[1:]):
        assert a <= b * 1.05, times
