"""Seeded synthetic workloads for the BASELINE.json configurations.

The paper measures on trained/pruned networks that are not available offline; the
configurations in BASELINE.json are therefore defined on synthetic tensors with the
stated shapes and value distributions, generated here with numpy's PCG64
``default_rng`` so that the GPU path, the CPU oracle and the reference all see the
same arrays.  All arrays are (N, C, H, W)- or (K, C, kh, kw)-indexed float32.

C1  sparse-filter conv 64->64 @56x56, x~N(0,1), W~N(0,0.05) with 95% i.i.d. zeros
C2  sparse-input conv 128->128 @28x28, x=|N(0,1)| with 90% i.i.d. zeros, W~N(0,0.05) dense
C3  VGG16 conv stack @224x224, x~N(0,1), W~N(0, sqrt(2/fan_in)) with 90% i.i.d. zeros
C4  per-layer sweep on the 13 VGG16 conv shapes at batch 32
C5  C3 at batch 256 with 95% zeros (batch-sharded across GPUs)
"""

from __future__ import annotations

import numpy as np

VGG16_PLAN = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]


def vgg16_conv_shapes(hw: int = 224, in_c: int = 3):
    """(C_in, K, H, W) of each of the 13 conv layers (network.py:541, :550-602)."""
    shapes = []
    c = in_c
    for item in VGG16_PLAN:
        if item == "M":
            hw //= 2
        else:
            shapes.append((c, item, hw, hw))
            c = item
    return shapes


def _rng(seed):
    return np.random.default_rng(seed)


def iid_mask_(arr: np.ndarray, rng, zero_frac: float) -> np.ndarray:
    """Zero each entry independently with probability ``zero_frac`` (in place)."""
    if zero_frac > 0.0:
        arr[rng.random(arr.shape, dtype=np.float32) < zero_frac] = 0.0
    return arr


def normal(rng, shape, std=1.0) -> np.ndarray:
    a = rng.standard_normal(shape, dtype=np.float32)
    if std != 1.0:
        a *= np.float32(std)
    return a


def c1(seed: int = 101):
    """Config 1: returns (x (1,64,56,56), W (64,64,3,3) 95% zeros, bias zeros)."""
    rng = _rng(seed)
    x = normal(rng, (1, 64, 56, 56))
    w = iid_mask_(normal(rng, (64, 64, 3, 3), 0.05), rng, 0.95)
    return x, w, np.zeros(64, np.float32)


def c2(seed: int = 102):
    """Config 2: returns (x (1,128,28,28) |N(0,1)| 90% zeros, dense W (128,128,3,3), bias zeros)."""
    rng = _rng(seed)
    x = iid_mask_(np.abs(normal(rng, (1, 128, 28, 28))), rng, 0.90)
    w = normal(rng, (128, 128, 3, 3), 0.05)
    return x, w, np.zeros(128, np.float32)


def vgg16_weights(seed: int = 103, zero_frac: float = 0.90, hw: int = 224, scale: float = 1.0):
    """Config 3/5 weights: per conv W ~ N(0, sqrt(2/(C*9))) with i.i.d. zeros, bias 0.

    ``scale`` narrows channel widths like build_benchmark_net (network.py:546-547).
    Returns a list of (filters (K,C,3,3), bias (K,)).
    """
    import math

    rng = _rng(seed)
    out = []
    c = 3
    for item in VGG16_PLAN:
        if item == "M":
            continue
        k = max(1, math.ceil(item * scale))
        w = iid_mask_(normal(rng, (k, c, 3, 3), math.sqrt(2.0 / (c * 9))), rng, zero_frac)
        out.append((w, np.zeros(k, np.float32)))
        c = k
    return out


def vgg16_input(n: int, seed: int = 104, hw: int = 224) -> np.ndarray:
    """Config 3/5 input batch x ~ N(0,1), shape (n, 3, hw, hw)."""
    return normal(_rng(seed), (n, 3, hw, hw))


def sweep_layer(layer: int, mode: str, zero_frac: float, n: int = 32, seed: int = 105, hw: int = 224):
    """Config 4 case: one VGG16 conv shape at batch n.

    mode 'sf': x ~ N(0,1), W ~ N(0, sqrt(2/fan_in)) with ``zero_frac`` i.i.d. zeros.
    mode 'si': x = |N(0,1)| with ``zero_frac`` i.i.d. zeros, dense W ~ N(0, 0.05).
    Returns (x (n,C,H,W), W (K,C,3,3), bias zeros).
    """
    import math

    c, k, h, w = vgg16_conv_shapes(hw)[layer]
    rng = _rng([seed, layer, int(zero_frac * 1000), 0 if mode == "sf" else 1])
    if mode == "sf":
        x = normal(rng, (n, c, h, w))
        wt = iid_mask_(normal(rng, (k, c, 3, 3), math.sqrt(2.0 / (c * 9))), rng, zero_frac)
    elif mode == "si":
        x = iid_mask_(np.abs(normal(rng, (n, c, h, w))), rng, zero_frac)
        wt = normal(rng, (k, c, 3, 3), 0.05)
    else:
        raise ValueError(f"unknown sweep mode {mode!r}")
    return x, wt, np.zeros(k, np.float32)
