"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

The reference package (sparse_infer, pure Python + numba) is imported read-only from
/root/reference/pkg/src with its numba cache redirected to /tmp so nothing is
written under /root/reference.  Every fixture stores the reference's own outputs
for seeded inputs; the oracle (oracle/) and the CUDA path are checked against them
by tests/.  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import hashlib
import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "fscnn_numba_cache"))
sys.dont_write_bytecode = True

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

import sparse_infer as si  # noqa: E402  (the reference)
from sparse_infer import network as nw  # noqa: E402

from paper_2212_08815_b200 import workloads as wl  # noqa: E402


def _nodes_i64(nodes) -> np.ndarray:
    """Node buffer as raw little-endian int64 words (bit-exact container)."""
    return np.ascontiguousarray(nodes).view(np.int64).copy()


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def rand_input(rng, dims, density=1.0):
    arr = rng.uniform(-0.5, 0.5, dims).astype(np.float32)
    if density < 1.0:
        arr[rng.random(dims) >= density] = 0.0
    return arr


def rand_filter(rng, dims, density=1.0):
    c, h, w = dims
    arr = rng.normal(0.0, np.sqrt(2.0 / (c * h * w)), dims).astype(np.float32)
    if density < 1.0:
        arr[rng.random(dims) >= density] = 0.0
    return arr


def rand_conv_case(rng, max_c=16, max_hw=32):
    while True:
        c = int(rng.integers(1, max_c + 1))
        h_i = int(rng.integers(1, max_hw + 1))
        w_i = int(rng.integers(1, max_hw + 1))
        k = int(rng.choice([1, 3, 5]))
        s = int(rng.choice([1, 2]))
        p = int(rng.choice([0, 1]))
        if k <= h_i + 2 * p and k <= w_i + 2 * p:
            return c, h_i, w_i, k, s, p, float(rng.choice([0.01, 0.05, 0.1, 0.5, 1.0]))


def gen_encoder(out):
    cases = {}
    # survey-worked example: -0.0 dropped, layout (w outer, h inner, c in fiber)
    ex = np.zeros((3, 2, 2), np.float32)
    ex[0, 0, 0], ex[2, 0, 0], ex[1, 1, 0], ex[2, 1, 1] = 1.0, 2.0, 3.0, 4.0
    ex[1, 0, 1] = -0.0
    cases["worked"] = (ex, "CHW")
    nan = np.zeros((4, 3, 2), np.float32)
    nan[1, 2, 1] = np.nan
    nan[3, 0, 0] = -0.0
    nan[0, 0, 0] = np.inf
    nan[2, 1, 0] = -np.inf
    cases["specials"] = (nan, "CHW")
    cases["zeros"] = (np.zeros((2, 2, 2), np.float32), "CHW")
    cases["ones"] = (np.ones((2, 2, 2), np.float32), "CHW")
    rng = np.random.default_rng(2001)
    orders = [o.name for o in si.AxisOrder3]
    for i in range(36):
        dims = tuple(int(x) for x in rng.integers(1, 10, 3))
        dens = float(rng.choice([0.0, 0.05, 0.3, 0.7, 1.0]))
        arr = rand_input(rng, dims, density=dens) if dens > 0 else np.zeros(dims, np.float32)
        cases[f"rand{i}"] = (arr, orders[i % 6])
    payload = {}
    for name, (arr, order) in cases.items():
        t = si.sparsify_tensor3(si.DenseTensor3.from_array(arr), si.AxisOrder3[order])
        t.validate()
        payload[f"{name}__input"] = arr
        payload[f"{name}__order"] = np.array(order)
        payload[f"{name}__nodes"] = _nodes_i64(t.nodes)
        payload[f"{name}__matrix_offsets"] = t.matrix_offsets.astype(np.int64)
        payload[f"{name}__segment_offsets"] = t.segment_offsets.astype(np.int64)
    # a filter bank through SparseTensor4.stack (network.prepare path)
    bank = np.stack([rand_filter(rng, (8, 3, 3), 0.3) for _ in range(16)])
    bank[3] = 0.0  # an all-zero filter
    t4 = si.SparseTensor4.stack(
        [si.sparsify_tensor3(si.DenseTensor3.from_array(f), si.AxisOrder3.CHW) for f in bank]
    )
    t4.validate()
    payload["bank__input"] = bank
    payload["bank__nodes"] = _nodes_i64(t4.nodes)
    payload["bank__tensor_offsets"] = t4.tensor_offsets.astype(np.int64)
    payload["bank__matrix_offsets"] = t4.matrix_offsets.astype(np.int64)
    payload["bank__segment_offsets"] = t4.segment_offsets.astype(np.int64)
    payload["names"] = np.array(list(cases))
    np.savez_compressed(os.path.join(out, "encoder.npz"), **payload)


def gen_sf(out):
    rng = np.random.default_rng(2002)
    payload = {}
    n_cases = 40
    for i in range(n_cases):
        c, h_i, w_i, k, s, p, dens = rand_conv_case(rng)
        n_f = int(rng.integers(1, 9))
        x = rand_input(rng, (c, h_i, w_i))
        bank = np.stack([rand_filter(rng, (c, k, k), dens) for _ in range(n_f)])
        bias = rng.uniform(-0.2, 0.2, n_f).astype(np.float32)
        t4 = si.SparseTensor4.stack(
            [si.sparsify_tensor3(si.DenseTensor3.from_array(f), si.AxisOrder3.CHW) for f in bank]
        )
        t_in = si.DenseTensor3.from_array(x)
        y2 = si.conv_forward_strategy_II(t_in, t4, s, p, bias)
        y1 = si.conv_forward_strategy_I(t_in, t4, s, p, bias)
        assert np.array_equal(y1.data, y2.data)
        geom = si.ConvGeometry((c, h_i, w_i), (c, k, k), s, p)
        mults = sum(
            si.conv_dense_input_sparse_filter_counted(t_in, t4.tensor(f), geom)[1] for f in range(n_f)
        )
        payload[f"c{i}__x"] = x
        payload[f"c{i}__w"] = bank
        payload[f"c{i}__bias"] = bias
        payload[f"c{i}__geom"] = np.array([s, p], np.int64)
        payload[f"c{i}__y"] = y2.to_array()
        payload[f"c{i}__mults"] = np.array(mults, np.int64)
    payload["n_cases"] = np.array(n_cases)
    np.savez_compressed(os.path.join(out, "sf_conv.npz"), **payload)


def gen_si(out):
    rng = np.random.default_rng(2003)
    payload = {}
    n_cases = 30
    for i in range(n_cases):
        c, h_i, w_i, k, s, p, _ = rand_conv_case(rng, max_c=12, max_hw=20)
        n_f = int(rng.integers(1, 7))
        dens = float(rng.choice([0.05, 0.2, 0.5]))
        x = rand_input(rng, (c, h_i, w_i), dens)
        bank = np.stack([rand_filter(rng, (c, k, k)) for _ in range(n_f)])
        with_bias = i % 5 == 4
        bias = rng.uniform(-0.2, 0.2, n_f).astype(np.float32) if with_bias else np.zeros(n_f, np.float32)
        sp = si.sparsify_tensor3(si.DenseTensor3.from_array(x), si.AxisOrder3.CHW)
        out_t = si.conv_forward_sparse_input(
            sp, [si.DenseTensor3.from_array(f) for f in bank], s, p, bias
        )
        payload[f"c{i}__x"] = x
        payload[f"c{i}__w"] = bank
        payload[f"c{i}__bias"] = bias
        payload[f"c{i}__geom"] = np.array([s, p], np.int64)
        if isinstance(out_t, si.DenseTensor3):
            payload[f"c{i}__kind"] = np.array("dense")
            payload[f"c{i}__y"] = out_t.to_array()
        else:
            payload[f"c{i}__kind"] = np.array("sparse")
            payload[f"c{i}__y"] = si.densify_tensor3(out_t).to_array()
            payload[f"c{i}__nodes"] = _nodes_i64(out_t.nodes)
            payload[f"c{i}__segment_offsets"] = out_t.segment_offsets.astype(np.int64)
            payload[f"c{i}__matrix_offsets"] = out_t.matrix_offsets.astype(np.int64)
    payload["n_cases"] = np.array(n_cases)
    np.savez_compressed(os.path.join(out, "si_conv.npz"), **payload)


def gen_configs(out):
    # C1: full config-1 sparse-filter conv through strategy II
    x, w, b = wl.c1()
    t4 = si.SparseTensor4.stack(
        [si.sparsify_tensor3(si.DenseTensor3.from_array(f), si.AxisOrder3.CHW) for f in w]
    )
    t_in = si.DenseTensor3.from_array(x[0])
    y = si.conv_forward_strategy_II(t_in, t4, 1, 1, b).to_array()
    geom = si.ConvGeometry((64, 56, 56), (64, 3, 3), 1, 1)
    mults = sum(si.conv_dense_input_sparse_filter_counted(t_in, t4.tensor(f), geom)[1] for f in range(64))
    np.savez_compressed(
        os.path.join(out, "c1.npz"),
        input_sha=np.array(sha(x, w)),
        y=y,
        mults=np.array(mults, np.int64),
        nodes_sha=np.array(sha(t4.nodes, t4.tensor_offsets, t4.matrix_offsets, t4.segment_offsets)),
        n_nodes=np.array(len(t4.nodes), np.int64),
    )
    # C2: full config-2 sparse-input conv layer (bias 0 -> CHW node output)
    x, w, b = wl.c2()
    sp = si.sparsify_tensor3(si.DenseTensor3.from_array(x[0]), si.AxisOrder3.CHW)
    out_t = si.conv_forward_sparse_input(sp, [si.DenseTensor3.from_array(f) for f in w], 1, 1, b)
    np.savez_compressed(
        os.path.join(out, "c2.npz"),
        input_sha=np.array(sha(x, w)),
        in_nodes_sha=np.array(sha(sp.nodes, sp.matrix_offsets, sp.segment_offsets)),
        y=si.densify_tensor3(out_t).to_array(),
        out_nodes_sha=np.array(sha(out_t.nodes, out_t.matrix_offsets, out_t.segment_offsets)),
        n_out_nodes=np.array(len(out_t.nodes), np.int64),
    )


def gen_vgg_small(out):
    """vgg16_desk at scale 0.125 on 32x32 (the reference's own desk config),
    sparse_filter variant, 90% i.i.d. zeros, batch 2."""
    net = nw.build_benchmark_net("vgg16_desk", 0.125, input_hw=32, variant=nw.VARIANT_SPARSE_FILTER)
    layers = wl.vgg16_weights(seed=2004, zero_frac=0.9, scale=0.125)
    weights = nw.NetworkWeights(entries=[nw.ConvParams(filters=f, bias=b) for f, b in layers])
    prepared = nw.prepare(net, weights)
    xs = wl.vgg16_input(2, seed=2005, hw=32)
    res = nw.forward(prepared, [si.DenseTensor3.from_array(a) for a in xs])
    ys = np.stack([o.to_array() for o in res.outputs])
    payload = {"x": xs, "y": ys, "n_layers": np.array(len(layers))}
    for i, (f, b) in enumerate(layers):
        payload[f"w{i}"] = f
        payload[f"b{i}"] = b
    np.savez_compressed(os.path.join(out, "vgg_small.npz"), **payload)


def gen_pool_relu(out):
    rng = np.random.default_rng(2006)
    payload = {}
    for i, (dims, pw, mode) in enumerate(
        [((3, 4, 6), (2, 2), "max"), ((2, 8, 8), (2, 2), "avg"), ((5, 6, 6), (3, 2), "max"), ((4, 4, 4), (1, 1), "max")]
    ):
        x = rand_input(rng, dims, 0.6)
        x[0, 0, 0] = np.nan
        y = si.pool_standalone(si.DenseTensor3.from_array(x), pw, mode).to_array()
        payload[f"p{i}__x"], payload[f"p{i}__y"] = x, y
        payload[f"p{i}__win"], payload[f"p{i}__mode"] = np.array(pw), np.array(mode)
    x = rand_input(rng, (3, 5, 5), 0.7)
    x[0, 0, :4] = [np.nan, -0.0, 0.0, -np.inf]
    payload["relu__x"] = x
    payload["relu__y"] = si.apply_activation(si.DenseTensor3.from_array(x), "relu").to_array()
    np.savez_compressed(os.path.join(out, "pool_relu.npz"), **payload)


def main():
    gen_encoder(HERE)
    gen_sf(HERE)
    gen_si(HERE)
    gen_configs(HERE)
    gen_vgg_small(HERE)
    gen_pool_relu(HERE)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
