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


def _put_sparse(payload, key, t):
    payload[f"{key}__order"] = np.array(t.order.name)
    payload[f"{key}__dims"] = np.array(t.dims, np.int64)
    payload[f"{key}__nodes"] = _nodes_i64(t.nodes)
    payload[f"{key}__matrix_offsets"] = np.asarray(t.matrix_offsets, np.int64)
    payload[f"{key}__segment_offsets"] = np.asarray(t.segment_offsets, np.int64)


def _with_special_nodes(t, rng):
    """Copy of t with some stored values replaced by +0.0, -0.0, NaN and negatives --
    explicit nodes the reference's own encoder never emits, but valid containers."""
    nodes = t.nodes.copy()
    data = np.nonzero(nodes["index"] != -1)[0]
    if data.size >= 4:
        pick = rng.choice(data, size=4, replace=False)
        nodes["value"][pick] = np.array([0.0, -0.0, np.nan, -1.5], np.float32)
    return si.SparseTensor3(order=t.order, dims=t.dims, nodes=nodes, matrix_offsets=t.matrix_offsets,
                            segment_offsets=t.segment_offsets)


def gen_pipeline(out):
    """The sparse-input pipeline and the remaining layer operators:
    node-format ReLU / LeakyReLU, pool_sparse, batch norm, pad, the dense baseline conv,
    dot_dense_sparse, the node-format transposes, the three network variants on the
    desk-scale VGG16 / YOLO stacks, and the density-evolution study."""
    rng = np.random.default_rng(2007)
    payload = {}
    orders = [o for o in si.AxisOrder3]
    # node-format activations, pooling, batch norm, pad
    for i in range(8):
        dims = (int(rng.integers(1, 6)), 2 * int(rng.integers(1, 5)), 2 * int(rng.integers(1, 5)))
        x = rand_input(rng, dims, 0.5)
        t = si.sparsify_tensor3(si.DenseTensor3.from_array(x), orders[i % 6])
        if i % 2:
            t = _with_special_nodes(t, rng)
        t.validate()
        key = f"n{i}"
        _put_sparse(payload, f"{key}_in", t)
        _put_sparse(payload, f"{key}_relu", si.apply_activation(t, "relu"))
        _put_sparse(payload, f"{key}_leaky", si.apply_activation(t, "leaky_relu", 0.1))
        _put_sparse(payload, f"{key}_pool", si.pool_sparse(t, (2, 2), "max" if i % 3 else "avg"))
        payload[f"{key}_pool__mode"] = np.array("max" if i % 3 else "avg")
        _put_sparse(payload, f"{key}_pad", si.pad_tensor(t, 1 + i % 2))
        payload[f"{key}_pad__p"] = np.array(1 + i % 2)
        bn = si.BatchNormParams(scale=rng.uniform(0.5, 1.5, dims[0]).astype(np.float32),
                                shift=rng.uniform(-0.5, 0.5, dims[0]).astype(np.float32),
                                mean=rng.uniform(-0.5, 0.5, dims[0]).astype(np.float32),
                                var=rng.uniform(0.5, 1.5, dims[0]).astype(np.float32), epsilon=1e-5)
        for f in ("scale", "shift", "mean", "var"):
            payload[f"{key}_bn__{f}"] = getattr(bn, f)
        _put_sparse(payload, f"{key}_bn", si.apply_batchnorm(t, bn))
        d = si.DenseTensor3.from_array(x)
        payload[f"{key}_dense__x"] = x
        payload[f"{key}_dense_bn__y"] = si.apply_batchnorm(d, bn).to_array()
        payload[f"{key}_dense_leaky__y"] = si.apply_activation(d, "leaky_relu", 0.1).to_array()
        payload[f"{key}_dense_pad__y"] = si.pad_tensor(d, 1 + i % 2).to_array()
    payload["n_node_cases"] = np.array(8)
    # dense baseline conv (layer + single filter) and the dot product
    for i in range(10):
        c, h_i, w_i, k, s, p, _ = rand_conv_case(rng, max_c=10, max_hw=16)
        n_f = int(rng.integers(1, 5))
        x = rand_input(rng, (c, h_i, w_i), 0.7)
        bank = np.stack([rand_filter(rng, (c, k, k), 0.6) for _ in range(n_f)])
        bias = rng.uniform(-0.2, 0.2, n_f).astype(np.float32)
        t_in = si.DenseTensor3.from_array(x)
        y = si.conv_forward_dense(t_in, [si.DenseTensor3.from_array(f) for f in bank], s, p, bias)
        geom = si.ConvGeometry((c, h_i, w_i), (c, k, k), s, p)
        payload[f"d{i}__x"], payload[f"d{i}__w"], payload[f"d{i}__bias"] = x, bank, bias
        payload[f"d{i}__geom"] = np.array([s, p], np.int64)
        payload[f"d{i}__y"] = y.to_array()
        payload[f"d{i}__y0"] = si.dense_conv_reference(t_in, si.DenseTensor3.from_array(bank[0]), geom)
    payload["n_dense_cases"] = np.array(10)
    for i in range(6):
        n = int(rng.integers(1, 40))
        dv = rand_input(rng, (n,))
        sv = si.SparseVector.from_dense(rand_input(rng, (int(rng.integers(1, n + 1)),), 0.4))
        payload[f"dot{i}__d"] = dv
        payload[f"dot{i}__length"] = np.array(sv.length)
        payload[f"dot{i}__nodes"] = _nodes_i64(sv.nodes)
        payload[f"dot{i}__y"] = np.array(si.dot_dense_sparse(dv, sv), np.float64)
    # transposes (explicit zero-valued nodes must move untouched)
    for i in range(6):
        r, c = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        a = rand_input(rng, (r, c), 0.5)
        order = si.AxisOrder2.WH if i % 2 == 0 else si.AxisOrder2.HW
        m = si.sparsify_matrix(a, order)
        if m.nnz >= 1:
            nodes = m.nodes.copy()
            nodes["value"][np.nonzero(nodes["index"] != -1)[0][0]] = 0.0
            m = si.SparseMatrix(order=m.order, n_rows=m.n_rows, n_cols=m.n_cols, nodes=nodes,
                                segment_offsets=m.segment_offsets)
        mt = si.transpose_matrix(m)
        for tag, mm in (("in", m), ("out", mt)):
            payload[f"tm{i}_{tag}__order"] = np.array(mm.order.name)
            payload[f"tm{i}_{tag}__shape"] = np.array([mm.n_rows, mm.n_cols], np.int64)
            payload[f"tm{i}_{tag}__nodes"] = _nodes_i64(mm.nodes)
            payload[f"tm{i}_{tag}__segment_offsets"] = np.asarray(mm.segment_offsets, np.int64)
    for i in range(4):
        dims = (int(rng.integers(1, 7)), int(rng.integers(1, 7)), int(rng.integers(1, 7)))
        t = si.sparsify_tensor3(si.DenseTensor3.from_array(rand_input(rng, dims, 0.5)), si.AxisOrder3.WHC)
        if i % 2:
            t = _with_special_nodes(t, rng)
        _put_sparse(payload, f"tt{i}_in", t)
        _put_sparse(payload, f"tt{i}_out", si.transpose_tensor3(t))
    # the three network variants (desk scale) with density recording
    cases = [("vgg16_desk", "sparse_input"), ("vgg16_desk_noact", "sparse_input"),
             ("vgg16_desk", "dense_baseline"), ("yolo_desk", "sparse_input"),
             ("yolo_desk", "dense_baseline"), ("yolo_desk", "sparse_filter"),
             ("yolo_desk_nobn", "sparse_input")]
    for i, (kind, variant) in enumerate(cases):
        net = nw.build_benchmark_net(kind, 0.125, input_hw=32, variant=variant)
        weights = nw.random_weights(net, 2008 + i)
        if variant == "sparse_filter":
            weights = nw.prune_weights(weights, 0.3, 2008 + i)
        prepared = nw.prepare(net, weights)
        base = nw.random_input(net.input_dims, 2008 + i)
        x = si.prune_random(base, 0.4, 2008 + i)
        inp = si.sparsify_tensor3(x, si.AxisOrder3.CHW) if variant == "sparse_input" else x
        res = nw.forward(prepared, [inp], record_density=True)
        o = res.outputs[0]
        key = f"net{i}"
        payload[f"{key}__kind"], payload[f"{key}__variant"] = np.array(kind), np.array(variant)
        payload[f"{key}__seed"] = np.array(2008 + i)
        payload[f"{key}__x"] = x.to_array()
        payload[f"{key}__densities"] = np.array(res.report.layer_densities, np.float64)
        if isinstance(o, si.SparseTensor3):
            _put_sparse(payload, f"{key}_out", o)
        else:
            payload[f"{key}_out__y"] = o.to_array()
        payload[f"{key}__weights_sha"] = np.array(sha(*[np.asarray(getattr(e, a)) for e in weights.entries
                                                         for a in (("filters", "bias") if hasattr(e, "filters")
                                                                   else ("scale", "shift", "mean", "var"))]))
    payload["n_net_cases"] = np.array(len(cases))
    net = nw.build_benchmark_net("vgg16_desk", 0.125, input_hw=32, variant="sparse_input")
    recs = nw.density_evolution(net, [0.1, 0.5, 1.0], 2020)
    payload["evo__input"] = np.array([r.input_density for r in recs], np.float64)
    payload["evo__layer"] = np.array([r.layer_index for r in recs], np.int64)
    payload["evo__kind"] = np.array([r.layer_kind for r in recs])
    payload["evo__density"] = np.array([r.output_density for r in recs], np.float64)
    np.savez_compressed(os.path.join(out, "pipeline.npz"), **payload)


def gen_formats(out):
    """The reference's on-disk formats: FSCT / FDT3 tensor blobs, FSNW
    weight files and the model text format, byte for byte."""
    import tempfile

    rng = np.random.default_rng(2009)
    payload = {}
    for i, o in enumerate(si.AxisOrder3):
        dims = tuple(int(v) for v in rng.integers(1, 6, 3))
        x = rand_input(rng, dims, 0.5)
        t = si.sparsify_tensor3(si.DenseTensor3.from_array(x), o)
        payload[f"t{i}__x"] = x
        payload[f"t{i}__order"] = np.array(o.name)
        payload[f"t{i}__fsct"] = np.frombuffer(si.sparse3_to_bytes(t), np.uint8)
        payload[f"t{i}__fdt3"] = np.frombuffer(si.dense3_to_bytes(si.DenseTensor3.from_array(x)), np.uint8)
    texts = [nw.format_model_text(nw.build_benchmark_net(kind, 0.125, input_hw=32)) for kind in nw.BENCH_KINDS]
    for j, kind in enumerate(("yolo_desk", "vgg16_desk")):
        net = nw.build_benchmark_net(kind, 0.0625, input_hw=32)
        w = nw.random_weights(net, 2010 + j)
        with tempfile.NamedTemporaryFile(suffix=".fsnw", delete=False) as fh:
            path = fh.name
        nw.save_weights(path, net, w)
        payload[f"w{j}__kind"] = np.array(kind)
        payload[f"w{j}__sha"] = np.array(sha(*[np.asarray(getattr(e, a)) for e in w.entries
                                               for a in (("filters", "bias") if hasattr(e, "filters")
                                                         else ("scale", "shift", "mean", "var"))]))
        payload[f"w{j}__fsnw"] = np.fromfile(path, np.uint8)
        os.unlink(path)
    payload["model_texts"] = np.array(texts)
    custom = "# a test stack\ninput c=3 h=14 w=14\nconv out=8 k=3 s=1 p=1  # first\nbatchnorm\nleaky_relu slope=0.1\npad p=1\nmaxpool k=2\nconv out=4 k=3 p=1\navgpool k=2\nrelu\n"
    payload["custom_text"] = np.array(custom)
    payload["custom_formatted"] = np.array(nw.format_model_text(nw.parse_model_text(custom, "custom")))
    np.savez_compressed(os.path.join(out, "formats.npz"), **payload)


def gen_harness(out):
    """The reference harness's density outputs (bench_cli.run_bench's probe rows and
    run_density_study) for small configs; timings are machine-specific and not kept."""
    from sparse_infer import bench_cli as bc

    payload = {}
    for i, (kind, variant) in enumerate((("vgg16_desk", "sparse_input"), ("vgg16_desk", "sparse_filter"))):
        cfg = bc.BenchConfig(net_kind=kind, scale=0.125, variant=variant, densities=[0.1, 0.5], reps=3,
                             timing_csv=None, density_csv=None)
        timing, dens = bc.run_bench(cfg)
        payload[f"b{i}__kind"], payload[f"b{i}__variant"] = np.array(kind), np.array(variant)
        payload[f"b{i}__timing_keys"] = np.array([f"{r.variant}|{r.density:g}|{r.batch}|{r.workers}|{r.strategy}|{r.rep}"
                                                  for r in timing])
        payload[f"b{i}__density"] = np.array([[r.input_density, r.layer_index, r.output_density] for r in dens])
        payload[f"b{i}__density_kind"] = np.array([r.layer_kind for r in dens])
    cfg = bc.BenchConfig(net_kind="yolo_desk", scale=0.125, variant="sparse_input", densities=[0.2, 1.0], reps=3)
    for kind, rows in bc.run_density_study(cfg).items():
        payload[f"study_{kind}"] = np.array([[r.input_density, r.layer_index, r.output_density] for r in rows])
    np.savez_compressed(os.path.join(out, "harness.npz"), **payload)


def main():
    gen_harness(HERE)
    gen_formats(HERE)
    gen_pipeline(HERE)
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
