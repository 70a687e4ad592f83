"""The sparse-input pipeline and the remaining layer operators on the GPU (SURVEY.md
§8f-1 and §8f-2), bit-exact against the reference's own outputs
(tests/golden/pipeline.npz, made by tests/golden/make_golden.py::gen_pipeline):

* node-format ReLU / LeakyReLU (rebuild_tensor3 semantics, incl. explicit +0.0 / -0.0 /
  NaN nodes), pool_sparse, batch norm, pad (CHW node pad keeps explicit zero nodes),
  all six axis orders;
* the dense baseline conv (layer and single filter) and dot_dense_sparse;
* transpose_matrix / transpose_tensor3 (values move untouched);
* prepare/forward of the sparse_input, dense_baseline and sparse_filter variants on
  the desk-scale VGG16 and YOLO stacks (incl. the conv+pool fusion rule and per-layer
  density recording), random_weights / prune_weights / prune_random, and
  density_evolution.
"""

import numpy as np
import pytest

from conftest import load_golden, nodes_from_i64, weights_sha

import paper_2212_08815_b200 as fs
from paper_2212_08815_b200 import network as nw

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    return load_golden("pipeline.npz")


def _sparse(g, key):
    return fs.SparseTensor3(fs.AxisOrder3[str(g[f"{key}__order"])], tuple(int(v) for v in g[f"{key}__dims"]),
                            nodes_from_i64(g[f"{key}__nodes"]), g[f"{key}__matrix_offsets"],
                            g[f"{key}__segment_offsets"])


def _same_sparse(t, g, key):
    assert t.order.name == str(g[f"{key}__order"]), key
    assert tuple(t.dims) == tuple(int(v) for v in g[f"{key}__dims"]), key
    assert np.ascontiguousarray(t.nodes).view(np.int64).tobytes() == g[f"{key}__nodes"].tobytes(), key
    assert np.array_equal(np.asarray(t.segment_offsets, np.int64), g[f"{key}__segment_offsets"]), key
    assert np.array_equal(np.asarray(t.matrix_offsets, np.int64), g[f"{key}__matrix_offsets"]), key


def _bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.int32)


def test_node_format_activation_pool_batchnorm_pad(g):
    for i in range(int(g["n_node_cases"])):
        key = f"n{i}"
        t = _sparse(g, f"{key}_in")
        _same_sparse(fs.apply_activation(t, "relu"), g, f"{key}_relu")
        _same_sparse(fs.apply_activation(t, "leaky_relu", 0.1), g, f"{key}_leaky")
        _same_sparse(fs.pool_sparse(t, (2, 2), str(g[f"{key}_pool__mode"])), g, f"{key}_pool")
        _same_sparse(fs.pad_tensor(t, int(g[f"{key}_pad__p"])), g, f"{key}_pad")
        bn = fs.BatchNormParams(scale=g[f"{key}_bn__scale"], shift=g[f"{key}_bn__shift"],
                                mean=g[f"{key}_bn__mean"], var=g[f"{key}_bn__var"], epsilon=1e-5)
        _same_sparse(fs.apply_batchnorm(t, bn), g, f"{key}_bn")
        d = fs.DenseTensor3.from_array(g[f"{key}_dense__x"])
        assert np.array_equal(_bits(fs.apply_batchnorm(d, bn).to_array()), _bits(g[f"{key}_dense_bn__y"])), key
        assert np.array_equal(_bits(fs.apply_activation(d, "leaky_relu", 0.1).to_array()),
                              _bits(g[f"{key}_dense_leaky__y"])), key
        assert np.array_equal(_bits(fs.pad_tensor(d, int(g[f"{key}_pad__p"])).to_array()),
                              _bits(g[f"{key}_dense_pad__y"])), key


def test_layer_op_validation_messages():
    t = fs.sparsify_tensor3(fs.DenseTensor3.from_array(np.ones((2, 4, 4), np.float32)), fs.AxisOrder3.CHW)
    with pytest.raises(ValueError, match="divisible"):
        fs.pool_sparse(t, (3, 3), "max")
    with pytest.raises(ValueError, match="positive"):
        fs.pool_sparse(t, (0, 2), "max")
    with pytest.raises(ValueError, match="non-negative"):
        fs.pad_tensor(t, -1)
    assert fs.pad_tensor(t, 0) is t
    with pytest.raises(ValueError, match="slope"):
        fs.apply_activation(t, "leaky_relu", -0.1)
    with pytest.raises(ValueError, match="shape"):
        fs.apply_batchnorm(t, fs.BatchNormParams(np.ones(3), np.zeros(3), np.zeros(3), np.ones(3)))
    with pytest.raises(fs.FormatError, match="WHC"):
        fs.transpose_tensor3(t)


def test_dense_baseline_conv_bitwise(g):
    for i in range(int(g["n_dense_cases"])):
        x, w, bias = g[f"d{i}__x"], g[f"d{i}__w"], g[f"d{i}__bias"]
        s, p = (int(v) for v in g[f"d{i}__geom"])
        t_in = fs.DenseTensor3.from_array(x)
        y = fs.conv_forward_dense(t_in, [fs.DenseTensor3.from_array(f) for f in w], s, p, bias)
        assert np.array_equal(_bits(y.to_array()), _bits(g[f"d{i}__y"])), i
        geom = fs.ConvGeometry(tuple(x.shape), tuple(w.shape[1:]), s, p)
        y0 = fs.dense_conv_reference(t_in, fs.DenseTensor3.from_array(w[0]), geom)
        assert np.array_equal(_bits(y0), _bits(g[f"d{i}__y0"])), i


def test_dot_dense_sparse_bitwise(g):
    for i in range(6):
        sv = fs.SparseVector(int(g[f"dot{i}__length"]), nodes_from_i64(g[f"dot{i}__nodes"]))
        again = fs.SparseVector.from_dense(sv.to_dense())  # the GPU encoder, 1-D
        assert again.length == sv.length and again.nodes.tobytes() == sv.nodes.tobytes()
        got = fs.dot_dense_sparse(g[f"dot{i}__d"], sv)
        assert np.float32(got).tobytes() == np.float32(g[f"dot{i}__y"]).tobytes(), i


def test_transposes_move_nodes_untouched(g):
    for i in range(6):
        m = fs.SparseMatrix(fs.AxisOrder2[str(g[f"tm{i}_in__order"])], *(int(v) for v in g[f"tm{i}_in__shape"]),
                            nodes_from_i64(g[f"tm{i}_in__nodes"]), g[f"tm{i}_in__segment_offsets"])
        mt = fs.transpose_matrix(m)
        assert mt.order.name == str(g[f"tm{i}_out__order"])
        assert np.ascontiguousarray(mt.nodes).view(np.int64).tobytes() == g[f"tm{i}_out__nodes"].tobytes(), i
        assert np.array_equal(np.asarray(mt.segment_offsets, np.int64), g[f"tm{i}_out__segment_offsets"]), i
        # and back: the round trip restores the input exactly
        back = fs.transpose_matrix(mt)
        assert np.ascontiguousarray(back.nodes).view(np.int64).tobytes() == g[f"tm{i}_in__nodes"].tobytes(), i
    for i in range(4):
        _same_sparse(fs.transpose_tensor3(_sparse(g, f"tt{i}_in")), g, f"tt{i}_out")


def test_network_variants_bitwise(g):
    fs.set_exact(True)  # the sparse_filter variant's bit-exact kernel
    try:
        for i in range(int(g["n_net_cases"])):
            key = f"net{i}"
            kind, variant, seed = str(g[f"{key}__kind"]), str(g[f"{key}__variant"]), int(g[f"{key}__seed"])
            net = nw.build_benchmark_net(kind, 0.125, input_hw=32, variant=variant)
            weights = nw.random_weights(net, seed)
            if variant == "sparse_filter":
                weights = nw.prune_weights(weights, 0.3, seed)
            assert weights_sha(weights) == str(g[f"{key}__weights_sha"]), key
            x = fs.prune_random(nw.random_input(net.input_dims, seed), 0.4, seed)
            assert np.array_equal(_bits(x.to_array()), _bits(g[f"{key}__x"])), key
            inp = fs.sparsify_tensor3(x, fs.AxisOrder3.CHW) if variant == "sparse_input" else x
            res = nw.forward(nw.prepare(net, weights), [inp], record_density=True)
            out = res.outputs[0]
            if isinstance(out, fs.SparseTensor3):
                _same_sparse(out, g, f"{key}_out")
            else:
                assert np.array_equal(_bits(out.to_array()), _bits(g[f"{key}_out__y"])), key
            assert np.array_equal(np.array(res.report.layer_densities, np.float64), g[f"{key}__densities"]), key
    finally:
        fs.set_exact(False)


def _same_output(a, b, key):
    assert type(a) is type(b), key
    if isinstance(a, fs.SparseTensor3):
        assert a.nodes.tobytes() == b.nodes.tobytes(), key
        assert np.array_equal(a.segment_offsets, b.segment_offsets), key
        assert np.array_equal(a.matrix_offsets, b.matrix_offsets), key
    else:
        assert np.array_equal(_bits(a.to_array()), _bits(b.to_array())), key


@pytest.mark.parametrize("exact", [True, False])
def test_batched_forward_equals_per_image(g, monkeypatch, exact):
    """forward() runs every variant as one batched device pass (activations resident in
    HBM between steps; the VGG16 sparse_filter engine aside); every image's output and
    recorded layer densities must be the per-image layer path's, bit for bit, with the
    bit-exact or the fast kernels, and (bit-exact kernels) the golden case's output the
    reference's.  Inputs with explicit zero-valued nodes take the per-image path."""
    import paper_2212_08815_b200.network as nwmod

    def per_image(prepared, inp):
        monkeypatch.setattr(nwmod, "_BATCHED", False)
        try:
            return nw.forward(prepared, inp, record_density=True)
        finally:
            monkeypatch.setattr(nwmod, "_BATCHED", True)

    fs.set_exact(exact)
    try:
        for i in range(int(g["n_net_cases"])):
            key = f"net{i}"
            kind, variant, seed = str(g[f"{key}__kind"]), str(g[f"{key}__variant"]), int(g[f"{key}__seed"])
            net = nw.build_benchmark_net(kind, 0.125, input_hw=32, variant=variant)
            weights = nw.random_weights(net, seed)
            if variant == "sparse_filter":
                weights = nw.prune_weights(weights, 0.3, seed)
            prepared = nw.prepare(net, weights)
            xs = [fs.prune_random(nw.random_input(net.input_dims, seed), 0.4, seed)]
            xs += [fs.prune_random(nw.random_input(net.input_dims, seed + j), 0.3 + 0.2 * j, seed + j)
                   for j in (1, 2)]
            inp = [fs.sparsify_tensor3(x, fs.AxisOrder3.CHW) if variant == "sparse_input" else x for x in xs]
            assert nwmod._batched_inputs_ok(prepared, inp)
            res_b = nw.forward(prepared, inp, record_density=True)
            res_s = per_image(prepared, inp)
            assert res_b.report.layer_densities == res_s.report.layer_densities, key
            for a, b in zip(res_b.outputs, res_s.outputs):
                _same_output(a, b, key)
            if exact:
                out = res_b.outputs[0]
                if isinstance(out, fs.SparseTensor3):
                    _same_sparse(out, g, f"{key}_out")
                else:
                    assert np.array_equal(_bits(out.to_array()), _bits(g[f"{key}_out__y"])), key
            if variant == "sparse_input":
                t = inp[0]
                nodes = t.nodes.copy()
                live = np.flatnonzero(nodes["index"] >= 0)
                nodes["value"][live[0]] = 0.0  # an explicit zero node
                z = fs.SparseTensor3(t.order, t.dims, nodes, t.matrix_offsets, t.segment_offsets)
                # the batched path declines it (device-side check) ...
                assert nwmod._forward_batched(prepared, [z, inp[1]]) is None
                # ... and forward() falls back to the per-image path, whose result it is
                got = nw.forward(prepared, [z, inp[1]]).outputs
                want = per_image(prepared, [z, inp[1]]).outputs
                for a, b in zip(got, want):
                    _same_output(a, b, key)
                # malformed structure (two live nodes of a segment out of channel order):
                # the batched path declines it on the device and the per-image path's
                # validation reports it, as the reference's format check would
                bad = t.nodes.copy()
                seg0 = int(t.segment_offsets[0])
                run = np.flatnonzero(bad["index"][seg0:] >= 0)
                j = next(r for r in range(len(run) - 1) if run[r + 1] == run[r] + 1)
                a0, a1 = seg0 + run[j], seg0 + run[j + 1]
                bad["index"][a0], bad["index"][a1] = bad["index"][a1], bad["index"][a0]
                zb = fs.SparseTensor3(t.order, t.dims, bad, t.matrix_offsets, t.segment_offsets)
                assert nwmod._forward_batched(prepared, [zb]) is None
                with pytest.raises(fs.FormatError):
                    nw.forward(prepared, [zb])
    finally:
        fs.set_exact(False)


def test_density_evolution_matches_reference(g):
    net = nw.build_benchmark_net("vgg16_desk", 0.125, input_hw=32, variant="sparse_input")
    recs = nw.density_evolution(net, [0.1, 0.5, 1.0], 2020)
    assert [r.input_density for r in recs] == list(g["evo__input"])
    assert [r.layer_index for r in recs] == list(g["evo__layer"])
    assert [r.layer_kind for r in recs] == [str(k) for k in g["evo__kind"]]
    assert np.array_equal(np.array([r.output_density for r in recs]), g["evo__density"])
    with pytest.raises(ValueError, match="sparse_input"):
        nw.density_evolution(net.with_variant("dense_baseline"), [0.5], 1)


def test_pipeline_ops_at_layer_size_vs_oracle(oracle):
    """The node-format ops on VGG16-layer-sized tensors (64 x 56 x 56, ~50 % dense, with
    explicit +0.0 / -0.0 / NaN nodes) against the oracle's restatements, byte for byte."""
    rng = np.random.default_rng(4242)
    x = rng.standard_normal((64, 56, 56)).astype(np.float32)
    x[rng.random(x.shape) < 0.5] = 0
    base = fs.sparsify_tensor3(fs.DenseTensor3.from_array(x), fs.AxisOrder3.CHW)
    nodes = base.nodes.copy()
    data = np.nonzero(nodes["index"] != -1)[0]
    pick = rng.choice(data, size=60, replace=False)
    nodes["value"][pick[:20]] = 0.0
    nodes["value"][pick[20:40]] = -0.0
    nodes["value"][pick[40:]] = np.nan
    t = fs.SparseTensor3(base.order, base.dims, nodes, base.matrix_offsets, base.segment_offsets)
    seg = np.asarray(t.segment_offsets, np.int64)
    for kind, slope in (("relu", 0.0), ("leaky_relu", 0.1)):
        got = fs.apply_activation(t, kind, slope)
        want_nodes, want_seg = oracle.rebuild(nodes, seg, "relu" if kind == "relu" else "leaky", slope)
        assert got.nodes.tobytes() == want_nodes.tobytes() and np.array_equal(got.segment_offsets, want_seg), kind
    got = fs.pad_tensor(t, 2)
    want_nodes, want_seg = oracle.pad_chw_nodes(nodes, seg, t.dims, 2)
    assert got.nodes.tobytes() == want_nodes.tobytes() and np.array_equal(got.segment_offsets, want_seg)
    dense = oracle.decode(nodes, seg, t.dims, "CHW")
    pooled = fs.pool_sparse(t, (2, 2), "max")
    want = oracle.pool(dense[None], 2, 2, "max")[0]
    p_nodes, _, _, p_seg = oracle.encode_batch(want[None], "CHW")
    assert pooled.nodes.tobytes() == p_nodes.tobytes() and np.array_equal(pooled.segment_offsets, p_seg[0])
    sc, sh, mu = (rng.uniform(-1, 1, 64).astype(np.float32) for _ in range(3))
    va = rng.uniform(0.5, 1.5, 64).astype(np.float32)
    d = fs.DenseTensor3.from_array(dense)
    got = fs.apply_batchnorm(d, fs.BatchNormParams(sc, sh, mu, va, 1e-5)).to_array()
    assert got.tobytes() == oracle.batchnorm(dense, sc, sh, mu, va, 1e-5).tobytes()
    whc = fs.sparsify_tensor3(d, fs.AxisOrder3.WHC)
    got = fs.transpose_tensor3(whc)
    want_nodes, want_seg = oracle.transpose_whc_to_chw(whc.nodes, np.asarray(whc.segment_offsets, np.int64), d.dims)
    assert got.nodes.tobytes() == want_nodes.tobytes() and np.array_equal(got.segment_offsets, want_seg)
