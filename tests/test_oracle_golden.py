"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz).

These run on CPU only.  They establish that oracle/ restates the reference
bit-for-bit (encoder, both conv paths, pooling, ReLU, the VGG stack), so the GPU
parity tests can trust it at sizes the golden fixtures do not cover.
"""

import numpy as np

from conftest import load_golden, nodes_from_i64
from paper_2212_08815_b200 import workloads as wl


def test_encoder_matches_reference_bitwise(oracle):
    g = load_golden("encoder.npz")
    for name in g["names"]:
        name = str(name)
        arr = g[f"{name}__input"]
        order = str(g[f"{name}__order"])
        nodes, mat, seg = oracle.encode(arr, order)
        assert nodes.view(np.int64).tobytes() == g[f"{name}__nodes"].tobytes(), name
        assert np.array_equal(mat, g[f"{name}__matrix_offsets"]), name
        assert np.array_equal(seg, g[f"{name}__segment_offsets"]), name
        back = oracle.decode(nodes, seg, arr.shape, order)
        # decode round trip is bit-exact except that -0.0 inputs come back +0.0
        want = np.where(arr == 0, np.float32(0), arr)
        assert np.array_equal(back.view(np.int32), want.view(np.int32)) or np.array_equal(
            back, want, equal_nan=True
        ), name


def test_encoder_bank_stack_matches_reference(oracle):
    g = load_golden("encoder.npz")
    nodes, tens, mat, seg = oracle.encode_batch(g["bank__input"], "CHW")
    assert nodes.view(np.int64).tobytes() == g["bank__nodes"].tobytes()
    assert np.array_equal(tens, g["bank__tensor_offsets"])
    assert np.array_equal(mat, g["bank__matrix_offsets"])
    assert np.array_equal(seg, g["bank__segment_offsets"])


def test_worked_example():
    """3x2x2 tensor with a -0.0 entry: the survey's hand-worked CHW encoding."""
    g = load_golden("encoder.npz")
    nodes = nodes_from_i64(g["worked__nodes"])
    assert [(int(n["index"]), float(n["value"])) for n in nodes] == [
        (0, 1.0), (2, 2.0), (-1, 0.0), (1, 3.0), (-1, 0.0), (-1, 0.0), (2, 4.0), (-1, 0.0)
    ]
    assert list(g["worked__segment_offsets"]) == [0, 3, 5, 6]
    assert list(g["worked__matrix_offsets"]) == [0, 5]


def test_sf_conv_matches_reference_bitwise(oracle):
    g = load_golden("sf_conv.npz")
    for i in range(int(g["n_cases"])):
        x, w, bias = g[f"c{i}__x"], g[f"c{i}__w"], g[f"c{i}__bias"]
        s, p = (int(v) for v in g[f"c{i}__geom"])
        k_n, _, h_f, w_f = w.shape
        nodes, seg = oracle.encode_bank(w)
        y = oracle.sf_conv(x[None], nodes, seg, k_n, h_f, w_f, s, p, bias, threads=2)[0]
        assert np.array_equal(y.view(np.int32), g[f"c{i}__y"].view(np.int32)), i
        mults = oracle.sf_count(x.shape[1], x.shape[2], seg, len(nodes), k_n, h_f, w_f, s, p)
        assert mults == int(g[f"c{i}__mults"]), i


def test_si_conv_matches_reference_bitwise(oracle):
    g = load_golden("si_conv.npz")
    for i in range(int(g["n_cases"])):
        x, w, bias = g[f"c{i}__x"], g[f"c{i}__w"], g[f"c{i}__bias"]
        s, p = (int(v) for v in g[f"c{i}__geom"])
        nodes, _, seg = oracle.encode(x, "CHW")
        y = oracle.si_conv([nodes], [seg], x.shape, w, s, p, threads=2)[0]
        if str(g[f"c{i}__kind"]) == "dense":
            y = y + bias[:, None, None]
        assert np.array_equal(y, g[f"c{i}__y"]), i
        if str(g[f"c{i}__kind"]) == "sparse":
            # the reference's CHW node output == encoding of the dense result
            on, om, os_ = oracle.encode(y, "CHW")
            assert on.view(np.int64).tobytes() == g[f"c{i}__nodes"].tobytes(), i
            assert np.array_equal(os_, g[f"c{i}__segment_offsets"]), i
            assert np.array_equal(om, g[f"c{i}__matrix_offsets"]), i


def test_config1_and_config2_match_reference(oracle):
    import hashlib

    def sha(*arrays):
        h = hashlib.sha256()
        for a in arrays:
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()

    g1 = load_golden("c1.npz")
    x, w, b = wl.c1()
    assert sha(x, w) == str(g1["input_sha"]), "workload generator drifted"
    nodes, tens, mat, seg = oracle.encode_batch(w, "CHW")
    assert sha(nodes, tens, mat, seg) == str(g1["nodes_sha"])
    y = oracle.sf_conv(x, nodes, seg, 64, 3, 3, 1, 1, b)[0]
    assert np.array_equal(y, g1["y"])
    assert oracle.sf_count(56, 56, seg, len(nodes), 64, 3, 3, 1, 1) == int(g1["mults"])

    g2 = load_golden("c2.npz")
    x, w, b = wl.c2()
    assert sha(x, w) == str(g2["input_sha"])
    n_in, m_in, s_in = oracle.encode(x[0], "CHW")
    assert sha(n_in, m_in, s_in) == str(g2["in_nodes_sha"])
    y = oracle.si_conv([n_in], [s_in], x.shape[1:], w, 1, 1)[0]
    assert np.array_equal(y, g2["y"])
    on, om, os_ = oracle.encode(y, "CHW")
    assert sha(on, om, os_) == str(g2["out_nodes_sha"])


def test_vgg_small_stack_matches_reference(oracle):
    g = load_golden("vgg_small.npz")
    banks = []
    for i in range(int(g["n_layers"])):
        w, b = g[f"w{i}"], g[f"b{i}"]
        nodes, seg = oracle.encode_bank(w)
        banks.append((nodes, seg, w.shape[0], b))
    y = oracle.vgg_forward(g["x"], banks)
    assert np.array_equal(y, g["y"])


def test_pool_and_relu_match_reference(oracle):
    g = load_golden("pool_relu.npz")
    for i in range(4):
        x, y = g[f"p{i}__x"], g[f"p{i}__y"]
        h_p, w_p = (int(v) for v in g[f"p{i}__win"])
        got = oracle.pool(x[None], h_p, w_p, str(g[f"p{i}__mode"]))[0]
        assert np.array_equal(got, y, equal_nan=True), i
    got = oracle.relu(g["relu__x"])
    assert np.array_equal(got.view(np.int32), g["relu__y"].view(np.int32))


def _g_sparse(g, key):
    from conftest import nodes_from_i64

    return (nodes_from_i64(g[f"{key}__nodes"]), g[f"{key}__segment_offsets"],
            tuple(int(v) for v in g[f"{key}__dims"]), str(g[f"{key}__order"]))


def test_oracle_pipeline_ops_pinned(oracle):
    """The oracle's restatements of the sparse-input pipeline ops reproduce the
    reference's own outputs byte for byte (tests/golden/pipeline.npz)."""
    g = load_golden("pipeline.npz")
    for i in range(int(g["n_node_cases"])):
        key = f"n{i}"
        nodes, seg, dims, order = _g_sparse(g, f"{key}_in")
        for kind, slope, tag in (("relu", 0.0, "relu"), ("leaky", 0.1, "leaky")):
            got_nodes, got_seg = oracle.rebuild(nodes, seg, kind, slope)
            assert got_nodes.tobytes() == g[f"{key}_{tag}__nodes"].tobytes(), (key, tag)
            assert np.array_equal(got_seg, g[f"{key}_{tag}__segment_offsets"]), (key, tag)
        x = g[f"{key}_dense__x"]
        bn = [g[f"{key}_bn__{f}"] for f in ("scale", "shift", "mean", "var")]
        assert oracle.batchnorm(x, *bn, 1e-5).tobytes() == g[f"{key}_dense_bn__y"].tobytes(), key
        p = int(g[f"{key}_pad__p"])
        assert oracle.pad_dense(x, p).tobytes() == g[f"{key}_dense_pad__y"].tobytes(), key
        if order == "CHW":
            got_nodes, got_seg = oracle.pad_chw_nodes(nodes, seg, dims, p)
            assert got_nodes.tobytes() == g[f"{key}_pad__nodes"].tobytes(), key
            assert np.array_equal(got_seg, g[f"{key}_pad__segment_offsets"]), key
    for i in range(6):
        from conftest import nodes_from_i64

        rows, cols = (int(v) for v in g[f"tm{i}_in__shape"])
        seg_len = cols if str(g[f"tm{i}_in__order"]) == "WH" else rows
        got_nodes, got_seg = oracle.transpose_segments(nodes_from_i64(g[f"tm{i}_in__nodes"]), seg_len)
        assert got_nodes.tobytes() == g[f"tm{i}_out__nodes"].tobytes(), i
        assert np.array_equal(got_seg, g[f"tm{i}_out__segment_offsets"]), i
    for i in range(4):
        nodes, seg, dims, _ = _g_sparse(g, f"tt{i}_in")
        got_nodes, got_seg = oracle.transpose_whc_to_chw(nodes, seg, dims)
        assert got_nodes.tobytes() == g[f"tt{i}_out__nodes"].tobytes(), i
        assert np.array_equal(got_seg, g[f"tt{i}_out__segment_offsets"]), i
