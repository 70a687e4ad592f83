"""The drop-in API (mirror of sparse_infer's hot-path surface) on the GPU, checked the
way the reference's own tests check the reference (pkg/tests/test_sparse_core.py,
test_kernels.py, test_layers.py, test_network.py), against its golden outputs and
the oracle.

Tolerances: bit-exact wherever the reference contract is (encoder/decoder, the
reference-order kernels, SI layer nodes, pooling, strategy I == II, worker and batch
invariance); the fast 3x3 path is held to north_star's max|err| <= 1e-4 max|ref|.
"""

import numpy as np
import pytest

from conftest import load_golden, nodes_from_i64, normwise_err

import paper_2212_08815_b200 as fs
from paper_2212_08815_b200 import network as nw, workloads as wl

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(autouse=True)
def _fast_kernels():
    fs.set_exact(False)
    yield
    fs.set_exact(False)


def test_encoder_api_all_orders_bitwise():
    g = load_golden("encoder.npz")
    for name in g["names"]:
        name = str(name)
        arr = g[f"{name}__input"]
        order = fs.AxisOrder3[str(g[f"{name}__order"])]
        t = fs.sparsify_tensor3(fs.DenseTensor3.from_array(arr), order)
        t.validate()
        assert t.nodes.view(np.int64).tobytes() == g[f"{name}__nodes"].tobytes(), name
        assert np.array_equal(t.segment_offsets, g[f"{name}__segment_offsets"]), name
        back = fs.densify_tensor3(t)
        want = np.where(arr == 0, np.float32(0), arr)
        assert np.array_equal(back.to_array(), want, equal_nan=True), name


def test_encoder_known_answers():
    z = fs.sparsify_tensor3(fs.DenseTensor3.from_array(np.zeros((2, 2, 2), np.float32)), fs.AxisOrder3.CHW)
    assert z.nnz == 0 and len(z.nodes) == 4 and len(z.segment_offsets) == 4
    o = fs.sparsify_tensor3(fs.DenseTensor3.from_array(np.ones((2, 2, 2), np.float32)), fs.AxisOrder3.CHW)
    for k in range(4):
        s = o.segment_offsets[k]
        assert list(o.nodes["index"][s : s + 3]) == [0, 1, -1]
    with pytest.raises(fs.FormatError):
        fs.sparsify_tensor3(fs.DenseTensor3.from_array(np.zeros((1, 1, 1), np.float32)), "chw")


def test_round_trip_random_tensors_bitwise():
    rng = np.random.default_rng(11)
    for _ in range(60):
        dims = tuple(int(x) for x in rng.integers(1, 9, 3))
        arr = rng.uniform(-0.5, 0.5, dims).astype(np.float32)
        arr[rng.random(dims) >= 0.1] = 0
        order = fs.AxisOrder3(int(rng.integers(0, 6)))
        t = fs.DenseTensor3.from_array(arr)
        s = fs.sparsify_tensor3(t, order)
        assert np.array_equal(fs.densify_tensor3(s).data, t.data)


def test_matrix_round_trip():
    rng = np.random.default_rng(17)
    arr = rng.uniform(-1, 1, (6, 9)).astype(np.float32)
    arr[rng.random(arr.shape) > 0.3] = 0.0
    for order in fs.AxisOrder2:
        m = fs.sparsify_matrix(arr, order)
        m.validate()
        assert np.array_equal(fs.densify_matrix(m), arr)


def _golden_bank(w):
    return fs.SparseTensor4.stack([fs.sparsify_tensor3(fs.DenseTensor3.from_array(f), fs.AxisOrder3.CHW) for f in w])


def test_sparse_filter_layers_match_reference():
    g = load_golden("sf_conv.npz")
    for i in range(int(g["n_cases"])):
        x, w, bias, y = g[f"c{i}__x"], g[f"c{i}__w"], g[f"c{i}__bias"], g[f"c{i}__y"]
        s, p = (int(v) for v in g[f"c{i}__geom"])
        t4 = _golden_bank(w)
        t_in = fs.DenseTensor3.from_array(x)
        a = fs.conv_forward_strategy_I(t_in, t4, s, p, bias)
        b = fs.conv_forward_strategy_II(t_in, t4, s, p, bias)
        assert a.dims == b.dims and np.array_equal(a.data, b.data), i  # strategies bit-equal
        fast = w.shape[2:] == (3, 3) and (s, p) == (1, 1)
        if fast:
            assert normwise_err(a.to_array(), y) <= TOL, i
        else:
            assert np.array_equal(a.to_array().view(np.int32), y.view(np.int32)), i
        fs.set_exact(True)
        e = fs.conv_forward_strategy_II(t_in, t4, s, p, bias)
        fs.set_exact(False)
        assert np.array_equal(e.to_array().view(np.int32), y.view(np.int32)), i


def test_single_filter_kernels_and_counted():
    g = load_golden("sf_conv.npz")
    for i in range(0, int(g["n_cases"]), 3):
        x, w, y = g[f"c{i}__x"], g[f"c{i}__w"], g[f"c{i}__y"]
        s, p = (int(v) for v in g[f"c{i}__geom"])
        bias = g[f"c{i}__bias"]
        t_in = fs.DenseTensor3.from_array(x)
        geom = fs.ConvGeometry(t_in.dims, w.shape[1:], s, p)
        total = 0
        for f in range(w.shape[0]):
            t_f = fs.sparsify_tensor3(fs.DenseTensor3.from_array(w[f]), fs.AxisOrder3.CHW)
            plain = fs.conv_dense_input_sparse_filter(t_in, t_f, geom)
            counted, n = fs.conv_dense_input_sparse_filter_counted(t_in, t_f, geom)
            assert np.array_equal(plain, counted)
            # per-filter plane + bias == layer output (same order, same roundings)
            assert np.array_equal((plain + bias[f]).view(np.int32), y[f].view(np.int32)), (i, f)
            total += n
        assert total == int(g[f"c{i}__mults"])
    with pytest.raises(fs.FormatError, match="CHW"):
        t_f = fs.sparsify_tensor3(fs.DenseTensor3.from_array(np.ones((1, 1, 1), np.float32)), fs.AxisOrder3.WHC)
        fs.conv_dense_input_sparse_filter(fs.DenseTensor3.from_array(np.ones((1, 3, 3), np.float32)), t_f,
                                          fs.ConvGeometry((1, 3, 3), (1, 1, 1)))


def test_sparse_input_layer_matches_reference_bitwise():
    g = load_golden("si_conv.npz")
    for i in range(int(g["n_cases"])):
        x, w, bias, y = g[f"c{i}__x"], g[f"c{i}__w"], g[f"c{i}__bias"], g[f"c{i}__y"]
        s, p = (int(v) for v in g[f"c{i}__geom"])
        sp = fs.sparsify_tensor3(fs.DenseTensor3.from_array(x), fs.AxisOrder3.CHW)
        filters = [fs.DenseTensor3.from_array(f) for f in w]
        out = fs.conv_forward_sparse_input(sp, filters, s, p, bias)
        if str(g[f"c{i}__kind"]) == "dense":
            assert isinstance(out, fs.DenseTensor3)
            assert np.array_equal(out.to_array(), y), i
        else:
            assert isinstance(out, fs.SparseTensor3)
            assert out.nodes.view(np.int64).tobytes() == g[f"c{i}__nodes"].tobytes(), i
            assert np.array_equal(out.segment_offsets, g[f"c{i}__segment_offsets"]), i
            geom = fs.ConvGeometry(sp.dims, filters[0].dims, s, p)
            m = fs.conv_sparse_input_dense_filter(sp, filters[0], geom)
            m.validate()
            assert np.array_equal(fs.densify_matrix(m), y[0]), i


def test_sparse_input_layer_fast_path(oracle):
    """A layer big enough for the channel-major SI kernel: within the north-star
    tolerance of the oracle; set_exact(True) routes it to the bit-exact kernel."""
    from paper_2212_08815_b200 import device

    rng = np.random.default_rng(57)
    c, k, h, w = 24, 128, 56, 112
    assert device.si_use_fast(h, w, k)  # the fast path is taken
    x = np.abs(rng.standard_normal((c, h, w))).astype(np.float32)
    x[rng.random(x.shape) < 0.9] = 0
    wt = rng.normal(0, 0.05, (k, c, 3, 3)).astype(np.float32)
    bias = rng.standard_normal(k).astype(np.float32)
    sp = fs.sparsify_tensor3(fs.DenseTensor3.from_array(x), fs.AxisOrder3.CHW)
    filters = [fs.DenseTensor3.from_array(f) for f in wt]
    nodes, _, seg = oracle.encode(x, "CHW")
    ref = oracle.si_conv([nodes], [seg], (c, h, w), wt, 1, 1)[0] + bias[:, None, None]
    fast = fs.conv_forward_sparse_input(sp, filters, 1, 1, bias).to_array()
    assert normwise_err(fast, ref) <= TOL
    fs.set_exact(True)
    exact = fs.conv_forward_sparse_input(sp, filters, 1, 1, bias).to_array()
    plane = oracle.si_conv([nodes], [seg], (c, h, w), wt, 1, 1)[0]
    want = (plane + bias[:, None, None]).astype(np.float32)  # layers.py:425-428, fp32 add
    assert np.array_equal(exact, want)


def test_fusion_equals_unfused_exactly():
    rng = np.random.default_rng(56)
    for mode in ("max", "avg"):
        x = rng.uniform(-0.5, 0.5, (3, 8, 8)).astype(np.float32)
        x[rng.random(x.shape) >= 0.3] = 0
        sp = fs.sparsify_tensor3(fs.DenseTensor3.from_array(x), fs.AxisOrder3.CHW)
        f = fs.DenseTensor3.from_array(rng.normal(0, 0.3, (3, 3, 3)).astype(np.float32))
        fused = fs.merged_conv_pool(sp, f, 1, (2, 2), mode, padding=1)
        conv = fs.conv_sparse_input_dense_filter(sp, f, fs.ConvGeometry((3, 8, 8), (3, 3, 3), 1, 1))
        pooled = fs.pool_standalone(fs.DenseTensor3.from_array(fs.densify_matrix(conv)[None]), (2, 2), mode)
        assert np.array_equal(fs.densify_matrix(fused), pooled.to_array()[0])
        zb = np.zeros(4, np.float32)
        filters = [fs.DenseTensor3.from_array(rng.normal(0, 0.3, (3, 3, 3)).astype(np.float32)) for _ in range(4)]
        a = fs.conv_forward_sparse_input(sp, filters, 1, 1, zb, fused_pool=(2, 2), pool_mode=mode)
        b = fs.conv_forward_sparse_input(sp, filters, 1, 1, zb)
        bp = fs.pool_standalone(fs.densify_tensor3(b), (2, 2), mode)
        assert np.array_equal(fs.densify_tensor3(a).data, bp.data)


def test_pool_and_relu_api():
    g = load_golden("pool_relu.npz")
    for i in range(4):
        x, y = g[f"p{i}__x"], g[f"p{i}__y"]
        got = fs.pool_standalone(fs.DenseTensor3.from_array(x), tuple(int(v) for v in g[f"p{i}__win"]), str(g[f"p{i}__mode"]))
        assert np.array_equal(got.to_array(), y, equal_nan=True), i
    r = fs.apply_activation(fs.DenseTensor3.from_array(g["relu__x"]), "relu")
    assert np.array_equal(r.to_array().view(np.int32), g["relu__y"].view(np.int32))
    with pytest.raises(ValueError, match="divisible"):
        fs.pool_standalone(fs.DenseTensor3.from_array(np.ones((1, 5, 4), np.float32)), (2, 2), "max")


def _small_vgg():
    g = load_golden("vgg_small.npz")
    layers = [(g[f"w{i}"], g[f"b{i}"]) for i in range(int(g["n_layers"]))]
    net = fs.build_benchmark_net("vgg16_desk", 0.125, input_hw=32, variant=nw.VARIANT_SPARSE_FILTER)
    weights = fs.NetworkWeights(entries=[fs.ConvParams(filters=f, bias=b) for f, b in layers])
    return g, net, weights


def test_vgg_stack_forward_matches_reference():
    g, net, weights = _small_vgg()
    prepared = fs.prepare(net, weights)
    assert prepared.engine is not None
    batch = [fs.DenseTensor3.from_array(a) for a in g["x"]]
    res = fs.forward(prepared, batch)
    got = np.stack([o.to_array() for o in res.outputs])
    assert normwise_err(got, g["y"]) <= TOL
    assert res.report.strategy == "strategy_i" and res.report.batch == 2
    # per-layer path (density recording) agrees with the fused engine
    rec = fs.forward(prepared, batch, record_density=True)
    assert rec.report.layer_densities is not None and len(rec.report.layer_densities) == len(net.layers)
    got2 = np.stack([o.to_array() for o in rec.outputs])
    assert normwise_err(got2, g["y"]) <= TOL


def test_vgg_engine_honours_set_exact_bitwise():
    """set_exact(True) routes the fused VGG engine (forward without record_density)
    through the reference-order kernels: bit-exact with the reference's own output
    (network.py:410-428 over layers.py:302-323)."""
    g, net, weights = _small_vgg()
    prepared = fs.prepare(net, weights)
    batch = [fs.DenseTensor3.from_array(a) for a in g["x"]]
    fs.set_exact(True)
    try:
        res = fs.forward(prepared, batch)
        got = np.stack([o.to_array() for o in res.outputs])
        assert got.tobytes() == np.ascontiguousarray(g["y"], np.float32).tobytes()
        # same through a pinned batch (the zero-copy source)
        pinned = fs.pinned_batch(len(batch), (3, 32, 32))
        for t, src in zip(pinned, batch):
            t.data[:] = src.data
        got_p = np.stack([o.to_array() for o in fs.forward(prepared, pinned).outputs])
        assert got_p.tobytes() == got.tobytes()
    finally:
        fs.set_exact(False)
    fast = np.stack([o.to_array() for o in fs.forward(prepared, batch).outputs])
    assert normwise_err(fast, g["y"]) <= TOL


def test_worker_strategy_and_batch_invariance_bitwise():
    g, net, weights = _small_vgg()
    prepared = fs.prepare(net, weights)
    rng = np.random.default_rng(86)
    xs = [fs.DenseTensor3.from_array(rng.standard_normal((3, 32, 32)).astype(np.float32)) for _ in range(6)]
    ref = [o.data.tobytes() for o in fs.forward(prepared, xs, workers=1).outputs]
    for workers in (2, 4, 8):
        assert [o.data.tobytes() for o in fs.forward(prepared, xs, workers=workers).outputs] == ref
    for st in (fs.ForwardStrategy(fs.StrategyKind.STRATEGY_I), fs.ForwardStrategy(fs.StrategyKind.STRATEGY_II)):
        assert [o.data.tobytes() for o in fs.forward(prepared, xs, strategy=st).outputs] == ref
    # an image's result does not depend on its batch position or batch size
    for i in (0, 3, 5):
        assert fs.forward(prepared, [xs[i]]).outputs[0].data.tobytes() == ref[i]


def test_pinned_batch_forward_equals_pageable():
    """network.pinned_batch inputs take the zero-copy DMA path; results are identical to
    the packed pageable path, including for a sub-list and a reordered list."""
    g, net, weights = _small_vgg()
    prepared = fs.prepare(net, weights)
    rng = np.random.default_rng(87)
    arrs = [rng.standard_normal((3, 32, 32)).astype(np.float32) for _ in range(5)]
    pageable = [fs.DenseTensor3.from_array(a) for a in arrs]
    pinned = fs.pinned_batch(5, (3, 32, 32))
    for t, a in zip(pinned, arrs):
        t.data[:] = fs.DenseTensor3.from_array(a).data
    ref = [o.data.tobytes() for o in fs.forward(prepared, pageable).outputs]
    assert nw._staging.pinned_source(pinned, 3 * 32 * 32) is not None  # zero-copy path recognised
    assert [o.data.tobytes() for o in fs.forward(prepared, pinned).outputs] == ref
    assert [o.data.tobytes() for o in fs.forward(prepared, pinned[:3]).outputs] == ref[:3]
    rev = pinned[::-1]  # not back to back in memory -> packed path, same results
    assert [o.data.tobytes() for o in fs.forward(prepared, rev).outputs] == ref[::-1]


def test_forward_rejects_mismatches():
    g, net, weights = _small_vgg()
    p = fs.prepare(net, weights)
    with pytest.raises(ValueError, match="nonempty"):
        fs.forward(p, [])
    with pytest.raises(ValueError, match="dims"):
        fs.forward(p, [fs.DenseTensor3.from_array(np.zeros((3, 16, 16), np.float32))])
    sp = fs.sparsify_tensor3(fs.DenseTensor3.from_array(np.ones((3, 32, 32), np.float32)), fs.AxisOrder3.CHW)
    with pytest.raises(ValueError, match="dense"):
        fs.forward(p, [sp])


def test_full_size_vgg16_config3_against_oracle(oracle):
    """BASELINE config 3 at full size (224x224, 90% zeros): 2 images through the
    engine vs the CPU oracle (normwise), plus the exact nnz-FLOP count."""
    import torch

    from paper_2212_08815_b200.engine import VGGEngine

    layers = wl.vgg16_weights(seed=103, zero_frac=0.9)
    x = wl.vgg16_input(2, seed=104)
    eng = VGGEngine(layers, batch=2, hw=224)
    y = eng.forward_device(torch.from_numpy(x).cuda()).cpu().numpy()
    banks = []
    mults = 0
    h = 224
    for (wt, b), item in zip(layers, [it for it in wl.VGG16_PLAN if it != "M"]):
        nodes, seg = oracle.encode_bank(wt)
        banks.append((nodes, seg, wt.shape[0], b))
    ref = oracle.vgg_forward(x, banks)
    assert normwise_err(y, ref) <= TOL
    # nnz-FLOPs per image from the engine == 2 x the oracle's exact multiply tally
    for st, (nodes, seg, k, _) in zip(eng.steps, banks):
        mults += oracle.sf_count(st.h, st.w, seg, len(nodes), k, 3, 3, 1, 1)
    assert eng.flops_per_image() == 2 * mults


def test_full_size_config5_batch_invariance(oracle):
    """BASELINE config 5 at full size (batch 256, 224x224, 95% zeros): a batch-sharded
    run is only correct if an image's output does not depend on its batch neighbours or
    position -- images 0, 137 and 255 of the 256-image pass equal their batch-1 passes
    bit for bit; image 0 against the oracle (normwise)."""
    import torch

    from paper_2212_08815_b200.engine import VGGEngine

    layers = wl.vgg16_weights(seed=103, zero_frac=0.95)
    x = torch.from_numpy(wl.vgg16_input(256, seed=105)).cuda()
    eng = VGGEngine(layers, batch=256, hw=224)
    y = eng.forward_device(x).clone()
    for i in (0, 137, 255):
        yi = eng.forward_device(x[i : i + 1].contiguous())
        assert torch.equal(y[i : i + 1].view(torch.int32), yi.view(torch.int32)), i
    banks = []
    for wt, b in layers:
        nodes, seg = oracle.encode_bank(wt)
        banks.append((nodes, seg, wt.shape[0], b))
    ref = oracle.vgg_forward(x[:1].cpu().numpy(), banks)
    assert normwise_err(y[:1].cpu().numpy(), ref) <= TOL


# -- batch-sharded multi-process stack (distributed.ShardedVGG) ----------------------


def _sharded_worker(rank, world, port, layers, xs, q, backend="gloo"):
    import os

    import torch
    import torch.distributed as dist

    from paper_2212_08815_b200 import distributed as pd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)  # both ranks share the one GPU: gloo carries the collectives
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        sh = pd.ShardedVGG(layers if rank == 0 else None, hw=32, device=torch.device("cuda", 0))
        outs, secs = sh.timed_forward([fs.DenseTensor3.from_array(a) for a in xs])
        lo, hi = sh.shard(len(xs))
        x_local = torch.from_numpy(np.stack(xs[lo:hi])).cuda()
        full = sh.forward_device(x_local, total=len(xs)).cpu().numpy()
        q.put((rank, [o.data.tobytes() for o in outs], full.tobytes(), secs > 0))
    finally:
        dist.destroy_process_group()


def test_sharded_forward_byte_identical_world2():
    """SPMD batch-sharded forward over two ranks (gloo; both on cuda:0) returns, on every
    rank, exactly the single-GPU outputs -- the north star's 'outputs byte-identical at
    1/2/4/8 GPUs' (reference worker invariance, pkg/tests/test_acceptance.py:311-351).
    Five images: unequal shards (3 + 2)."""
    import socket

    import torch
    import torch.multiprocessing as mp

    from paper_2212_08815_b200.engine import VGGEngine

    layers = wl.vgg16_weights(seed=21, zero_frac=0.95, scale=0.125)
    rng = np.random.default_rng(22)
    xs = [rng.standard_normal((3, 32, 32)).astype(np.float32) for _ in range(5)]
    eng = VGGEngine(layers, batch=5, hw=32)
    prepared = nw.prepared_from_engine(eng)
    ref = [o.data.tobytes() for o in fs.forward(prepared, [fs.DenseTensor3.from_array(a) for a in xs]).outputs]
    ref_dev = eng.forward_device(torch.from_numpy(np.stack(xs)).cuda()).contiguous().cpu().numpy().tobytes()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, layers, xs, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        outs, full, timed = res[r]
        assert outs == ref, r
        assert full == ref_dev, r
        assert timed


def test_sharded_forward_nccl_world1():
    """The same SPMD flow with the production backend: NCCL collectives on device buffers
    (bank broadcast of the int32 node pairs / int64 offset tables / f32 bias, the padded
    rank-ordered all-gather, the max-over-ranks reduce).  One GPU is reachable, so the
    NCCL group has one rank; the outputs must equal the plain single-GPU forward byte for
    byte."""
    import socket

    import torch
    import torch.multiprocessing as mp

    from paper_2212_08815_b200.engine import VGGEngine

    layers = wl.vgg16_weights(seed=23, zero_frac=0.9, scale=0.125)
    rng = np.random.default_rng(24)
    xs = [rng.standard_normal((3, 32, 32)).astype(np.float32) for _ in range(3)]
    eng = VGGEngine(layers, batch=3, hw=32)
    prepared = nw.prepared_from_engine(eng)
    ref = [o.data.tobytes() for o in fs.forward(prepared, [fs.DenseTensor3.from_array(a) for a in xs]).outputs]
    ref_dev = eng.forward_device(torch.from_numpy(np.stack(xs)).cuda()).contiguous().cpu().numpy().tobytes()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_sharded_worker, args=(0, 1, port, layers, xs, q, "nccl"))
    p.start()
    _, outs, full, timed = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert outs == ref
    assert full == ref_dev
    assert timed
