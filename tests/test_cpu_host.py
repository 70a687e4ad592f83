"""Host-side checks that need no GPU: the C ABI's exported surface, the Python
mirror's validation/shape logic, the launch planner, and the batch-sharded
multi-process driver over gloo (world size 2)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_2212_08815_b200 as fs
from paper_2212_08815_b200 import _lib, device, kernels, network, workloads as wl
from paper_2212_08815_b200.sparse_core import NODE_DTYPE


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "fscnn_b200.h")).read()
    return sorted(set(re.findall(r"\b(fscnn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.exported_symbols())
    assert lib.fscnn_abi_version() == 1
    assert lib.fscnn_sf_pack_kt() in (2, 4, 8)
    assert lib.fscnn_encode_workspace_bytes(10**6) >= 8 * (10**6 // 4096)


def test_abi_rejects_bad_arguments_without_gpu():
    """Argument validation happens before any CUDA call, so it runs here."""
    with pytest.raises(_lib.FscnnError, match="negative extent"):
        _lib.call("fscnn_encode_offsets", None, -1, 1, 1, 1, 0, 0, 0, 0, None, None, None, 0, None)
    with pytest.raises(_lib.FscnnError, match="pool window"):
        _lib.call("fscnn_pool2d", None, 1, 1, 4, 4, 0, 2, 1, None, None)
    with pytest.raises(_lib.FscnnError, match="exceeds"):
        _lib.call("fscnn_sf_conv_exact", None, 1, 1, 2, 2, None, None, 1, 5, 5, 1, 0, None, 0, None, None)
    with pytest.raises(_lib.FscnnError, match="exceeds"):
        _lib.call("fscnn_dense_conv_exact", None, 1, 1, 2, 2, None, 1, 5, 5, 1, 0, None, None, None)
    with pytest.raises(_lib.FscnnError, match="activation kind"):
        _lib.call("fscnn_activation", None, 0, 7, 0.0, None, None)
    with pytest.raises(_lib.FscnnError, match="non-negative"):
        _lib.call("fscnn_pad2d", None, 1, 1, 2, 2, -1, None, None)
    with pytest.raises(_lib.FscnnError, match="null"):
        _lib.call("fscnn_batchnorm", None, 1, 1, 2, 2, None, None, None, None, 1e-5, None, None)
    with pytest.raises(_lib.FscnnError, match="negative extent"):
        _lib.call("fscnn_encode_masked_offsets", None, None, -1, 1, 1, 1, 0, 0, 0, 0, None, None, None, 0, None)
    with pytest.raises(_lib.FscnnError, match="negative extent"):
        _lib.call("fscnn_remap_segments_offsets", None, -1, 0, None, 1, None, None, None, 0, None)
    with pytest.raises(_lib.FscnnError, match="row pitch"):
        _lib.call("fscnn_sf_conv3x3_ex", None, 1, 4, 8, 8, 6, None, None, 0, 1, 1, 4, None, 0, 0, None, 12,
                  0, 4, None)
    with pytest.raises(_lib.FscnnError, match="row pitch"):
        _lib.call("fscnn_whc_to_nchw_ex", None, 1, 1, 4, 8, None, 8, 1, None)
    # the channel-major sparse-input entries
    with pytest.raises(_lib.FscnnError, match="bad SI pack"):
        _lib.call("fscnn_si_pack_fast", None, 0, 4, None, None)
    with pytest.raises(_lib.FscnnError, match="bad extents"):
        _lib.call("fscnn_si_conv3x3_fast", None, None, 0, 1, 0, 4, 4, None, 8, None, None, None)
    with pytest.raises(_lib.FscnnError, match="null buffer"):
        _lib.call("fscnn_si_conv3x3_fast", None, None, 4, 1, 2, 4, 4, None, 8, None, None, None)
    with pytest.raises(_lib.FscnnError, match="too large"):
        _lib.call("fscnn_si_conv3x3_fast", 8, 8, 4, 70000, 2, 4, 4, 8, 8, None, 8, None)
    lib = _lib.load()
    assert lib.fscnn_si_fast_bank_floats(0, 4) == 0
    # K padded to whole CTAs: 40 filters -> 1 per lane, 2 warps of 32 = 64
    assert lib.fscnn_si_fast_bank_floats(40, 3) == 3 * 9 * 64
    # 512 filters -> 2 per lane, 8 warps = 512
    assert lib.fscnn_si_fast_bank_floats(512, 2) == 2 * 9 * 512
    # the sparse-filter kernel accepts 1, 2, 4 and 8 filters per warp, not 3
    with pytest.raises(_lib.FscnnError, match="kt must be"):
        _lib.call("fscnn_sf_pack_offsets", 8, 4, 4, 3, 8, 8, None, 0, None)  # dummy non-null pointers


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present: the no-fallback path is exercised by the GPU suite")
    t = fs.DenseTensor3.from_array(np.ones((2, 3, 3), np.float32))
    with pytest.raises(RuntimeError, match="CUDA"):
        fs.sparsify_tensor3(t, fs.AxisOrder3.CHW)


def test_geometry_and_layer_contracts():
    g = kernels.ConvGeometry((4, 9, 11), (4, 3, 3), stride=2, padding=1)
    assert (g.n_h, g.n_w) == (5, 6)
    for kw, msg in (({"filter_dims": (3, 3, 3)}, "channel"), ({"stride": 0}, "stride"),
                    ({"padding": -1}, "padding")):
        args = dict(input_dims=(2, 5, 5), filter_dims=(2, 3, 3))
        args.update(kw)
        with pytest.raises(ValueError, match=msg):
            kernels.ConvGeometry(**args)
    with pytest.raises(ValueError, match="exceeds"):
        kernels.ConvGeometry((2, 3, 3), (2, 5, 5))
    conv = fs.LayerSpec(kind="conv", out_channels=8, kernel=(3, 3), stride=1, padding=1)
    assert conv.out_dims((3, 32, 32)) == (8, 32, 32)
    with pytest.raises(ValueError, match="divisible"):
        fs.LayerSpec(kind="maxpool", kernel=(2, 2)).out_dims((8, 31, 32))
    s = fs.ForwardStrategy()
    assert s.resolve(4) is fs.StrategyKind.STRATEGY_I and s.resolve(5) is fs.StrategyKind.STRATEGY_II


def test_vgg16_net_and_plan():
    net = fs.build_benchmark_net("vgg16_desk", 1.0, input_hw=224, variant=network.VARIANT_SPARSE_FILTER)
    convs = [l for l in net.layers if l.kind == "conv"]
    assert len(convs) == 13 and sum(l.kind == "maxpool" for l in net.layers) == 5
    assert net.shape_chain()[-1] == (512, 7, 7)
    assert network._vgg_plan(net) == wl.VGG16_PLAN
    assert [s[:3] for s in wl.vgg16_conv_shapes()][-1] == (512, 512, 14)
    with pytest.raises(ValueError, match="unknown"):
        fs.build_benchmark_net("lenet", 1.0)
    with pytest.raises(ValueError, match="scale"):
        fs.build_benchmark_net("vgg16_desk", 0.0)


def test_stack_and_validate_on_oracle_encoding(oracle):
    rng = np.random.default_rng(5)
    parts = []
    for _ in range(4):
        a = rng.standard_normal((3, 4, 5)).astype(np.float32)
        a[rng.random(a.shape) < 0.6] = 0
        nodes, mat, seg = oracle.encode(a, "CHW")
        parts.append(fs.SparseTensor3(fs.AxisOrder3.CHW, (3, 4, 5), nodes, mat, seg))
    t4 = fs.SparseTensor4.stack(parts)
    t4.validate()
    assert t4.dims == (4, 3, 4, 5)
    for i in range(4):
        assert np.array_equal(t4.tensor(i).nodes, parts[i].nodes)
    bad = parts[0].nodes.copy()
    bad["index"][-1] = 0
    with pytest.raises(fs.FormatError):
        fs.SparseTensor3(fs.AxisOrder3.CHW, (3, 4, 5), bad, parts[0].matrix_offsets, parts[0].segment_offsets).validate()
    with pytest.raises(fs.FormatError):
        fs.SparseTensor4.stack([])


def test_multiply_count_matches_oracle(oracle):
    rng = np.random.default_rng(9)
    w = rng.standard_normal((1, 16, 5, 5)).astype(np.float32)
    w[rng.random(w.shape) < 0.9] = 0
    nodes, mat, seg = oracle.encode(w[0], "CHW")
    t_f = fs.SparseTensor3(fs.AxisOrder3.CHW, (16, 5, 5), nodes, mat, seg)
    for s, p in ((1, 0), (2, 1)):
        geom = kernels.ConvGeometry((16, 12, 12), (16, 5, 5), s, p)
        want = oracle.sf_count(12, 12, seg, len(nodes), 1, 5, 5, s, p)
        assert kernels.multiply_count(t_f, geom) == want


def test_launch_planner():
    assert device.pick_ly(64, 224) == 4 and device.pick_ly(3, 224) == 2 and device.pick_ly(512, 14) == 4
    counts = np.full((16, 512), 5, np.int64)  # 16 groups x 512 channels, 4 nodes + sentinel
    bank = device.PackedBank(64, 512, 4, None, None, int(counts.sum()), counts, 0)
    cc, mx = bank.chunk_plan(4)
    assert cc == 16 and mx == 80  # 16-channel chunks keep two CTAs per SM
    assert device.sf3x3_smem_bytes(4, cc, mx + 4, 512) <= device.SMEM_2CTA
    shallow = device.PackedBank(64, 3, 4, None, None, 0, np.full((16, 3), 2, np.int64), 0)
    assert shallow.chunk_plan(2) == (3, 6)  # one chunk holds all channels
    dense = device.PackedBank(64, 512, 4, None, None, 0, np.full((16, 512), 37, np.int64), 0)
    cc2, mx2 = dense.chunk_plan(2)  # a fully dense bank still fits (smaller chunks if needed)
    assert device.sf3x3_smem_bytes(2, cc2, mx2 + 4, 512) <= device.SMEM_LIMIT


def test_workload_shapes_and_determinism():
    x1, w1, b1 = wl.c1()
    assert x1.shape == (1, 64, 56, 56) and w1.shape == (64, 64, 3, 3)
    frac = float((w1 == 0).mean())
    assert 0.93 < frac < 0.97
    x2, w2, _ = wl.c2()
    assert float((x2 == 0).mean()) > 0.88 and (x2 >= 0).all()
    layers = wl.vgg16_weights(seed=1, zero_frac=0.9, scale=0.125)
    assert [f.shape[0] for f, _ in layers] == [8, 8, 16, 16, 32, 32, 32, 64, 64, 64, 64, 64, 64]
    x, w, _ = wl.sweep_layer(3, "si", 0.75, n=2)
    assert x.shape == (2, 128, 112, 112) and 0.72 < float((x == 0).mean()) < 0.78


# -- multi-process driver over gloo -------------------------------------------------


def _dist_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2212_08815_b200 import distributed as pd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cpu")
        banks = None
        if rank == 0:
            rng = np.random.default_rng(0)
            banks = []
            for k in (3, 5):
                n = int(rng.integers(10, 40))
                nodes = torch.from_numpy(rng.integers(-1, 9, (n, 2)).astype(np.int32))
                banks.append((nodes, torch.arange(k * 9, dtype=torch.int64), torch.arange(k, dtype=torch.int64),
                               torch.arange(k * 3, dtype=torch.int64), torch.rand(k)))
        got = pd.broadcast_banks(banks, dev)
        sig = [tuple(t.numpy().tobytes() for t in b) for b in got]
        lo, hi = pd.shard_range(10, rank, world)
        y = torch.full((2, 3), float(rank))
        gathered = [g.numpy().tolist() for g in pd.gather_outputs(y)]
        mx = pd.max_over_ranks(float(rank + 1), dev)
        # unequal shards (5 items over 2 ranks: 3 + 2) gathered in rank order
        a, b = pd.shard_range(5, rank, world)
        full = pd.gather_batch(torch.arange(a, b, dtype=torch.float32).repeat_interleave(4).view(b - a, 2, 2), 5)
        # equal shards (6 over 2): the single-collective path, into a caller-owned buffer
        a, b = pd.shard_range(6, rank, world)
        buf = torch.full((6, 2, 2), -1.0)
        eq = pd.gather_batch(torch.arange(a, b, dtype=torch.float32).repeat_interleave(4).view(b - a, 2, 2), 6, out=buf)
        assert eq.data_ptr() == buf.data_ptr()
        q.put((rank, sig, (lo, hi), gathered, mx, full.numpy().tolist(), str(pd.comm_device(dev)),
               eq.numpy().tolist()))
    finally:
        dist.destroy_process_group()


def test_batch_sharded_driver_gloo_world2():
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] == res[1][0]  # identical banks on every rank after the broadcast
    assert res[0][1] == (0, 5) and res[1][1] == (5, 10)
    assert res[0][2] == [[[0.0] * 3] * 2, [[1.0] * 3] * 2]  # rank-ordered gather
    assert res[0][3] == res[1][3] == 2.0
    want = [[[float(i)] * 2] * 2 for i in range(5)]
    assert res[0][4] == res[1][4] == want
    assert res[0][5] == "cpu"
    assert res[0][6] == res[1][6] == [[[float(i)] * 2] * 2 for i in range(6)]


def test_shard_range_covers_batch():
    from paper_2212_08815_b200.distributed import shard_range

    for total in (1, 7, 32, 256):
        for world in (1, 2, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_node_dtype_is_reference_layout():
    assert NODE_DTYPE.itemsize == 8 and NODE_DTYPE.names == ("index", "value")
    assert fs.AxisOrder3.CHW.axes == (0, 1, 2) and fs.AxisOrder3.WHC.axes == (2, 1, 0)


def test_weight_and_input_generators_match_reference():
    """random_weights / prune_weights / random_input / prune_random are host-side
    workload generators; they must reproduce the reference's draws exactly
    (tests/golden/pipeline.npz, made by the reference)."""
    from conftest import load_golden, weights_sha

    from paper_2212_08815_b200 import network as nw
    from paper_2212_08815_b200.sparse_core import prune_random

    g = load_golden("pipeline.npz")
    for i in range(int(g["n_net_cases"])):
        key = f"net{i}"
        kind, variant, seed = str(g[f"{key}__kind"]), str(g[f"{key}__variant"]), int(g[f"{key}__seed"])
        net = nw.build_benchmark_net(kind, 0.125, input_hw=32, variant=variant)
        weights = nw.random_weights(net, seed)
        if variant == "sparse_filter":
            weights = nw.prune_weights(weights, 0.3, seed)
        assert weights_sha(weights) == str(g[f"{key}__weights_sha"]), key
        x = prune_random(nw.random_input(net.input_dims, seed), 0.4, seed)
        assert x.to_array().tobytes() == g[f"{key}__x"].tobytes(), key


def test_sfjit_generator_emits_valid_ptx_and_compiles():
    """The per-layer code generator (csrc/sfjit.cu) on CPU: its PTX for both CTA modes
    (parts of an image / whole images) assembles with ptxas, and the nvJitLink compile
    jobs behind fscnn_sfjit_create finish without a GPU."""
    import ctypes
    import shutil
    import subprocess
    import tempfile

    lib = _lib.load()
    ptxas = shutil.which("ptxas") or "/usr/local/cuda/bin/ptxas"
    rng = np.random.default_rng(0)
    for c, k, h, pool in ((16, 72, 16, 1), (8, 32, 112, 0)):
        w = (rng.standard_normal((k, c, 3, 3)) * 0.1).astype(np.float32)
        w[rng.random(w.shape) < 0.9] = 0
        b = rng.standard_normal(k).astype(np.float32)
        g = 1 if k > 48 else 0  # the last (partial) group of 72 filters, or the only one
        n = lib.fscnn_sfjit_ptx(w.ctypes.data, b.ctypes.data, k, c, h, h, 1, pool, 0, g, None, 0)
        assert n > 0
        buf = ctypes.create_string_buffer(n + 1)
        assert lib.fscnn_sfjit_ptx(w.ctypes.data, b.ctypes.data, k, c, h, h, 1, pool, 0, g, buf, n + 1) == n
        text = buf.value.decode()
        assert ".entry sfjit" in text and "fma.rn.f32x2" in text
        if os.path.exists(ptxas):
            with tempfile.TemporaryDirectory() as d:
                src = os.path.join(d, "g.ptx")
                open(src, "w").write(text)
                r = subprocess.run([ptxas, "-arch=sm_100a", "-O3", src, "-o", os.path.join(d, "g.cubin")],
                                   capture_output=True, text=True)
                assert r.returncode == 0, r.stderr[-2000:]
        h_ = ctypes.c_void_p()
        os.environ["FSCNN_JIT_CACHE"] = "off"
        try:
            assert lib.fscnn_sfjit_create(w.ctypes.data, b.ctypes.data, k, c, h, h, 1, pool, 0, ctypes.byref(h_)) == 0
            assert lib.fscnn_sfjit_compiled(h_) == 0, lib.fscnn_last_error()
            info = (ctypes.c_int64 * 12)()
            assert lib.fscnn_sfjit_info(h_, info, None) == 0
            assert info[0] == -(-k // info[3])  # groups = ceil(k / filters per group)
        finally:
            del os.environ["FSCNN_JIT_CACHE"]
            lib.fscnn_sfjit_destroy(h_)
    # every VGG16 conv shape plans and generates (C = 3: a box that is not a 128-byte
    # multiple; 14x14: whole-image CTAs whose chunk is ONE TMA operation over 4 images)
    for c, k, h, pool in ((3, 64, 224, 0), (64, 64, 224, 1), (64, 128, 112, 0), (128, 256, 56, 0),
                          (256, 512, 28, 0), (512, 512, 28, 1), (512, 512, 14, 0), (512, 512, 14, 1)):
        w = (rng.standard_normal((k, c, 3, 3)) * 0.1).astype(np.float32)
        w[rng.random(w.shape) < 0.9] = 0
        b = np.zeros(k, np.float32)
        n = lib.fscnn_sfjit_ptx(w.ctypes.data, b.ctypes.data, k, c, h, h, 1, pool, 48, 0, None, 0)
        assert n > 0, (c, k, h, lib.fscnn_last_error())
        if h == 14:
            buf = ctypes.create_string_buffer(n + 1)
            lib.fscnn_sfjit_ptx(w.ctypes.data, b.ctypes.data, k, c, h, h, 1, pool, 48, 0, buf, n + 1)
            text = buf.value.decode()
            # one TMA per chunk: the issue loop runs once (not once per image)
            assert "setp.lt.u32 pl, qbi, 1;" in text and "setp.lt.u32 pl, qbi, nbox;" not in text
    # odd extents are refused with a message (the engine then keeps the jump-table kernel)
    w = np.ones((8, 4, 3, 3), np.float32)
    assert lib.fscnn_sfjit_ptx(w.ctypes.data, None, 8, 4, 15, 15, 1, 0, 0, 0, None, 0) == -1
    assert b"even" in lib.fscnn_last_error()


def test_device_twin_host_logic():
    """Device twins: host tensors pass through to_host, unsupported
    types are refused, and DeviceSparseTensor3.validate applies the host validate()'s
    rules (exercised here on CPU torch tensors holding a reference-encoded tensor)."""
    import torch

    t = fs.DenseTensor3.from_array(np.zeros((2, 3, 4), np.float32))
    assert fs.to_host(t) is t
    with pytest.raises(TypeError):
        fs.to_device(np.zeros(3))
    # a 2-channel 2x2 CHW tensor: segments (w*H + h) each a channel fiber + sentinel
    nodes = np.array([(0, 1.0), (1, 2.0), (-1, 0.0), (-1, 0.0), (1, 3.0), (-1, 0.0), (0, 4.0), (-1, 0.0)],
                     dtype=fs.NODE_DTYPE)
    seg = np.array([0, 3, 4, 6], np.int64)
    host = fs.SparseTensor3(fs.AxisOrder3.CHW, (2, 2, 2), nodes, seg[::2].copy(), seg)
    host.validate()

    def twin(nd, sg, mat=None):
        words = torch.from_numpy(np.ascontiguousarray(nd).view(np.int32).reshape(-1, 2).copy())
        sg_t = torch.from_numpy(np.asarray(sg, np.int64))
        return fs.DeviceSparseTensor3(fs.AxisOrder3.CHW, (2, 2, 2), words,
                                      sg_t[::2].clone() if mat is None else torch.tensor(mat), sg_t)

    d = twin(nodes, seg)
    d.validate()
    assert d.n_segments == 4 and d.nnz == 4
    bad = nodes.copy()
    bad["index"][0], bad["index"][1] = 1, 0  # channels out of order
    with pytest.raises(fs.FormatError, match="increase"):
        twin(bad, seg).validate()
    with pytest.raises(fs.FormatError, match="strictly increase"):
        twin(nodes, [0, 3, 3, 6]).validate()
    bad = nodes.copy()
    bad["index"][4] = 2  # out of [0, C)
    with pytest.raises(fs.FormatError, match="out of"):
        twin(bad, seg).validate()
    with pytest.raises(fs.FormatError, match="matrix"):
        twin(nodes, seg, mat=[0, 3]).validate()
