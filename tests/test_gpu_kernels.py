"""CUDA kernels (through the C ABI) against the oracle and the reference's golden outputs.

Bit-exact where the reference contract is bit-exact (encoder, decoder, reference-order
sparse-filter conv, sparse-input conv, pooling, ReLU); the fast 3x3 sparse-filter
kernel reassociates the fp32 sum, so it is held to the north-star tolerance
max|err| <= 1e-4 * max|ref| (BASELINE.json).
"""

import numpy as np
import pytest

from conftest import load_golden, normwise_err
from paper_2212_08815_b200 import workloads as wl

pytestmark = pytest.mark.gpu

FAST_TOL = 1e-4  # north_star: conv outputs within max|err| <= 1e-4 * max|ref|


@pytest.fixture(scope="module")
def dev():
    import torch

    from paper_2212_08815_b200 import device

    assert torch.cuda.is_available()
    return device


def _t(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_encoder_matches_reference_bitwise(dev):
    g = load_golden("encoder.npz")
    for name in g["names"]:
        name = str(name)
        arr, order = g[f"{name}__input"], str(g[f"{name}__order"])
        enc = dev.encode_order(_t(arr[None]), order)
        nodes = enc.nodes[: enc.n_nodes].cpu().numpy()
        assert nodes.tobytes() == g[f"{name}__nodes"].tobytes(), name
        assert np.array_equal(enc.seg_off.cpu().numpy(), g[f"{name}__segment_offsets"]), name
        assert np.array_equal(enc.matrix_off.cpu().numpy(), g[f"{name}__matrix_offsets"]), name
        back = dev.decode_order(enc.nodes, enc.seg_off, (1,) + arr.shape, order).cpu().numpy()[0]
        want = np.where(arr == 0, np.float32(0), arr)
        assert np.array_equal(back, want, equal_nan=True), name


def test_encoder_stack_and_warp_walker(dev, oracle):
    g = load_golden("encoder.npz")
    enc = dev.encode_order(_t(g["bank__input"]), "CHW")
    assert enc.nodes[: enc.n_nodes].cpu().numpy().tobytes() == g["bank__nodes"].tobytes()
    assert np.array_equal(enc.tensor_off.cpu().numpy(), g["bank__tensor_offsets"])
    assert np.array_equal(enc.matrix_off.cpu().numpy().reshape(16, -1), g["bank__matrix_offsets"])
    assert np.array_equal(enc.seg_off.cpu().numpy().reshape(16, -1), g["bank__segment_offsets"])
    # long contiguous fibers take the warp-ballot walker: channel-innermost source
    rng = np.random.default_rng(7)
    x = rng.standard_normal((3, 70, 5, 6)).astype(np.float32)
    x[rng.random(x.shape) < 0.8] = 0
    x[0, :, 0, 0] = -0.0
    whc = _t(x.transpose(0, 3, 2, 1)).permute(0, 3, 2, 1)  # logical NCHW, c contiguous
    enc = dev.encode_order(whc, "CHW")
    ref_nodes, ref_ten, ref_mat, ref_seg = oracle.encode_batch(x, "CHW")
    assert enc.nodes[: enc.n_nodes].cpu().numpy().tobytes() == ref_nodes.view(np.int32).tobytes()
    assert np.array_equal(enc.seg_off.cpu().numpy(), ref_seg.ravel())
    assert np.array_equal(enc.tensor_off.cpu().numpy(), ref_ten)


@pytest.mark.parametrize("shape,zf", [((4, 16, 96, 100), 0.9), ((3, 45, 13, 37), 0.5), ((2, 70, 9, 16), 0.97)])
def test_encoder_large_scan(dev, oracle, shape, zf):
    """Many segments: exercises the multi-tile int64 scan and the tiled writer (ragged
    channel chunks and position tiles, -0.0 / NaN / inf entries)."""
    rng = np.random.default_rng(8)
    x = rng.standard_normal(shape).astype(np.float32)
    x[rng.random(x.shape) < zf] = 0
    flat = x.reshape(-1)
    idx = rng.choice(flat.size, 12, replace=False)
    flat[idx[:4]] = -0.0
    flat[idx[4:8]] = np.nan
    flat[idx[8:]] = np.inf
    enc = dev.encode_order(_t(x), "CHW")
    ref_nodes, _, _, ref_seg = oracle.encode_batch(x, "CHW")
    assert enc.n_nodes == len(ref_nodes)
    assert enc.nodes[: enc.n_nodes].cpu().numpy().tobytes() == ref_nodes.view(np.int32).tobytes()
    assert np.array_equal(enc.seg_off.cpu().numpy(), ref_seg.ravel())


def _bank(dev, w):
    enc = dev.encode_order(_t(w), "CHW")
    return enc


def test_sf_exact_matches_reference_bitwise(dev):
    g = load_golden("sf_conv.npz")
    for i in range(int(g["n_cases"])):
        x, w, bias = g[f"c{i}__x"], g[f"c{i}__w"], g[f"c{i}__bias"]
        s, p = (int(v) for v in g[f"c{i}__geom"])
        enc = _bank(dev, w)
        y = dev.sf_conv_exact(_t(x[None]), enc.nodes, enc.seg_off, w.shape[0], w.shape[2],
                              w.shape[3], s, p, _t(bias)).cpu().numpy()[0]
        assert np.array_equal(y.view(np.int32), g[f"c{i}__y"].view(np.int32)), i


def test_sf_fast_config1_within_tolerance(dev):
    import torch

    x, w, b = wl.c1()
    gold = load_golden("c1.npz")["y"]
    bank = dev.sf_pack(_t(w))
    y = dev.sf_conv3x3(dev.to_halo(_t(x)), bank, _t(b), relu=False, pool=False, w=56)
    torch.cuda.synchronize()
    got = dev.from_halo(y, 56)[0].cpu().numpy()
    assert normwise_err(got, gold) <= FAST_TOL


@pytest.mark.parametrize(
    "n,c,k,h,w,zf,ly",
    [
        (2, 64, 64, 56, 56, 0.9, 0),
        (1, 3, 64, 32, 32, 0.9, 0),
        (3, 13, 19, 14, 14, 0.5, 0),
        (2, 20, 72, 28, 28, 0.9, 2),
        (1, 17, 8, 9, 23, 0.0, 4),
        (2, 8, 130, 40, 36, 0.95, 8),
        (1, 5, 3, 1, 1, 0.0, 0),
        (3, 40, 40, 28, 28, 0.9, 4),
        (2, 33, 32, 56, 56, 0.9, 4),
        (4, 24, 12, 14, 14, 0.5, 4),
        (2, 9, 16, 27, 30, 0.8, 0),
        (1, 12, 8, 50, 41, 0.9, 8),
        # runs of empty channels (one dispatch skips a run, clipped to the chunk)
        (2, 48, 40, 20, 20, 0.99, 4),
        (1, 37, 12, 16, 16, 1.0, 4),
        (2, 70, 8, 12, 12, 0.97, 2),
    ],
)
def test_sf_fast_matches_oracle(dev, oracle, n, c, k, h, w, zf, ly):
    import torch

    rng = np.random.default_rng(n * 1000 + c * 10 + k)
    x = rng.standard_normal((n, c, h, w)).astype(np.float32)
    wt = rng.standard_normal((k, c, 3, 3)).astype(np.float32)
    wt[rng.random(wt.shape) < zf] = 0
    bias = rng.standard_normal(k).astype(np.float32)
    nodes, seg = oracle.encode_bank(wt)
    ref = oracle.sf_conv(x, nodes, seg, k, 3, 3, 1, 1, bias)
    bank = dev.sf_pack(_t(wt))
    xp = dev.to_halo(_t(x))
    y = dev.sf_conv3x3(xp, bank, _t(bias), relu=False, pool=False, w=w, ly=ly)
    got = dev.from_halo(y, w).cpu().numpy()
    assert normwise_err(got, ref) <= FAST_TOL
    # fused relu + 2x2 max-pool against relu -> pool on the oracle result
    if h % 2 == 0 and w % 2 == 0:
        yp = dev.sf_conv3x3(xp, bank, _t(bias), relu=True, pool=True, w=w, ly=ly)
        want = oracle.pool(oracle.relu(ref), 2, 2, "max")
        assert normwise_err(dev.from_halo(yp, w // 2).cpu().numpy(), want) <= FAST_TOL


@pytest.mark.parametrize("k", [36, 64, 8])
def test_sf_fast_filters_per_warp_agree_bitwise(dev, k):
    """2, 4 or 8 filters per warp only regroup the filters: bit-identical outputs (the
    engine picks KT = 2 for grids that cannot fill the GPU)."""
    rng = np.random.default_rng(k)
    x = rng.standard_normal((2, 24, 28, 28)).astype(np.float32)
    wt = rng.standard_normal((k, 24, 3, 3)).astype(np.float32)
    wt[rng.random(wt.shape) < 0.9] = 0
    bias = rng.standard_normal(k).astype(np.float32)
    xp = dev.to_halo(_t(x))
    outs = []
    for kt, warps in ((2, 0), (4, 0), (8, 0), (2, 4), (1, 0)):  # (2, 4), kt 1: 4-warp CTAs
        bank = dev.sf_pack(_t(wt), kt)
        for pool in (False, True):
            y = dev.sf_conv3x3(xp, bank, _t(bias), relu=True, pool=pool, w=28, cta_warps=warps)
            outs.append(((kt, warps), pool, y.cpu().numpy()))
    for cfg, pool, o in outs:
        ref = [q for kk, pp, q in outs if kk == (4, 0) and pp == pool][0]
        assert o.tobytes() == ref.tobytes(), (cfg, pool)


@pytest.mark.parametrize("n,h,w", [(3, 28, 28), (2, 56, 56), (5, 14, 14), (2, 27, 30)])
def test_sf_fast_layouts_agree_bitwise(dev, n, h, w):
    """Every sub-region height runs the same per-lane arithmetic: bit-identical outputs."""
    rng = np.random.default_rng(h * w + n)
    x = rng.standard_normal((n, 40, h, w)).astype(np.float32)
    wt = rng.standard_normal((36, 40, 3, 3)).astype(np.float32)
    wt[rng.random(wt.shape) < 0.9] = 0
    bias = rng.standard_normal(36).astype(np.float32)
    bank = dev.sf_pack(_t(wt))
    xp = dev.to_halo(_t(x))
    for pool in ((False, True) if h % 2 == 0 and w % 2 == 0 else (False,)):
        wo = w // 2 if pool else w
        outs = [dev.from_halo(dev.sf_conv3x3(xp, bank, _t(bias), relu=True, pool=pool, w=w, ly=ly), wo)
                .cpu().numpy().tobytes() for ly in (2, 4, 8)]
        assert outs[0] == outs[1] == outs[2]


def test_sf_fast_fuzz_against_oracle(dev, oracle):
    """Seeded random geometries through the fast kernel (every layout, ragged sizes,
    densities from empty to dense, bias/ReLU/fused pool) against the oracle."""
    rng = np.random.default_rng(20261020)
    for case in range(24):
        n = int(rng.integers(1, 4))
        c = int(rng.integers(1, 70))
        k = int(rng.integers(1, 80))
        h = int(rng.integers(1, 40))
        w = int(rng.integers(1, 40))
        zf = float(rng.choice([0.0, 0.5, 0.9, 0.97, 1.0]))
        ly = int(rng.choice([0, 2, 4, 8]))
        relu = bool(rng.integers(0, 2))
        pool = bool(rng.integers(0, 2)) and h % 2 == 0 and w % 2 == 0
        x = rng.standard_normal((n, c, h, w)).astype(np.float32)
        wt = rng.standard_normal((k, c, 3, 3)).astype(np.float32)
        wt[rng.random(wt.shape) < zf] = 0
        bias = rng.standard_normal(k).astype(np.float32)
        nodes, seg = oracle.encode_bank(wt)
        ref = oracle.sf_conv(x, nodes, seg, k, 3, 3, 1, 1, bias)
        if relu:
            ref = oracle.relu(ref)
        if pool:
            ref = oracle.pool(ref, 2, 2, "max")
        bank = dev.sf_pack(_t(wt))
        y = dev.sf_conv3x3(dev.to_halo(_t(x)), bank, _t(bias), relu=relu, pool=pool, w=w, ly=ly)
        got = dev.from_halo(y, w // 2 if pool else w).cpu().numpy()
        assert got.shape == ref.shape, case
        assert normwise_err(got, ref) <= FAST_TOL, (case, n, c, k, h, w, zf, ly, relu, pool)


def test_sf_fast_is_deterministic_and_batch_invariant(dev):
    import torch

    rng = np.random.default_rng(3)
    x = rng.standard_normal((5, 32, 28, 28)).astype(np.float32)
    wt = rng.standard_normal((64, 32, 3, 3)).astype(np.float32)
    wt[rng.random(wt.shape) < 0.9] = 0
    bank = dev.sf_pack(_t(wt))
    full = dev.sf_conv3x3(dev.to_halo(_t(x)), bank, None, relu=True, pool=False).cpu().numpy()
    again = dev.sf_conv3x3(dev.to_halo(_t(x)), bank, None, relu=True, pool=False).cpu().numpy()
    assert full.tobytes() == again.tobytes()
    for i in range(5):
        one = dev.sf_conv3x3(dev.to_halo(_t(x[i : i + 1])), bank, None, relu=True, pool=False).cpu().numpy()
        assert one.tobytes() == full[i : i + 1].tobytes()
    torch.cuda.synchronize()


def test_si_conv_matches_reference_bitwise(dev, oracle):
    g = load_golden("si_conv.npz")
    for i in range(int(g["n_cases"])):
        x, w, bias = g[f"c{i}__x"], g[f"c{i}__w"], g[f"c{i}__bias"]
        s, p = (int(v) for v in g[f"c{i}__geom"])
        enc = dev.encode_order(_t(x[None]), "CHW")
        wt = dev.kcrs_to_crsk(_t(w))
        dense = str(g[f"c{i}__kind"]) == "dense"
        y = dev.si_conv(enc.nodes, enc.seg_off, 1, *x.shape, wt, w.shape[0], w.shape[2],
                        w.shape[3], s, p, _t(bias) if dense else None).cpu().numpy()[0]
        assert np.array_equal(y.view(np.int32), g[f"c{i}__y"].view(np.int32)), i


def test_si_strip_kernel_bitwise(dev, oracle):
    """3x3/s1/p1 strip kernel == reference order, bit for bit (incl. ragged widths)."""
    g = load_golden("si_conv.npz")
    hit = 0
    for i in range(int(g["n_cases"])):
        x, w, bias = g[f"c{i}__x"], g[f"c{i}__w"], g[f"c{i}__bias"]
        s, p = (int(v) for v in g[f"c{i}__geom"])
        if w.shape[2:] != (3, 3) or (s, p) != (1, 1):
            continue
        hit += 1
        enc = dev.encode_order(_t(x[None]), "CHW")
        dense = str(g[f"c{i}__kind"]) == "dense"
        y = dev.si_conv3x3(enc.nodes, enc.seg_off, 1, *x.shape, dev.si_pack3x3(_t(w)), w.shape[0],
                           _t(bias) if dense else None).cpu().numpy()[0]
        assert np.array_equal(y.view(np.int32), g[f"c{i}__y"].view(np.int32)), i
    assert hit >= 3
    rng = np.random.default_rng(12)
    for (n, c, k, h, wd) in ((2, 37, 70, 13, 29), (1, 5, 3, 1, 1), (3, 64, 33, 28, 28)):
        x = np.abs(rng.standard_normal((n, c, h, wd))).astype(np.float32)
        x[rng.random(x.shape) < 0.8] = 0
        wt = rng.standard_normal((k, c, 3, 3)).astype(np.float32)
        enc = dev.encode_order(_t(x), "CHW")
        got = dev.si_conv3x3(enc.nodes, enc.seg_off, n, c, h, wd, dev.si_pack3x3(_t(wt)), k).cpu().numpy()
        ref = dev.si_conv(enc.nodes, enc.seg_off, n, c, h, wd, dev.kcrs_to_crsk(_t(wt)), k, 3, 3, 1, 1).cpu().numpy()
        assert np.array_equal(got.view(np.int32), ref.view(np.int32))
        segs = [oracle.encode(x[b], "CHW") for b in range(n)]
        oref = oracle.si_conv([s[0] for s in segs], [s[2] for s in segs], (c, h, wd), wt, 1, 1)
        assert np.array_equal(got, oref)


def test_si_strip_paths_agree_bitwise(dev, monkeypatch):
    """Every SI strip variant (shared-memory or L2 weights, strip width 8/4/2 picked by
    problem size) computes the same bits as the gather kernel."""
    rng = np.random.default_rng(31)
    for (n, c, k, h, wd) in ((1, 64, 40, 20, 23), (4, 16, 96, 30, 30), (1, 130, 32, 9, 9), (6, 48, 64, 28, 28)):
        x = np.abs(rng.standard_normal((n, c, h, wd))).astype(np.float32)
        x[rng.random(x.shape) < 0.85] = 0
        wt = rng.standard_normal((k, c, 3, 3)).astype(np.float32)
        enc = dev.encode_order(_t(x), "CHW")
        ref = dev.si_conv(enc.nodes, enc.seg_off, n, c, h, wd, dev.kcrs_to_crsk(_t(wt)), k, 3, 3, 1, 1).cpu().numpy()
        wq = dev.si_pack3x3(_t(wt))
        for nosmem in (False, True):
            if nosmem:
                monkeypatch.setenv("FSCNN_SI_NOSMEM", "1")
            else:
                monkeypatch.delenv("FSCNN_SI_NOSMEM", raising=False)
            got = dev.si_conv3x3(enc.nodes, enc.seg_off, n, c, h, wd, wq, k).cpu().numpy()
            assert np.array_equal(got.view(np.int32), ref.view(np.int32)), (n, c, k, h, wd, nosmem)


def test_si_fast_within_tolerance(dev, oracle):
    """Channel-major SI kernel (one and two filters per lane) vs the bit-exact kernels /
    oracle: north-star tolerance, ragged tiles, K and C off multiples of 32 / 64, empty
    and fully dense inputs, several 32-channel chunks, bias."""
    rng = np.random.default_rng(41)
    cases = [(2, 37, 70, 13, 29, 0.8), (1, 5, 3, 1, 1, 0.5), (3, 64, 33, 28, 28, 0.9), (1, 130, 257, 9, 17, 0.95),
             (2, 16, 64, 8, 8, 0.0), (1, 40, 32, 10, 12, 1.0), (4, 96, 128, 14, 14, 0.5),
             (1, 70, 200, 11, 9, 0.0), (2, 100, 160, 7, 13, 0.9), (2, 64, 300, 10, 14, 0.5),
             (1, 33, 512, 6, 9, 0.9)]
    for (n, c, k, h, wd, zf) in cases:
        x = np.abs(rng.standard_normal((n, c, h, wd))).astype(np.float32)
        x[rng.random(x.shape) < zf] = 0
        wt = rng.standard_normal((k, c, 3, 3)).astype(np.float32)
        bias = rng.standard_normal(k).astype(np.float32)
        enc = dev.encode_order(_t(x), "CHW")
        ref = dev.si_conv(enc.nodes, enc.seg_off, n, c, h, wd, dev.kcrs_to_crsk(_t(wt)), k, 3, 3, 1, 1,
                          _t(bias)).cpu().numpy()
        wf = dev.si_pack_fast(_t(wt))
        got = dev.si_conv3x3_fast(enc.nodes, enc.seg_off, n, c, h, wd, wf, k, _t(bias)).cpu().numpy()
        assert normwise_err(got, ref) <= FAST_TOL, (n, c, k, h, wd, zf, normwise_err(got, ref))
        # deterministic
        again = dev.si_conv3x3_fast(enc.nodes, enc.seg_off, n, c, h, wd, wf, k, _t(bias)).cpu().numpy()
        assert np.array_equal(got.view(np.int32), again.view(np.int32))
        if zf == 1.0:
            assert np.array_equal(got, np.broadcast_to(bias[None, :, None, None], got.shape))
    # against the oracle directly (no bias: dense plane, +0.0 where the sum is zero)
    n, c, k, h, wd = 2, 48, 40, 12, 20
    x = np.abs(rng.standard_normal((n, c, h, wd))).astype(np.float32)
    x[rng.random(x.shape) < 0.9] = 0
    wt = rng.standard_normal((k, c, 3, 3)).astype(np.float32)
    enc = dev.encode_order(_t(x), "CHW")
    got = dev.si_conv3x3_fast(enc.nodes, enc.seg_off, n, c, h, wd, dev.si_pack_fast(_t(wt)), k).cpu().numpy()
    segs = [oracle.encode(x[b], "CHW") for b in range(n)]
    oref = oracle.si_conv([s[0] for s in segs], [s[2] for s in segs], (c, h, wd), wt, 1, 1)
    assert normwise_err(got, oref) <= FAST_TOL


def test_si_conv_config2(dev):
    import hashlib

    x, w, b = wl.c2()
    g = load_golden("c2.npz")
    enc = dev.encode_order(_t(x), "CHW")
    y = dev.si_conv(enc.nodes, enc.seg_off, 1, 128, 28, 28, dev.kcrs_to_crsk(_t(w)), 128, 3, 3, 1, 1)
    assert np.array_equal(y.cpu().numpy()[0], g["y"])
    y2 = dev.si_conv3x3(enc.nodes, enc.seg_off, 1, 128, 28, 28, dev.si_pack3x3(_t(w)), 128)
    assert np.array_equal(y2.cpu().numpy()[0], g["y"])
    out = dev.encode_order(y, "CHW")
    h = hashlib.sha256()
    for a in (out.nodes[: out.n_nodes].cpu().numpy(), out.matrix_off.cpu().numpy(), out.seg_off.cpu().numpy()):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(g["out_nodes_sha"])


def test_pool_relu_and_layouts(dev):
    g = load_golden("pool_relu.npz")
    for i in range(4):
        x, y = g[f"p{i}__x"], g[f"p{i}__y"]
        h_p, w_p = (int(v) for v in g[f"p{i}__win"])
        got = dev.pool2d(_t(x[None]), h_p, w_p, str(g[f"p{i}__mode"]) == "max").cpu().numpy()[0]
        assert np.array_equal(got, y, equal_nan=True), i
    r = dev.relu(_t(g["relu__x"])).cpu().numpy()
    assert np.array_equal(r.view(np.int32), g["relu__y"].view(np.int32))
    rng = np.random.default_rng(5)
    # narrow (q-tiled) and wide (column-tiled) kernels, ragged channel / row / column tiles
    for shape in [(3, 37, 11, 13), (2, 45, 7, 70), (1, 64, 9, 32), (2, 8, 5, 33)]:
        x = rng.standard_normal(shape).astype(np.float32)
        n, c, h, w = shape
        whc = dev.nchw_to_whc(_t(x))
        assert np.array_equal(whc.cpu().numpy(), x.transpose(0, 3, 2, 1)), shape
        back = dev.whc_to_nchw(whc, n, c, h, w)
        assert np.array_equal(back.cpu().numpy(), x), shape
        # halo-column buffers: logical column j at memory column j + 1, zero columns kept
        hal = dev.halo_empty(n, c, h, w)
        dev.whc_to_halo(whc.view(-1), n, c, h, w, hal)
        hn = hal.cpu().numpy()
        assert np.array_equal(hn[..., 1 : w + 1], x), shape
        assert not hn[..., 0].any() and not hn[..., w + 1 :].any(), shape
        assert np.array_equal(dev.halo_to_whc(hal, w).cpu().numpy(), x.transpose(0, 3, 2, 1)), shape


@pytest.mark.parametrize("layer,zf", [(8, 0.9), (5, 0.5), (1, 0.75)])
def test_si_fast_at_vgg_layer_size(dev, layer, zf):
    """BASELINE config 4 shapes (batch 4): the channel-major SI kernel against the
    bit-exact strip kernel (itself pinned to the reference), north-star tolerance; and
    linearity in the weights (W1 + W2 applied = the two results added, to fp32
    reassociation)."""
    import torch

    x, wt, _ = wl.sweep_layer(layer, "si", zf, n=4)
    n, c, h, w = x.shape
    k = wt.shape[0]
    enc = dev.encode_order(_t(x), "CHW")
    ref = dev.si_conv3x3(enc.nodes, enc.seg_off, n, c, h, w, dev.si_pack3x3(_t(wt)), k)
    got = dev.si_conv3x3_fast(enc.nodes, enc.seg_off, n, c, h, w, dev.si_pack_fast(_t(wt)), k)
    assert normwise_err(got.cpu().numpy(), ref.cpu().numpy()) <= FAST_TOL
    w2 = np.random.default_rng(layer).normal(0, 0.05, wt.shape).astype(np.float32)
    a = dev.si_conv3x3_fast(enc.nodes, enc.seg_off, n, c, h, w, dev.si_pack_fast(_t(w2)), k)
    s = dev.si_conv3x3_fast(enc.nodes, enc.seg_off, n, c, h, w, dev.si_pack_fast(_t(wt + w2)), k)
    assert normwise_err(s.cpu().numpy(), (got + a).cpu().numpy()) <= FAST_TOL
    torch.cuda.synchronize()


# -- per-layer specialised sparse-filter kernels (sfjit.cu) ----------------------------

SFJIT_CASES = [
    # c, k, h, n, relu, pool, zero fraction: part mode (large images, several CTAs per
    # image), multi-image mode (small ones, ragged last CTA), partial filter groups,
    # bias/ReLU/pool combinations, dense and nearly empty banks
    (3, 8, 8, 1, True, False, 0.5),
    (16, 32, 16, 2, True, True, 0.9),
    (24, 40, 12, 3, False, False, 0.9),
    (64, 64, 28, 5, True, True, 0.9),
    (32, 64, 14, 33, True, False, 0.95),
    (8, 32, 56, 2, True, True, 0.0),
    (64, 32, 224, 1, True, False, 0.9),
    (40, 72, 30, 2, True, True, 0.99),
]


@pytest.mark.parametrize("c,k,h,n,relu,pool,zf", SFJIT_CASES)
def test_sfjit_bitwise_equals_jump_table_kernel(dev, oracle, c, k, h, n, relu, pool, zf):
    """The specialised kernels accumulate in the jump-table kernel's order (channels
    ascending, then each filter's taps), so the two agree bit for bit; both are checked
    against the oracle at the north-star tolerance."""
    rng = np.random.default_rng(c * 1000 + k + h)
    w = (rng.standard_normal((k, c, 3, 3)) * 0.1).astype(np.float32)
    w[rng.random(w.shape) < zf] = 0
    b = (rng.standard_normal(k) * 0.1).astype(np.float32)
    x = rng.standard_normal((n, c, h, h)).astype(np.float32)
    xd = dev.to_halo(_t(x))
    ref = dev.sf_conv3x3(xd, dev.sf_pack(_t(w)), _t(b), relu=relu, pool=pool, w=h)
    got = dev.SfJit(w, b, h, h, relu=relu, pool=pool)(xd)
    assert ref.cpu().numpy().tobytes() == got.cpu().numpy().tobytes()
    if n * c * h * h <= 200_000:
        nodes, seg = oracle.encode_bank(w)
        want = oracle.sf_conv(x, nodes, seg, k, 3, 3, 1, 1, b)
        if relu:
            want = oracle.relu(want)
        if pool:
            want = oracle.pool(want, 2, 2, "max")
        wo = h // 2 if pool else h
        y = dev.from_halo(got, wo).cpu().numpy()
        assert normwise_err(y, want) <= FAST_TOL


def test_sfjit_batch_invariant(dev):
    rng = np.random.default_rng(5)
    c, k, h = 16, 64, 14
    w = (rng.standard_normal((k, c, 3, 3)) * 0.1).astype(np.float32)
    w[rng.random(w.shape) < 0.9] = 0
    x = rng.standard_normal((7, c, h, h)).astype(np.float32)
    j = dev.SfJit(w, None, h, h, relu=True, pool=True)
    full = j(dev.to_halo(_t(x))).cpu().numpy()
    for i in range(7):
        one = j(dev.to_halo(_t(x[i : i + 1]))).cpu().numpy()
        assert one.tobytes() == full[i : i + 1].tobytes()


@pytest.mark.parametrize("layer", list(range(13)))
def test_c4_sweep_points_against_exact_kernel(dev, layer):
    """BASELINE config 4's sparse-filter points at batch 2: every VGG16 layer shape at
    {50, 75, 90, 95, 99} % filter zeros, the fast jump-table kernel against the
    reference-order exact kernel (pinned bit-exact to the reference) at the north-star
    tolerance; the specialised kernels equal the jump-table kernel bit for bit on the
    sparsest and densest points of a few shapes (their compile time is per bank)."""
    import torch

    c, k, h, w = wl.vgg16_conv_shapes()[layer]
    for zf in (0.5, 0.75, 0.9, 0.95, 0.99):
        x, wt, b = wl.sweep_layer(layer, "sf", zf, n=2)
        wd, bias = _t(wt), _t(b)
        xh = dev.to_halo(_t(x))
        enc = dev.encode_order(wd, "CHW")
        ex = dev.sf_conv_exact(_t(x), enc.nodes, enc.seg_off, k, 3, 3, 1, 1, bias, relu=True)
        jt = dev.sf_conv3x3(xh, dev.sf_pack(wd), bias, relu=True, pool=False, w=w)
        got = dev.from_halo(jt, w)
        err = float((got - ex).abs().max() / ex.abs().max().clamp_min(1e-30))
        assert err <= FAST_TOL, (layer, zf, err)
        if layer in (0, 4, 12) and zf in (0.5, 0.99):
            sj = dev.SfJit(wt, b, h, w, relu=True, pool=False)(xh)
            assert torch.equal(sj.view(torch.int32), jt.view(torch.int32)), (layer, zf)


@pytest.mark.parametrize("mode", ["max", "avg"])
def test_si_fast_fused_pool_equals_conv_then_pool(dev, mode):
    """Alg. 7 in the channel-major kernel's epilogue (layers.py:345-390) gives exactly the
    conv followed by the standalone pool (_pool_dense_kernel order), bias added after."""
    import torch

    rng = np.random.default_rng(17 if mode == "max" else 18)
    for n, c, k, h, w in ((2, 40, 72, 12, 20), (1, 128, 128, 28, 28), (3, 16, 200, 10, 14)):
        x = np.abs(rng.standard_normal((n, c, h, w))).astype(np.float32)
        x[rng.random(x.shape) < 0.85] = 0
        if mode == "max":
            x[0, 0, 1, 1] = -0.0  # explicit -0.0 inputs behave like absent nodes
        wt = (rng.standard_normal((k, c, 3, 3)) * 0.05).astype(np.float32)
        b = (rng.standard_normal(k) * 0.01).astype(np.float32)
        enc = dev.encode_order(_t(x), "CHW")
        wf = dev.si_pack_fast(_t(wt))
        conv = dev.si_conv3x3_fast(enc.nodes, enc.seg_off, n, c, h, w, wf, k)
        want = dev.pool2d(conv, 2, 2, mode == "max") + _t(b).view(1, -1, 1, 1)
        got = dev.si_conv3x3_fast(enc.nodes, enc.seg_off, n, c, h, w, wf, k, bias=_t(b), pool=mode)
        assert tuple(got.shape) == (n, k, h // 2, w // 2)
        assert torch.equal(got.view(torch.int32), want.view(torch.int32)), (n, c, k, h, w)


@pytest.mark.parametrize("k,pool", [(64, None), (96, "max"), (128, None), (256, "avg"), (130, "max")])
def test_si_fast_dense_input_equals_node_input(dev, k, pool):
    """fscnn_si_conv3x3_fast_dense (tile streams straight from a dense activation) is bit
    for bit the node-input kernel on the encoded activation: +-0.0 not stored, NaN and
    inf stored, ragged tiles, several images."""
    rng = np.random.default_rng(k)
    n, c, h, w = 3, 40, 18, 22
    x = np.abs(rng.standard_normal((n, c, h, w))).astype(np.float32)
    x[rng.random(x.shape) < 0.6] = 0
    x[0, 1, 2, 3] = -0.0
    x[1, 5, 0, 0] = np.nan
    x[2, 7, 17, 21] = np.inf
    x[2, 8, 4, 4] = -1.5
    wt = rng.standard_normal((k, c, 3, 3)).astype(np.float32)
    bias = rng.standard_normal(k).astype(np.float32)
    xd = _t(x)
    wf = dev.si_pack_fast(_t(wt))
    enc = dev.encode_order(xd, "CHW")
    ref = dev.si_conv3x3_fast(enc.nodes, enc.seg_off, n, c, h, w, wf, k, _t(bias), pool=pool).cpu().numpy()
    got = dev.si_conv3x3_fast_dense(xd, wf, k, _t(bias), pool=pool).cpu().numpy()
    assert np.array_equal(got.view(np.int32), ref.view(np.int32))
