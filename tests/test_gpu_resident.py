"""Device-resident twins of the reference tensors: DeviceDenseTensor3 /
DeviceSparseTensor3 go through every operator that takes the host types and come back
as twins, so a chain stays on the GPU; .to_host() must give exactly the host chain's
result (the same kernels run either way), and malformed twins are rejected like
malformed host tensors."""
import numpy as np
import pytest

import paper_2212_08815_b200 as fs
from paper_2212_08815_b200 import layers as ly

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.asarray(a, np.float32).view(np.int32)


def _same(host, dev):
    got = fs.to_host(dev)
    assert type(got) is type(host)
    assert tuple(got.dims) == tuple(host.dims)
    if isinstance(host, fs.SparseTensor3):
        assert got.order is host.order
        assert got.nodes.tobytes() == host.nodes.tobytes()
        assert np.array_equal(got.segment_offsets, host.segment_offsets)
        assert np.array_equal(got.matrix_offsets, host.matrix_offsets)
    else:
        assert np.array_equal(_bits(got.data), _bits(host.data))


def _bank(rng, k, c, zf):
    w = rng.normal(0, 0.2, (k, c, 3, 3)).astype(np.float32)
    w[rng.random(w.shape) < zf] = 0
    return w


def test_round_trips_all_orders():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((5, 7, 9)).astype(np.float32)
    x[rng.random(x.shape) < 0.6] = 0
    x[0, 0, 0] = -0.0
    t = fs.DenseTensor3.from_array(x)
    d = fs.to_device(t)
    assert isinstance(d, fs.DeviceDenseTensor3)
    _same(t, d)
    for order in fs.AxisOrder3:
        hs = fs.sparsify_tensor3(t, order)
        ds = fs.sparsify_tensor3(d, order)
        assert isinstance(ds, fs.DeviceSparseTensor3)
        _same(hs, ds)
        _same(hs, fs.to_device(hs))
        assert ds.nnz == hs.nnz
        _same(fs.densify_tensor3(hs), fs.densify_tensor3(ds))


def test_chain_stays_on_device_and_matches_host():
    """encoder -> sparse-input conv -> ReLU -> node pool -> decode -> sparse-filter conv
    -> ReLU -> pool -> pad -> batch norm, host objects vs device twins."""
    rng = np.random.default_rng(11)
    c, k1, k2, h = 16, 32, 24, 12
    x = np.abs(rng.standard_normal((c, h, h))).astype(np.float32)
    x[rng.random(x.shape) < 0.8] = 0
    w1 = rng.normal(0, 0.1, (k1, c, 3, 3)).astype(np.float32)
    filt1 = [fs.DenseTensor3.from_array(f) for f in w1]
    t4 = fs.SparseTensor4.stack([fs.sparsify_tensor3(fs.DenseTensor3.from_array(f), fs.AxisOrder3.CHW)
                                 for f in _bank(rng, k2, k1, 0.9)])
    bias2 = rng.normal(0, 0.1, k2).astype(np.float32)
    bn = ly.BatchNormParams(scale=rng.uniform(0.5, 1.5, k2), shift=rng.normal(0, 0.1, k2),
                            mean=rng.normal(0, 0.1, k2), var=rng.uniform(0.5, 1.5, k2))

    def chain(t):
        s = fs.sparsify_tensor3(t, fs.AxisOrder3.CHW)
        y = fs.conv_forward_sparse_input(s, filt1, 1, 1, np.zeros(k1, np.float32))
        y = fs.apply_activation(y, "relu")
        y = fs.pool_sparse(y, (2, 2), "max")
        d = fs.densify_tensor3(y)
        z = fs.conv_forward_strategy_II(d, t4, 1, 1, bias2)
        z = fs.apply_activation(z, "relu")
        z = fs.pool_standalone(z, (2, 2), "avg")
        z = fs.pad_tensor(z, 1)
        return y, fs.apply_batchnorm(z, bn)

    for exact in (False, True):
        fs.set_exact(exact)
        try:
            t = fs.DenseTensor3.from_array(x)
            hy, hz = chain(t)
            dy, dz = chain(fs.to_device(t))
            assert isinstance(dy, fs.DeviceSparseTensor3) and isinstance(dz, fs.DeviceDenseTensor3)
            _same(hy, dy)
            _same(hz, dz)
        finally:
            fs.set_exact(False)
    # node-format pad keeps every node (a device segment gather for the twin too)
    s = fs.sparsify_tensor3(fs.DenseTensor3.from_array(x), fs.AxisOrder3.CHW)
    _same(fs.pad_tensor(s, 2), fs.pad_tensor(fs.to_device(s), 2))


def test_malformed_twin_rejected():
    rng = np.random.default_rng(5)
    x = np.abs(rng.standard_normal((8, 6, 6))).astype(np.float32)
    x[rng.random(x.shape) < 0.3] = 0
    s = fs.to_device(fs.sparsify_tensor3(fs.DenseTensor3.from_array(x), fs.AxisOrder3.CHW))
    s.validate()
    nodes = s.nodes.clone()
    idx = nodes[:, 0].cpu().numpy()
    j = next(i for i in range(len(idx) - 1) if idx[i] >= 0 and idx[i + 1] >= 0)
    nodes[j, 0], nodes[j + 1, 0] = int(idx[j + 1]), int(idx[j])
    bad = fs.DeviceSparseTensor3(s.order, s.dims, nodes, s.matrix_offsets, s.segment_offsets)
    with pytest.raises(fs.FormatError, match="increase"):
        bad.validate()
    filt = [fs.DenseTensor3.from_array(rng.normal(0, 0.1, (8, 3, 3)).astype(np.float32)) for _ in range(4)]
    with pytest.raises(fs.FormatError):
        fs.conv_forward_sparse_input(bad, filt, 1, 1, np.zeros(4, np.float32))
    nodes = s.nodes.clone()
    nodes[-1, 0] = 3  # last segment loses its sentinel
    with pytest.raises(fs.FormatError, match="sentinel"):
        fs.DeviceSparseTensor3(s.order, s.dims, nodes, s.matrix_offsets, s.segment_offsets).validate()
