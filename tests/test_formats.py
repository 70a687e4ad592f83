"""The reference's on-disk formats, byte for byte against files the
reference wrote (tests/golden/formats.npz, tests/golden/make_golden.py::gen_formats):
FSCT / FDT3 tensor blobs, FSNW weight files, the model text format -- and their
error messages (test_sparse_core.py:223-237 / test_network.py's "magic", "truncated",
"order tag" cases).  Host-side I/O: runs on CPU.
"""

import os

import numpy as np
import pytest

from conftest import load_golden, weights_sha

import paper_2212_08815_b200 as fs
from paper_2212_08815_b200 import network as nw


@pytest.fixture(scope="module")
def g():
    return load_golden("formats.npz")


def test_fsct_fdt3_roundtrip_bytes(g):
    for i in range(6):
        blob = g[f"t{i}__fsct"].tobytes()
        t = fs.sparse3_from_bytes(blob)
        assert t.order.name == str(g[f"t{i}__order"])
        assert fs.sparse3_to_bytes(t) == blob
        d = fs.dense3_from_bytes(g[f"t{i}__fdt3"].tobytes())
        assert np.array_equal(d.to_array(), g[f"t{i}__x"])
        assert fs.dense3_to_bytes(d) == g[f"t{i}__fdt3"].tobytes()


def test_fsct_fdt3_errors(g):
    blob = g["t0__fsct"].tobytes()
    with pytest.raises(fs.FormatError, match="magic"):
        fs.sparse3_from_bytes(b"XXXX" + blob[4:])
    with pytest.raises(fs.FormatError, match="truncated"):
        fs.sparse3_from_bytes(blob[:10])
    with pytest.raises(fs.FormatError, match="truncated"):
        fs.sparse3_from_bytes(blob[:-3])
    bad = bytearray(blob)
    bad[4] = 9
    with pytest.raises(fs.FormatError, match="order tag"):
        fs.sparse3_from_bytes(bytes(bad))
    d = g["t0__fdt3"].tobytes()
    with pytest.raises(fs.FormatError, match="magic"):
        fs.dense3_from_bytes(b"FSCT" + d[4:])
    with pytest.raises(fs.FormatError, match="payload"):
        fs.dense3_from_bytes(d[:-4])


def test_fsnw_weight_files(g, tmp_path):
    for j in range(2):
        kind = str(g[f"w{j}__kind"])
        net = nw.build_benchmark_net(kind, 0.0625, input_hw=32)
        ref_file = tmp_path / f"ref{j}.fsnw"
        ref_file.write_bytes(g[f"w{j}__fsnw"].tobytes())
        w = nw.load_weights(str(ref_file), net)
        assert weights_sha(w) == str(g[f"w{j}__sha"])
        # our writer reproduces the reference's file exactly
        mine = tmp_path / f"mine{j}.fsnw"
        nw.save_weights(str(mine), net, nw.random_weights(net, 2010 + j))
        assert mine.read_bytes() == ref_file.read_bytes()
    raw = g["w0__fsnw"].tobytes()
    net = nw.build_benchmark_net("yolo_desk", 0.0625, input_hw=32)
    for blob, msg in ((b"NOPE" + raw[4:], "magic"), (raw[:8], "truncated"), (raw[:-5], "truncated"),
                      (raw + b"\0\0", "trailing")):
        p = tmp_path / "bad.fsnw"
        p.write_bytes(blob)
        with pytest.raises(fs.FormatError, match=msg):
            nw.load_weights(str(p), net)
    other = nw.build_benchmark_net("vgg16_desk", 0.0625, input_hw=32)
    p = tmp_path / "mismatch.fsnw"
    p.write_bytes(raw)
    with pytest.raises(fs.FormatError, match="parameterized layers"):
        nw.load_weights(str(p), other)


def test_model_text(g):
    for kind, text in zip(nw.BENCH_KINDS, g["model_texts"]):
        net = nw.build_benchmark_net(kind, 0.125, input_hw=32)
        assert nw.format_model_text(net) == str(text)
        back = nw.parse_model_text(str(text), kind)
        assert back.layers == net.layers and back.input_dims == net.input_dims
    custom = nw.parse_model_text(str(g["custom_text"]), "custom")
    assert nw.format_model_text(custom) == str(g["custom_formatted"])
    with pytest.raises(fs.FormatError, match="missing"):
        nw.parse_model_text("conv out=3 k=3\n")
    with pytest.raises(fs.FormatError, match="unknown layer kind"):
        nw.parse_model_text("input c=1 h=4 w=4\nfoo\n")
    with pytest.raises(fs.FormatError, match="malformed"):
        nw.parse_model_text("input c=1 h=4 w=4\nconv out 3\n")
    with pytest.raises(fs.FormatError, match="line 2"):
        nw.parse_model_text("input c=1 h=4 w=4\nconv k=3\n")
