"""Device-side operators: thin typed wrappers over the C ABI on torch CUDA tensors.

Everything here is stream-ordered on torch's current stream and allocates its outputs
with torch (the caching allocator).  The only host synchronisations are the ones the
node format forces: an encoder must learn its node count before it can size the node
buffer (count -> scan -> read total -> write), exactly the reference's two-pass
_build_segmented (sparse_core.py:319-331).

Tensor conventions
  dense activations   torch.float32 [N, C, H, W] (row pitch may exceed W, see ldw)
  node buffers        torch.int32 [n_nodes, 2]  -- byte-identical to NODE_DTYPE
  offset tables       torch.int64
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream

NODE_DTYPE = np.dtype([("index", "<i4"), ("value", "<f4")])


def _dev():
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def nodes_to_numpy(nodes: torch.Tensor, count: int | None = None) -> np.ndarray:
    """Device node buffer -> reference NODE_DTYPE array (bit copy)."""
    t = nodes if count is None else nodes[:count]
    return t.cpu().numpy().view(NODE_DTYPE).reshape(-1)


def nodes_from_numpy(nodes: np.ndarray, slack: int = 0) -> torch.Tensor:
    """Reference NODE_DTYPE array -> device int32 [n + slack, 2] (bit copy)."""
    a = np.ascontiguousarray(nodes).view(np.int32).reshape(-1, 2)
    out = torch.empty((a.shape[0] + slack, 2), dtype=torch.int32, device=_dev())
    if a.shape[0]:
        out[: a.shape[0]].copy_(torch.from_numpy(a), non_blocking=False)
    if slack:
        out[a.shape[0]:].fill_(-1)
    return out


# -- encoder / decoder ---------------------------------------------------------------


@dataclass
class Encoded:
    """Output of the device encoder for a batch of arranged tensors."""

    nodes: torch.Tensor          # int32 [n_nodes (+slack), 2]
    n_nodes: int
    seg_off: torch.Tensor        # int64 [batch*outer*mid]
    matrix_off: torch.Tensor     # int64 [batch*outer]
    tensor_off: torch.Tensor     # int64 [batch]


def encode(src: torch.Tensor, batch: int, outer: int, mid: int, inner: int,
           strides: tuple[int, int, int, int], slack: int = 0, mask: torch.Tensor | None = None) -> Encoded:
    """Node-format encoding of ``batch`` arranged (outer, mid, inner) views of ``src``.

    strides = (s_b, s_o, s_m, s_i) in elements.  Restates sparsify_tensor3 /
    SparseTensor4.stack (sparse_core.py:273-353) on the device; see fscnn_encode_*.
    With ``mask`` (uint8, same element offsets as ``src``) an entry is stored iff its
    mask byte is set (fscnn_encode_masked_*), whatever its value.
    """
    dev = _dev()
    s_b, s_o, s_m, s_i = (int(v) for v in strides)
    n_seg = batch * outer * mid
    seg = torch.empty(max(n_seg, 1), dtype=torch.int64, device=dev)
    total = torch.empty(1, dtype=torch.int64, device=dev)
    ws_bytes = int(_lib.load().fscnn_encode_workspace_bytes(n_seg))
    ws = torch.empty(ws_bytes // 8 + 1, dtype=torch.int64, device=dev)
    st = stream()
    geo = (batch, outer, mid, inner, s_b, s_o, s_m, s_i)
    if mask is None:
        call("fscnn_encode_offsets", ptr(src), *geo, ptr(seg), ptr(total), ptr(ws), ws_bytes, st)
    else:
        call("fscnn_encode_masked_offsets", ptr(src), ptr(mask), *geo, ptr(seg), ptr(total), ptr(ws),
             ws_bytes, st)
    n_nodes = int(total.item())  # the format's one forced sync: size the node buffer
    nodes = torch.empty((n_nodes + slack, 2), dtype=torch.int32, device=dev)
    if slack:
        nodes[n_nodes:].fill_(-1)
    mat = torch.empty(max(batch * outer, 1), dtype=torch.int64, device=dev)
    ten = torch.empty(max(batch, 1), dtype=torch.int64, device=dev)
    if mask is None:
        call("fscnn_encode_nodes", ptr(src), *geo, ptr(seg), ptr(nodes), ptr(mat), ptr(ten), st)
    else:
        call("fscnn_encode_masked_nodes", ptr(src), ptr(mask), *geo, ptr(seg), ptr(nodes), ptr(mat),
             ptr(ten), st)
    return Encoded(nodes, n_nodes, seg[:n_seg], mat[: batch * outer], ten[:batch])


# (inner, mid, outer) axis ids 0=C 1=H 2=W per order name (sparse_core.py:44-66)
ORDER_AXES = {
    "WHC": (2, 1, 0),
    "WCH": (2, 0, 1),
    "HWC": (1, 2, 0),
    "HCW": (1, 0, 2),
    "CHW": (0, 1, 2),
    "CWH": (0, 2, 1),
}


def _order_geometry(shape, strides, order: str):
    """(outer, mid, inner, s_b, s_o, s_m, s_i) of a [B, C, H, W]-indexed view in ``order``."""
    inner_ax, mid_ax, outer_ax = ORDER_AXES[order]
    dims = shape[1:]
    es = (strides[1], strides[2], strides[3])  # element strides of c, h, w
    return (int(dims[outer_ax]), int(dims[mid_ax]), int(dims[inner_ax]),
            int(strides[0]), int(es[outer_ax]), int(es[mid_ax]), int(es[inner_ax]))


def encode_order(x: torch.Tensor, order: str, slack: int = 0, mask: torch.Tensor | None = None) -> Encoded:
    """Encode a [B, C, H, W]-indexed tensor (any strides) in the named axis order; with
    ``mask`` (same strides) the stored set is the mask, not the nonzeros."""
    assert x.dim() == 4
    if mask is not None:
        assert mask.stride() == x.stride() and mask.dtype == torch.uint8
    o, m, i, s_b, s_o, s_m, s_i = _order_geometry(x.shape, x.stride(), order)
    return encode(x, x.shape[0], o, m, i, (s_b, s_o, s_m, s_i), slack, mask)


def decode(nodes: torch.Tensor, seg_off: torch.Tensor, batch: int, outer: int, mid: int,
           inner: int, out: torch.Tensor, strides: tuple[int, int, int, int],
           mask: torch.Tensor | None = None) -> torch.Tensor:
    """Write every element of the strided destination view from node format (and, with
    ``mask``, 1 where a node is stored / 0 elsewhere at the same element offsets)."""
    d_b, d_o, d_m, d_i = (int(v) for v in strides)
    if mask is None:
        call("fscnn_decode", ptr(nodes), ptr(seg_off), batch, outer, mid, inner, ptr(out),
             d_b, d_o, d_m, d_i, stream())
    else:
        call("fscnn_decode_masked", ptr(nodes), ptr(seg_off), batch, outer, mid, inner, ptr(out),
             ptr(mask), d_b, d_o, d_m, d_i, stream())
    return out


def decode_order(nodes, seg_off, dims_bchw, order: str, out: torch.Tensor | None = None,
                 mask: torch.Tensor | None = None):
    """Inverse of encode_order: returns a dense [B, C, H, W] tensor."""
    if out is None:
        out = torch.empty(tuple(dims_bchw), dtype=torch.float32, device=_dev())
    o, m, i, s_b, s_o, s_m, s_i = _order_geometry(out.shape, out.stride(), order)
    return decode(nodes, seg_off, int(dims_bchw[0]), o, m, i, out, (s_b, s_o, s_m, s_i), mask)


# -- sparse-filter conv ------------------------------------------------------------------

STAGES, BOXW, SUBW, TILE = 2, 20, 16, 4  # STAGES: the minimum ring the kernel runs with
# filters per CTA (CTA_FILTERS // kt warps); must match the library's build
# (-DFSCNN_SF3_CTA_FILTERS, default 32 = two CTAs per SM, 64 = one)
CTA_FILTERS = int(os.environ.get("FSCNN_SF3_CTA_FILTERS", "32"))
SMEM_LIMIT = 227 * 1024


def _align(v: int, a: int) -> int:
    return (v + a - 1) // a * a


SMEM_2CTA = 113 * 1024  # per-CTA budget that keeps two CTAs resident per SM


def sf3x3_smem_bytes(ly: int, cc: int, ent_cap: int, c: int, kt: int = 4, stages: int = STAGES) -> int:
    NWARP = {1: 4, 2: 8}.get(kt, CTA_FILTERS // kt)  # mirrors SfCfg in sf_conv.cu
    li, box = 8 // ly, _align(BOXW * (TILE * ly + 2) * cc, 32)
    n_chunks = math.ceil(c / cc)
    return (stages * li * box * 4 + stages * NWARP * ent_cap * 8 + 2 * stages * 8
            + NWARP * (n_chunks + 1) * 4)


def pick_ly(c: int, h: int) -> int:
    """Sub-region height 4*ly (mirrors the auto rule of fscnn_sf_conv3x3_ex): 16x16
    sub-regions measured fastest on every VGG16 width with 16-channel chunks (also at
    56/28/14, where they pad more rows than 8x16); 8x16 for shallow inputs (c < 8) and
    short images."""
    return 2 if (c < 8 or h <= 8) else 4


def sf_ctas(n: int, h: int, w: int, k: int, ly: int, kt: int) -> int:
    """CTAs of one fast sparse-filter launch (mirrors launch_sf3x3 in sf_conv.cu)."""
    li = 8 // ly
    n_sub = n * -(-h // (TILE * ly)) * -(-w // SUBW)
    filters_per_cta = {1: 4, 2: 16}.get(kt, CTA_FILTERS)  # default warps per CTA
    return -(-n_sub // li) * -(-k // filters_per_cta)


def sf_grid_plan(n: int, h: int, w: int, k: int, ly: int) -> tuple[int, int]:
    """(filters per warp, warps per CTA; 0 = default) for a launch over n images.  When
    the 4-filters-per-warp grid cannot give every SM a CTA (deep layers at small batch),
    fewer filters per warp -- more CTAs, a shorter dispatch chain per warp, more patch
    reloads per nonzero; bit-identical results -- are faster: 2 per warp below 148 CTAs,
    1 per warp in 4-warp CTAs at <= 32 (VGG16 layer 8 at batch 1: 213 -> 157 -> 114 us;
    layer 10: 204 -> 151 -> 96 us); both lose once the grid fills the GPU
    (tools/kt_check.py)."""
    g4 = sf_ctas(n, h, w, k, ly, 4)
    if g4 >= 148:
        return 4, 0
    return (2, 0) if g4 > 32 else (1, 4)


@dataclass
class PackedBank:
    """A filter bank in the fast kernel's channel-major packed stream (device)."""

    k: int
    c: int
    kt: int                    # filters per group (4 or 8)
    nodes: torch.Tensor        # int32 [total + 2, 2]
    seg_off: torch.Tensor      # int64 [groups * c]
    total: int
    counts: np.ndarray         # host: nodes per (group, channel) incl. sentinel
    nnz: int                   # nonzero weights
    _cache: dict = None

    def chunk_plan(self, ly: int) -> tuple[int, int]:
        """(cc, max_chunk_entries) for sub-region height 4*ly: the largest channel chunk
        whose 2-stage ring keeps two CTAs per SM (per-chunk ring coupling costs ~25% at 4
        vs 8 channels, ~8% at 8 vs 16), else the largest that fits at all."""
        if self._cache is None:
            self._cache = {}
        if ly in self._cache:
            return self._cache[ly]
        forced = int(os.environ.get("FSCNN_SF3_CC", "0"))
        cands = []
        sizes = sorted({16, 8, 4, 2, 1} | ({self.c} if self.c < 16 else set()), reverse=True)
        for cc in ((forced,) if forced else sizes):
            if cc > self.c and not forced:
                continue
            n_chunks = math.ceil(self.c / cc)
            pad = n_chunks * cc - self.c
            cnt = np.pad(self.counts, ((0, 0), (0, pad)))
            mx = int(cnt.reshape(cnt.shape[0], n_chunks, cc).sum(axis=2).max())
            ent_cap = (mx + 4) & ~1
            cands.append((cc, mx, sf3x3_smem_bytes(ly, cc, ent_cap, self.c, self.kt)))
        for limit in ((SMEM_2CTA, SMEM_LIMIT) if CTA_FILTERS == 32 else (SMEM_LIMIT,)):
            for cc, mx, need in cands:
                if need <= limit:
                    self._cache[ly] = (cc, mx)
                    return cc, mx
        raise RuntimeError("filter bank too dense for the fast kernel's shared memory")


def default_kt(c: int) -> int:
    """Filters per warp group: 8 halves the per-channel patch reloads (shared-memory
    bound at 4) at half the resident warps; the env var FSCNN_SF3_KT overrides."""
    forced = int(os.environ.get("FSCNN_SF3_KT", "0"))
    return forced if forced in (1, 2, 4, 8) else int(_lib.load().fscnn_sf_pack_kt())


def sf_pack(w_kc33: torch.Tensor, kt: int | None = None) -> PackedBank:
    """Pack a dense [K, C, 3, 3] bank (device) into the fast kernel's stream."""
    assert w_kc33.dim() == 4 and tuple(w_kc33.shape[2:]) == (3, 3)
    w = w_kc33.contiguous()
    k, c = int(w.shape[0]), int(w.shape[1])
    kt = int(kt or default_kt(c))
    groups = math.ceil(k / kt)
    dev = _dev()
    seg = torch.empty(groups * c, dtype=torch.int64, device=dev)
    total = torch.empty(1, dtype=torch.int64, device=dev)
    ws_bytes = int(_lib.load().fscnn_encode_workspace_bytes(groups * c))
    ws = torch.empty(ws_bytes // 8 + 1, dtype=torch.int64, device=dev)
    st = stream()
    call("fscnn_sf_pack_offsets", ptr(w), k, c, kt, ptr(seg), ptr(total), ptr(ws), ws_bytes, st)
    n = int(total.item())
    nodes = torch.empty((n + 2, 2), dtype=torch.int32, device=dev)
    nodes[n:].fill_(-1)
    call("fscnn_sf_pack_nodes", ptr(w), k, c, kt, ptr(seg), n, ptr(nodes), st)
    so = seg.cpu().numpy()
    ends = np.append(so[1:], n)
    counts = (ends - so).reshape(groups, c)
    return PackedBank(k, c, kt, nodes, seg, n, counts, int(n - groups * c))


def halo_pitch(w: int) -> int:
    """Row pitch of the halo-column layout: logical column j at memory column j+1,
    column 0 and columns > w zero, pitch a multiple of 4 floats (16 B, TMA stride)."""
    return _align(w + 1, 4)


def halo_empty(n: int, c: int, h: int, w: int, device=None) -> torch.Tensor:
    """Zeroed [N, C, H, halo_pitch(w)] buffer (the kernels never write the halo columns)."""
    return torch.zeros((n, c, h, halo_pitch(w)), dtype=torch.float32, device=device or _dev())


def to_halo(x: torch.Tensor) -> torch.Tensor:
    """Dense [N, C, H, W] -> halo-column layout copy."""
    n, c, h, w = (int(v) for v in x.shape)
    out = halo_empty(n, c, h, w, x.device)
    out[..., 1 : w + 1] = x
    return out


def pitch_copy(x: torch.Tensor, rows: int, w: int, ldx: int, colx: int, y: torch.Tensor, ldy: int,
               coly: int) -> torch.Tensor:
    call("fscnn_pitch_copy", ptr(x), rows, w, ldx, colx, ptr(y), ldy, coly, stream())
    return y


def nchw_into_halo(x: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """Dense [N, C, H, W] into a halo-column buffer [N, C, H, pitch] (one kernel)."""
    x = x.contiguous()
    n, c, h, w = (int(v) for v in x.shape)
    assert out.is_contiguous() and tuple(out.shape[:3]) == (n, c, h) and out.shape[3] >= w + 1
    return pitch_copy(x, n * c * h, w, w, 0, out, int(out.shape[3]), 1)


def halo_to_nchw(xh: torch.Tensor, w: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """Logical [N, C, H, w] of a halo-column buffer -> dense contiguous [N, C, H, w]."""
    assert xh.is_contiguous()
    n, c, h, ld = (int(v) for v in xh.shape)
    if out is None:
        out = torch.empty((n, c, h, w), dtype=torch.float32, device=xh.device)
    return pitch_copy(xh, n * c * h, w, ld, 1, out, w, 0)


def from_halo(xh: torch.Tensor, w: int) -> torch.Tensor:
    """View of the logical [N, C, H, W] data inside a halo-column buffer."""
    return xh[..., 1 : w + 1]


def sf_conv3x3(x: torch.Tensor, bank: PackedBank, bias: torch.Tensor | None, relu: bool,
               pool: bool, out: torch.Tensor | None = None, w: int | None = None,
               ly: int = 0, cta_warps: int = 0) -> torch.Tensor:
    """Fast 3x3/s1/p1 sparse-filter conv (+ReLU, +fused 2x2 max-pool).

    ``x`` is a halo-column buffer [N, C, H, pitch] (see halo_pitch) holding a logical
    width ``w`` (default pitch - 1).  Returns the halo-column output buffer
    [N, K, H', pitch'] (H' = H/2 with the fused pool); use from_halo to view it.
    """
    n, c, h = int(x.shape[0]), int(x.shape[1]), int(x.shape[2])
    ldi = int(x.stride(2))
    w = ldi - 1 if w is None else int(w)
    assert x.stride(3) == 1 and x.stride(1) == ldi * h and x.stride(0) == ldi * h * c
    assert c == bank.c and ldi >= w + 1
    if ly <= 0:
        ly = pick_ly(c, h)
    cc, mx = bank.chunk_plan(ly)
    ho, wo = (h // 2, w // 2) if pool else (h, w)
    if out is None:
        out = halo_empty(n, bank.k, ho, wo, x.device)
    ldo = int(out.stride(2))
    call("fscnn_sf_conv3x3_ex", ptr(x), n, c, h, w, ldi, ptr(bank.nodes), ptr(bank.seg_off),
         bank.total, mx, cc, bank.k, ptr(bias), int(relu), int(pool), ptr(out), ldo, ly,
         bank.kt | (int(cta_warps) << 8), stream())
    return out


def sfjit_enabled() -> bool:
    """The VGG engine compiles each bank into specialised kernels unless FSCNN_SFJIT=0."""
    return os.environ.get("FSCNN_SFJIT", "1") != "0"


class SfJit:
    """Per-layer specialised sparse-filter conv (fscnn_sfjit_*): the filter bank is
    compiled into straight-line kernels (one per group of 32 filters).  Bit-identical to
    sf_conv3x3 on the same bank (same accumulation order).  Construction submits the
    compile jobs and returns; the first call (or wait()) joins them."""

    INFO = ("groups", "ctas_per_image_or_minus_images_per_cta", "warps", "filters_per_group", "channels_per_chunk", "stages",
            "smem_bytes", "box_rows", "row_pitch", "boxes_per_cta", "registers", "cached_groups")

    def __init__(self, w_kc33, bias, h: int, w: int, relu: bool = True, pool: bool = False, flags: int = 0):
        import ctypes

        wt = np.ascontiguousarray(w_kc33.detach().cpu().numpy() if torch.is_tensor(w_kc33) else w_kc33,
                                  dtype=np.float32)
        self.k, self.c = int(wt.shape[0]), int(wt.shape[1])
        assert wt.shape[2:] == (3, 3)
        b = None
        if bias is not None:
            b = np.ascontiguousarray(bias.detach().cpu().numpy() if torch.is_tensor(bias) else bias, dtype=np.float32)
        self.h, self.w, self.relu, self.pool = h, w, bool(relu), bool(pool)
        handle = ctypes.c_void_p()
        call("fscnn_sfjit_create", wt.ctypes.data, b.ctypes.data if b is not None else None, self.k, self.c, h, w,
             int(relu), int(pool), int(flags), ctypes.byref(handle))
        self._h = handle
        self._lib = _lib.load()

    def wait(self) -> "SfJit":
        call("fscnn_sfjit_wait", self._h)
        return self

    def info(self) -> dict:
        import ctypes

        v = (ctypes.c_int64 * 12)()
        sec = (ctypes.c_double * 2)()
        call("fscnn_sfjit_info", self._h, v, sec)
        d = dict(zip(self.INFO, list(v)))
        d["compile_seconds_total"] = sec[1]
        return d

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None, n: int | None = None) -> torch.Tensor:
        """x: halo-column buffer [N, C, H, pitch] -> halo-column output [N, K, H', pitch']."""
        n = int(x.shape[0]) if n is None else n
        assert int(x.shape[1]) == self.c and int(x.shape[2]) == self.h and x.stride(3) == 1
        ldi = int(x.stride(2))
        ho, wo = (self.h // 2, self.w // 2) if self.pool else (self.h, self.w)
        if out is None:
            out = halo_empty(n, self.k, ho, wo, x.device)
        call("fscnn_sfjit_launch", self._h, ptr(x), n, ldi, ptr(out), int(out.stride(2)), stream())
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and getattr(self, "_lib", None) is not None:
            self._lib.fscnn_sfjit_destroy(h)
            self._h = None


def sf_conv_exact(x: torch.Tensor, nodes: torch.Tensor, seg_off: torch.Tensor, k: int, h_f: int,
                  w_f: int, stride_: int, pad: int, bias: torch.Tensor | None, relu: bool = False,
                  out: torch.Tensor | None = None) -> torch.Tensor:
    """Reference-order sparse-filter conv (bit-exact with layers.py:170-180)."""
    x = x.contiguous()
    n, c, h, w = (int(v) for v in x.shape)
    n_h = (h + 2 * pad - h_f) // stride_ + 1
    n_w = (w + 2 * pad - w_f) // stride_ + 1
    if out is None:
        out = torch.empty((n, k, n_h, n_w), dtype=torch.float32, device=x.device)
    call("fscnn_sf_conv_exact", ptr(x), n, c, h, w, ptr(nodes), ptr(seg_off), k, h_f, w_f,
         stride_, pad, ptr(bias), int(relu), ptr(out), stream())
    return out


# -- sparse-input conv --------------------------------------------------------------------


def kcrs_to_crsk(w: torch.Tensor) -> torch.Tensor:
    w = w.contiguous()
    k, c, r, s = (int(v) for v in w.shape)
    out = torch.empty((c, r, s, k), dtype=torch.float32, device=w.device)
    call("fscnn_kcrs_to_crsk", ptr(w), k, c, r, s, ptr(out), stream())
    return out


def si_conv(nodes: torch.Tensor, seg_off: torch.Tensor, n: int, c: int, h: int, w: int,
            wt_crsk: torch.Tensor, k: int, h_f: int, w_f: int, stride_: int, pad: int,
            bias: torch.Tensor | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Sparse-input conv over CHW node tensors (bit-exact with kernels.py:136-166)."""
    n_h = (h + 2 * pad - h_f) // stride_ + 1
    n_w = (w + 2 * pad - w_f) // stride_ + 1
    if out is None:
        out = torch.empty((n, k, n_h, n_w), dtype=torch.float32, device=nodes.device)
    call("fscnn_si_conv", ptr(nodes), ptr(seg_off), n, c, h, w, ptr(wt_crsk), k, h_f, w_f,
         stride_, pad, ptr(bias), ptr(out), stream())
    return out


def si_pack3x3(w_kc33: torch.Tensor) -> torch.Tensor:
    """Dense [K, C, 3, 3] bank -> the strip kernel's [C][3][K] float4 layout."""
    w = w_kc33.contiguous()
    k, c = int(w.shape[0]), int(w.shape[1])
    out = torch.empty((c, 3, k, 4), dtype=torch.float32, device=w.device)
    call("fscnn_si_pack3x3", ptr(w), k, c, ptr(out), stream())
    return out


def si_conv3x3(nodes: torch.Tensor, seg_off: torch.Tensor, n: int, c: int, h: int, w: int,
               wq: torch.Tensor, k: int, bias: torch.Tensor | None = None,
               out: torch.Tensor | None = None) -> torch.Tensor:
    """3x3/s1/p1 sparse-input conv (strip kernel), bit-exact with kernels.py:136-166."""
    if out is None:
        out = torch.empty((n, k, h, w), dtype=torch.float32, device=nodes.device)
    call("fscnn_si_conv3x3", ptr(nodes), ptr(seg_off), n, c, h, w, ptr(wq), k, ptr(bias), ptr(out), stream())
    return out


def si_pack_fast(w_kc33: torch.Tensor) -> torch.Tensor:
    """Dense [K, C, 3, 3] bank -> the channel-major kernel's [C][Kp/(32 KT)][9][32][KT]
    layout (KT = filters per lane: 4 from K = 128, 2 from K = 64, else 1; Kp = K rounded
    up to 32 KT, 64 at least)."""
    w = w_kc33.contiguous()
    k, c = int(w.shape[0]), int(w.shape[1])
    n = int(_lib.load().fscnn_si_fast_bank_floats(k, c))
    out = torch.empty(n, dtype=torch.float32, device=w.device)
    call("fscnn_si_pack_fast", ptr(w), k, c, ptr(out), stream())
    return out


def si_fast_warps(n: int, h: int, w: int, k: int) -> int:
    """Warps of the two-pass channel-major SI kernel (K >= 64): one per (output tile,
    filter group) -- 4x8 tiles x 64 filters below K = 128, 4x4 tiles x 128 filters from
    there -- mirroring si3x3_tl_kernel's grid in si_fast.cu."""
    if k < 128:
        return n * -(-h // 4) * -(-w // 8) * -(-k // 64)
    return n * -(-h // 4) * -(-w // 4) * -(-k // 128)


def si_use_fast(h: int, w: int, k: int) -> bool:
    """The layer API's choice for a 3x3/s1/p1 sparse-input conv of one h x w image with k
    filters: the channel-major kernel when one image already gives every SM two warps
    and the filter count fills its 64-filter lane pairs (K >= 64), else the bit-exact
    strip kernel.  Deep layers (K >= 256: VGG16's 512-filter 28x28 and 14x14 convs) take
    the channel-major kernel from 64 warps per image: one image then runs 0.96-1.8x the
    strip kernel's time, a batch of 32 3.7-4.3x faster (measured,
    profiles/r02_si_rule_n1.txt).  Depends on the image shape only, never on the batch,
    so batched and per-image runs agree bitwise."""
    warps = si_fast_warps(1, h, w, k)
    return k >= 64 and (warps >= 2 * 148 or (k >= 256 and warps >= 64))


def si_conv3x3_fast(nodes: torch.Tensor, seg_off: torch.Tensor, n: int, c: int, h: int, w: int,
                    wf: torch.Tensor, k: int, bias: torch.Tensor | None = None,
                    out: torch.Tensor | None = None, pool: str | None = None) -> torch.Tensor:
    """3x3/s1/p1 sparse-input conv, channel-major (fp32 reassociation of kernels.py:136-166,
    held to the north-star 1e-4 normwise tolerance).  ``pool`` = 'max' / 'avg' fuses
    Alg. 7's 2x2 pooling (layers.py:345-390) into the epilogue: [n, k, h/2, w/2]."""
    mode = {None: 0, "max": 1, "avg": 2}[pool]
    if out is None:
        shape = (n, k, h // 2, w // 2) if mode else (n, k, h, w)
        out = torch.empty(shape, dtype=torch.float32, device=nodes.device)
    n_nodes = int(nodes.numel() // 2)
    call("fscnn_si_conv3x3_fast_pool", ptr(nodes), ptr(seg_off), n_nodes, n, c, h, w, ptr(wf), k, ptr(bias), mode,
         ptr(out), stream())
    return out


def si_conv3x3_fast_dense(x: torch.Tensor, wf: torch.Tensor, k: int, bias: torch.Tensor | None = None,
                          out: torch.Tensor | None = None, pool: str | None = None) -> torch.Tensor:
    """si_conv3x3_fast straight from a dense [n, c, h, w] activation: bit-identical to
    encoding x in CHW order and calling si_conv3x3_fast (same tile streams), without
    the encode (and its host sync) between sparse-input layers.  K >= 64."""
    x = x.contiguous()
    n, c, h, w = (int(v) for v in x.shape)
    mode = {None: 0, "max": 1, "avg": 2}[pool]
    if out is None:
        shape = (n, k, h // 2, w // 2) if mode else (n, k, h, w)
        out = torch.empty(shape, dtype=torch.float32, device=x.device)
    call("fscnn_si_conv3x3_fast_dense", ptr(x), n, c, h, w, ptr(wf), k, ptr(bias), mode, ptr(out), stream())
    return out


# -- dense layers / layout ----------------------------------------------------------------


def relu(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    x = x.contiguous()
    if out is None:
        out = torch.empty_like(x)
    call("fscnn_relu", ptr(x), x.numel(), ptr(out), stream())
    return out


ACT_RELU, ACT_LEAKY, ACT_RELU_NODES = 0, 1, 2


def activation(x: torch.Tensor, kind: int, slope: float = 0.0, out: torch.Tensor | None = None) -> torch.Tensor:
    """ACT_RELU: np.maximum(x, 0); ACT_LEAKY: np.where(x > 0, x, slope*x);
    ACT_RELU_NODES: x > 0 ? x : 0 (the node-format keep rule, layers.py:488-489)."""
    x = x.contiguous()
    if out is None:
        out = torch.empty_like(x)
    call("fscnn_activation", ptr(x), x.numel(), int(kind), float(np.float32(slope)), ptr(out), stream())
    return out


def batchnorm(x: torch.Tensor, scale, shift, mean, var, eps: float, out=None) -> torch.Tensor:
    """apply_batchnorm (layers.py:507-509) on NCHW, numpy float32 op order."""
    x = x.contiguous()
    n, c, h, w = (int(v) for v in x.shape)
    dev = x.device
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).to(dev)
    sc, sh, mu, va = t(scale), t(shift), t(mean), t(var)
    if out is None:
        out = torch.empty_like(x)
    call("fscnn_batchnorm", ptr(x), n, c, h, w, ptr(sc), ptr(sh), ptr(mu), ptr(va),
         float(np.float32(eps)), ptr(out), stream())
    return out


def pad2d(x: torch.Tensor, p: int, out=None) -> torch.Tensor:
    x = x.contiguous()
    n, c, h, w = (int(v) for v in x.shape)
    if out is None:
        out = torch.empty((n, c, h + 2 * p, w + 2 * p), dtype=torch.float32, device=x.device)
    call("fscnn_pad2d", ptr(x), n, c, h, w, int(p), ptr(out), stream())
    return out


def remap_segments(nodes: torch.Tensor, seg_off: torch.Tensor, n_nodes: int, seg_map: torch.Tensor):
    """Segment gather (see fscnn_remap_segments_*): returns (nodes, n_nodes, seg_off)."""
    dev = _dev()
    n_old, n_new = int(seg_off.numel()), int(seg_map.numel())
    new_off = torch.empty(max(n_new, 1), dtype=torch.int64, device=dev)
    total = torch.empty(1, dtype=torch.int64, device=dev)
    ws_bytes = int(_lib.load().fscnn_encode_workspace_bytes(n_new))
    ws = torch.empty(ws_bytes // 8 + 1, dtype=torch.int64, device=dev)
    m = seg_map.to(dev, torch.int64).contiguous()
    call("fscnn_remap_segments_offsets", ptr(seg_off), n_old, n_nodes, ptr(m), n_new, ptr(new_off),
         ptr(total), ptr(ws), ws_bytes, stream())
    count = int(total.item())
    out = torch.empty((max(count, 1), 2), dtype=torch.int32, device=dev)
    call("fscnn_remap_segments_nodes", ptr(nodes), ptr(seg_off), n_old, n_nodes, ptr(m), n_new,
         ptr(new_off), ptr(out), stream())
    return out[:count], count, new_off[:n_new]


def dense_conv_exact(x: torch.Tensor, wt: torch.Tensor, stride_: int, pad: int, bias: torch.Tensor | None,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """Dense baseline conv, bit-exact with _dense_conv_kernel (kernels.py:169-192)."""
    x, wt = x.contiguous(), wt.contiguous()
    n, c, h, w = (int(v) for v in x.shape)
    k, _, h_f, w_f = (int(v) for v in wt.shape)
    n_h = (h + 2 * pad - h_f) // stride_ + 1
    n_w = (w + 2 * pad - w_f) // stride_ + 1
    if out is None:
        out = torch.empty((n, k, n_h, n_w), dtype=torch.float32, device=x.device)
    call("fscnn_dense_conv_exact", ptr(x), n, c, h, w, ptr(wt), k, h_f, w_f, stride_, pad, ptr(bias),
         ptr(out), stream())
    return out


def pool2d(x: torch.Tensor, h_p: int, w_p: int, use_max: bool, out=None) -> torch.Tensor:
    x = x.contiguous()
    n, c, h, w = (int(v) for v in x.shape)
    if out is None:
        out = torch.empty((n, c, h // h_p, w // w_p), dtype=torch.float32, device=x.device)
    call("fscnn_pool2d", ptr(x), n, c, h, w, h_p, w_p, int(use_max), ptr(out), stream())
    return out


def whc_to_nchw(x_whc: torch.Tensor, n: int, c: int, h: int, w: int, out=None) -> torch.Tensor:
    if out is None:
        out = torch.empty((n, c, h, w), dtype=torch.float32, device=x_whc.device)
    call("fscnn_whc_to_nchw", ptr(x_whc), n, c, h, w, ptr(out), stream())
    return out


def whc_to_halo(x_whc: torch.Tensor, n: int, c: int, h: int, w: int, out: torch.Tensor) -> torch.Tensor:
    """(W,H,C)-memory images straight into a halo-column buffer [N, C, H, pitch]."""
    assert out.is_contiguous() and tuple(out.shape[:3]) == (n, c, h) and out.shape[3] >= w + 1
    call("fscnn_whc_to_nchw_ex", ptr(x_whc), n, c, h, w, ptr(out), int(out.shape[3]), 1, stream())
    return out


def halo_to_whc(xh: torch.Tensor, w: int, out=None) -> torch.Tensor:
    """Logical [N, C, H, w] of a halo-column buffer -> (W,H,C)-memory images [N, W, H, C]."""
    assert xh.is_contiguous()
    n, c, h, ld = (int(v) for v in xh.shape)
    if out is None:
        out = torch.empty((n, w, h, c), dtype=torch.float32, device=xh.device)
    call("fscnn_nchw_to_whc_ex", ptr(xh), n, c, h, w, ld, 1, ptr(out), stream())
    return out


def nchw_to_whc(x: torch.Tensor, out=None) -> torch.Tensor:
    x = x.contiguous()
    n, c, h, w = (int(v) for v in x.shape)
    if out is None:
        out = torch.empty((n, w, h, c), dtype=torch.float32, device=x.device)
    call("fscnn_nchw_to_whc", ptr(x), n, c, h, w, ptr(out), stream())
    return out
