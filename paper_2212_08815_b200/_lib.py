"""ctypes binding of libfscnn_b200.so (the C ABI declared in include/fscnn_b200.h).

The package has no CPU fallback: importing a compute entry point without the built
library, or calling one without a CUDA device, raises immediately.  Device memory
and streams come from PyTorch (torch.cuda tensors, the current stream); the C ABI
sees plain pointers.
"""

from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfscnn_b200.so")


class FscnnError(RuntimeError):
    """A CUDA-side failure reported by libfscnn_b200."""


_i64, _i32, _vp, _sz = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/fscnn_b200.h
_SIGNATURES = {
    "fscnn_abi_version": (_i32, []),
    "fscnn_last_error": (ctypes.c_char_p, []),
    "fscnn_launch_count": (_i64, []),
    "fscnn_reset_launch_count": (None, []),
    "fscnn_add_launch_count": (None, [_i64]),
    "fscnn_encode_workspace_bytes": (_sz, [_i64]),
    "fscnn_encode_offsets": (_i32, [_vp] + [_i64] * 8 + [_vp, _vp, _vp, _sz, _vp]),
    "fscnn_encode_nodes": (_i32, [_vp] + [_i64] * 8 + [_vp, _vp, _vp, _vp, _vp]),
    "fscnn_decode": (_i32, [_vp, _vp] + [_i64] * 4 + [_vp] + [_i64] * 4 + [_vp]),
    "fscnn_decode_masked": (_i32, [_vp, _vp] + [_i64] * 4 + [_vp, _vp] + [_i64] * 4 + [_vp]),
    "fscnn_encode_masked_offsets": (_i32, [_vp, _vp] + [_i64] * 8 + [_vp, _vp, _vp, _sz, _vp]),
    "fscnn_encode_masked_nodes": (_i32, [_vp, _vp] + [_i64] * 8 + [_vp, _vp, _vp, _vp, _vp]),
    "fscnn_remap_segments_offsets": (_i32, [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "fscnn_remap_segments_nodes": (_i32, [_vp, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp]),
    "fscnn_sf_conv_exact": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp]),
    "fscnn_sf_pack_kt": (_i32, []),
    "fscnn_sf_pack_offsets": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp, _vp, _sz, _vp]),
    "fscnn_sf_pack_nodes": (_i32, [_vp, _i32, _i32, _i32, _vp, _i64, _vp, _vp]),
    "fscnn_sf_conv3x3_ex": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _i32, _i32, _i32, _vp]),
    "fscnn_si_conv": (_i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp]),
    "fscnn_kcrs_to_crsk": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "fscnn_si_pack3x3": (_i32, [_vp, _i32, _i32, _vp, _vp]),
    "fscnn_si_conv3x3": (_i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp, _vp]),
    "fscnn_si_fast_bank_floats": (_i64, [_i32, _i32]),
    "fscnn_si_pack_fast": (_i32, [_vp, _i32, _i32, _vp, _vp]),
    "fscnn_si_conv3x3_fast": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp, _vp]),
    "fscnn_si_conv3x3_fast_pool": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _i32, _vp, _vp]),
    "fscnn_si_conv3x3_fast_dense": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _i32, _vp, _vp]),
    "fscnn_dense_conv_exact": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp]),
    "fscnn_relu": (_i32, [_vp, _i64, _vp, _vp]),
    "fscnn_activation": (_i32, [_vp, _i64, _i32, ctypes.c_float, _vp, _vp]),
    "fscnn_batchnorm": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, ctypes.c_float, _vp, _vp]),
    "fscnn_pad2d": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "fscnn_pool2d": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "fscnn_whc_to_nchw": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "fscnn_nchw_to_whc": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "fscnn_whc_to_nchw_ex": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _vp]),
    "fscnn_nchw_to_whc_ex": (_i32, [_vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "fscnn_sfjit_create": (_i32, [_vp, _vp] + [_i32] * 7 + [_vp]),
    "fscnn_sfjit_compiled": (_i32, [_vp]),
    "fscnn_sfjit_wait": (_i32, [_vp]),
    "fscnn_sfjit_ptx": (_i64, [_vp, _vp] + [_i32] * 8 + [_vp, _i64]),
    "fscnn_sfjit_launch": (_i32, [_vp, _vp, _i32, _i32, _vp, _i32, _vp]),
    "fscnn_sfjit_info": (_i32, [_vp, _vp, _vp]),
    "fscnn_sfjit_destroy": (None, [_vp]),
    "fscnn_pitch_copy": (_i32, [_vp, _i64, _i32, _i32, _i32, _vp, _i32, _i32, _vp]),
    "fscnn_fp32_probe": (_i32, [_vp, _i32, _i32, _vp]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the C-ABI library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2212_08815_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point; raise FscnnError on failure."""
    fn = getattr(load(), name)
    rc = fn(*args)
    if rc != 0:
        msg = load().fscnn_last_error().decode(errors="replace")
        raise FscnnError(f"{name} failed (status {rc}): {msg}")


def ptr(t) -> int | None:
    """Device pointer of a tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream() -> int:
    """The current torch CUDA stream as a cudaStream_t handle."""
    return torch.cuda.current_stream().cuda_stream


def launch_count() -> int:
    return int(load().fscnn_launch_count())


def reset_launch_count() -> None:
    load().fscnn_reset_launch_count()
