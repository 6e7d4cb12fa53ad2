"""ctypes binding of the C-ABI in include/hyena_b200.h (libhyena_b200.so, built in-tree).

There is no fallback: if the shared library is missing or a CUDA device is not
available, every compute entry point raises. The library is loaded from this
package directory only (never from site-packages or a JIT cache).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhyena_b200.so")

MIXER_HISTORY = 144  # HY_MIXER_HISTORY

HY_OK, HY_ERR_INVALID, HY_ERR_INELIGIBLE, HY_ERR_UNSUPPORTED, HY_ERR_CUDA = range(5)
HY_F32, HY_BF16, HY_F64 = 0, 1, 2

_P = ctypes.c_void_p
_I = ctypes.c_int
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); must match include/hyena_b200.h
SIGNATURES = {
    "hy_version": (_I, []),
    "hy_last_error": (ctypes.c_char_p, []),
    "hy_causal_conv_fwd": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "hy_gated_conv_fwd": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "hy_two_stage_fwd": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "hy_hyena_mixer_fwd": (_I, [_P, _P, _P, _P, _P, _I, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "hy_feat_pack_size": (_SZ, [_I, _I]),
    "hy_feat_pack": (_I, [_P, _I, _I, _P, _P]),
    "hy_se_mixer_fwd": (_I, [_P, _P, _P, _I, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "hy_fft_conv_workspace_size": (_SZ, [_I, _I, _I, _I, _I, _I]),
    "hy_fft_conv_fwd": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _SZ, _P]),
    "hy_fft_spectrum_size": (_SZ, [_I, _I, _I]),
    "hy_fft_spectrum": (_I, [_P, _I, _I, _I, _P, _P, _SZ, _P]),
    "hy_fft_conv_spec_fwd": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _SZ, _P]),
    "hy_halo_correction_fwd": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "hy_debug_two_stage_trace": (_I, [_P, _I]),
    "hy_li_mixer_fwd": (_I, [_P, _P, _P, _P, _I, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "hy_li_conv_fwd": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "hy_li_conv_segmented_fwd": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _I, ctypes.c_longlong, _I, _P]),
    "hy_causal_conv_bwd_workspace_size": (_SZ, [_I, _I, _I, _I, _I]),
    "hy_causal_conv_bwd": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _SZ, _P]),
    "hy_featurize_fwd": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P]),
    "hy_mixer_bwd_prep": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P]),
    "hy_featurizer_bwd_workspace_size": (_SZ, [_I, _I]),
    "hy_featurizer_bwd": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _SZ, _I, _P]),
    "hy_two_stage_taps_grad_workspace_size": (_SZ, [_I, _I]),
    "hy_two_stage_taps_grad": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _SZ, _P]),
    "hy_toeplitz_taps_reduce": (_I, [_P, _P, _P, _P, _SZ, _I, _I, _I, _I, _P]),
    "hy_li_param_grad_workspace_size": (_SZ, [_I, _I]),
    "hy_li_param_grad": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _SZ, _P]),
    "hy_block_conv_fwd": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "hy_li_scan_fwd": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "hy_li_scan_mixer_fwd": (_I, [_P, _P, _P, _I, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "hy_fft_c2c_workspace_size": (_SZ, [ctypes.c_longlong, ctypes.c_longlong, _I]),
    "hy_fft_c2c": (_I, [_P, _P, ctypes.c_longlong, ctypes.c_longlong, _I, _I, _P, _SZ, _P]),
    "hy_gate_mul": (_I, [_P, _P, _P, ctypes.c_longlong, _I, _P]),
    "hy_split3_cat": (_I, [_P, _P, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong, _P]),
    "hy_qkv_feat_gemm": (_I, [_P, _P, _P, _I, _P, _P, _I, _I, _I, _I, _I, _P]),
}

_lib = None


class HyenaLibError(RuntimeError):
    """The native library is missing or a kernel launch failed."""


def load() -> ctypes.CDLL:
    """Load (once) and return the native library; raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise HyenaLibError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_2503_01868_b200/csrc` (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().hy_last_error().decode(errors="replace")


_LAUNCHES = [0]


def launch_count() -> int:
    """Kernel-launching C-ABI calls that returned HY_OK in this process (bench accounting)."""
    return _LAUNCHES[0]


def check(status: int, what: str) -> None:
    """Map an hy_status to the reference's exception types."""
    if status == HY_OK:
        _LAUNCHES[0] += 1
        return
    msg = f"{what}: {last_error()}"
    if status == HY_ERR_INVALID:
        raise ValueError(msg)
    if status == HY_ERR_INELIGIBLE:
        from .blockconv import TwoStageIneligibleError
        raise TwoStageIneligibleError(msg)
    if status == HY_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise HyenaLibError(msg)
