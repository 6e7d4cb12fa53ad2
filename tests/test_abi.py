"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every
symbol include/hyena_b200.h declares, with matching ctypes signatures. No kernel
is launched (there is no GPU here)."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from paper_2503_01868_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hyena_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return re.findall(r"HY_API\s+[\w\s\*]+?\b(hy_\w+)\s*\(", text)


def test_header_declares_entry_points():
    syms = header_symbols()
    for want in ("hy_causal_conv_fwd", "hy_gated_conv_fwd", "hy_two_stage_fwd", "hy_hyena_mixer_fwd",
                 "hy_fft_conv_fwd", "hy_fft_conv_workspace_size", "hy_halo_correction_fwd", "hy_last_error"):
        assert want in syms


def test_library_exports_every_header_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail(f"{_lib.LIB_PATH} not built (run __graft_entry__.build())")
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert set(header_symbols()) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"


def test_arity_matches_header():
    text = open(HEADER).read()
    for name, (_, args) in _lib.SIGNATURES.items():
        m = re.search(r"HY_API[\w\s\*]+?\b" + name + r"\s*\(([^)]*)\)", text)
        assert m, name
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), name


def test_no_compute_without_gpu_errors_cleanly():
    # host-only call: version and the error string are usable without a device
    lib = _lib.load()
    assert lib.hy_version() >= 100
    assert isinstance(lib.hy_last_error(), (bytes, type(None)))


def test_status_mapping():
    from paper_2503_01868_b200 import TwoStageIneligibleError
    with pytest.raises(ValueError):
        _lib.check(_lib.HY_ERR_INVALID, "x")
    with pytest.raises(TwoStageIneligibleError):
        _lib.check(_lib.HY_ERR_INELIGIBLE, "x")
    with pytest.raises(NotImplementedError):
        _lib.check(_lib.HY_ERR_UNSUPPORTED, "x")
    with pytest.raises(_lib.HyenaLibError):
        _lib.check(_lib.HY_ERR_CUDA, "x")


def test_invalid_args_rejected_before_launch():
    # argument validation happens host-side inside the library, no device needed
    lib = _lib.load()
    st = lib.hy_causal_conv_fwd(ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16),
                                1, 6, 8, 3, 4, _lib.HY_F32, None)
    assert st == _lib.HY_ERR_INVALID  # group_size 4 does not divide 6
    assert "group_size" in _lib.last_error()
    st = lib.hy_two_stage_fwd(None, None, ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16), None,
                              1, 4, 1024, 200, 1, _lib.HY_BF16, None)
    assert st == _lib.HY_ERR_INELIGIBLE
