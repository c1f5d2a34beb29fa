"""The C-ABI library builds, loads and exports every symbol include/pmx.h declares
(no compute calls: this tier runs without a GPU)."""

import ctypes
import subprocess

import pytest

from paper_2601_12638_b200 import _native as N


def test_header_and_binding_agree():
    declared = set(N.header_symbols())
    assert declared == set(N.SIGNATURES), declared ^ set(N.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = N.load()
    for name in N.header_symbols():
        assert hasattr(lib, name), name
    assert lib.pmx_abi_version() == 3
    assert lib.pmx_conv_backend(2, 0).decode() in ("tcgen05", "simt")


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_path_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2601_12638_b200 import quant

    with pytest.raises(RuntimeError, match="CUDA device"):
        quant.fake_quant([1.0, 2.0], quant.QuantParams(scale=0.5))


def test_observer_key_decoding():
    import numpy as np

    vals = np.array([-3.5, -0.0, 0.0, 1e-30, 7.25, np.inf, -np.inf], np.float32)
    bits = vals.view(np.uint32)
    keys = np.where(bits & 0x80000000, ~bits, bits | 0x80000000).astype(np.uint32)
    np.testing.assert_array_equal(N.decode_keys(keys), vals)
    order = np.argsort(keys, kind="stable")
    assert list(vals[order][[0, -1]]) == [-np.inf, np.inf]
