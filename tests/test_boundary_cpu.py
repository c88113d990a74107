"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/sigkernel.h declares, and reports errors the way the
reference does (InvalidArgument / InvalidState).  No compute calls (no GPU)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "sigkernel.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sk_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2509_10613_b200 import _lib
    if not os.path.exists(_lib.SO_PATH):
        from paper_2509_10613_b200 import build
        build.build()
    return _lib.load(require_device=False)


def test_exports_every_header_symbol(lib):
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/sigkernel.h but not exported"
    from paper_2509_10613_b200 import _lib
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync with the header"


def test_abi_version(lib):
    assert lib.sk_abi_version() == 1


def test_errors_map_to_reference_exceptions(lib):
    from paper_2509_10613_b200 import _lib
    from paper_2509_10613_b200.errors import InvalidArgument
    # L < 2 -> InvalidArgument before any device work (kernel.py:55-56)
    rc = lib.sk_forward_batch(None, None, 1, 1, 5, 2, 0, 0, 0, 1.0, None, None, 0, None)
    assert rc == _lib.SK_INVALID_ARGUMENT
    assert b"at least 2 points" in lib.sk_last_error()
    with pytest.raises(InvalidArgument):
        _lib.check(rc)
    assert issubclass(InvalidArgument, ValueError)
    rc = lib.sk_forward_batch(None, None, 1, 5, 5, 2, -1, 0, 0, 1.0, None, None, 0, None)
    assert rc == _lib.SK_INVALID_ARGUMENT
    rc = lib.sk_forward_batch(None, None, 1, 5, 5, 2, 0, 0, 1, 0.0, None, None, 0, None)
    assert rc == _lib.SK_INVALID_ARGUMENT  # RBF sigma must be > 0
    rc = lib.sk_backward_gram(None, None, 2, 2, 5, 5, 2, 0, 0, 0, 1.0, 0, 2, None, None, None,
                              None, 0, None)
    assert rc == _lib.SK_INVALID_ARGUMENT  # cotangent required
    import ctypes
    dummy = ctypes.c_double(0.0)
    rc = lib.sk_value_and_grad_gram(None, None, 2, 2, 5, 5, 2, 0, 0, 0, 1.0, 0, 2,
                                    ctypes.addressof(dummy), None, None, None, None, 0, None)
    assert rc == _lib.SK_INVALID_ARGUMENT and b"values" in lib.sk_last_error()
    rc = lib.sk_value_and_grad_gram(None, None, 2, 3, 5, 5, 2, 0, 0, 0, 1.0, 0, 2,
                                    ctypes.addressof(dummy), None, None, None, None, 0, None)
    assert rc == _lib.SK_INVALID_ARGUMENT  # symmetric needs n2 == n1


def test_workspace_queries_positive(lib):
    # few short pairs (BASELINE config 1) take the small-pair kernel: no workspace
    assert lib.sk_forward_batch_workspace_bytes(32, 64, 64, 4, 0, 0, 0) == 0
    assert lib.sk_forward_batch_workspace_bytes(32, 128, 128, 4, 0, 0, 0) > 0
    assert lib.sk_forward_gram_workspace_bytes(16, 16, 30, 30, 3, 1, 1, 0, 1) > 0
    assert lib.sk_backward_batch_workspace_bytes(8, 40, 50, 8, 2, 2, 1) > 0
    assert lib.sk_backward_gram_workspace_bytes(8, 8, 40, 40, 16, 0, 0, 0, 1) > 0
    assert lib.sk_solve_delta_workspace_bytes(3, 4, 5, 1, 1) > 0


def test_product_path_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2509_10613_b200 as sk
    x = torch.zeros(2, 5, 3, dtype=torch.float64)
    with pytest.raises((sk.InvalidArgument, sk.NativeUnavailable)):
        sk.sig_kernel(x, x)


def test_no_oracle_on_product_path():
    pkg = os.path.join(ROOT, "paper_2509_10613_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace(
                    "the C oracle", ""), f"{f} references the oracle"
