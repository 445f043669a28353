"""CPU checks of the drop-in boundary: libnnm.so loads without a GPU and exports
every symbol include/nnm.h declares; compute entry points fail loudly (no CPU
fallback) when no device is present."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from nnm_testutil import ROOT

HEADER = os.path.join(ROOT, "include", "nnm.h")
LIB = os.path.join(ROOT, "paper_1402_3789_b200", "libnnm.so")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(nnm_\w+)\(", src, re.M)))


def test_header_declares_expected_surface():
    from paper_1402_3789_b200._native import EXPORTED

    assert set(declared_symbols()) == set(EXPORTED)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.skip("libnnm.so not built")
    lib = ctypes.CDLL(LIB)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    lib.nnm_abi_version.restype = ctypes.c_int
    assert lib.nnm_abi_version() == 4


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    if not os.path.exists(LIB):
        pytest.skip("libnnm.so not built")
    import paper_1402_3789_b200 as nnm
    from paper_1402_3789_b200._native import NativeError

    with pytest.raises(NativeError, match="no CUDA device"):
        nnm.fit(np.zeros((4, 2)))


def test_validation_errors_before_device():
    import paper_1402_3789_b200 as nnm

    with pytest.raises(nnm.ValidationError):
        nnm.ConstraintSet(kl2=5, kl3=5)
    with pytest.raises(nnm.ValidationError):
        nnm.RunConfig(pairs_per_batch=0)
    with pytest.raises(nnm.ValidationError):
        nnm.Dataset(values=np.array([[np.nan]]))


def test_dataset_finite_check_host_only():
    """nnm_first_nonfinite is host code (no GPU): the Dataset check of model.py:29-76 with the
    reference's message, for NaN / +-inf anywhere, at sizes that use several threads."""
    if not os.path.exists(LIB):
        pytest.skip("libnnm.so not built")
    from paper_1402_3789_b200 import Dataset, ValidationError
    from paper_1402_3789_b200 import _native

    rng = np.random.default_rng(3)
    X = rng.normal(size=(300_001, 7))
    assert _native.first_nonfinite(np.ascontiguousarray(X)) == -1
    Dataset(values=X)
    for flat, bad in ((0, np.nan), (5, np.inf), (X.size // 2 + 3, -np.inf), (X.size - 1, np.nan)):
        Y = X.copy()
        Y.reshape(-1)[flat] = bad
        assert _native.first_nonfinite(Y) == flat
        with pytest.raises(ValidationError, match=f"non-finite feature value in row {flat // 7 + 1}$"):
            Dataset(values=Y)
    Z = X.copy()
    Z[10, 2] = np.nan
    Z[200_000, 1] = np.inf  # the first one wins
    assert _native.first_nonfinite(Z) == 10 * 7 + 2
