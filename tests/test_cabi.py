"""The C-ABI library loads without a GPU and exports every symbol the header declares."""
import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2210_15874_b200 import _native as N


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "qtn_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(qtn_\w+)\s*\(", hdr, re.M))
    assert declared == set(N.EXPORTS)
    lib = N.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.qtn_abi_version() == N.ABI_VERSION


def test_struct_layouts_match_header():
    assert N.BUCKET_DT.itemsize == 64
    assert N.MEMBER_DT.itemsize == 24
    assert ctypes.sizeof(N.ProgramC) == 6 * 4 + 8 * 8 + 8 + 8 + 8   # + inputs_hi, n_in_elems
    assert N.NODE_DT.itemsize == 32


def test_errors_cross_abi_as_codes():
    lib = N.load()
    assert lib.qtn_node_launch(None, None, 0, None) == N.QTN_E_INVALID
    assert b"null program" in lib.qtn_last_error()
    n = ctypes.c_int(-1)
    assert lib.qtn_device_count(ctypes.byref(n)) == 0 and n.value >= 0
    bad = (ctypes.c_int64 * 1)(1)
    assert lib.qtn_permute(0, None, 0, 0, None, 1, bad, None) == N.QTN_E_INVALID


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    import paper_2210_15874_b200 as Q
    tn = Q.TensorNetwork([Q.Tensor((0,), [1, 2]), Q.Tensor((0,), [3, 4])])
    with pytest.raises(N.NativeUnavailable):
        Q.contract_network(tn, [0])
