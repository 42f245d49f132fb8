"""The C-ABI library (libfgfrft_b200.so) without a GPU: it loads, exports every symbol that
include/fgfrft_b200.h declares, its host-side coefficient / fingerprint code is bit-exact
against the reference's golden vectors, and argument validation raises the reference's
exception types before any device work (errors.hpp:36-62, transform.hpp:43-53)."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import paper_2602_20870_b200 as fg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "fgfrft_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|uint64_t)\s+(fgfrft_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(fg.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(fg.exported_symbols()) == declared


def test_sinc_coeffs_bit_exact_vs_reference_golden():
    data = json.load(open(os.path.join(GOLDEN, "sinc_coeffs.json")))
    for case in data["cases"]:
        c, dc = fg.sinc_coeffs(float.fromhex(case["alpha"]), case["l"])
        assert [float(v).hex() for v in c] == case["c"]
        assert [float(v).hex() for v in dc] == case["dc"]


def test_sinc_rejects_bad_truncation():
    with pytest.raises(fg.ParameterError):
        fg.sinc_coeffs(0.5, 0)


def test_fnv_bit_exact_vs_reference_golden():
    data = json.load(open(os.path.join(GOLDEN, "fnv1a64.json")))
    for case in data["cases"]:
        n = case["n"]
        buf = (np.arange(n, dtype=np.uint64) * 2654435761 % 251).astype(np.uint8)
        assert fg.fnv1a64(buf) == int(case["value"])


def test_cache_parameter_errors_before_device_work():
    f = np.eye(8, dtype=complex)
    with pytest.raises(fg.ParameterError):
        fg.PowerCache(f, 0)
    with pytest.raises(fg.CapacityError):   # transform.hpp:46-53: budget is checked first
        fg.PowerCache(f, 10, 1024)
    with pytest.raises(fg.ParameterError):
        fg.PowerCache(np.zeros((6, 6), dtype=complex), 2, dtype=fg.C64 + 5)


def test_capacity_error_message_matches_reference_text():
    with pytest.raises(fg.CapacityError, match=r"PowerCache: 10 powers of a 64x64 matrix need 655360 bytes"):
        fg.PowerCache(np.eye(64, dtype=complex), 10, 1024)
