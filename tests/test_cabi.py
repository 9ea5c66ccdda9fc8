"""The C-ABI library loads and exports every symbol include/hmx.h declares;
host-side entry points validate their arguments (no GPU needed)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1706_09384_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "hmx.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void)\s+(hmx_\w+)\s*\(", text, re.M)))


def test_every_declared_symbol_is_exported_and_bound():
    L = _lib.lib()
    decl = _declared()
    assert len(decl) >= 25
    for name in decl:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"
    assert L.hmx_abi_version() == 3


def test_host_error_paths():
    L = _lib.lib()
    h = C.c_void_p()
    pts = np.zeros((0, 3))
    assert L.hmx_tree_build(_lib.ptr(np.zeros((1, 3))), 0, 4, C.byref(h)) == 1
    assert "empty input" in _lib.last_error()
    assert L.hmx_tree_build(_lib.ptr(np.zeros((4, 3))), 4, 0, C.byref(h)) == 1
    del pts
    with pytest.raises(ValueError):
        _lib.check(1, "x")


def test_struct_layouts_match_header():
    # hmx_kernel: int32 kind, int32 pad, 6 doubles
    assert C.sizeof(_lib.HmxKernel) == 8 + 6 * 8
    assert C.sizeof(_lib.HmxAcaCfg) == 8 + 8 + 8 + 4 + 4 + 8 + 4 + 4 + 8 + 8
    text = open(os.path.join(ROOT, "include", "hmx.h")).read()
    body = re.search(r"typedef struct \{([^{}]*)\} hmx_stats;", text).group(1)
    n_i64 = sum(len(re.findall(r"\w+", l.split("int64_t", 1)[1].split(";")[0]))
                for l in body.splitlines() if l.strip().startswith("int64_t"))
    n_f64 = sum(len(re.findall(r"\w+", l.split("double", 1)[1].split(";")[0]))
                for l in body.splitlines() if l.strip().startswith("double"))
    assert C.sizeof(_lib.HmxStats) == 8 * (n_i64 + n_f64)
