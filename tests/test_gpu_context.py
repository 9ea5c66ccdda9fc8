"""Context memory utilities of the C-ABI: the opt-in reserved region (hmx_ctx_reserve) serves the
assemblies' workspaces and streams without changing results, survives a cache release while an
H-matrix lives in it, and goes back to the driver afterwards."""

import numpy as np
import pytest
import torch

import paper_1706_09384_b200 as hmx
from paper_1706_09384_b200 import _lib
from tests._problems import Problem

pytestmark = pytest.mark.gpu


def test_reserved_region_serves_assemblies_bitwise():
    pb = Problem("U8k", 1024)
    x = pb.rhs(3)
    _lib.release_cached(0)
    H0, _ = pb.device_h()
    y0 = hmx.matvec(H0, x)
    r0 = H0.block_info()["rank_after"].copy()
    del H0
    _lib.release_cached(0)
    free0 = torch.cuda.mem_get_info(0)[0]
    t = _lib.reserve(0, 8.0)
    assert t >= 0.0
    free1 = torch.cuda.mem_get_info(0)[0]
    assert free0 - free1 >= 7.9e9
    with pytest.raises(Exception):  # one region per context
        _lib.reserve(0, 1.0)
    H1, _ = pb.device_h()
    # the assembly's workspaces and streams came out of the region: no further device allocation of that size
    assert free1 - torch.cuda.mem_get_info(0)[0] < 0.5e9
    assert np.array_equal(H1.block_info()["rank_after"], r0)
    assert np.array_equal(hmx.matvec(H1, x), y0)
    _lib.release_cached(0)  # H1 lives in the region: it must stay
    assert np.array_equal(hmx.matvec(H1, x), y0)
    H2, _ = pb.device_h()   # a second H next to it
    assert np.array_equal(hmx.matvec(H2, x), y0)
    del H1, H2
    _lib.release_cached(0)  # empty now: handed back
    assert torch.cuda.mem_get_info(0)[0] >= free0 - 0.5e9


def test_requests_beyond_the_region_fall_back():
    pb = Problem("U8k", 1024)
    x = pb.rhs(4)
    _lib.release_cached(0)
    H0, _ = pb.device_h()
    y0 = hmx.matvec(H0, x)
    del H0
    _lib.release_cached(0)
    _lib.reserve(0, 0.05)  # 50 MB: far too small for the workspaces
    H1, _ = pb.device_h()
    assert np.array_equal(hmx.matvec(H1, x), y0)
    del H1
    _lib.release_cached(0)
