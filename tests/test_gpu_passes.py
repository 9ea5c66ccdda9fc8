"""ACA capacity overflow: a workspace budget far below the rank model forces
most leaves through rerun passes (2x column capacity each, on the
high-priority rerun stream).  The ACA does not depend on the capacity, so the
steps, ranks and the H-matvec must equal the single-pass assembly's bit for
bit."""

import numpy as np
import pytest

import paper_1706_09384_b200 as hmx
from tests._problems import Problem

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag,n", [("U8k", 2048), ("T65k", 2048), ("H4k", 4096)])
def test_overflow_reruns_match_single_pass(tag, n):
    pb = Problem(tag, n)
    H1, _ = pb.device_h()
    assert H1.stats()["aca_passes"] == 1
    H2, _ = pb.device_h(mem_budget_gb=0.002)
    assert H2.stats()["aca_passes"] >= 2
    b1, b2 = H1.block_info(), H2.block_info()
    for k in ("steps", "rank_before", "rank_after"):
        np.testing.assert_array_equal(b1[k], b2[k])
    x = pb.rhs(2)
    np.testing.assert_array_equal(hmx.matvec(H1, x), hmx.matvec(H2, x))
