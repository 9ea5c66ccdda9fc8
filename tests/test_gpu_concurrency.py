"""Concurrent matvec on one assembled H ("An assembled HMatrix is
immutable and safe for concurrent matvec") and the device-resident GMRES.

* two CUDA streams x 50 matvecs interleaved on one H: every result bitwise
  equal to the serial one (per-stream workspaces, ``hmx_matvec_on``);
* host threads on the context stream and on private streams: bitwise equal;
* GMRES: iterations, history and solution against the oracle GMRES
  (oracle/solve.py) on the same device matvec, with restarts forced, the
  iteration cap and b = 0.
"""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_1706_09384_b200 as hmx
from oracle import solve as OS
from tests._problems import Problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def prob():
    pb = Problem("U8k", 2048)
    H, _ = pb.device_h()
    return pb, H


def test_two_streams_bitwise(prob):
    import torch

    pb, H = prob
    xs = [torch.from_numpy(pb.rhs(s)).cuda() for s in range(50)]
    ref = [hmx.matvec(H, x).clone() for x in xs]
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    o1, o2 = [None] * 50, [None] * 50
    for i in range(50):  # interleaved launches: both streams busy at once
        with torch.cuda.stream(s1):
            o1[i] = hmx.matvec(H, xs[i])
        with torch.cuda.stream(s2):
            o2[i] = hmx.matvec(H, xs[49 - i])
    torch.cuda.synchronize()
    for i in range(50):
        assert torch.equal(o1[i], ref[i])
        assert torch.equal(o2[i], ref[49 - i])


def test_threads_bitwise(prob):
    import torch

    pb, H = prob
    xs = [pb.rhs(100 + s) for s in range(24)]
    ref = [hmx.matvec(H, x) for x in xs]
    with ThreadPoolExecutor(6) as ex:   # all on the context stream: serialised by the workspace lock
        got = list(ex.map(lambda x: hmx.matvec(H, x), xs))
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)
    streams = [torch.cuda.Stream() for _ in range(3)]

    def on_stream(i):
        return hmx.matvec(H, xs[i], stream=streams[i % 3].cuda_stream)

    with ThreadPoolExecutor(6) as ex:   # private streams: concurrent on the device
        got = list(ex.map(on_stream, range(len(xs))))
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("restart", [50, 3])
def test_device_gmres_vs_oracle(prob, restart):
    pb, H = prob
    b = pb.rhs(7)
    tol = 1e-8 if restart == 3 else 1e-6
    res = hmx.solve_gmres(H, b, hmx.GmresConfig(tol=tol, restart=restart, max_iters=300))
    xo, it_o, hist_o, conv_o = OS.gmres(lambda v: hmx.matvec(H, v), b, tol, restart, 300)
    assert res.converged and conv_o
    assert abs(res.iters - it_o) <= 1
    k = min(len(res.history), len(hist_o))
    np.testing.assert_allclose(res.history[:k], hist_o[:k], rtol=1e-6)
    assert np.linalg.norm(res.x - xo) <= 1e-6 * np.linalg.norm(xo)
    r = b - hmx.matvec(H, res.x)
    assert np.linalg.norm(r) <= 1.01 * tol * np.linalg.norm(b)


def test_device_gmres_cap_and_zero(prob):
    pb, H = prob
    b = pb.rhs(8)
    res = hmx.solve_gmres(H, b, hmx.GmresConfig(tol=1e-14, restart=4, max_iters=6))
    xo, it_o, hist_o, conv_o = OS.gmres(lambda v: hmx.matvec(H, v), b, 1e-14, 4, 6)
    assert not res.converged and not conv_o
    assert res.iters == it_o == 6 and len(res.history) == 6
    np.testing.assert_allclose(res.history, hist_o, rtol=1e-6)
    z = hmx.solve_gmres(H, np.zeros_like(b))
    assert z.iters == 0 and z.converged and not np.any(z.x)


def test_device_gmres_deterministic(prob):
    pb, H = prob
    b = pb.rhs(9)
    r1 = hmx.solve_gmres(H, b, hmx.GmresConfig(tol=1e-8, restart=5))
    r2 = hmx.solve_gmres(H, b, hmx.GmresConfig(tol=1e-8, restart=5))
    assert r1.iters == r2.iters
    np.testing.assert_array_equal(r1.x, r2.x)
