"""Snapshot format: bit-exact round trip, version and
checksum errors (errors.py:23-32)."""

import struct

import numpy as np
import pytest

import paper_1706_09384_b200 as hmx
from paper_1706_09384_b200 import snapfile as S

from ._problems import Problem


def test_wrong_magic_and_version(tmp_path):
    p = tmp_path / "bad.hmx"
    p.write_bytes(b"NOTASNAP" + b"\0" * 64)
    with pytest.raises(hmx.SnapshotVersionError):
        S.load(str(p))
    p.write_bytes(S.MAGIC + struct.pack("<IQ", S.VERSION + 1, 2) + b"{}" + b"\0" * 32)
    with pytest.raises(hmx.SnapshotVersionError):
        S.load(str(p))
    assert issubclass(hmx.SnapshotVersionError, hmx.SnapshotError)


def test_corrupt_payload(tmp_path):
    import hashlib

    body = S.MAGIC + struct.pack("<IQ", S.VERSION, 2) + b"{}" + b"payload"
    p = tmp_path / "c.hmx"
    p.write_bytes(body + hashlib.sha256(body).digest())
    flipped = bytearray(p.read_bytes())
    flipped[-40] ^= 1  # one bit of the payload
    p.write_bytes(bytes(flipped))
    with pytest.raises(hmx.SnapshotCorruptError):
        S.load(str(p))


@pytest.mark.gpu
@pytest.mark.parametrize("tag,n", [("H4k", 2048), ("U8k", 1024), ("T65k", 1024)])
def test_round_trip_bitwise(tmp_path, tag, n):
    pb = Problem(tag, n)
    H, _ = pb.device_h()
    path = str(tmp_path / f"{tag}.hmx")
    hmx.snapshot("save", path, H)
    H2 = hmx.snapshot("load", path)
    x = pb.rhs(3)
    np.testing.assert_array_equal(hmx.matvec(H2, x), hmx.matvec(H, x))  # bitwise
    for b in (0, len(pb.table) // 2, len(pb.table) - 1):
        p1, p2 = H.block(b), H2.block(b)
        if pb.table[b, 0] == 0:
            np.testing.assert_array_equal(p1, p2)
        else:
            np.testing.assert_array_equal(p1.u, p2.u)
            np.testing.assert_array_equal(p1.v, p2.v)
    assert H2.stats()["n_stored"] == H.stats()["n_stored"]
    # the assembly record and the block tree travel with the snapshot
    i1, i2 = H.block_info(), H2.block_info()
    for k in ("steps", "rank_before", "rank_after", "flags"):
        np.testing.assert_array_equal(i1[k], i2[k])
    assert hmx.storage_report(H2) == hmx.storage_report(H)
    np.testing.assert_array_equal(H2.block_tree.table, H.block_tree.table)
    # the loaded H carries its kernel: the estimator regenerates the same leaves
    e1, _ = hmx.block_errors(H, pb.spec, pb.cloud)
    e2, _ = hmx.block_errors(H2, H2.spec, pb.cloud)
    np.testing.assert_array_equal(e1, e2)
    # reused for a new right-hand side: same GMRES result as in-process
    r1 = hmx.solve_gmres(H, pb.rhs(4), hmx.GmresConfig(tol=1e-6))
    r2 = hmx.solve_gmres(H2, pb.rhs(4), hmx.GmresConfig(tol=1e-6))
    assert r1.iters == r2.iters
    np.testing.assert_array_equal(r1.x, r2.x)


@pytest.mark.gpu
def test_loaded_h_factorises(tmp_path):
    """hlu needs the block tree: a snapshot carries it (version 2)."""
    pb = Problem("H4k", 1024)
    H, _ = pb.device_h()
    path = str(tmp_path / "h.hmx")
    hmx.snapshot("save", path, H)
    H2 = hmx.snapshot("load", path)
    f1 = hmx.hlu(H, 1e-6)
    f2 = hmx.hlu(H2, 1e-6)
    b = pb.rhs(5)
    np.testing.assert_array_equal(hmx.triangular_solve(f1, b), hmx.triangular_solve(f2, b))
