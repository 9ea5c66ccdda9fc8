"""H-matrix snapshots (SPEC.md:563-571 ``snapshot(save|load, path)``; SURVEY
8(f) row 3): a versioned, checksummed binary image of an assembled H-matrix
(or, ``save_lu``, of H-LU factors).

Layout (little endian)::

    b"HMXSNAP\\0" | u32 version | u64 header length | header (JSON)
    | arrays: perm, table (nb x 7: kind, r0, r1, c0, c1, row node, col node),
      steps, rank_before, rank_after, flags
      [+ version 2 with a block tree: the cluster tree (nodes nn x 5, boxes nn x 6)
       and the cloud (points N x 3, normals N x 3 when present)]
    | payload: every leaf in leaves() order -- dense (d m) x (d n), or
      U (d m) x r then V (d n) x r, complex128 row-major
    | SHA-256 of everything before it (32 bytes)

``load`` rebuilds the device H-matrix through ``hmx_hmatrix_load`` with the
same leaf table and ranks, so the streams, the matvec plan and therefore the
matvec output are bitwise identical to the saved H-matrix's; the per-leaf
assembly record (ACA steps, rank before recompression, flags) is restored
through ``hmx_hmatrix_set_block_info`` and, for version 2, the block tree is
rebuilt so ``storage_report`` and ``hlu`` work on a loaded H.  Version 1
files (no tree) still load.  Errors
(``errors.py:23-32``): wrong magic / version -> ``SnapshotVersionError``,
checksum or size mismatch -> ``SnapshotCorruptError``.
"""

import hashlib
import io
import json
import struct

import numpy as np

from .errors import SnapshotCorruptError, SnapshotVersionError
from .hmatrix import HMatrix
from .kernels import KernelSpec, Material

MAGIC = b"HMXSNAP\0"
VERSION = 2
_READS = (1, 2)
_ARRAYS = ("perm", "table", "steps", "rank_before", "rank_after", "flags")
_TREE_ARRAYS = ("nodes", "boxes", "points", "normals")


def _spec_json(spec):
    if spec is None:
        return None
    m = spec.material
    return {"variant": spec.variant, "kappa": spec.kappa,
            "material": None if m is None else {"rho": m.rho, "mu": m.mu, "nu": m.nu, "omega": m.omega}}


def _spec_from(js):
    if js is None:
        return None
    m = js["material"]
    return KernelSpec(js["variant"], js["kappa"], None if m is None else Material(**m))


class _HashWriter:
    def __init__(self, f):
        self.f = f
        self.h = hashlib.sha256()

    def write(self, b):
        b = memoryview(b).cast("B")
        self.h.update(b)
        self.f.write(b)


def save(h, path):
    """Write ``h`` to ``path``."""
    info = h.block_info()
    table = np.asarray(h.table)
    if table.shape[1] < 7:   # no node columns (an imported H without a tree)
        table = np.concatenate([table[:, :5], np.full((len(table), 2), -1, np.int64)], axis=1)
    table = np.ascontiguousarray(table[:, :7], dtype=np.int64)
    perm = np.ascontiguousarray(h.perm, dtype=np.int64)
    arrays = {"perm": perm, "table": table, "steps": info["steps"], "rank_before": info["rank_before"],
              "rank_after": info["rank_after"], "flags": info["flags"]}
    bt = h.block_tree
    tree = None
    if bt is not None and (bt.rows is bt.cols or np.array_equal(bt.rows.permutation, bt.cols.permutation)):
        ct = bt.rows
        tree = {"n_leaf": int(ct.n_leaf), "eta": float(bt.eta), "has_normals": ct.cloud.normals is not None,
                "cloud_d": int(ct.cloud.d)}
        arrays["nodes"] = np.ascontiguousarray(ct.nodes_array, dtype=np.int64)
        arrays["boxes"] = np.ascontiguousarray(ct.boxes_array, dtype=np.float64)
        arrays["points"] = np.ascontiguousarray(ct.cloud.points, dtype=np.float64)
        if ct.cloud.normals is not None:
            arrays["normals"] = np.ascontiguousarray(ct.cloud.normals, dtype=np.float64)
    header = {"d": h.d, "n_points": h.n_points, "n_blocks": len(table), "self_shift": h.self_shift,
              "spec": _spec_json(h.spec), "tree": tree,
              "arrays": {k: {"dtype": str(v.dtype), "shape": list(v.shape)} for k, v in arrays.items()}}
    hb = json.dumps(header, sort_keys=True).encode()
    with open(path, "wb") as f:
        w = _HashWriter(f)
        w.write(MAGIC)
        w.write(struct.pack("<IQ", VERSION, len(hb)))
        w.write(hb)
        for k in _ARRAYS + _TREE_ARRAYS:
            if k in arrays:
                w.write(np.ascontiguousarray(arrays[k]).tobytes())
        for b in range(len(table)):
            p = h.block(b)
            if table[b, 0] == 0:
                w.write(np.ascontiguousarray(p).tobytes())
            else:
                w.write(np.ascontiguousarray(p.u).tobytes())
                w.write(np.ascontiguousarray(p.v).tobytes())
        f.write(w.h.digest())


def load(path, device=0):
    """Read a snapshot written by :func:`save` (an HMatrix) or :func:`save_lu` (LUFactors) back onto
    ``device``."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < len(MAGIC) + 12 + 32 or raw[:len(MAGIC)] != MAGIC:
        raise SnapshotVersionError("not an hmx snapshot")
    version, hlen = struct.unpack_from("<IQ", raw, len(MAGIC))
    if version not in _READS:
        raise SnapshotVersionError(f"snapshot version {version}, this build reads {_READS}")
    body, digest = raw[:-32], raw[-32:]
    if hashlib.sha256(body).digest() != digest:
        raise SnapshotCorruptError("snapshot checksum mismatch")
    buf = io.BytesIO(body)
    buf.seek(len(MAGIC) + 12)
    header = json.loads(buf.read(hlen))
    if header.get("kind") == "lu":
        return _load_lu(header, buf, len(body), device)
    arrays = {}
    for k in _ARRAYS + _TREE_ARRAYS:
        meta = header["arrays"].get(k)
        if meta is None:
            continue
        dt = np.dtype(meta["dtype"])
        n = int(np.prod(meta["shape"])) if meta["shape"] else 1
        raw_k = buf.read(n * dt.itemsize)
        if len(raw_k) != n * dt.itemsize:
            raise SnapshotCorruptError("snapshot payload size mismatch")
        arrays[k] = np.frombuffer(raw_k, dtype=dt).reshape(meta["shape"])
    d, table, ranks = header["d"], arrays["table"], arrays["rank_after"]
    payload = []
    for b in range(len(table)):
        dm, dn = d * int(table[b, 2] - table[b, 1]), d * int(table[b, 4] - table[b, 3])
        if table[b, 0] == 0:
            payload.append(np.frombuffer(buf.read(16 * dm * dn), np.complex128).reshape(dm, dn))
        else:
            r = int(ranks[b])
            u = np.frombuffer(buf.read(16 * dm * r), np.complex128).reshape(dm, r)
            v = np.frombuffer(buf.read(16 * dn * r), np.complex128).reshape(dn, r)
            payload.append((u, v))
    if buf.tell() != len(body):
        raise SnapshotCorruptError("snapshot payload size mismatch")
    H = HMatrix.from_factors(d, header["n_points"], arrays["perm"], table, payload, device=device)
    from . import _lib

    steps = np.ascontiguousarray(arrays["steps"], dtype=np.int64)
    rb = np.ascontiguousarray(arrays["rank_before"], dtype=np.int64)
    fl = np.ascontiguousarray(arrays["flags"], dtype=np.int32)
    _lib.check(_lib.lib().hmx_hmatrix_set_block_info(H.handle, _lib.ptr(steps), _lib.ptr(rb), _lib.ptr(fl)),
               "hmx_hmatrix_set_block_info")
    H.spec = _spec_from(header["spec"])
    H.self_shift = header["self_shift"]
    tree = header.get("tree")
    if tree is not None and table.shape[1] >= 7:
        from .geometry import BlockTree, PointCloud, cluster_tree_from_arrays

        cloud = PointCloud(np.array(arrays["points"]), None if "normals" not in arrays else np.array(arrays["normals"]),
                           d=tree["cloud_d"])
        ct = cluster_tree_from_arrays(cloud, np.array(arrays["perm"]), np.array(arrays["nodes"]),
                                      np.array(arrays["boxes"]), tree["n_leaf"])
        H.block_tree = BlockTree(rows=ct, cols=ct, table=np.ascontiguousarray(table, dtype=np.int64), eta=tree["eta"])
        H.table = H.block_tree.table
    return H


# ---- LU factors ("-> HMatrix or LUFactors") ------------------------------------
# Same envelope (magic, version, JSON header, SHA-256 trailer); header "kind": "lu" carries the
# factor tree's structure, the payload every leaf in tree order: a factored diagonal leaf as
# L, U (m x m) and its row permutation (int64), any other dense leaf as its block, a low-rank leaf
# as U then V -- complex128 row-major.

def _lu_struct(x, leaves):
    from . import hierarchical_lu as HL

    box = [x.r0, x.r1, x.c0, x.c1]
    if isinstance(x, HL.Sub):
        return {"S": box, "rs": x.rs, "cs": x.cs, "ch": [[_lu_struct(c, leaves) for c in row] for row in x.ch]}
    leaves.append(x)
    if isinstance(x, HL.Dense):
        return {"D": box, "f": int(x.factored)}
    return {"R": box, "k": x.rank}


def save_lu(f, path):
    """Write LU factors (``hierarchical_lu.LUFactors``) to ``path``."""
    from . import hierarchical_lu as HL

    leaves = []
    tree = _lu_struct(f.root, leaves)
    perm = np.ascontiguousarray(f.perm, dtype=np.int64)
    header = {"kind": "lu", "d": f.d, "n": f.n, "eps_lu": f.eps_lu, "n_points": len(perm), "tree": tree}
    hb = json.dumps(header, sort_keys=True).encode()
    with open(path, "wb") as fh:
        w = _HashWriter(fh)
        w.write(MAGIC)
        w.write(struct.pack("<IQ", VERSION, len(hb)))
        w.write(hb)
        w.write(perm.tobytes())
        for x in leaves:
            if isinstance(x, HL.Dense):
                mats = [x.L, x.U] if x.factored else [x.a]
                for m in mats:
                    w.write(np.ascontiguousarray(m.cpu().numpy()).tobytes())
                if x.factored:
                    w.write(np.ascontiguousarray(x.pidx.cpu().numpy().astype(np.int64)).tobytes())
            else:
                w.write(np.ascontiguousarray(x.u.cpu().numpy()).tobytes())
                w.write(np.ascontiguousarray(x.v.cpu().numpy()).tobytes())
        fh.write(w.h.digest())


def _load_lu(header, buf, nbody, device):
    import torch

    from . import hierarchical_lu as HL

    dev = torch.device("cuda", device)
    perm = np.frombuffer(buf.read(8 * header["n_points"]), np.int64).copy()

    def arr(shape, dtype=np.complex128):
        n = int(np.prod(shape))
        a = np.frombuffer(buf.read(np.dtype(dtype).itemsize * n), dtype)
        if a.size != n:
            raise SnapshotCorruptError("snapshot payload size mismatch")
        return torch.as_tensor(a.reshape(shape).copy(), device=dev)

    def rec(js):
        if "S" in js:
            r0, r1, c0, c1 = js["S"]
            return HL.Sub(r0, r1, c0, c1, [tuple(q) for q in js["rs"]], [tuple(q) for q in js["cs"]],
                          [[rec(c) for c in row] for row in js["ch"]])
        if "D" in js:
            r0, r1, c0, c1 = js["D"]
            m, n = r1 - r0, c1 - c0
            if js["f"]:
                lo, up = arr((m, m)), arr((m, m))
                return HL.Dense(r0, r1, c0, c1, torch.tril(lo, -1) + up, True, arr((m,), np.int64))
            return HL.Dense(r0, r1, c0, c1, arr((m, n)))
        r0, r1, c0, c1 = js["R"]
        k = js["k"]
        return HL.LowRank(r0, r1, c0, c1, arr((r1 - r0, k)), arr((c1 - c0, k)))

    root = rec(header["tree"])
    if buf.tell() != nbody:
        raise SnapshotCorruptError("snapshot payload size mismatch")
    tree = HL.HTree.from_nodes(root, device)   # the engine copies the leaves into its own pool
    return HL._factors(tree, header["eps_lu"], header["d"], perm, header["n"])


def snapshot(op, path, h=None, device=0):
    """SPEC.md:563 ``snapshot(save|load, path) -> HMatrix or LUFactors``."""
    if op == "save":
        if h is None:
            raise ValueError("snapshot('save', path, h): no H-matrix / LU factors given")
        from .hierarchical_lu import LUFactors

        if isinstance(h, LUFactors):
            save_lu(h, path)
        else:
            save(h, path)
        return h
    if op == "load":
        return load(path, device=device)
    raise ValueError(f"unknown snapshot op {op!r}")
