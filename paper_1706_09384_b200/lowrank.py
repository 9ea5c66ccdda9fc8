"""Low-rank layer of the hmatx API: types (LowRankFactor,
BlockGenerator, ACAConfig) and operations.  The ACA / recompression arithmetic
runs batched on the device inside ``hmatrix.assemble`` (``csrc/aca.cu``,
``csrc/recompress.cu``); the one-block operations below call the same kernels."""

from dataclasses import dataclass

import numpy as np

TRUNC_RULES = {"frobenius": 0, "spectral": 1}
ACA_KERNELS = {"auto": 0, "cuda_core": 1}


@dataclass(frozen=True)
class ACAConfig:
    """eps_aca, max_rank (None = min(d m, d n)), sigma3_floor
    (SPEC.md:337), trunc_rule for recompression (oracle/lowrank.py decision 8)."""

    eps_aca: float = 1e-4
    max_rank: int | None = None
    sigma3_floor: float = 1e-12
    trunc_rule: str = "frobenius"
    mem_budget_gb: float = 0.0
    # device-path options (no reference counterpart): ACA kernel for the wide d = 3 leaves
    # ("auto" = tensor-core DMMA, "cuda_core"), its copy-ring depth (0 = deepest that fits),
    # the seed of the randomized-SVD fallback's Gaussian test matrices, a separate recompression
    # tolerance (0: eps_aca, the reference), and opt-in per-leaf certification: after assembly
    # every admissible leaf is regenerated and the ones with ||A_b - U V^H||_F > eps ||A_b||_F are
    # re-compressed at tighter tolerances until none is (hmatrix.assemble)
    aca_kernel: str = "auto"
    tc_stages: int = 0
    rsvd_seed: int = 0
    eps_recompress: float = 0.0
    certify: bool = False

    def __post_init__(self):
        if not (0.0 < self.eps_aca < 1.0):
            raise ValueError("eps_aca must be in (0, 1)")
        if self.max_rank is not None and self.max_rank < 1:
            raise ValueError("max_rank must be >= 1")
        if self.trunc_rule not in TRUNC_RULES:
            raise ValueError(f"trunc_rule must be one of {sorted(TRUNC_RULES)}")
        if self.aca_kernel not in ACA_KERNELS:
            raise ValueError(f"aca_kernel must be one of {sorted(ACA_KERNELS)}")
        if self.tc_stages not in (0, 2, 3):
            raise ValueError("tc_stages must be 0, 2 or 3")

    def c_struct(self, mem_budget_gb=None):
        """The hmx_aca_cfg of include/hmx.h."""
        c = _lib.HmxAcaCfg()
        c.eps = self.eps_aca
        c.max_rank = self.max_rank or 0
        c.sigma3_floor = self.sigma3_floor
        c.trunc_rule = TRUNC_RULES[self.trunc_rule]
        c.aca_kernel = ACA_KERNELS[self.aca_kernel]
        c.mem_budget_gb = self.mem_budget_gb if mem_budget_gb is None else mem_budget_gb
        c.tc_stages = self.tc_stages
        c.rsvd_seed = int(self.rsvd_seed)
        c.eps_recompress = self.eps_recompress
        return c


@dataclass
class LowRankFactor:
    """block ~= u v^* (SPEC.md:248-253)."""

    u: np.ndarray
    v: np.ndarray

    def __post_init__(self):
        if self.u.shape[1] != self.v.shape[1]:
            raise ValueError("factor column counts differ")

    @property
    def rank(self):
        return self.u.shape[1]

    def dense(self):
        return self.u @ self.v.conj().T


# ---- one-block operations of the reference's lowrank module ----------
#
# aca_partial / aca_vector / recompress run the device kernels of the batched
# assembly on a single block (C-ABI hmx_aca_block / hmx_recompress).  The
# dense-matrix utilities numerical_rank / aca_full / randomized_svd are not on
# the assembly or matvec path; they run on the GPU through torch.linalg.

import ctypes as _C  # noqa: E402

from . import _lib  # noqa: E402
from .errors import FallbackNeeded  # noqa: E402


class BlockGenerator:
    """On-demand entries of the kernel block rows x cols:
    ``block_entry(i, j)`` (d x d), ``row(i)`` (d x d n), ``col(j)`` (d m x d);
    ``m``, ``n`` in points, ``shape`` in scalar entries.  Entries come from the
    device kernel-core (``hmx_eval_block``)."""

    def __init__(self, spec, rows, cols, col_normals=None, self_shift=None):
        self.spec = spec
        self.d = spec.d
        self.X = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 3)
        self.Y = np.ascontiguousarray(cols, dtype=np.float64).reshape(-1, 3)
        self.NY = None if col_normals is None else np.ascontiguousarray(col_normals, dtype=np.float64).reshape(-1, 3)
        if spec.variant == "elasto_t" and self.NY is None:
            raise ValueError("ElastoT requires column normals")
        self.self_shift = self_shift
        self.m, self.n = self.X.shape[0], self.Y.shape[0]

    @property
    def shape(self):
        return (self.d * self.m, self.d * self.n)

    def _eval(self, X, Y, NY):
        from .kernels import _eval

        out = _eval(self.spec.c_kernel(), X, Y, NY, self.self_shift)
        if out is None:
            from .errors import SingularEvaluationError

            raise SingularEvaluationError("coincident points without a self-block rule")
        return out

    def block_entry(self, i, j):
        return self._eval(self.X[i:i + 1], self.Y[j:j + 1], None if self.NY is None else self.NY[j:j + 1])

    def row(self, i):
        return self._eval(self.X[i:i + 1], self.Y, self.NY)

    def col(self, j):
        return self._eval(self.X, self.Y[j:j + 1], None if self.NY is None else self.NY[j:j + 1])

    def dense(self):
        return self._eval(self.X, self.Y, self.NY)


@dataclass
class ACAResult(LowRankFactor):
    """LowRankFactor plus the ACA bookkeeping (a max-rank stop is a
    flagged result, ``converged`` false)."""

    steps: int = 0
    converged: bool = True


def _c_cfg(cfg):
    return cfg.c_struct(mem_budget_gb=0.0)


def _aca_block(gen, cfg, recompress_too, device=0):
    if not isinstance(gen, BlockGenerator):
        raise TypeError("the device ACA takes a kernel BlockGenerator (paper_1706_09384_b200.lowrank)")
    d, m, n = gen.d, gen.m, gen.n
    cap = min(d * m, d * n) if cfg.max_rank is None else min(cfg.max_rank, d * m, d * n)
    cap = max(cap, 1)
    U = np.zeros((d * m, cap), np.complex128)
    V = np.zeros((d * n, cap), np.complex128)
    rank, steps, status = _C.c_int64(), _C.c_int64(), _C.c_int32()
    shift = gen.self_shift
    st = _lib.lib().hmx_aca_block(
        _lib.context(device), _C.byref(gen.spec.c_kernel()), _lib.ptr(gen.X), m, _lib.ptr(gen.Y), n,
        _lib.ptr(gen.NY), 0 if shift is None else 1, 0.0 if shift is None else float(shift),
        _C.byref(_c_cfg(cfg)), 1 if recompress_too else 0, cap, _lib.ptr(U), _lib.ptr(V), _C.byref(rank),
        _C.byref(steps), _C.byref(status))
    if st == 3:  # HMX_EPIVOT: every sigma_3 pivot below the floor
        raise FallbackNeeded(_lib.last_error())
    _lib.check(st, "hmx_aca_block")
    r = int(rank.value)
    return ACAResult(np.ascontiguousarray(U[:, :r]), np.ascontiguousarray(V[:, :r]), steps=int(steps.value),
                     converged=bool(status.value & 1))


def aca_partial(gen, cfg=ACAConfig()):
    """Scalar partially pivoted ACA on the device."""
    if gen.d != 1:
        raise ValueError("aca_partial needs a scalar (d = 1) generator")
    return _aca_block(gen, cfg, False)


def aca_vector(gen, cfg=ACAConfig()):
    """sigma_3-pivoted rank-3 ACA on the device; raises
    FallbackNeeded when every candidate sigma_3 is below the floor."""
    if gen.d != 3:
        raise ValueError("aca_vector needs a d = 3 generator")
    return _aca_block(gen, cfg, False)


def recompress(f, eps, rule="frobenius", device=0):
    """SPEC.md:318-326 on the device: Gram pair, scaled Cholesky, Hermitian
    eigen-decomposition, truncation, U' = U W_U, V' = V W_V."""
    u = np.ascontiguousarray(f.u, dtype=np.complex128)
    v = np.ascontiguousarray(f.v, dtype=np.complex128)
    K = u.shape[1]
    if K == 0:
        return LowRankFactor(u, v)
    uo = np.empty((u.shape[0], K), np.complex128)
    vo = np.empty((v.shape[0], K), np.complex128)
    r = _C.c_int64()
    _lib.check(_lib.lib().hmx_recompress(_lib.context(device), u.shape[0], v.shape[0], K, _lib.ptr(u), _lib.ptr(v),
                                         float(eps), TRUNC_RULES[rule], _C.byref(r), _lib.ptr(uo), _lib.ptr(vo)),
               "hmx_recompress")
    r = int(r.value)
    # row-major with leading dimension r
    uo = uo.reshape(-1)[: u.shape[0] * r].reshape(u.shape[0], r).copy()
    vo = vo.reshape(-1)[: v.shape[0] * r].reshape(v.shape[0], r).copy()
    return LowRankFactor(uo, vo)


def _torch_dev(device=0):
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("CUDA device required")
    from . import _lib

    _lib.release_cached(device)  # cuSOLVER workspaces must not compete with the assembly cache
    return torch, torch.device("cuda", device)


def numerical_rank(a, eps):
    """smallest r with sigma_{r+1} <= eps sigma_1 (2-norm rule)."""
    torch, dev = _torch_dev()
    s = torch.linalg.svdvals(torch.as_tensor(np.asarray(a, dtype=np.complex128), device=dev))
    if s.numel() == 0 or float(s[0]) == 0.0:
        return 0
    return int((s > eps * s[0]).sum())


def aca_full(a, cfg=ACAConfig()):
    """Fully pivoted ACA on an explicit matrix, on the GPU."""
    torch, dev = _torch_dev()
    R = torch.as_tensor(np.array(a, dtype=np.complex128), device=dev)
    m, n = R.shape
    na = float(torch.linalg.norm(R))
    max_rank = min(m, n) if cfg.max_rank is None else min(cfg.max_rank, m, n)
    us, vs = [], []
    converged = True
    while float(torch.linalg.norm(R)) > cfg.eps_aca * na:
        if len(us) >= max_rank:
            converged = False
            break
        k = int(torch.argmax(R.abs()))
        i, j = divmod(k, n)
        p = R[i, j]
        u = R[:, j] / p
        v = R[i, :].conj().clone()
        R = R - torch.outer(u, v.conj())
        us.append(u)
        vs.append(v)
    if not us:
        return ACAResult(np.zeros((m, 0), np.complex128), np.zeros((n, 0), np.complex128), steps=0, converged=True)
    U = torch.stack(us, 1).cpu().numpy()
    V = torch.stack(vs, 1).cpu().numpy()
    return ACAResult(U, V, steps=len(us), converged=converged)


def randomized_svd(a, eps, oversample=10, max_rank=None, seed=0, device=0):
    """SPEC.md:308-316 on the device (hmx_rsvd, csrc/rsvd.cu): Gaussian range finder with
    8 + oversample columns, doubling until ||A - Q Q^H A||_F <= eps ||A||_F; ``a`` is a dense
    matrix or a BlockGenerator (densified on the device).  Returns the un-truncated factors
    U = Q, V = (Q^H A)^H (``recompress`` trims them, as after ACA); ``converged`` is False when
    the column cap min(max_rank, m, n) stopped the doubling (a flagged result)."""
    A = a.dense() if isinstance(a, BlockGenerator) else np.asarray(a, dtype=np.complex128)
    A = np.ascontiguousarray(A, dtype=np.complex128)
    if A.ndim != 2 or A.size == 0:
        raise ValueError("randomized_svd needs a non-empty 2-D block")
    m, n = A.shape
    cap = min(m, n) if max_rank is None else min(int(max_rank), m, n)
    U = np.zeros((m, cap), np.complex128)
    V = np.zeros((n, cap), np.complex128)
    k = _C.c_int64()
    conv = _C.c_int32()
    _lib.check(_lib.lib().hmx_rsvd(_lib.context(device), _lib.ptr(A), m, n, float(eps), int(oversample), cap,
                                   int(seed), _lib.ptr(U), _lib.ptr(V), _C.byref(k), _C.byref(conv)), "hmx_rsvd")
    K = int(k.value)
    U = U.reshape(-1)[: m * K].reshape(m, K).copy()
    V = V.reshape(-1)[: n * K].reshape(n, K).copy()
    return ACAResult(U, V, steps=0, converged=bool(conv.value))
