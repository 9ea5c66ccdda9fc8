"""Low-rank types of the hmatx API.  The ACA / recompression
arithmetic itself runs batched on the device inside ``hmatrix.assemble``
(``csrc/aca.cu``, ``csrc/recompress.cu``)."""

from dataclasses import dataclass

import numpy as np

TRUNC_RULES = {"frobenius": 0, "spectral": 1}


@dataclass(frozen=True)
class ACAConfig:
    """eps_aca, max_rank (None = min(d m, d n)), sigma3_floor
    (SPEC.md:337), trunc_rule for recompression (oracle/lowrank.py decision 8)."""

    eps_aca: float = 1e-4
    max_rank: int | None = None
    sigma3_floor: float = 1e-12
    trunc_rule: str = "frobenius"
    mem_budget_gb: float = 0.0

    def __post_init__(self):
        if not (0.0 < self.eps_aca < 1.0):
            raise ValueError("eps_aca must be in (0, 1)")
        if self.max_rank is not None and self.max_rank < 1:
            raise ValueError("max_rank must be >= 1")
        if self.trunc_rule not in TRUNC_RULES:
            raise ValueError(f"trunc_rule must be one of {sorted(TRUNC_RULES)}")


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
