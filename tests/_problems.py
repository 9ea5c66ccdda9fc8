"""Shared problem construction for the tests: the product path
(``paper_1706_09384_b200``) and the oracle get identical inputs."""

import numpy as np

import paper_1706_09384_b200 as hmx
from paper_1706_09384_b200.configs import WORKLOADS


def spec_for(w):
    return w.spec()


def oracle_params(spec):
    """Oracle parameter dict carrying exactly the values the device receives."""
    k = spec.c_kernel()
    if spec.d == 1:
        return {"kappa": k.kappa}
    return {"kp": k.kp, "ks": k.ks, "lam": k.lam, "mu": k.mu, "scale": k.scale}


class Problem:
    def __init__(self, tag, n_points=None):
        base = WORKLOADS[tag]
        w = base if n_points in (None, base.n_points) else base.with_points(n_points)
        self.w = w
        self.kind = w.kind
        self.d = w.d
        self.N = w.n_points
        self.cloud = hmx.make_geometry("sphere", w.n_points, 1.0, d=w.d)
        self.ct = hmx.build_cluster_tree(self.cloud, w.n_leaf)
        self.bt = hmx.build_block_tree(self.ct, self.ct, w.eta)
        self.spec = spec_for(w)
        self.params = oracle_params(self.spec)
        self.table = self.bt.leaf_table
        self.pts = self.ct.points_tree
        self.nrm = self.ct.normals_tree if w.kind == "T" else None

    def rhs(self, seed=0):
        rng = np.random.default_rng(seed)
        n = self.d * self.N
        return rng.standard_normal(n) + 1j * rng.standard_normal(n)

    def oracle_h(self, workers=8, rule="frobenius"):
        from oracle import hmatrix as OH

        return OH.assemble(self.kind, self.params, self.pts, self.nrm, self.ct.permutation, self.table,
                           self.w.eps, self_shift=float(self.N), workers=workers, rule=rule,
                           n_leaf=self.w.n_leaf)

    def device_h(self, **cfg):
        return hmx.assemble(self.spec, self.cloud, self.ct, self.bt, hmx.ACAConfig(eps_aca=self.w.eps, **cfg))
