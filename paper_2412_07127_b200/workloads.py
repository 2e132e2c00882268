"""The BASELINE.json systems as seeded synthetic inputs.

configs[0]  3-D 7-point Poisson, 32^3, uniform[-1,1] RHS, GNN seed 0
configs[1]  Q1 elasticity, 40^3 elements, lognormal(0,1) moduli
configs[2]  Q1 elasticity, 118^3 elements (5.01M dofs after clamping)
configs[3]  Q1 elasticity, 149^3 elements (10.06M dofs), lognormal(0,1.5)
configs[4]  7-point FV diffusion, 256^3, k = 10^u, u ~ U[-3,3]

Inputs are drawn from the reference's counter RNG (rng.hpp): element moduli
and the RHS from derive_seed(seed, tag) streams; GNN weights from
GnnModel::init(gnn_seed) (gnn.cpp:96). The oracle side of the tests builds
the same inputs through oracle/ from the same seeds.
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

TAG_MODULI = 0x4D4F44  # "MOD"
TAG_RHS = 0x524853  # "RHS"


@dataclass(frozen=True)
class Workload:
    name: str
    family: str  # poisson | diffusion | elasticity
    m: int
    seed: int
    gnn_seed: int
    rel_tol: float = 1e-8
    max_iters: int = -1
    dim: int = 3
    variable: bool = False
    log10_lo: float = -1.0
    log10_hi: float = 1.0
    sigma: float = 1.0
    nu: float = 0.3
    rhs: str = "normal"  # normal | uniform

    def scaled(self, m: int) -> "Workload":
        return replace(self, m=m, name=f"{self.name}@m{m}")

    @property
    def n(self) -> int:
        if self.family == "elasticity":
            return 3 * (self.m + 1) ** 2 * self.m
        return self.m ** self.dim


CONFIGS = [
    Workload("poisson3d_7pt_32", "poisson", 32, seed=0, gnn_seed=0, max_iters=1000, rhs="uniform"),
    Workload("elasticity_q1_40", "elasticity", 40, seed=1, gnn_seed=1),
    Workload("elasticity_q1_118", "elasticity", 118, seed=2, gnn_seed=1),
    Workload("elasticity_q1_149", "elasticity", 149, seed=3, gnn_seed=1, sigma=1.5),
    Workload("diffusion_fv_256", "diffusion", 256, seed=4, gnn_seed=1, max_iters=5000, rhs="uniform",
             variable=True, log10_lo=-3.0, log10_hi=3.0),
]


def moduli(w: Workload, field_lognormal, derive_seed) -> np.ndarray:
    return field_lognormal(w.m ** 3, derive_seed(w.seed, TAG_MODULI), w.sigma)


def rhs(w: Workload, n: int, field_normal, field_uniform_pm1, derive_seed) -> np.ndarray:
    s = derive_seed(w.seed, TAG_RHS)
    return field_normal(n, s) if w.rhs == "normal" else field_uniform_pm1(n, s)


def build(w: Workload):
    """(Matrix on the device, host RHS, Model) for the product path."""
    from . import Matrix, Model, derive_seed, field_lognormal, field_normal, field_uniform_pm1

    if w.family == "elasticity":
        a = Matrix.gen_elasticity(w.m, moduli(w, field_lognormal, derive_seed), w.nu)
    elif w.family == "diffusion" or w.variable:
        a = Matrix.gen_diffusion(w.dim, w.m, w.log10_lo, w.log10_hi, w.seed)
    else:
        a = Matrix.gen_poisson(w.dim, w.m)
    b = rhs(w, a.n, field_normal, field_uniform_pm1, derive_seed)
    return a, b, Model.init(w.gnn_seed)


def build_oracle(w: Workload):
    """The same system through the CPU oracle (test infrastructure)."""
    from oracle import oracle as O

    if w.family == "elasticity":
        a = O.gen_elasticity(w.m, moduli(w, O.lognormal_field, O.derive_seed), w.nu)
    elif w.family == "diffusion" or w.variable:
        a = O.gen_poisson(w.dim, w.m, O.cell_coeffs(w.m ** w.dim, w.seed, w.log10_lo, w.log10_hi))
    else:
        a = O.gen_poisson(w.dim, w.m)
    b = rhs(w, a.n, O.normal_field, O.uniform_pm1_field, O.derive_seed)
    return a, b, O.gnn_init(w.gnn_seed)


def by_name(name: str) -> Optional[Workload]:
    for w in CONFIGS:
        if w.name == name:
            return w
    return None
