"""Seeded synthetic instance generator for the spatial hypercube queueing model.

This module is shared by the CPU oracle (``oracle/``), the tests and ``bench.py``.
It holds NONE of the method's arithmetic: it only draws the problem data
(per-atom arrival rates lambda_j, per-unit service rates nu_i and the
distance-ordered preference lists zeta_j) that the paper's problem statement
takes as input ("Model", Table 1 notation).  No transition
rate, no probability and no measure is computed here.

Recipe (SURVEY.md §8(d) "Generator"; numpy ``default_rng(seed)``, draws in this
exact order):
  1. unit coordinates U = rng.random((N, 2)); clustered variant: cluster centres
     C = rng.random((4, 2)), U[i] = clip(C[i % 4] + sigma * z_i, 0, 1) with
     z = rng.standard_normal((N, 2)) (round-robin clusters, sigma = 0.1);
  2. atom coordinates X = rng.random((J, 2));
  3. demand fractions f = rng.dirichlet(ones(J));
  4. service rates nu = rng.uniform(lo, hi, N);
  5. total arrival rate Lambda = rho * sum(nu), lambda_j = Lambda * f_j;
  6. pref[j] = units sorted by (Euclidean distance |X_j - U_i|, unit index i)
     (ties by unit index), truncated to L entries and
     padded with -1.

The five BASELINE.json configs stand in for the paper's St. Paul / Greenville
EMS data, which are not available here.
"""
from __future__ import annotations

import dataclasses
import hashlib
from typing import Optional

import numpy as np

__all__ = [
    "Instance",
    "CONFIGS",
    "generate",
    "config_instance",
    "homogeneous_copy",
    "ordered_hunt",
    "from_arrays",
]


@dataclasses.dataclass(frozen=True)
class Instance:
    """One problem instance in ABI form.

    lam   : float64 [J]   per-atom arrival rates lambda_j = Lambda * f_j
    mu    : float64 [N]   per-unit service rates nu_i (the paper's nu_i)
    pref  : int32  [J, N] 0-based unit ids in preference order, -1 padded
    """

    name: str
    N: int
    J: int
    lam: np.ndarray
    mu: np.ndarray
    pref: np.ndarray
    rho: float
    seed: int

    @property
    def states(self) -> int:
        return 1 << self.N

    def sha256(self) -> str:
        h = hashlib.sha256()
        h.update(np.int64([self.N, self.J]).tobytes())
        h.update(np.ascontiguousarray(self.lam, dtype=np.float64).tobytes())
        h.update(np.ascontiguousarray(self.mu, dtype=np.float64).tobytes())
        h.update(np.ascontiguousarray(self.pref, dtype=np.int32).tobytes())
        return h.hexdigest()

    def describe(self) -> dict:
        return {
            "name": self.name,
            "N": self.N,
            "J": self.J,
            "rho": self.rho,
            "seed": self.seed,
            "truncated": bool((self.pref < 0).any()),
            "sha256": self.sha256()[:16],
        }


# BASELINE.json "configs" (N, J, placement, mu range, rho, list length, seed).
CONFIGS = {
    1: dict(N=10, J=20, clustered=False, mu_lo=0.5, mu_hi=1.5, rho=0.5, L=None, seed=1),
    2: dict(N=18, J=100, clustered=False, mu_lo=0.5, mu_hi=1.5, rho=0.6, L=None, seed=2),
    3: dict(N=24, J=200, clustered=True, mu_lo=0.3, mu_hi=2.0, rho=0.7, L=None, seed=3),
    4: dict(N=28, J=500, clustered=False, mu_lo=0.5, mu_hi=1.5, rho=0.8, L=8, seed=4),
    5: dict(N=31, J=1000, clustered=False, mu_lo=0.5, mu_hi=1.5, rho=0.6, L=None, seed=5),
}
CONFIG5_RHOS = (0.3, 0.6, 0.9)


def generate(
    N: int,
    J: int,
    *,
    seed: int,
    rho: float,
    mu_lo: float = 0.5,
    mu_hi: float = 1.5,
    clustered: bool = False,
    L: Optional[int] = None,
    sigma: float = 0.1,
    name: str = "synthetic",
) -> Instance:
    """Draw one EMS-shaped instance following the recipe in the module docstring."""
    if N < 1 or J < 1:
        raise ValueError("N and J must be >= 1")
    rng = np.random.default_rng(seed)
    if clustered:
        centres = rng.random((4, 2))
        z = rng.standard_normal((N, 2))
        U = np.clip(centres[np.arange(N) % 4] + sigma * z, 0.0, 1.0)
    else:
        U = rng.random((N, 2))
    X = rng.random((J, 2))
    f = rng.dirichlet(np.ones(J))
    nu = rng.uniform(mu_lo, mu_hi, N)
    total = rho * float(nu.sum())
    lam = total * f
    pref = _distance_prefs(U, X, L)
    return Instance(name, N, J, lam.astype(np.float64), nu.astype(np.float64), pref, float(rho), int(seed))


def _distance_prefs(U: np.ndarray, X: np.ndarray, L: Optional[int]) -> np.ndarray:
    N = U.shape[0]
    J = X.shape[0]
    d = np.sqrt(((X[:, None, :] - U[None, :, :]) ** 2).sum(axis=2))  # [J, N]
    pref = np.full((J, N), -1, dtype=np.int32)
    units = np.arange(N)
    keep = N if L is None else min(L, N)
    for j in range(J):
        order = np.lexsort((units, d[j]))  # primary: distance, secondary: unit index
        pref[j, :keep] = order[:keep]
    return pref


def config_instance(cfg: int, *, rho: Optional[float] = None, N: Optional[int] = None,
                    J: Optional[int] = None) -> Instance:
    """BASELINE.json config ``cfg`` (1..5).  ``N``/``J`` override gives the
    shrunk variants of the same generator used by the small-N tests."""
    c = dict(CONFIGS[cfg])
    if rho is not None:
        c["rho"] = rho
    if N is not None:
        c["N"] = N
    if J is not None:
        c["J"] = J
    name = f"cfg{cfg}" if (N is None and J is None) else f"cfg{cfg}-N{c['N']}J{c['J']}"
    return generate(c["N"], c["J"], seed=c["seed"], rho=c["rho"], mu_lo=c["mu_lo"], mu_hi=c["mu_hi"],
                    clustered=c["clustered"], L=c["L"], name=name)


def homogeneous_copy(inst: Instance) -> Instance:
    """same geometry, lists and demand fractions;
    nu_i = 1 and Lambda = rho * N."""
    total = inst.rho * inst.N
    f = inst.lam / inst.lam.sum()
    return Instance(inst.name + "-homog", inst.N, inst.J, total * f, np.ones(inst.N), inst.pref.copy(),
                    inst.rho, inst.seed)


def ordered_hunt(N: int, rho: float, *, J: int = 1, order: Optional[np.ndarray] = None) -> Instance:
    """Every atom uses the same full list (an 'ordered hunt'), nu_i = 1,
    Lambda = rho * N split evenly over J atoms."""
    if order is None:
        order = np.arange(N, dtype=np.int32)
    total = rho * N
    lam = np.full(J, total / J)
    pref = np.tile(np.asarray(order, dtype=np.int32), (J, 1))
    return Instance(f"hunt-N{N}", N, J, lam, np.ones(N), pref, float(rho), 0)


def from_arrays(lam, mu, pref, *, name: str = "custom", rho: float = float("nan")) -> Instance:
    lam = np.asarray(lam, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    pref = np.asarray(pref, dtype=np.int32)
    if pref.ndim != 2:
        raise ValueError("pref must be [J][N]")
    J, N = pref.shape
    return Instance(name, N, J, lam, mu, pref, rho, 0)
