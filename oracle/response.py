"""Oracle for the response-time measures.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Follows the definitions state by
state: for every atom j and state m the dispatched unit is the first free unit of
zeta_j (m in S_ij); m belongs to E(j, T) iff that unit's tau_ij < T (strict).
    MRT   = sum_ij rho_ij tau_ij,  rho_ij = sum_{m in S_ij} f_j P{B_m} / (1 - Pi)
    F(T)  = sum_j sum_{m in E(j,T)} f_j P{B_m} / (1 - Pi)
    MRT_j = sum_i rho_ij tau_ij / sum_i rho_ij
    F_j(T)= sum_{m in E(j,T)} P{B_m} / (1 - Pi)
with 1 - Pi the served fraction (reading R10: Pi = sum_j f_j P(list j all busy), the
paper's P{all busy} for full lists).
"""
from __future__ import annotations

import numpy as np


def response_times(lam, mu, pref, pi, tau, T):
    lam = np.asarray(lam, dtype=np.float64)
    pref = np.asarray(pref)
    tau = np.asarray(tau, dtype=np.float64)
    J, N = pref.shape
    f = lam / lam.sum()
    S = 1 << N
    rho = np.zeros((J, N))      # sum over S_ij of f_j P{B_m}
    E = np.zeros(J)             # sum over E(j, T) of P{B_m}
    lost = 0.0
    for m in range(S):
        for j in range(J):
            unit = -1
            for u in pref[j]:
                if u < 0:
                    break
                if not (m >> int(u)) & 1:
                    unit = int(u)
                    break
            if unit < 0:
                lost += f[j] * pi[m]
                continue
            rho[j, unit] += f[j] * pi[m]
            if tau[j, unit] < T:
                E[j] += pi[m]
    served = 1.0 - lost
    rho /= served
    mrt = float((rho * tau).sum())
    frac = float((f * E).sum() / served)
    rs = rho.sum(axis=1)
    mrt_j = np.where(rs > 0, (rho * tau).sum(axis=1) / np.where(rs > 0, rs, 1.0), 0.0)
    frac_j = np.where(f > 0, E / served, 0.0)
    return mrt, frac, mrt_j, frac_j
