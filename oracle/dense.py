"""Dense brute-force oracle: the plain definition of the stationary distribution.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Independent of both the C
oracle (oracle/hq_oracle.c) and the CUDA path: the generator matrix is built
here from the model definition with its own code.

The model: states B_m in {0,1}^N, bit u of m set iff unit u
is busy (reading C5).  An arrival at atom j (rate lambda_j = lambda f_j) is
served by the first free unit of its preference list zeta_j (PAPER.md:76,
PAPER.md:175); if every unit of the list is busy the call is lost (C = 0,
PAPER.md:78).  A busy unit i completes service at rate nu_i
(PAPER.md:169).  pi solves pi Q = 0 with sum(pi) = 1 (Eqs. balance_eq_heter
and sumto1_intial); one balance row is replaced by the
normalisation ("eliminating one balance equation as
redundant").
"""
from __future__ import annotations

import numpy as np


def generator_matrix(lam, mu, pref) -> np.ndarray:
    lam = np.asarray(lam, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    pref = np.asarray(pref)
    J, N = pref.shape
    S = 1 << N
    Q = np.zeros((S, S))
    for m in range(S):
        for j in range(J):
            for u in pref[j]:
                if u < 0:
                    break          # truncated list exhausted: call lost
                if not (m >> int(u)) & 1:
                    Q[m, m | (1 << int(u))] += lam[j]   # first free unit serves the call
                    break
        for i in range(N):
            if (m >> i) & 1:
                Q[m, m & ~(1 << i)] += mu[i]            # service completion of unit i
        Q[m, m] = -Q[m].sum()
    return Q


def stationary(lam, mu, pref) -> np.ndarray:
    """pi with pi Q = 0, sum(pi) = 1, by LU (numpy.linalg.solve)."""
    Q = generator_matrix(lam, mu, pref)
    S = Q.shape[0]
    A = Q.T.copy()
    A[0, :] = 1.0          # replace the balance equation of state 0 by sum(pi) = 1
    rhs = np.zeros(S)
    rhs[0] = 1.0
    return np.linalg.solve(A, rhs)


def measures(lam, mu, pref, pi):
    """Workload rho_i, dispatch rho_ij over the sets S_ij
     and the lost fraction, by enumeration."""
    lam = np.asarray(lam, dtype=np.float64)
    pref = np.asarray(pref)
    J, N = pref.shape
    S = 1 << N
    f = lam / lam.sum()
    work = np.zeros(N)
    disp = np.zeros((J, N))
    loss = 0.0
    for m in range(S):
        for i in range(N):
            if (m >> i) & 1:
                work[i] += pi[m]
        for j in range(J):
            served = False
            for u in pref[j]:
                if u < 0:
                    break
                if not (m >> int(u)) & 1:
                    disp[j, int(u)] += f[j] * pi[m]
                    served = True
                    break
            if not served:
                loss += f[j] * pi[m]
    return work, disp / (1.0 - loss), loss
