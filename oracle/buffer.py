"""Oracle for the waiting-room extension.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares no code with the CUDA
path.  Two independent constructions:

* ``stationary_buffer`` -- the plain definition: the dense generator of the
  queued system on the 2^N hypercube states plus the C waiting states, solved
  by LU.  The queued model: the balance equations of the
  loss system hold for every state except the all-busy one, which also moves
  to "1 call waiting" at rate lambda (arrival) and is entered from it at rate
  sum nu; waiting states c = 1..C form a birth-death chain with birth rate
  lambda (for c < C) and death rate sum nu (Eq. finite_buffer_queue).
  Calls that arrive with C calls waiting are lost.

* ``tail_from_loss`` -- Proposition "Reformulation, Finite Buffer"
   and the Remark on unlimited capacity,
  step by step: the conditional probabilities are the loss system's, the
  layer masses p(n) = G(n) p(0) of the extended birth-death chain with
  G(n) = lambda(0)..lambda(n-1) / (mu(1)..mu(N-1) mu(N)^(n-N+1)) for n > N.
  Reading R16: in the queued system the all-busy state's arrival
  rate is lambda (the call joins the queue), so lambda(N) = lambda and
  lambda(n) = lambda for N < n < N + C; mu(N) = sum nu because p_N(all busy)
  = 1.

* ``measures_buffer`` -- workload, dispatch and loss by enumeration over the
  hypercube states plus the waiting states, with reading R14 for queued calls:
  a waiting call is served by the unit that completes service first, unit i
  with probability nu_i / sum nu (FCFS queue; the paper gives no dispatch
  rule for queued calls).
"""
from __future__ import annotations

import numpy as np

UNLIMITED = -1


def generator_matrix_buffer(lam, mu, pref, C: int) -> np.ndarray:
    """Dense generator of the queued system: index m < 2^N is hypercube state m,
    index 2^N + c - 1 is "c calls waiting" (c = 1..C)."""
    lam = np.asarray(lam, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    pref = np.asarray(pref)
    J, N = pref.shape
    if (pref < 0).any():
        raise ValueError("a waiting room needs full preference lists")
    S = 1 << N
    full = S - 1
    Lam = lam.sum()
    snu = mu.sum()
    Q = np.zeros((S + C, S + C))
    for m in range(S):
        for j in range(J):
            for u in pref[j]:
                if not (m >> int(u)) & 1:
                    Q[m, m | (1 << int(u))] += lam[j]   # first free unit of the list
                    break
        for i in range(N):
            if (m >> i) & 1:
                Q[m, m & ~(1 << i)] += mu[i]
    if C > 0:
        Q[full, S] += Lam                  # all busy -> one call waiting
        Q[S, full] += snu                  # the first completion takes the waiting call
        for c in range(1, C + 1):
            k = S + c - 1
            if c < C:
                Q[k, k + 1] += Lam         # another call waits
            if c > 1:
                Q[k, k - 1] += snu
    for k in range(S + C):
        Q[k, k] = -Q[k].sum()
    return Q


def stationary_buffer(lam, mu, pref, C: int):
    """(pi over the hypercube states, tail[c-1] = P~{c}) by LU of the dense
    generator (one balance row replaced by the normalisation)."""
    Q = generator_matrix_buffer(lam, mu, pref, C)
    n = Q.shape[0]
    A = Q.T.copy()
    A[0, :] = 1.0
    rhs = np.zeros(n)
    rhs[0] = 1.0
    x = np.linalg.solve(A, rhs)
    S = 1 << np.asarray(pref).shape[1]
    return x[:S], x[S:]


def tail_from_loss(pi_loss, Lam: float, mu, C: int):
    """Proposition (finite buffer) / Remark (unlimited): the queued system's
    hypercube pi and tail from the loss system's pi (same p_n(B_m)).

    p(n), n <= N, are the loss system's layer masses up to the common factor
    p(0); G(n) = p_loss(n) / p_loss(0) for n <= N; for n = N + c,
    G(n) = lambda(0)..lambda(n-1) / (mu(1)..mu(N-1) mu(N)^(c+1)) = G(N) (lambda/mu(N))^c
    with lambda(N..n-1) = lambda and mu(N) = sum nu (reading R16)."""
    pi_loss = np.asarray(pi_loss, dtype=np.float64)
    S = pi_loss.size
    N = S.bit_length() - 1
    pc = np.array([bin(m).count("1") for m in range(S)])
    p_loss = np.bincount(pc, weights=pi_loss, minlength=N + 1)
    G = p_loss / p_loss[0]
    muN = float(np.sum(mu))
    if C == UNLIMITED:
        if not Lam < muN:
            raise ValueError("unlimited buffer: lambda < mu(N) required (PAPER.md:296)")
        # Remark: p(0) = [1 + sum_{n<N} G(n) + G(N) / (1 - lambda / mu(N))]^-1
        p0 = 1.0 / (1.0 + G[1:N].sum() + G[N] / (1.0 - Lam / muN))
        ctail = 2000   # geometric tail, truncated where (lambda/mu(N))^c underflows the fp64 sum
        Gt = np.array([G[N] * (Lam / muN) ** c for c in range(1, ctail + 1)])
    else:
        Gt = np.array([G[N] * (Lam / muN) ** c for c in range(1, C + 1)])
        p0 = 1.0 / (1.0 + G[1:].sum() + Gt.sum())
    scale = p0 / p_loss[0]            # P{B_m} = p(n) p_n(B_m) = scale * pi_loss(m)
    return scale * pi_loss, p0 * Gt


def measures_buffer(lam, mu, pref, pi, tail, C: int):
    """(workload[N], dispatch[J][N], loss) of the queued system by enumeration."""
    lam = np.asarray(lam, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    pref = np.asarray(pref)
    J, N = pref.shape
    S = 1 << N
    f = lam / lam.sum()
    tail = np.asarray(tail, dtype=np.float64)
    work = np.zeros(N)
    served = np.zeros((J, N))
    for m in range(S):
        for i in range(N):
            if (m >> i) & 1:
                work[i] += pi[m]
        for j in range(J):
            for u in pref[j]:
                if not (m >> int(u)) & 1:
                    served[j, int(u)] += f[j] * pi[m]
                    break
    work += tail.sum()                         # every unit is busy while calls wait
    if C == 0:                                 # the loss system: a call finding all busy is lost
        loss, p_wait = pi[S - 1], 0.0
    elif C == UNLIMITED:
        loss, p_wait = 0.0, pi[S - 1] + tail.sum()
    else:                                      # lost iff C calls wait; waits iff all busy and room
        loss, p_wait = tail[C - 1], pi[S - 1] + tail.sum() - tail[C - 1]
    served += np.outer(f, mu / mu.sum()) * p_wait
    return work, served / (1.0 - loss), loss
