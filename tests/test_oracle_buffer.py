"""Pins of the waiting-room oracle (oracle/buffer.py) against
closed forms and brute force (-m "not gpu").

* N = 1: the M/M/1/K queue (K = C + 1 places), pi_k proportional to r^k.
* homogeneous service rates: the M/M/N/N+C queue, p(n) = a^n/n! p(0) for n <= N and
  p(N + c) = p(N) (a/N)^c; unlimited: the Erlang-C waiting probability.
* heterogeneous instances: the Proposition (loss-system conditional probabilities +
  the extended birth-death tail, oracle.buffer.tail_from_loss applied to the
  Algorithm-1 oracle) equals the dense LU of the queued generator (brute force).
* measures: flow identities that hold for any stationary distribution of the queued
  system (sum rho_ij = 1, nu_i rho_i = Lambda (1 - loss) sum_j rho_ij, loss = P~{C}).
"""
import math

import numpy as np
import pytest

import hqinst
import oracle
from oracle import buffer, dense

U = buffer.UNLIMITED


def layer_mass(pi, N):
    pc = np.array([bin(m).count("1") for m in range(1 << N)])
    return np.bincount(pc, weights=pi, minlength=N + 1)


@pytest.mark.parametrize("C", [1, 2, 5])
@pytest.mark.parametrize("r", [0.5, 1.0, 1.7])
def test_mm1k_closed_form(C, r):
    lam, mu, pref = np.array([r]), np.array([1.0]), np.array([[0]])
    pi, tail = buffer.stationary_buffer(lam, mu, pref, C)
    K = C + 1
    w = np.array([r ** k for k in range(K + 1)])
    w /= w.sum()
    np.testing.assert_allclose(np.concatenate([pi, tail]), w, rtol=0, atol=1e-15)
    pi2, tail2 = buffer.tail_from_loss(dense.stationary(lam, mu, pref), r, mu, C)
    np.testing.assert_allclose(np.concatenate([pi2, tail2]), w, rtol=0, atol=1e-15)


@pytest.mark.parametrize("C", [1, 4, 12])
@pytest.mark.parametrize("rho", [0.4, 0.9, 1.3])
def test_homogeneous_mmnc_closed_form(C, rho):
    inst = hqinst.homogeneous_copy(hqinst.generate(4, 6, seed=11, rho=0.5))
    N = inst.N
    a = rho * N
    lam = inst.lam * (a / inst.lam.sum())
    pi, tail = buffer.stationary_buffer(lam, inst.mu, inst.pref, C)
    w = [a ** n / math.factorial(n) for n in range(N + 1)]
    w += [w[N] * (a / N) ** c for c in range(1, C + 1)]
    w = np.array(w) / sum(w)
    np.testing.assert_allclose(layer_mass(pi, N), w[: N + 1], rtol=0, atol=1e-14)
    np.testing.assert_allclose(tail, w[N + 1:], rtol=0, atol=1e-14)


@pytest.mark.parametrize("N", [2, 3, 5])
@pytest.mark.parametrize("rho", [0.3, 0.8])
def test_unlimited_erlang_c(N, rho):
    a = rho * N
    inst = hqinst.homogeneous_copy(hqinst.generate(N, 4, seed=5, rho=0.5))
    lam = inst.lam * (a / inst.lam.sum())
    pi_loss = oracle.solve(hqinst.from_arrays(lam, inst.mu, inst.pref), tol=1e-15)["pi"]
    pi, tail = buffer.tail_from_loss(pi_loss, a, inst.mu, U)
    # Erlang C: P(wait) = (a^N/N! N/(N-a)) / (sum_{k<N} a^k/k! + a^N/N! N/(N-a))
    top = a ** N / math.factorial(N) * N / (N - a)
    erlang_c = top / (sum(a ** k / math.factorial(k) for k in range(N)) + top)
    assert abs(pi[-1] + tail.sum() - erlang_c) <= 1e-14
    assert abs(pi.sum() + tail.sum() - 1.0) <= 1e-14
    # the truncated dense chain converges to the unlimited one (error ~ r^C)
    pi_d, tail_d = buffer.stationary_buffer(lam, inst.mu, inst.pref, 160)
    np.testing.assert_allclose(pi_d, pi, rtol=0, atol=1e-14)
    np.testing.assert_allclose(tail_d[:40], tail[:40], rtol=0, atol=1e-14)


@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("C", [1, 3, 10, U])
@pytest.mark.parametrize("rho", [0.3, 0.7])
def test_proposition_matches_dense_lu(seed, C, rho):
    inst = hqinst.generate(7, 15, seed=seed, rho=rho, mu_lo=0.5, mu_hi=1.5)
    pi_loss = oracle.solve(inst, tol=1e-15, max_iter=5000)["pi"]
    pi, tail = buffer.tail_from_loss(pi_loss, inst.lam.sum(), inst.mu, C)
    pi_d, tail_d = buffer.stationary_buffer(inst.lam, inst.mu, inst.pref, 200 if C == U else C)
    np.testing.assert_allclose(pi, pi_d, rtol=0, atol=1e-13)
    n = min(len(tail_d), 50)
    np.testing.assert_allclose(tail[:n], tail_d[:n], rtol=0, atol=1e-13)


@pytest.mark.parametrize("C", [0, 1, 6, U])
def test_measures_flow_identities(C):
    inst = hqinst.generate(6, 12, seed=4, rho=0.6, mu_lo=0.5, mu_hi=1.5)
    pi, tail = buffer.stationary_buffer(inst.lam, inst.mu, inst.pref, 200 if C == U else C)
    w, d, loss = buffer.measures_buffer(inst.lam, inst.mu, inst.pref, pi, tail, C)
    Lam = inst.lam.sum()
    assert abs(d.sum() - 1.0) <= 1e-13
    # unit i is busy a fraction rho_i of the time and completes nu_i rho_i calls per unit time
    np.testing.assert_allclose(inst.mu * w, Lam * (1.0 - loss) * d.sum(axis=0), rtol=1e-12, atol=0)
    if C == 0:
        w0, d0, l0 = dense.measures(inst.lam, inst.mu, inst.pref, pi)
        np.testing.assert_allclose(w, w0, atol=1e-15)
        np.testing.assert_allclose(d, d0, atol=1e-15)
        assert abs(loss - l0) <= 1e-15
    elif C > 0:
        assert loss == tail[C - 1]
