"""GPU parity at BASELINE.json's full sizes (-m gpu), through the C-ABI.

The oracle cannot re-run N = 24..31 inside a test session, so at these sizes
the CUDA result is checked against:
  * cfg3 (N = 24): a committed oracle fixture (tests/golden/oracle_cfg3.npz,
    written by tests/golden/make_oracle_fixtures.py, which calls only oracle/):
    pi at 6.6k sampled states, layer masses, workloads, dispatch, loss;
  * cfg4 (N = 28, truncated lists) and cfg5 (N = 31): the oracle's own
    balance equation (Eq. balance_eq_heter) evaluated state by
    state at seeded samples of the GPU pi, plus properties that hold at any
    size: sum pi = 1, pi >= 0, the loss ordering (truncated lists: loss > P(all busy)),
    sum rho_ij = 1 and the unit flow identity nu_i rho_i = Lambda (1 - loss) sum_j rho_ij;
    (the whole-vector checks at these sizes are in test_gpu_fullsize.py);
  * N = 31 ordered hunt: the Erlang-B closed forms for the layer masses, the
    per-unit workloads and the loss (textbook, independent of the method).
"""
import math
import os

import numpy as np
import pytest
import torch

import hqinst
import oracle

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "oracle_cfg3.npz")
TOL = 1e-13


def solve(hq, inst, tol=TOL):
    s = hq.Solver.from_instance(inst)
    r = s.solve(tol=tol, max_iter=20000)
    m = s.measures(r["pi"])
    out = dict(pi=r["pi"], status=r["status"], iters=r["iters"], residual=r["residual"],
               workload=m["workload"].cpu().numpy(), dispatch=m["dispatch"].cpu().numpy(), loss=m["loss"])
    s.close()
    return out


def layer_masses(pi, N, chunk_bits=26):
    """sum of pi over each popcount layer (chunked, on the device)."""
    out = torch.zeros(N + 1, dtype=torch.float64, device=pi.device)
    S = 1 << N
    step = min(S, 1 << chunk_bits)
    for base in range(0, S, step):
        idx = torch.arange(base, base + step, device=pi.device, dtype=torch.int64)
        pc = torch.zeros_like(idx)
        x = idx.clone()
        while True:
            nz = x != 0
            if not bool(nz.any()):
                break
            pc += x & 1
            x >>= 1
        out += torch.bincount(pc, weights=pi[base:base + step], minlength=N + 1)[: N + 1]
    return out.cpu().numpy()


def sampled_balance(inst, pi, nsamp=3000, seed=7):
    """Relative balance residual of the GPU pi over seeded sample states,
    evaluated by the oracle's independent per-state code."""
    rng = np.random.default_rng(seed)
    N = inst.N
    states = np.unique(rng.integers(0, 1 << N, size=nsamp, dtype=np.int64))
    st = torch.from_numpy(states).to(pi.device)
    cols = [pi[st]] + [pi[st ^ (1 << i)] for i in range(N)]
    nbr = torch.stack(cols, dim=1).cpu().numpy()
    out, inn = oracle.state_balance(inst, states.astype(np.uint64), nbr)
    return float(np.abs(out - inn).sum() / out.sum()), float(np.max(np.abs(out - inn) / np.maximum(out, 1e-300)))


def measure_identities(inst, g):
    lam = inst.lam
    Lam = lam.sum()
    d = g["dispatch"]
    assert abs(d.sum() - 1.0) <= 1e-12
    # unit flow balance: nu_i rho_i = Lambda (1 - loss) sum_j rho_ij (exact at the fixed point)
    lhs = inst.mu * g["workload"]
    rhs = Lam * (1.0 - g["loss"]) * d.sum(axis=0)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-10, atol=1e-12)


def test_cfg3_against_oracle_fixture(hq):
    inst = hqinst.config_instance(3)
    f = np.load(GOLD)
    assert str(f["sha256"]) == inst.sha256(), "fixture was written for another instance"
    g = solve(hq, inst)
    assert g["status"] == 0 and g["residual"] <= TOL
    pi = g["pi"]
    st = torch.from_numpy(f["states"].astype(np.int64)).to(pi.device)
    got = pi[st].cpu().numpy()
    assert np.abs(got - f["pi_states"]).max() <= 1e-12
    np.testing.assert_allclose(layer_masses(pi, inst.N), f["masses"], rtol=0, atol=1e-12)
    assert np.abs(g["workload"] - f["workload"]).max() <= 1e-10
    assert np.abs(g["dispatch"] - f["dispatch"]).max() <= 1e-10
    assert abs(g["loss"] - float(f["loss"])) <= 1e-10
    measure_identities(inst, g)


def test_cfg3_homogeneous_erlang(hq):
    inst = hqinst.homogeneous_copy(hqinst.config_instance(3))
    g = solve(hq, inst)
    a = inst.lam.sum()
    w = np.array([a ** n / math.factorial(n) for n in range(inst.N + 1)])
    np.testing.assert_allclose(layer_masses(g["pi"], inst.N), w / w.sum(), rtol=0, atol=1e-12)


def _large_checks(inst, g):
    assert g["status"] == 0 and g["residual"] <= TOL
    pi = g["pi"]
    assert abs(float(pi.sum()) - 1.0) <= 1e-12
    assert float(pi.min()) >= 0.0
    rel, _ = sampled_balance(inst, pi)
    assert rel <= 1e-11, rel
    measure_identities(inst, g)
    return pi


def test_cfg4_truncated_n28(hq):
    inst = hqinst.config_instance(4)
    g = solve(hq, inst)
    _large_checks(inst, g)
    # loss with truncated lists = sum_j f_j P(list_j all busy) > P(all busy)
    assert g["loss"] > float(g["pi"][-1])


def test_ordered_hunt_n31_closed_form(hq):
    N = 31
    order = np.random.default_rng(31).permutation(N).astype(np.int32)
    inst = hqinst.ordered_hunt(N, 0.6, J=1, order=order)
    g = solve(hq, inst)
    assert g["status"] == 0
    a = inst.lam.sum()
    B = [1.0]
    for k in range(1, N + 1):
        B.append(a * B[-1] / (k + a * B[-1]))
    ref = np.zeros(N)
    for k, u in enumerate(order, start=1):
        ref[u] = a * (B[k - 1] - B[k])
    np.testing.assert_allclose(g["workload"], ref, rtol=0, atol=1e-11)
    assert abs(g["loss"] - B[N]) <= 1e-12
    w = np.array([math.exp(n * math.log(a) - math.lgamma(n + 1)) for n in range(N + 1)])
    np.testing.assert_allclose(layer_masses(g["pi"], N), w / w.sum(), rtol=0, atol=1e-12)


def test_cfg3_bitwise_deterministic(hq):
    """The N >= 21 path (folded scalar step, double-buffered partials, fixed-order sums) gives
    bitwise identical results on two handles."""
    inst = hqinst.config_instance(3)
    a = solve(hq, inst)
    b = solve(hq, inst)
    assert torch.equal(a["pi"], b["pi"]) and a["iters"] == b["iters"] and a["residual"] == b["residual"]
