"""Pins of the response-time oracle (oracle/response.py) -m "not gpu"."""
import json
import os

import numpy as np
import pytest

import hqinst
from oracle import dense, response


def test_hand_example_n2():
    """N2_homogeneous (tests/golden/spec_n2_examples.json): pi = (0.4, 0.3, 0.1, 0.2), one atom
    with list (unit 0, unit 1).  S_00 = {00, 10} (mass 0.5), S_01 = {01} (0.3), Pi = 0.2:
    rho = (0.625, 0.375).  tau = (4, 10): MRT = 0.625*4 + 0.375*10 = 6.25; F(6) = 0.625
    (strict: F(10) = 0.625, F(11) = 1)."""
    ex = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_n2_examples.json")))
    e = next(x for x in ex["examples"] if x["name"] == "N2_homogeneous")
    tau = np.array([[4.0, 10.0]])
    for T, F in [(6.0, 0.625), (10.0, 0.625), (11.0, 1.0), (4.0, 0.0)]:
        mrt, frac, mj, fj = response.response_times(e["lam"], e["mu"], e["pref"], np.array(e["pi"]), tau, T)
        assert abs(mrt - 6.25) < 1e-15 and abs(frac - F) < 1e-15
        assert abs(mj[0] - 6.25) < 1e-15 and abs(fj[0] - F) < 1e-15


@pytest.mark.parametrize("L", [None, 3])
def test_limits_and_dispatch_agreement(L):
    inst = hqinst.generate(6, 9, seed=2, rho=0.7, L=L)
    pi = dense.stationary(inst.lam, inst.mu, inst.pref)
    rng = np.random.default_rng(0)
    tau = rng.uniform(1.0, 9.0, size=(inst.J, inst.N))
    # MRT equals sum rho_ij tau_ij with the independently enumerated dispatch of dense.measures
    _, d, _ = dense.measures(inst.lam, inst.mu, inst.pref, pi)
    mrt, frac, mj, fj = response.response_times(inst.lam, inst.mu, inst.pref, pi, tau, 5.0)
    assert abs(mrt - (d * tau).sum()) < 1e-14
    assert abs(frac - d[tau < 5.0].sum()) < 1e-14
    # every call within a threshold above all tau; none below all tau; constant tau
    assert abs(response.response_times(inst.lam, inst.mu, inst.pref, pi, tau, 10.0)[1] - 1.0) < 1e-14
    assert response.response_times(inst.lam, inst.mu, inst.pref, pi, tau, 1.0)[1] == 0.0
    c = response.response_times(inst.lam, inst.mu, inst.pref, pi, np.full_like(tau, 3.5), 2.0)
    assert abs(c[0] - 3.5) < 1e-14 and np.abs(c[2] - 3.5).max() < 1e-14
    # F = sum_j f_j F_j
    f = inst.lam / inst.lam.sum()
    assert abs((f * fj).sum() - frac) < 1e-14
