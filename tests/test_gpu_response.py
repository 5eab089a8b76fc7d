"""GPU parity of the response-time measures (row f3, include/hq.h hq_response_times) against
oracle/response.py on the oracle's pi, through the C-ABI."""
import numpy as np
import pytest
import torch

import hqinst
import oracle
from oracle import response

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("which", ["cfg1", "trunc", "cfg2"])
def test_response_parity(hq, which):
    inst = {"cfg1": lambda: hqinst.config_instance(1),
            "trunc": lambda: hqinst.generate(11, 40, seed=9, rho=0.6, L=4),
            "cfg2": lambda: hqinst.config_instance(2)}[which]()
    s = hq.Solver.from_instance(inst)
    r = s.solve(tol=1e-13)
    m = s.measures(r["pi"])
    rng = np.random.default_rng(5)
    tau = rng.uniform(2.0, 12.0, size=(inst.J, inst.N))
    pi_o = oracle.solve(inst, tol=1e-14, max_iter=20000)["pi"]
    for T in (6.0, 9.0):
        g = s.response_times(m["dispatch"].reshape(-1), tau, T)
        mrt, frac, mj, fj = response.response_times(inst.lam, inst.mu, inst.pref, pi_o, tau, T)
        assert abs(g["mrt"] - mrt) <= 1e-10 and abs(g["frac_within"] - frac) <= 1e-10
        assert np.abs(g["mrt_j"].cpu().numpy() - mj).max() <= 1e-10
        assert np.abs(g["frac_within_j"].cpu().numpy() - fj).max() <= 1e-10
    s.close()


def test_response_rejects_buffer(hq):
    inst = hqinst.config_instance(1)
    s = hq.Solver.from_instance(inst)
    s.set_buffer(3)
    r = s.solve(tol=1e-13)
    m = s.measures(r["pi"])
    with pytest.raises(hq.HQError, match="zero-capacity"):
        s.response_times(m["dispatch"].reshape(-1), np.ones((inst.J, inst.N)), 5.0)
    s.close()
