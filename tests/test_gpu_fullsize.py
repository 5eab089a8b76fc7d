"""Whole-vector GPU parity at the mid and full sizes (-m gpu), through the C-ABI.

Bar (BASELINE.json north_star): both sides run to relative residual 1e-13; pi within
1e-10 L1 and 1e-12 max-abs; measures within 1e-10.  What each size is compared with
(DESIGN.md §3):

  * N = 19..23 (every warp-count / fold variant of the CTA-tiled path: nW = 2, 3, 4 and
    both sides of the folded scalar step at N = 21): a full oracle run in the session,
    whole vector;
  * cfg3 (N = 24): a full oracle run in the session (a few minutes on the box's host
    cores), whole vector, plus the measures;
  * cfg4 (N = 28, truncated lists): the committed oracle fixture
    (tests/golden/oracle_cfg4.npz, written by tests/golden/make_oracle_fixtures.py, which
    calls only oracle/): pi at 20k seeded states plus every state of layers 0-2 and
    N-2..N, sums of pi over all 2^14 blocks of 2^14 states, layer masses, measures; and
    the oracle's memory-lean residual of the whole GPU pi;
  * cfg5 (N = 31) at rho 0.3 / 0.6 / 0.9: the oracle's memory-lean residual
    (oracle_residual_stream, Eq. balance_eq_heter, reading C3) over all 2^31 states of
    the GPU pi, sum pi = 1, pi >= 0; and the homogeneous copy against the Erlang-B
    layer masses (aggregate M/M/N/N, independent of the method).
"""
import math
import os

import numpy as np
import pytest
import torch

import hqinst
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-13
PI_L1 = 1e-10
PI_MAX = 1e-12
MEAS = 1e-10
GOLD4 = os.path.join(os.path.dirname(__file__), "golden", "oracle_cfg4.npz")


def gpu_solve(hq, inst, host=True):
    s = hq.Solver.from_instance(inst)
    r = s.solve(tol=TOL, max_iter=20000)
    m = s.measures(r["pi"])
    out = dict(iters=r["iters"], residual=r["residual"], status=r["status"], stats=s.stats(),
               workload=m["workload"].cpu().numpy(), dispatch=m["dispatch"].cpu().numpy(), loss=m["loss"])
    out["pi"] = r["pi"].cpu().numpy() if host else r["pi"]
    s.close()
    del r, m
    torch.cuda.empty_cache()
    return out


def layer_masses_np(pi, N):
    """sum of pi per popcount layer, in 2^20-state chunks (host)."""
    tab = np.array([bin(b).count("1") for b in range(256)], dtype=np.int8)
    out = np.zeros(N + 1)
    step = 1 << min(N, 22)
    for base in range(0, 1 << N, step):
        idx = np.arange(base, base + step, dtype=np.uint32)
        pc = np.zeros(step, dtype=np.int8)
        for sh in range(0, 32, 8):
            pc += tab[(idx >> sh) & 0xFF]
        out += np.bincount(pc, weights=pi[base:base + step], minlength=N + 1)
    return out


def whole_vector(g, o, inst):
    assert g["status"] == 0 and g["residual"] <= TOL, (g["status"], g["residual"])
    d = np.abs(g["pi"] - o["pi"])
    assert d.sum() <= PI_L1, d.sum()
    assert d.max() <= PI_MAX, d.max()
    w, disp, loss = oracle.measures(inst, o["pi"])
    assert np.abs(g["workload"] - w).max() <= MEAS
    assert np.abs(g["dispatch"] - disp).max() <= MEAS
    assert abs(g["loss"] - loss) <= MEAS
    r, _, _ = oracle.residual_stream(inst, g["pi"])
    assert r <= 1.5 * TOL, r


# (N, generator config, J, list length): N = 19/20 -> nW = 2/3, N >= 21 -> nW = 4 (folded
# scalar step); uniform, clustered and truncated (top-8) shapes
_MID = [
    (19, 2, 100, None),
    (20, 3, 120, None),
    (21, 4, 150, 8),
    (22, 2, 100, None),
    (23, 4, 200, 8),
]


@pytest.mark.parametrize("N,cfg,J,L", _MID)
def test_mid_sizes_whole_vector(hq, N, cfg, J, L):
    inst = hqinst.config_instance(cfg, N=N, J=J)
    assert (L is None) == bool((inst.pref >= 0).all())
    g = gpu_solve(hq, inst)
    assert g["stats"]["path"] == 3
    o = oracle.solve(inst, tol=TOL, max_iter=5000)
    assert o["status"] == 0
    whole_vector(g, o, inst)


def gpu_solve_loop(hq, inst, loop):
    """gpu_solve with the host-looped or the device-resident solve (HQ_LOOP is read at hq_create)."""
    old = os.environ.get("HQ_LOOP")
    os.environ["HQ_LOOP"] = loop
    try:
        g = gpu_solve(hq, inst)
    finally:
        if old is None:
            os.environ.pop("HQ_LOOP")
        else:
            os.environ["HQ_LOOP"] = old
    assert g["stats"]["device_loop"] == (1.0 if loop == "device" else 0.0)
    return g


def test_cfg3_whole_vector(hq):
    """cfg3 (N = 24, 16.8M states): the oracle run in the session, every state compared, for
    both the host-looped and the device-resident solve (one cooperative launch)."""
    inst = hqinst.config_instance(3)
    o = oracle.solve(inst, tol=TOL, max_iter=5000)
    assert o["status"] == 0
    for loop in ("host", "device"):
        g = gpu_solve_loop(hq, inst, loop)
        whole_vector(g, o, inst)


def gpu_solve_env(hq, inst, env):
    """gpu_solve with development switches set in the environment (read at hq_create)."""
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return gpu_solve(hq, inst)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("order", [
    {"HQ_ORDER": "group", "HQ_GROUP_BITS": "3"},                          # cfg4/cfg5 default path
    {"HQ_ORDER": "group", "HQ_GROUP_BITS": "4", "HQ_PFH": "0", "HQ_PFO": "0"},
    {"HQ_ORDER": "chunk", "HQ_CHUNK_BITS": "2"},   # 256 chunks >= the 148-CTA grid
    {"HQ_ORDER": "group", "HQ_GROUP_BITS": "3", "HQ_GLAG": "1"},          # group progress bound
])
def test_tile_orders_whole_vector(hq, order):
    """The tile visit orders of N >= 27 (group order: Gray-code groups, round-robin CTAs, L2
    prefetch of the tile-unit slices; chunked order) at N = 23, where the oracle runs in the
    session: the order only changes which CTA sums which tile, never a state's arithmetic."""
    inst = hqinst.config_instance(4, N=23, J=200)
    g = gpu_solve_env(hq, inst, order)
    assert g["stats"]["path"] == 3 and g["stats"]["chunk_bits"] >= 0
    o = oracle.solve(inst, tol=TOL, max_iter=5000)
    assert o["status"] == 0
    whole_vector(g, o, inst)


@pytest.mark.parametrize("N,cfg,J", [(12, 2, 60), (18, 2, 100), (21, 4, 150)])
def test_device_loop_matches_host_loop(hq, N, cfg, J):
    """The device-resident solve performs the same half-sweeps as the host-looped one: after a
    fixed number of sweeps (tol = 0) the iterates agree to rounding (the per-layer sums are
    added in a different order), and both converge to the oracle's pi."""
    inst = hqinst.config_instance(cfg, N=N, J=J)
    for K in (1, 7):
        its = []
        for loop in ("host", "device"):
            old = os.environ.get("HQ_LOOP")
            os.environ["HQ_LOOP"] = loop
            try:
                s = hq.Solver.from_instance(inst)
            finally:
                if old is None:
                    os.environ.pop("HQ_LOOP")
                else:
                    os.environ["HQ_LOOP"] = old
            r = s.solve(tol=0.0, max_iter=K)
            assert r["iters"] == K and s.stats()["device_loop"] == (1.0 if loop == "device" else 0.0)
            its.append(r["pi"].cpu().numpy())
            s.close()
        assert np.abs(its[0] - its[1]).max() <= 1e-14
    o = oracle.solve(inst, tol=TOL)
    for loop in ("host", "device"):
        whole_vector(gpu_solve_loop(hq, inst, loop), o, inst)


def _mem_available():
    try:
        with open("/proc/meminfo") as fh:
            return [int(x.split()[1]) * 1024 for x in fh if x.startswith("MemAvailable")][0]
    except (OSError, IndexError):
        return 0


def test_n28_iterates_whole_vector(hq):
    """The N >= 27 launch configuration (group tile order, L2 prefetch, 2^28 states: cfg4's
    generator with full lists) element by element: after exactly K sweeps the GPU iterate
    equals the oracle's K-th Algorithm-1 iterate over the WHOLE vector.
    The oracle needs its rate table here (60 GB + ~20 GB of arrays; list scans take hours)."""
    inst = hqinst.generate(28, 500, seed=4, rho=0.8, name="cfg4-full-lists")
    need = (1 << inst.N) * inst.N * 8 + (1 << inst.N) * 8 * 10
    if _mem_available() < 1.2 * need:
        pytest.skip("host memory below %.0f GB" % (1.2 * need / 2**30))
    K = 3
    o = oracle.solve(inst, tol=0.0, max_iter=K, use_table=True)
    s = hq.Solver.from_instance(inst)
    r = s.solve(tol=0.0, max_iter=K)
    assert r["iters"] == K
    pi = r["pi"].cpu().numpy()
    s.close()
    d = np.abs(pi - o["pi"])
    assert d.max() <= 1e-14 and d.sum() <= 1e-12, (d.max(), d.sum())
    # entries are ~4e-9 at this size: also element by element in relative terms
    rel = float((d / o["pi"]).max())
    assert o["pi"].min() > 0 and rel <= 1e-9, rel


def test_cfg4_against_oracle_fixture(hq):
    if not os.path.exists(GOLD4):
        pytest.skip("tests/golden/oracle_cfg4.npz not generated")
    inst = hqinst.config_instance(4)
    f = np.load(GOLD4)
    assert str(f["sha256"]) == inst.sha256(), "fixture was written for another instance"
    assert int(f["status"]) == 0 and float(f["residual"]) <= TOL
    g = gpu_solve(hq, inst)
    assert g["status"] == 0 and g["residual"] <= TOL
    pi = g["pi"]
    st = f["states"].astype(np.int64)
    assert np.abs(pi[st] - f["pi_states"]).max() <= PI_MAX
    bb = int(f["block_bits"])
    bs = pi.reshape(-1, 1 << bb).sum(axis=1)
    assert np.abs(bs - f["block_sums"]).sum() <= PI_L1, np.abs(bs - f["block_sums"]).sum()
    np.testing.assert_allclose(layer_masses_np(pi, inst.N), f["masses"], rtol=0, atol=PI_MAX)
    assert np.abs(g["workload"] - f["workload"]).max() <= MEAS
    assert np.abs(g["dispatch"] - f["dispatch"]).max() <= MEAS
    assert abs(g["loss"] - float(f["loss"])) <= MEAS
    r, _, _ = oracle.residual_stream(inst, pi)
    assert r <= 1.5 * TOL, r


def test_cfg4_full_residual(hq):
    """cfg4 (N = 28, top-8 lists, 2^28 states): the oracle's residual of the WHOLE GPU pi
    (Eq. balance_eq_heter; unique solution PAPER.md:1438) -- runs with or
    without the committed fixture."""
    inst = hqinst.config_instance(4)
    g = gpu_solve(hq, inst)
    assert g["status"] == 0 and g["residual"] <= TOL, (g["status"], g["residual"])
    pi = g.pop("pi")
    assert abs(pi.sum() - 1.0) <= 1e-12
    assert pi.min() >= 0.0
    r, num, den = oracle.residual_stream(inst, pi)
    assert r <= 1.5 * TOL, r
    # truncated lists: calls are lost in more states than the all-busy one
    assert g["loss"] > pi[-1]
    lhs = inst.mu * g["workload"]
    rhs = inst.lam.sum() * (1.0 - g["loss"]) * g["dispatch"].sum(axis=0)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-10, atol=1e-12)
    del pi


@pytest.mark.parametrize("rho", [0.3, 0.6, 0.9])
def test_cfg5_full_residual(hq, rho):
    """cfg5 (N = 31, 2^31 states, 17 GB pi): the oracle's residual of the whole GPU pi."""
    inst = hqinst.config_instance(5, rho=rho)
    g = gpu_solve(hq, inst)
    assert g["status"] == 0 and g["residual"] <= TOL, (g["status"], g["residual"])
    pi = g.pop("pi")
    assert abs(pi.sum() - 1.0) <= 1e-12
    assert pi.min() >= 0.0
    r, num, den = oracle.residual_stream(inst, pi)
    assert r <= 1.5 * TOL, r
    # full lists: loss = P(all busy); unit flow identity nu_i rho_i = Lambda (1 - loss) sum_j rho_ij
    assert abs(g["loss"] - pi[-1]) <= 1e-15
    lhs = inst.mu * g["workload"]
    rhs = inst.lam.sum() * (1.0 - g["loss"]) * g["dispatch"].sum(axis=0)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-10, atol=1e-12)
    del pi


def test_cfg5_homogeneous_erlang(hq):
    """Homogeneous copy of cfg5 (nu_i = 1, Lambda = 0.6 N; reading C10): the layer masses are
    the truncated Poisson (Erlang loss) distribution for any preference lists."""
    inst = hqinst.homogeneous_copy(hqinst.config_instance(5))
    g = gpu_solve(hq, inst)
    assert g["status"] == 0 and g["residual"] <= TOL
    a = inst.lam.sum()
    N = inst.N
    w = np.array([math.exp(n * math.log(a) - math.lgamma(n + 1)) for n in range(N + 1)])
    np.testing.assert_allclose(layer_masses_np(g["pi"], N), w / w.sum(), rtol=0, atol=PI_MAX)


@pytest.mark.parametrize("gb,lag", [(3, 1), (3, 2), (6, 1)])
def test_group_lag_bitwise(hq, gb, lag):
    """The group progress bound (HQ_GLAG: a CTA starts a tile of group g only when every CTA
    is done with group g - lag) changes when a CTA visits its tiles, never which tiles or in
    which order it sums them: pi and the measures are bitwise those of the unbounded run."""
    inst = hqinst.config_instance(4, N=23, J=200)
    base = {"HQ_ORDER": "group", "HQ_GROUP_BITS": str(gb)}
    g0 = gpu_solve_env(hq, inst, dict(base, HQ_GLAG="0"))   # the default is lag 2 with >= 32 groups
    g1 = gpu_solve_env(hq, inst, dict(base, HQ_GLAG=str(lag)))
    assert g0["stats"]["group_lag"] == 0 and g1["stats"]["group_lag"] == lag
    assert g0["iters"] == g1["iters"] and g0["residual"] == g1["residual"]
    assert np.array_equal(g0["pi"], g1["pi"])
    assert np.array_equal(g0["workload"], g1["workload"]) and g0["loss"] == g1["loss"]
