"""Write oracle fixtures for GPU parity at sizes too slow to re-run the oracle
in every GPU test session.  Calls only ``oracle`` and ``hqinst``.

  python tests/golden/make_oracle_fixtures.py cfg3

writes tests/golden/oracle_cfg3.npz with: the instance hash, the oracle's
sweeps and residual, the layer masses, the measures, and pi at a seeded
sample of states (every state of the three lowest and three highest layers,
plus uniform random states).
"""
import itertools
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import hqinst  # noqa: E402
import oracle  # noqa: E402


def edge_states(N):
    """every state of the layers 0, 1, 2, N-2, N-1, N (enumerated by combinations)"""
    full = (1 << N) - 1
    low = [0] + [1 << a for a in range(N)] + [(1 << a) | (1 << b) for a, b in itertools.combinations(range(N), 2)]
    return sorted(set(low) | {full ^ m for m in low})


def sample_states(N, nrand=6000, seed=123):
    rng = np.random.default_rng(seed)
    S = 1 << N
    if N <= 26:
        edge = [m for m in range(S) if bin(m).count("1") in (0, 1, 2, N - 2, N - 1, N)]
    else:
        edge = edge_states(N)
    rnd = rng.integers(0, S, size=nrand)
    return np.unique(np.concatenate([np.array(edge, dtype=np.int64), rnd.astype(np.int64)]))


def popcounts(N):
    idx = np.arange(1 << N, dtype=np.uint32)
    pc = np.zeros(1 << N, dtype=np.int8)
    tab = np.array([bin(b).count("1") for b in range(256)], dtype=np.int8)
    for sh in range(0, 32, 8):
        pc += tab[(idx >> sh) & 0xFF]
    return pc


def main(which):
    extra = {}
    if which == "cfg3":
        inst = hqinst.config_instance(3)
        nrand = 6000
    elif which == "cfg4":
        inst = hqinst.config_instance(4)
        nrand = 20000
    else:
        raise SystemExit("unknown fixture " + which)
    # the oracle's Algorithm-3 rate table (2^N N doubles, same arithmetic as its list scans)
    # when the host has the memory for it: cfg4 needs 60 GB + ~20 GB of other arrays
    need = (1 << inst.N) * inst.N * 8 + (1 << inst.N) * 8 * 10
    use_table = None
    try:
        with open("/proc/meminfo") as fh:
            avail = [int(x.split()[1]) * 1024 for x in fh if x.startswith("MemAvailable")][0]
        use_table = avail > 1.2 * need
    except (OSError, IndexError):
        pass
    if inst.N >= 27 and not use_table:
        raise SystemExit(f"{which}: the list-scan oracle at N = {inst.N} takes days; needs "
                         f"{1.2 * need / 2**30:.0f} GB of host memory for the rate table")
    print(f"{which}: N={inst.N} J={inst.J} use_table={use_table} threads={oracle.num_threads()}", flush=True)
    t = time.time()
    r = oracle.solve(inst, tol=1e-13, max_iter=3000, use_table=use_table)
    dt = time.time() - t
    pi = r["pi"]
    N = inst.N
    pc = popcounts(N)
    masses = np.bincount(pc, weights=pi, minlength=N + 1)
    del pc
    if N >= 26:
        # sums of pi over consecutive blocks of 2^14 natural indices (whole-vector check at
        # sizes whose pi is too large to commit), in ascending order within a block
        extra["block_bits"] = 14
        extra["block_sums"] = pi.reshape(-1, 1 << 14).sum(axis=1)
    w, d, loss = oracle.measures(inst, pi)
    st = sample_states(N, nrand=nrand)
    out = os.path.join(HERE, f"oracle_{which}.npz")
    np.savez_compressed(out, sha256=inst.sha256(), iters=r["iters"], residual=r["residual"], status=r["status"],
                        masses=masses, workload=w, dispatch=d, loss=loss, states=st, pi_states=pi[st],
                        oracle_seconds=dt, oracle_threads=oracle.num_threads(), tol=1e-13,
                        oracle_table=bool(use_table), **extra)
    print(f"wrote {out}: iters={r['iters']} residual={r['residual']:.3e} time={dt:.1f}s threads={oracle.num_threads()}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
