#!/usr/bin/env python
"""Benchmark: state-updates/s and time-to-1e-13 residual (fp64) on one B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--secondary C,..]
                    [--impl ours|reference]

Headline workload: BASELINE.json config 5 (N = 31, J = 1000, rho = 0.6; 2^31 states,
17 GB of pi), the largest configuration that fits one GPU; config 3 (N = 24) is measured
after it with the same protocol and reported under "secondary".

A "step" is one pass of the whole hot path on the resident instance: hq_solve
from the uniform initial iterate to relative residual <= 1e-13 (Algorithm 1
sweeps, verification residual, assembly of pi) followed by hq_measures.
value = state updates (sum over updated layers of C(N,n), i.e. 2^N - 2 per
sweep) / device time of the K steps (CUDA events, max over ranks).

Multi-GPU: the solve does not shard ("replicas only"): under
torchrun every rank solves its own replica and value is the sum over ranks /
the max time ("scaling": "weak").

--impl reference times the CPU oracle (oracle/, the test-infrastructure
reference implementation written from the paper) on a bounded sample of the
same workload, on rank 0 only (N >= 27: per-state extrapolation, the oracle
cannot hold 2^N states).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "state-updates/sec and time-to-1e-13 residual (fp64) vs HBM roofline, 1 B200"
UNIT = "state-updates/s"
BYTES_PER_UPDATE = 32  # read p_{n-1}, p_{n+1} (16 B amortised), read + write p_n (16 B)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5,
                    help="BASELINE.json config 1..5 (default 5: N=31, the largest single-GPU config)")
    ap.add_argument("--secondary", default="3",
                    help="comma-separated configs measured after the headline and reported under "
                         "'secondary' ('' to skip)")
    ap.add_argument("--rho", type=float, default=None)
    ap.add_argument("--tol", type=float, default=1e-13)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    return ap.parse_args()


def workload_desc(inst, cfg):
    return {"workload": f"cfg{cfg}: {inst.name} N={inst.N} J={inst.J} rho={inst.rho:g} "
                        f"{'top-8 truncated' if (inst.pref < 0).any() else 'full'} lists, 2^{inst.N} states",
            "N": inst.N, "J": inst.J, "rho": inst.rho, "seed": inst.seed, "tol": None,
            "instance_sha256": inst.sha256()[:16]}


# ------------------------------------------------------------------ clocks

class Clocks:
    def __init__(self, enabled=True, index=0):
        self.enabled = enabled
        self.proc = None
        self.path = None
        self.index = index

    def start(self):
        if not self.enabled:
            return
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 9:
                    rows.append(p)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows)}


# ------------------------------------------------------------------ peaks / profiles

def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy test)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_summary(cfg):
    """Counters of one steady-state sweep-kernel launch (k_sweep3, one half-sweep with every
    layer of the class active) of this config from the committed `ncu --set full` capture
    (profiles/ncu_summary.json, written by tools/ncu_summary.py): dram bytes per launch
    (dram__bytes_read.sum + dram__bytes_write.sum), DRAM throughput, issue-slot and FP64-pipe
    utilisation, warp instructions per launch.  None if absent."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(f"cfg{cfg}")


# ------------------------------------------------------------------ reference arm (CPU oracle)

def oracle_sample(inst, sweeps=3):
    """Time `sweeps` oracle sweeps on this host, excluding the one-off rate
    table build: t(1 + sweeps) - t(1)."""
    import oracle

    t0 = time.perf_counter()
    oracle.solve(inst, tol=0.0, max_iter=1)
    t1 = time.perf_counter()
    oracle.solve(inst, tol=0.0, max_iter=1 + sweeps)
    t2 = time.perf_counter()
    dt = (t2 - t1) - (t1 - t0)
    updates = ((1 << inst.N) - 2) * sweeps
    return updates / dt, dt, oracle.num_threads()


def oracle_state_sample(inst, nstates, seed=11):
    """Per-state oracle work at sizes where the oracle cannot hold the state space (N >= 27:
    eight 2^N arrays): the balance equation of Eq. balance_eq_heter at seeded random states
    (oracle_state_balance: Algorithm-3 list scan, lambda_m list scan, the N-neighbour
    gather), about the work of one oracle sweep per state (update + residual pass, each a
    list scan and a gather).  Returns (states/s, seconds, threads)."""
    import numpy as np

    import oracle

    rng = np.random.default_rng(seed)
    done, dt = 0, 0.0
    while done < nstates:
        n = min(1 << 18, nstates - done)
        st = rng.integers(0, 1 << inst.N, size=n, dtype=np.int64).astype(np.uint64)
        nbr = rng.random((n, inst.N + 1))
        t0 = time.perf_counter()
        oracle.state_balance(inst, st, nbr)
        dt += time.perf_counter() - t0
        done += n
    return done / dt, dt, oracle.num_threads()


def cpu_sample(inst, cfg):
    """(value, seconds, threads, sample text) of the oracle on this host: full sweeps for
    N <= 26, per-state extrapolation above."""
    if inst.N <= 26:
        ns = cpu_sample_sweeps(inst.N)
        v, dt, cores = oracle_sample(inst, ns)
        return v, dt, cores, (f"{ns} Algorithm-1 sweeps of cfg{cfg} (each with the oracle's full residual pass), "
                              f"rate-table build excluded, {dt:.1f} s")
    nst = 1 << 22
    v, dt, cores = oracle_state_sample(inst, nst)
    return v, dt, cores, (f"extrapolated: {nst} seeded random cfg{cfg} states through the oracle's per-state "
                          f"balance code (list-scan rates + N-neighbour gather, about one oracle sweep's work per "
                          f"state; the oracle cannot hold 2^{inst.N} states), {dt:.1f} s")


def cpu_sample_sweeps(N):
    """Oracle sweeps per sample: about 10-20 s of CPU work on a 16-core host."""
    return max(1, min(64, 16 << max(0, 24 - N)))


def arm_config(inst, args, world):
    """The config block both arms print (same workload, tolerance and L2 statement)."""
    return dict(workload_desc(inst, args.config), tol=args.tol,
                l2="inputs larger than L2: per half-sweep the kernel streams %.0f MB (both classes of p, "
                   "omega/kappa, rate programs) vs 126 MB L2; no explicit flush"
                   % ((8 + 8 + 16) * (1 << inst.N) / 2 / 2 ** 20),
                parallelism="replicas" if world > 1 else "single GPU")


def reduce_over_ranks(t, work, device):
    """Replicas only: the job takes as long as the slowest rank and does the
    work of all ranks -> (max over ranks of t, sum over ranks of work).  Works for any
    torch.distributed backend (nccl with a CUDA device, gloo with the CPU)."""
    import torch
    import torch.distributed as dist

    x = torch.tensor([t, work], dtype=torch.float64, device=device)
    mx = x.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = x.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return float(mx[0]), float(sm[1])


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import hqinst

    inst = hqinst.config_instance(args.config, rho=args.rho)
    vals = []
    tt = 0.0
    if inst.N <= 26:
        sweeps = cpu_sample_sweeps(inst.N)
        for _ in range(args.warmup if inst.N <= 20 else 0):
            oracle_sample(inst, 1)
        for _ in range(args.steps):
            v, dt, cores = oracle_sample(inst, sweeps)
            vals.append(v)
            tt += dt
        sample = (f"{sweeps} Algorithm-1 sweeps of cfg{args.config} per step (each with the oracle's full residual "
                  f"pass), rate-table build excluded")
    else:
        nst = 1 << 20
        for step in range(args.steps):
            v, dt, cores = oracle_state_sample(inst, nst, seed=100 + step)
            vals.append(v)
            tt += dt
        sample = (f"extrapolated: {nst} seeded random cfg{args.config} states per step through the oracle's "
                  f"per-state balance code (list-scan rates + N-neighbour gather, about one oracle sweep's work "
                  f"per state; the oracle cannot hold 2^{inst.N} states)")
    value = statistics.median(vals)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": arm_config(inst, args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm

def measure(args, inst, steps, warmup, dev, dist, clocks=None):
    """Warm up, then time `steps` solves (+ measures) of the resident instance with CUDA events
    on the solve stream.  Returns the per-config measurement (this rank)."""
    import torch

    from paper_2603_03019_b200 import hq

    solver = hq.Solver.from_instance(inst)
    pi = torch.empty(1 << inst.N, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        r = solver.solve(tol=args.tol, max_iter=100000, pi=pi, stream=stream)
        solver.measures(pi, stream=stream)
        if r["status"] != 0:
            raise RuntimeError(f"solve did not converge: {r}")
        return r

    for _ in range(max(warmup, 0)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    if clocks:
        clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0.record(stream)
    acc = dict(updates=0.0, sweep_ms=0.0, sweep_launches=0.0, launches=0.0)
    iters, res, solve_ms = [], [], []
    for _ in range(steps):
        r = step()
        st = solver.stats()
        acc["updates"] += st["state_updates"]
        acc["sweep_ms"] += st["sweep_ms"]
        acc["sweep_launches"] += st["sweep_launches"]
        acc["launches"] += st["launches"] + 3 + inst.N   # + measures: copy, N zeta passes, measures kernel
        iters.append(r["iters"])
        res.append(r["residual"])
        solve_ms.append(st["solve_ms"])
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ck = clocks.stop() if clocks else None
    ms = e0.elapsed_time(e1)
    ms_max, updates_tot = reduce_over_ranks(ms, acc["updates"], dev) if dist else (ms, acc["updates"])
    out = dict(acc, ms=ms, ms_max=ms_max, updates_tot=updates_tot, iters=iters, res=res, solve_ms=solve_ms,
               clocks=ck, stats=solver.stats())
    solver.close()
    del pi
    torch.cuda.empty_cache()
    return out


def roofline_block(cfg, m, steps):
    """Roofline of the dominant kernel (k_sweep3, one launch per half-sweep), timed live by
    the CUDA events hq_solve records around every sweep launch on its stream (hq_stats).
    HBM: algorithmic bytes (32 B per state update) / launch time against
    the measured copy bandwidth.  The binding unit comes from the committed ncu counters of
    this config (profiles/ncu_summary.json): "hbm" when DRAM throughput is the highest
    utilisation, else "alu" (the issue slots: warp instructions per launch from ncu / the
    live launch time against 4 issue slots per SM per cycle at the measured SM clock)."""
    peak, peak_src = measured_peaks()
    sweep_ms, nl = m["sweep_ms"], max(m["sweep_launches"], 1.0)
    launch_ms = sweep_ms / nl
    upl = m["updates"] / nl
    achieved = BYTES_PER_UPDATE * upl / (launch_ms * 1e-3) / 1e9 if sweep_ms > 0 else None
    hbm = {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
           "peak_source": peak_src, "algorithmic_bytes_per_state_update": BYTES_PER_UPDATE,
           "algorithmic_bytes_per_launch": BYTES_PER_UPDATE * upl}
    ncu = ncu_summary(cfg)
    block = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": hbm["frac"],
             "traffic": ncu.get("dram_bytes_per_launch") if ncu else None,
             "kernel": "k_sweep3 (one launch per half-sweep of the red-black schedule)",
             "launch_ms": launch_ms, "launches_per_step": nl / steps, "sweep_ms_per_step": sweep_ms / steps,
             "sweep_share_of_step": sweep_ms / m["ms"] if m["ms"] else None, "hbm_algorithmic": hbm}
    if ncu:
        ck = m.get("clocks") or {}
        mhz = ck.get("sm_mhz") or 1965.0
        issue_peak = 4 * 148 * mhz * 1e6 / 1e9   # G warp instructions / s
        inst_rate = ncu["warp_inst_per_launch"] / (launch_ms * 1e-3) / 1e9 if ncu.get("warp_inst_per_launch") else None
        block["ncu"] = {k: ncu.get(k) for k in ("dram_bytes_per_launch", "dram_throughput_frac", "issue_active",
                                                "fp64_pipe_frac", "warp_inst_per_launch", "l2_hit_rate",
                                                "launch_us_under_ncu", "source")}
        block["issue"] = {"achieved": inst_rate, "peak": issue_peak, "unit": "G warp-inst/s",
                          "frac": (inst_rate / issue_peak) if inst_rate else None,
                          "peak_source": "4 issue slots/SM/cycle x 148 SMs x median SM clock of the run"}
        dram_frac = ncu.get("dram_throughput_frac") or 0.0
        if (ncu.get("issue_active") or 0.0) > dram_frac and inst_rate:
            block.update(bound="alu", achieved=inst_rate, peak=issue_peak, unit="G warp-inst/s",
                         frac=inst_rate / issue_peak)
    return block


def run_ours(args, rank, world, local_rank):
    import torch

    import hqinst
    from paper_2603_03019_b200 import hq

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

    inst = hqinst.config_instance(args.config, rho=args.rho)
    clocks = Clocks(enabled=(not args.no_clocks) and rank == 0, index=local_rank)
    m = measure(args, inst, args.steps, args.warmup, dev, dist, clocks)

    # ---- e2e: through the C-ABI with host buffers, h2d + d2h inside the timed region
    e2e = None
    if not args.no_e2e:
        lam_h = torch.from_numpy(inst.lam.copy()).pin_memory()
        mu_h = torch.from_numpy(inst.mu.copy()).pin_memory()
        pref_h = torch.from_numpy(inst.pref.copy()).pin_memory()
        pi_h = torch.empty(1 << inst.N, dtype=torch.float64).pin_memory()
        w_h = torch.empty(inst.N, dtype=torch.float64).pin_memory()
        d_h = torch.empty(inst.J * inst.N, dtype=torch.float64).pin_memory()
        pi = torch.empty(1 << inst.N, dtype=torch.float64, device=dev)
        stream = torch.cuda.current_stream()
        e2e_steps = max(1, min(args.steps, 3 if inst.N <= 26 else 2))
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_updates = 0.0
        for _ in range(e2e_steps):
            s2 = hq.Solver(lam_h.numpy(), mu_h.numpy(), pref_h.numpy())
            s2.solve(tol=args.tol, max_iter=100000, pi=pi, stream=stream)
            m2 = s2.measures(pi, stream=stream)
            pi_h.copy_(pi, non_blocking=True)
            w_h.copy_(m2["workload"], non_blocking=True)
            d_h.copy_(m2["dispatch"].reshape(-1), non_blocking=True)
            torch.cuda.synchronize()
            e2e_updates += s2.stats()["state_updates"]
            s2.close()
        t_e2e = time.perf_counter() - t0
        if dist:
            t_e2e, e2e_updates = reduce_over_ranks(t_e2e, e2e_updates, dev)
        h2d = inst.lam.nbytes + inst.mu.nbytes + inst.pref.nbytes
        d2h = (8 << inst.N) + 8 * inst.N + 8 * inst.J * inst.N + 8 + 8
        e2e = {"value": e2e_updates / t_e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1000.0 * t_e2e / e2e_steps, "steps": e2e_steps,
               "timing": "host wall clock around create (incl. the one-off rate-program precompute) + solve + "
                         "measures + d2h of pi and the measures + sync, max over ranks"}
        del pi, pi_h
        torch.cuda.empty_cache()

    # ---- secondary configs (same protocol, fewer steps)
    secondary = []
    for c in [int(x) for x in args.secondary.split(",") if x.strip()]:
        if c == args.config:
            continue
        i2 = hqinst.config_instance(c)
        m2 = measure(args, i2, min(args.steps, 5) if i2.N >= 26 else max(args.steps, 5), args.warmup, dev, dist)
        secondary.append({"config": workload_desc(i2, c), "value": m2["updates_tot"] / (m2["ms_max"] * 1e-3),
                          "unit": UNIT, "ms_per_step": m2["ms_max"] / len(m2["iters"]),
                          "time_to_tol_ms": statistics.median(m2["solve_ms"]),
                          "sweeps": statistics.median(m2["iters"]), "residual": max(m2["res"]),
                          "roofline": roofline_block(c, m2, len(m2["iters"]))})

    if rank != 0:
        return 0
    line = {"metric": METRIC, "value": m["updates_tot"] / (m["ms_max"] * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": m["ms_max"] / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded EMS-shaped instance, hqinst)",
            "config": arm_config(inst, args, world),
            "time_to_tol_ms": statistics.median(m["solve_ms"]), "sweeps": statistics.median(m["iters"]),
            "residual": max(m["res"]), "roofline": roofline_block(args.config, m, args.steps),
            "gpu_launches": int(m["launches"]), "e2e": e2e}
    if m["clocks"]:
        line["clocks"] = m["clocks"]
    if not args.no_cpu_baseline and world == 1:
        try:
            v, dt, cores, sample = cpu_sample(inst, args.config)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}
        except Exception as ex:  # the oracle is a reported baseline, never the product
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": None, "kind": "oracle",
                                    "sample": f"failed: {ex}"}
    if secondary:
        line["secondary"] = secondary
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
