"""State-space sharding plan for N beyond one GPU.

Host-side plumbing only (partition, halo exchange, exact cross-rank sums); the sweep itself
stays in the CUDA kernels.  The paper's own parallel scheme (Algorithm 2, master/worker over
the states of a layer) rests on the two properties used here: the states of
a layer are independent, and a layer step needs only layers n - 1 and n + 1.

Partition.  With G = 2^s ranks, rank r owns every state whose top s bits of the compressed
index j = m >> 1 equal r (both parity classes): a sub-cube of 2^(N-1-s) compressed states per
class.  A neighbour m ^ e_u of a state is local for the N - s low units and lives on rank
r ^ 2^(u - (N - s)) for each of the s top units -- at the SAME local index.  So the halo of a
half-sweep along top unit u is the partner's whole slice of the read class, 8 B x 2^(N-1-s),
and the exchange is a pairwise swap (hypercube pattern, no all-to-all).

Scalars.  The per-layer sums of a half-sweep (sum p, sum p omega, sum p kappa
[, sum p lambda_m, |dp|]) are kept in the device loop's fixed-point format (HQ_XL 32-bit limbs
in 64-bit words); summing those integers across ranks with an all-reduce is exact and
independent of the reduction order, so every rank takes the same scalar step bit for bit.

Cost per half-sweep and rank (N = 33, G = 2: 2^31 states per rank): halo 8.6 GB over NVLink 5
(~900 GB/s per direction, ~10 ms) against ~40 ms of local sweep: overlappable by streaming the
tile-unit neighbour loads of the top unit from the partner's buffer (or peer memory) while
the low units are gathered.  One rank must hold 8 B (p) + 16 B (omega, kappa) + ~4 B (rate
programs) per owned state + the halo (8 B x 2^(N-1-s) per top unit): N = 31 needs ~77 GB on
one GPU; N = 32 ~154 GB (fits 180 GB, but the layer-slot arrays cap N at 31); N >= 33
requires s >= 1.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

HQ_XL = 5   # limbs of the exact per-layer sums (include/hq_v3.h)


@dataclasses.dataclass(frozen=True)
class ShardPlan:
    N: int          # units
    world: int      # ranks G = 2^s
    rank: int

    @property
    def s(self) -> int:
        s = int(math.log2(self.world))
        if 1 << s != self.world:
            raise ValueError("the number of ranks must be a power of two")
        if s > self.N - 10:
            raise ValueError("too many ranks for N: a rank must keep at least one CTA tile per class")
        return s

    @property
    def local_states(self) -> int:
        """compressed states per class on this rank"""
        return 1 << (self.N - 1 - self.s)

    @property
    def top_units(self) -> list:
        """(internal) units whose neighbours live on another rank, with that rank"""
        low = self.N - self.s
        return [(u, self.rank ^ (1 << (u - low))) for u in range(low, self.N)]

    def owner(self, j: int) -> tuple:
        """(rank, local index) of compressed index j"""
        return j >> (self.N - 1 - self.s), j & (self.local_states - 1)

    def global_index(self, local: np.ndarray) -> np.ndarray:
        return (np.uint64(self.rank) << np.uint64(self.N - 1 - self.s)) | local.astype(np.uint64)

    def halo_bytes_per_halfsweep(self) -> int:
        return 8 * self.local_states * self.s

    def rank_bytes(self, truncated: bool = False, prog_bytes_per_state: float = 4.0) -> float:
        """device memory of one rank: p, omega/kappa (+ lambda_m), programs, halo, caller's pi"""
        owned = 2 * self.local_states
        per = 8 + 16 + (8 if truncated else 0) + prog_bytes_per_state + 8
        return owned * per + self.halo_bytes_per_halfsweep()


def exchange_halo(plan: ShardPlan, read_class, group=None):
    """Swap the read class slice with every top-unit partner (pairwise send/recv in a fixed
    order: lower rank sends first).  Returns {unit: partner slice} (same dtype / device)."""
    import torch
    import torch.distributed as dist

    out = {}
    for u, partner in plan.top_units:
        buf = torch.empty_like(read_class)
        if plan.rank < partner:
            dist.send(read_class, partner, group=group)
            dist.recv(buf, partner, group=group)
        else:
            dist.recv(buf, partner, group=group)
            dist.send(read_class, partner, group=group)
        out[u] = buf
    return out


def to_limbs(x: float, xe: int) -> np.ndarray:
    """Fixed-point limbs of a sum x >= 0 (the device loop's xadd_g format, unit
    2^(xe - 32 HQ_XL)): the bits below the unit are dropped."""
    if x < 0 or not math.isfinite(x):
        raise ValueError("sums are non-negative and finite")
    v = int(math.floor(math.ldexp(x, 32 * HQ_XL - xe)))
    if v >> (32 * HQ_XL):
        raise OverflowError("sum out of range for xe")
    return np.array([(v >> (32 * k)) & 0xFFFFFFFF for k in range(HQ_XL)], dtype=np.int64)


def from_limbs(limbs: np.ndarray, xe: int) -> float:
    v = sum(int(limbs[k]) << (32 * k) for k in range(len(limbs)))
    return math.ldexp(float(v), xe - 32 * HQ_XL) if v.bit_length() <= 1000 else math.inf


def allreduce_exact(limbs, group=None):
    """Sum fixed-point limb vectors (int64 tensor [..., HQ_XL]) over the ranks: integer
    addition, so every rank gets the same bits whatever the reduction order."""
    import torch.distributed as dist

    dist.all_reduce(limbs, op=dist.ReduceOp.SUM, group=group)
    return limbs
