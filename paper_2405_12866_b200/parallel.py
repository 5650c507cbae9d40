"""Host-side multi-GPU logic for QFactor-Sample instantiation.

One process per GPU (torchrun), torch.distributed for the plumbing.  Two ways
the path shards:

* multistart (independent units, "multistarts"): rank r owns the starts
  ``start_slice(S, r, world)``; no data-path collective.  At the end the ranks
  all-gather their per-start results and every rank applies the same winner
  rule (lowest global start index among the earliest converged sweep, else the
  minimum c_train, ties to the lower index — DESIGN.md R16).
* sample axis (one exchange per gate): rank r holds the pool rows m with
  m ≡ r (mod world) (``sample_rows``), so every prefix of M rows splits evenly
  (M divisible by world); the partial environments are all-reduced per gate
  inside libqfs (``qfs_create_dist`` mode 1, NCCL).

This module is argument plumbing only: the arithmetic of the sweep runs in
libqfs (one ``Context`` per rank).  Engines are injected so the same host
logic can be exercised on CPU with the gloo backend (tests/test_parallel_gloo.py).
"""
from __future__ import annotations

import math
from typing import Callable, Sequence

import numpy as np


def start_slice(s_total: int, rank: int, world: int) -> range:
    """Contiguous block of global start indices owned by ``rank`` (balanced)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = s_total * rank // world
    hi = s_total * (rank + 1) // world
    return range(lo, hi)


def sample_rows(m_pool: int, rank: int, world: int) -> np.ndarray:
    """Pool rows held by ``rank`` in sample-sharded mode: m ≡ rank (mod world)."""
    if m_pool % world:
        raise ValueError("pool size must be divisible by world in sample mode")
    return np.arange(rank, m_pool, world)


def local_prefix(m_global: int, world: int) -> int:
    """Local rows of a global training prefix of ``m_global`` rows (QFS_ERR_CAPACITY otherwise)."""
    if m_global % world:
        raise ValueError("M must be divisible by world in sample mode")
    return m_global // world


TERM_RANK = {"CONVERGED": 0}


def select_winner(results: Sequence[dict]) -> int:
    """Winner rule over GLOBAL start order (R16).

    ``results[s]`` needs keys term, sweeps, c_train.  The converged start with
    the fewest sweeps (earliest converging global sweep: starts run in
    lockstep) and the lowest index wins; if none converged, the minimum
    c_train, ties to the lower index."""
    best, best_sweep = -1, math.inf
    for s, r in enumerate(results):
        if r["term"] == "CONVERGED" and r["sweeps"] < best_sweep:
            best, best_sweep = s, r["sweeps"]
    if best >= 0:
        return best
    vals = [r["c_train"] for r in results]
    return int(min(range(len(vals)), key=lambda s: (vals[s], s)))


def gather_results(local_results: list, local_gates: np.ndarray, rank: int, world: int, group=None):
    """All-gather per-start results and gates in global start order."""
    if world == 1:
        return list(local_results), np.asarray(local_gates)
    import torch.distributed as dist
    objs = [None] * world
    dist.all_gather_object(objs, (rank, list(local_results), np.asarray(local_gates)), group=group)
    objs.sort(key=lambda t: t[0])
    res, gates = [], []
    for _, r, g in objs:
        res.extend(r)
        gates.append(g)
    return res, np.concatenate(gates, axis=0)


def any_flag(local: bool, world: int, group=None) -> bool:
    """'Any converged' across ranks (allreduce MAX of an int)."""
    if world == 1:
        return bool(local)
    import torch
    import torch.distributed as dist
    t = torch.tensor([1 if local else 0], dtype=torch.int32)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return bool(t.item())


def run_multistart(engine: Callable[[np.ndarray, dict], tuple], init_all: np.ndarray, params: dict,
                   rank: int, world: int, group=None):
    """Multistart-sharded instantiation.

    ``engine(init_gates_local, params) -> (gates_local, results_local, winner_local)``
    is this rank's instantiation (libqfs ``Context.instantiate`` in production).
    Returns (global results, global gates, global winner), identical on all ranks.

    stop_on_first across ranks: each rank's engine already stops its own starts
    at its first converged sweep; a start of another rank converging later does
    not change the winner because the winner is taken over the global results by
    (earliest sweep, lowest index).  Results of ranks that ran past the global
    first converged sweep are reported as STOPPED there (their costs are those
    of their last sweep).
    """
    sl = start_slice(init_all.shape[0], rank, world)
    gates_l, res_l, _ = engine(np.ascontiguousarray(init_all[sl.start:sl.stop]), params)
    res, gates = gather_results(res_l, gates_l, rank, world, group)
    if params.get("stop_on_first", 0):
        conv = [r["sweeps"] for r in res if r["term"] == "CONVERGED"]
        if conv:
            first = min(conv)
            for r in res:
                if r["term"] == "CONVERGED" and r["sweeps"] > first:
                    r["term"] = "STOPPED"
    return res, gates, select_winner(res)
