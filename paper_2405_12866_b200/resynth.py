"""Gate-deletion re-instantiation of circuit partitions.

The paper's second workload (Table 2): a large circuit is cut into
small partitions; for each partition, "a uni-directional sweep aimed at
deleting one gate at a time while re-instantiating the reduced partition to
its original unitary form".  Partitions are independent, so they are
spread over GPUs (one process per GPU; partition p goes to rank p mod world)
with no collective on the data path.

This module is host logic only: every instantiation runs through libqfs
(``qfs.Context.instantiate``) on the GPU; the partitioner itself is out of
scope (an external tool in the paper), so callers pass partitions
as (n, pairs, kinds, gates) blocks.  Readings (SPEC-style, the paper is
terse): a deletion is kept only when the reduced block CONVERGES (the P:188
success condition, not merely a low cost); the sweep is single-pass, left to
right, no retry of earlier gates; fixed gates may be deleted like any other
(Table 2 counts CNOT deletions); the reduced block starts from the current
gates (start 0) plus seeded Haar multistarts.
"""
from __future__ import annotations

import dataclasses
import time
from typing import Callable, List, Sequence

import numpy as np

from . import inputs as I


@dataclasses.dataclass
class Block:
    """One partition: n qubits, K gates on pairs with kinds, gate matrices."""
    n: int
    pairs: np.ndarray   # int32 [K][2]
    kinds: np.ndarray   # int32 [K] (inputs.GATE_*)
    gates: np.ndarray   # complex128 [K][4][4]

    @property
    def k(self) -> int:
        return int(self.pairs.shape[0])


@dataclasses.dataclass
class DeletionReport:
    kept: List[int]          # original indices of the gates that remain
    deleted: List[int]       # original indices deleted, in deletion order
    attempts: int
    instantiations_s: float  # wall time inside instantiate calls
    c_train: float           # training cost of the final block
    block: Block


def _samples(n: int, m: int, v: int, seed: int):
    x = I.haar_states(I.rng_for(seed, 1, 0), n, m)
    xv = I.haar_states(I.rng_for(seed, 2, 0), n, v)
    return x, xv


def _local_device() -> int:
    """This process's GPU: LOCAL_RANK under torchrun (one process per GPU), else 0."""
    import os
    return int(os.environ.get("LOCAL_RANK", "0"))


def delete_gates_pass(block: Block, params: dict, starts: int = 4, m_pool: int | None = None,
                      v: int = 16, seed: int = 0, context_factory: Callable | None = None,
                      device: int | None = None) -> DeletionReport:
    """Single left-to-right pass: tentatively remove each gate and keep the
    removal if the reduced block re-instantiates (CONVERGED) to the original
    block's action on the training states (the re-instantiate protocol of P:198).

    ``context_factory(n, pairs)`` returns a fresh qfs.Context (default: the GPU
    library on ``device``, default LOCAL_RANK); ``params`` are qfs_instantiate
    parameters (m_init, dist_tol, ...)."""
    shared = None
    dev = _local_device() if device is None else int(device)
    if context_factory is None:
        # one GPU context per partition: each attempt swaps the structure in
        # (qfs_set_structure) and keeps the samples and device buffers
        from . import qfs
        shared = {}

        def context_factory(n, pairs):
            if "ctx" not in shared:
                shared["ctx"] = qfs.Context(n, pairs, device=dev)
                shared["fresh"] = True
            else:
                shared["ctx"].set_structure(pairs)
                shared["fresh"] = False
            return shared["ctx"]
    n = block.n
    N = 1 << n
    m_pool = min(N, m_pool or N)
    x, xv = _samples(n, m_pool, min(v, N), seed)
    y = I.apply_circuit_tensor(n, block.pairs, block.gates, x)
    yv = I.apply_circuit_tensor(n, block.pairs, block.gates, xv)
    idx = list(range(block.k))
    cur_gates = np.array(block.gates)
    deleted: List[int] = []
    attempts, t_inst, c_last = 0, 0.0, float("nan")
    pos = 0
    while pos < len(idx):
        trial = idx[:pos] + idx[pos + 1:]
        if not trial:
            break
        attempts += 1
        pairs = block.pairs[trial]
        kinds = block.kinds[trial]
        keep = [q for q in range(len(idx)) if q != pos]
        init = np.empty((starts, len(trial), 4, 4), dtype=np.complex128)
        init[0] = cur_gates[keep]
        rng = I.rng_for(seed, 5, attempts)
        for st in range(1, starts):
            for j, kd in enumerate(kinds):
                if kd == I.GATE_FIXED:
                    init[st, j] = block.gates[trial[j]]
                elif kd == I.GATE_VAR1:
                    init[st, j] = I._embed1(I.haar_unitary(rng, 2))
                else:
                    init[st, j] = I.haar_unitary(rng)
        ctx = context_factory(n, pairs)
        try:
            if hasattr(ctx, "set_gate_kinds"):
                ctx.set_gate_kinds(kinds)
            if shared is None or shared["fresh"]:  # the samples stay on a shared context
                ctx.set_samples(x, y, xv, yv)
            t0 = time.perf_counter()
            g, res, win = ctx.instantiate(init, params)
            t_inst += time.perf_counter() - t0
        finally:
            if shared is None and hasattr(ctx, "close"):
                ctx.close()
        if res[win]["term"] == "CONVERGED":
            deleted.append(idx[pos])
            idx = trial
            cur_gates = np.asarray(g[win])
            c_last = res[win]["c_train"]
        else:
            pos += 1
    if shared and "ctx" in shared:
        shared["ctx"].close()
    out = Block(n=n, pairs=block.pairs[idx], kinds=block.kinds[idx], gates=cur_gates)
    return DeletionReport(kept=idx, deleted=deleted, attempts=attempts, instantiations_s=t_inst,
                          c_train=c_last, block=out)


def partitions_for_rank(n_parts: int, rank: int, world: int) -> List[int]:
    """Partition p is processed by rank p mod world (independent units, no collective)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_parts, world))


def resynth_partitions(blocks: Sequence[Block], params: dict, rank: int = 0, world: int = 1,
                       gather: Callable | None = None, workers: int = 1, **kw) -> list:
    """Run delete_gates_pass on this rank's partitions; ``gather`` (e.g. a
    torch.distributed all_gather_object wrapper) merges the per-rank reports
    into partition order.  ``workers`` > 1 runs that many partitions at once
    from host threads (each with its own contexts and stream; small
    partitions are latency-bound, so they overlap on one GPU).  Returns
    [(partition index, DeletionReport)]."""
    parts = partitions_for_rank(len(blocks), rank, world)
    if workers > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=workers) as ex:
            reps = list(ex.map(lambda p: delete_gates_pass(blocks[p], params, seed=p, **kw), parts))
        mine = list(zip(parts, reps))
    else:
        mine = [(p, delete_gates_pass(blocks[p], params, seed=p, **kw)) for p in parts]
    if gather is None or world == 1:
        return mine
    allr = gather(mine)
    return sorted((item for part in allr for item in part), key=lambda t: t[0])


def redundant_block(n: int, layers: int, seed: int, extra: int = 2) -> Block:
    """Synthetic partition with known redundancy (stand-in for Table 1's
    circuits, which are not in this container): a U3 + CNOT template with
    ``extra`` additional one-qubit gates, each placed right after a template
    one-qubit gate on the same qubit and set to the identity in the target —
    one of each such adjacent pair is deletable by construction (two
    consecutive one-qubit unitaries on a qubit merge into one)."""
    pairs, kinds = I.u3_cnot_template(n, layers)
    pairs, kinds = [tuple(map(int, p)) for p in pairs], [int(k) for k in kinds]
    rng = I.rng_for(seed, 0, 0)
    gates = [I._embed1(I.haar_unitary(rng, 2)) if kd == I.GATE_VAR1 else I.CNOT for kd in kinds]
    var1 = [j for j, kd in enumerate(kinds) if kd == I.GATE_VAR1]
    picks = sorted(rng.choice(len(var1), size=min(extra, len(var1)), replace=False))
    for off, v in enumerate(picks):
        j = var1[v] + off + 1                  # right after it (earlier insertions shift indices)
        pairs.insert(j, pairs[j - 1])
        kinds.insert(j, I.GATE_VAR1)
        gates.insert(j, np.eye(4, dtype=np.complex128))
    return Block(n=n, pairs=np.asarray(pairs, np.int32), kinds=np.asarray(kinds, np.int32),
                 gates=np.stack(gates))
