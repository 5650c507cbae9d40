"""NEXT-4 demo on the GPU: the gate-deletion pass over synthetic
partitions with constructed redundancy (U3 + CNOT templates plus identity
one-qubit gates next to a one-qubit gate on the same qubit), one partition
after another on one GPU (bench.py-style multi-GPU sharding of partitions is
resynth.resynth_partitions with p mod world).  Prints one JSON line per
partition: qubits, gates before/after, deletions, attempts, seconds."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12866_b200 import build, resynth as R, inputs as I  # noqa: E402

build.build()
prm = dict(dist_tol=1e-10, diff_tol_r=1e-3, plateau_window=5, min_iter=6, max_iter=300, m_init=4,
           overtrain_ratio=0.1, beta=0.0, stop_on_first=1)
for q, (n, layers, extra) in enumerate([(4, 4, 2), (5, 4, 3), (6, 5, 3), (7, 5, 4), (8, 6, 4), (9, 6, 4)]):
    b = R.redundant_block(n, layers, seed=100 + q, extra=extra)
    t0 = time.perf_counter()
    rep = R.delete_gates_pass(b, prm, starts=4, seed=q)
    dt = time.perf_counter() - t0
    u3 = lambda blk: int(np.sum(blk.kinds == I.GATE_VAR1))
    cx = lambda blk: int(np.sum(blk.kinds == I.GATE_FIXED))
    print(json.dumps(dict(partition=q, n=n, gates_before=b.k, gates_after=rep.block.k,
                          u3_before=u3(b), u3_after=u3(rep.block), cnot_before=cx(b), cnot_after=cx(rep.block),
                          constructed_redundant=extra, deleted=len(rep.deleted), attempts=rep.attempts,
                          seconds=round(dt, 3), instantiate_seconds=round(rep.instantiations_s, 3),
                          c_train=rep.c_train)), flush=True)

# all partitions at once from host threads (resynth_partitions(workers=...)): wall time
blocks = [R.redundant_block(n, layers, seed=100 + q, extra=extra)
          for q, (n, layers, extra) in enumerate([(4, 4, 2), (5, 4, 3), (6, 5, 3), (7, 5, 4), (8, 6, 4), (9, 6, 4)])]
for workers in (1, 6):
    t0 = time.perf_counter()
    out = R.resynth_partitions(blocks, prm, workers=workers, starts=4)
    dt = time.perf_counter() - t0
    print(json.dumps(dict(workers=workers, partitions=len(blocks), seconds=round(dt, 3),
                          deleted=[len(r.deleted) for _, r in out])), flush=True)
