"""Sweep throughput across partition sizes (north_star: "synthetic circuits
shaped like the paper's 3-14-qubit partitions"): brick-wall circuits with
K = 10 n blocks, M = 16 training states (capped at 2^n), 16 starts, R init,
fixed-M sweeps through qfs_bench_sweeps (CUDA events), on the auto path
(cluster-resident where the states fit) and the streamed path.
One JSON line per (n, path)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12866_b200 import build, inputs as I, qfs  # noqa: E402

build.build()
S = 16
for n in range(3, 15):
    K = 10 * n
    M = min(16, 1 << n)
    pairs = I.brick_pairs(n, K)
    rng = I.rng_for(90 + n, 0, 0)
    init = np.stack([np.stack([I.haar_unitary(rng) for _ in range(K)]) for _ in range(S)])
    x = I.haar_states(I.rng_for(90 + n, 1, 0), n, M)
    target = np.stack([I.haar_unitary(rng) for _ in range(K)])
    y = I.apply_circuit_tensor(n, pairs, target, x)
    for path in ("auto", "streamed"):
        ctx = qfs.Context(n, pairs)
        ctx.set_path(path)
        ctx.set_samples(x, y)
        ctx.bench_sweeps(init, M, 3)
        sweeps = 20 if n <= 12 else 5
        sec = ctx.bench_sweeps(init, M, sweeps)
        rate = S * sweeps / sec
        print(json.dumps(dict(n=n, k=K, m=M, starts=S, path=path, start_sweeps_per_s=round(rate, 1),
                              ms_per_sweep=round(sec / sweeps * 1e3, 4),
                              amp_gate_updates_per_s=rate * M * (1 << n) * K)), flush=True)
        ctx.close()
