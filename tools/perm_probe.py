"""Per-gate environment error of the streamed sweep against the oracle on small
shapes (perm-mode layout debugging)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import oracle
from paper_2405_12866_b200 import inputs as I, qfs


def run(n, k, m, s, pool, brick=True, seed=1):
    rng = np.random.default_rng(seed)
    pairs = I.brick_pairs(n, k) if brick else I.c4_pairs(n, k, rng)
    target = np.stack([I.haar_unitary(rng) for _ in pairs])
    x = I.haar_states(rng, n, pool)
    y = I.apply_circuit_tensor(n, pairs, target, x)
    init = np.stack([np.stack([I.haar_unitary(rng) for _ in pairs]) for _ in range(s)])
    ctx = qfs.Context(n, pairs)
    ctx.set_path("streamed")
    ctx.set_samples(x, y)
    gt = ctx.trace_sweeps(init, m, 1)
    ot = oracle.trace_sweeps(n, pairs, init, x, y, m, 1)
    e = [float(np.abs(gt["env"][0, i] - ot["env"][0, i]).max() / np.abs(ot["env"][0, i]).max()) for i in range(k)]
    ctx.close()
    return e, pairs


for args in [(9, 4, 32, 1, 32), (10, 4, 32, 1, 32), (11, 4, 32, 1, 32), (12, 4, 32, 1, 32), (12, 4, 32, 1, 256),
             (9, 4, 32, 1, 256), (12, 4, 32, 2, 32), (12, 4, 16, 1, 16), (12, 3, 32, 1, 32), (12, 6, 64, 1, 64)]:
    e, pairs = run(*args)
    print(args, " ".join(f"{v:.1e}" for v in e), pairs.tolist(), flush=True)
