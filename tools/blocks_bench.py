"""Sweep throughput of multi-qubit block circuits (qfs_create_blocks, NEXT-3)
vs the same-size two-qubit brick circuit, fixed M, CUDA-event timing
(qfs_bench_sweeps).  One JSON line per case.

    python tools/blocks_bench.py [n ...]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12866_b200 import build, inputs as I, qfs  # noqa: E402


def main():
    build.build()
    ns = [int(a) for a in sys.argv[1:]] or [6, 9, 12]
    for n in ns:
        k, s = 10 * n, 16
        m = min(32, 1 << n)
        qubits, arity, tgt, x, y, xv, yv, g0 = I.block_problem(n, k, s=s, m_pool=m, v=0, init="R")
        ctx = qfs.BlockContext(n, qubits, arity)
        ctx.set_samples(x, y)
        ctx.bench_sweeps(g0, m, 2)
        sweeps = 10
        sec = ctx.bench_sweeps(g0, m, sweeps)
        ctx.close()
        # streamed algorithmic bytes per start-sweep: forward write B 16 B per amp (K-1 gates),
        # backward per gate: chi apply 32 B + environment reads 32 B
        amps = m * (1 << n)
        byt = amps * (16 * (k - 1) + 64 * k)
        v = s * sweeps / sec
        print(json.dumps(dict(n=n, k=k, m=m, s=s, three_qubit_blocks=int((arity == 3).sum()),
                              start_sweeps_per_s=round(v, 1), ms_per_sweep=round(sec / sweeps * 1e3, 3),
                              algorithmic_gbs=round(v * byt / 1e9, 1))), flush=True)
        # two-qubit brick circuit of the same n, k, m through the pair path
        p = I.brick_pairs(n, k)
        rng = np.random.default_rng(1)
        gp = np.stack([[I.haar_unitary(rng) for _ in range(k)] for _ in range(s)])
        c2 = qfs.Context(n, p)
        c2.set_samples(x, y)
        c2.bench_sweeps(gp, m, 2)
        sec2 = c2.bench_sweeps(gp, m, sweeps)
        c2.close()
        print(json.dumps(dict(n=n, k=k, m=m, s=s, pairs_only=True,
                              start_sweeps_per_s=round(s * sweeps / sec2, 1))), flush=True)


if __name__ == "__main__":
    main()
