"""QFactor (full unitary, M = 2^n) vs QFactor-Sample on B200 — SURVEY.md §8(f) NEXT-1.

The paper's central comparison (17.7x mean, 69x above 8 qubits, QF-J vs
QFS-J on A100) on synthetic solvable block circuits, both modes through the
same libqfs (qfs_instantiate):

  QF  : training inputs = the computational basis (M = 2^n: the sample
        cost is then the full Hilbert-Schmidt cost), IMPLICIT (qfs_set_samples_basis:
        x_m = e_m generated in the kernels, only y = U's columns stored), no
        validation, QFactor's single-iteration plateau rule (plateau_window = 1)
  QFS : Haar training states, number_of_training_states = 2, double-and-restart
        on overtrain_ratio = 0.1 with min(16, 2^n) validation states, plateau window 5

Hyperparameters: the paper's evaluation values: dist_tol 1e-10,
diff_tol_r 1e-3, min_iter 6, beta 0.  Circuits: brick wall of K = 4n Haar 4x4
blocks; S = 4 multistarts from W initial gates (target * exp(i eps H), eps 0.3)
so both modes can reach the target; stop at the first converged start.

    python tools/qf_vs_qfs.py [n ...]      -> one JSON line per n (stdout)
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12866_b200 import build, inputs as I, qfs  # noqa: E402

CFG = 40  # seed namespace of this tool


def problem(n, k, s):
    pairs = I.brick_pairs(n, k)
    target = np.stack([I.haar_unitary(I.rng_for(CFG + n, 0, j)) for j in range(k)])
    N = 1 << n
    init = np.stack([np.stack([I.warm_gate(I.rng_for(CFG + n, 3, st), target[j], 0.3) for j in range(k)])
                     for st in range(s)])
    basis = np.eye(N, dtype=np.complex128)
    qf = dict(y=I.apply_circuit_tensor(n, pairs, target, basis))
    del basis
    xs = I.haar_states(I.rng_for(CFG + n, 1, 0), n, min(N, 512))   # QFS pool (final M was <= 32 at n >= 9)
    xv = I.haar_states(I.rng_for(CFG + n, 2, 0), n, min(16, N))
    qs = dict(x=xs, y=I.apply_circuit_tensor(n, pairs, target, xs), xv=xv,
              yv=I.apply_circuit_tensor(n, pairs, target, xv))
    return pairs, init, qf, qs


def run(ctx, init, prm):
    ctx.instantiate(init, dict(prm, max_iter=2))  # graph shapes, warm
    t0 = time.perf_counter()
    g, res, w = ctx.instantiate(init, prm)
    dt = time.perf_counter() - t0
    r = res[w]
    return dict(seconds=round(dt, 4), sweeps=int(r["sweeps"]), term=r["term"], c_train=r["c_train"],
                final_m=int(r["final_m"]), restarts=int(r["restarts"]),
                converged=sum(x["term"] == "CONVERGED" for x in res))


def main():
    build.build()
    ns = [int(a) for a in sys.argv[1:]] or list(range(3, 14))
    base = dict(dist_tol=1e-10, diff_tol_r=1e-3, min_iter=6, max_iter=3000, beta=0.0, stop_on_first=1)
    for n in ns:
        k = 4 * n
        s = 4 if n <= 12 else 1   # n = 13: the QF B cache is (K-1) GB per start
        pairs, init, qf, qs = problem(n, k, s)
        N = 1 << n
        ctx = qfs.Context(n, pairs)
        ctx.set_samples_basis(qf["y"])
        r_qf = run(ctx, init, dict(base, plateau_window=1, m_init=N, overtrain_ratio=1e300))
        ctx.close()
        ctx = qfs.Context(n, pairs)
        ctx.set_samples(qs["x"], qs["y"], qs["xv"], qs["yv"])
        r_qs = run(ctx, init, dict(base, plateau_window=5, m_init=2, overtrain_ratio=0.1))
        ctx.close()
        print(json.dumps(dict(n=n, k=k, starts=s, qf=r_qf, qfs=r_qs,
                              speedup=round(r_qf["seconds"] / r_qs["seconds"], 2))), flush=True)


if __name__ == "__main__":
    main()
