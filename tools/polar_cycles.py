"""Diagnostic: cycles of the half-warp polar (qfs_op_polar) per environment
class, from a library built with -DQFS_DIAG_POLAR (sigma sum replaced by
path * 1e7 + clock64 cycles; path 100 = Newton-Schulz, else Jacobi sweeps).

    QFS_LIB=ab_so/libqfs_diag.so python tools/polar_cycles.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12866_b200 import inputs as I, qfs  # noqa: E402


def with_kappa(rng, cnt, kappa):
    out = []
    for _ in range(cnt):
        u, v = I.haar_unitary(rng), I.haar_unitary(rng)
        s = np.exp(np.linspace(0, -np.log(kappa), 4))
        out.append(u @ np.diag(s) @ v)
    return np.stack(out)


def main():
    rng = np.random.default_rng(1)
    ctx = qfs.Context(2, [[0, 1]])
    cnt = 512
    G0 = np.stack([I.haar_unitary(rng) for _ in range(cnt)])
    cases = {"random": rng.standard_normal((cnt, 4, 4)) + 1j * rng.standard_normal((cnt, 4, 4))}
    for kap in (1.05, 1.4, 1.8, 3.0):
        cases[f"kappa {kap}"] = with_kappa(rng, cnt, kap)
    for name, E in cases.items():
        _, s = ctx.op_polar(E, G0)
        path = np.floor(s / 1e7)
        cyc = s - path * 1e7
        ns = path == 100
        print(f"{name:12s} NS {ns.mean():.2f}  cycles NS mean {cyc[ns].mean() if ns.any() else 0:.0f}  "
              f"Jacobi mean {cyc[~ns].mean() if (~ns).any() else 0:.0f} (sweeps {path[~ns].mean() if (~ns).any() else 0:.1f})",
              flush=True)


if __name__ == "__main__":
    main()
