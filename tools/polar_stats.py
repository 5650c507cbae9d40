"""Diagnostic (build with QFS_NVCC_DEFINES=-DQFS_DIAG_POLAR): Jacobi sweeps and
cycles of the half-warp polar on cold random E and on near-unitary E."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12866_b200 import build, qfs, inputs as I

build.build(force=True)
rng = np.random.default_rng(1)
ctx = qfs.Context(2, [[0, 1]])
cnt = 256
G0 = np.stack([I.haar_unitary(rng) for _ in range(cnt)])
cases = {"random": rng.standard_normal((cnt, 4, 4)) + 1j * rng.standard_normal((cnt, 4, 4))}
for eps in (1e-1, 1e-3, 1e-6):
    cases[f"unitary+{eps:g}"] = 32 * G0 + eps * (rng.standard_normal((cnt, 4, 4)) + 1j * rng.standard_normal((cnt, 4, 4)))
for name, E in cases.items():
    _, s = ctx.op_polar(E, G0)
    sw = np.floor(s / 1e7); cyc = s - sw * 1e7
    print(f"{name:16s} sweeps mean {sw.mean():.2f} max {sw.max():.0f}  cycles mean {cyc.mean():.0f} "
          f"per sweep {np.mean(cyc / sw):.0f}")
