"""Probe the bulk-copy backward kernel on small shapes, each case in its own
process under a hard timeout (a hang is reported, not waited out).

    python tools/bt_probe.py [timeout_s]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASE = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import oracle
from paper_2405_12866_b200 import inputs as I, qfs
n, k, m, s, inst = map(int, sys.argv[2:7])
rng = np.random.default_rng(1)
pairs = I.brick_pairs(n, k)
target = np.stack([I.haar_unitary(rng) for _ in pairs])
x = I.haar_states(rng, n, m)
y = I.apply_circuit_tensor(n, pairs, target, x)
init = np.stack([np.stack([I.haar_unitary(rng) for _ in pairs]) for _ in range(s)])
ctx = qfs.Context(n, pairs)
ctx.set_path("streamed")
xv = I.haar_states(rng, n, 16)
yv = I.apply_circuit_tensor(n, pairs, target, xv)
ctx.set_samples(x, y, xv, yv)
if inst:
    prm = dict(dist_tol=-1.0, diff_tol_r=1e-3, plateau_window=0, min_iter=10**6, max_iter=inst, m_init=m,
               overtrain_ratio=1e300, beta=0.0, stop_on_first=0)
    g, r, w = ctx.instantiate(init, prm)
    print("inst", r[0])
    sys.exit(0)
gt = ctx.trace_sweeps(init, m, 1)
ot = oracle.trace_sweeps(n, pairs, init, x, y, m, 1, threads=min(s, 8))
err = np.abs(gt["env"] - ot["env"]).max() / np.abs(ot["env"]).max()
print("err", err)
"""

CASES = [  # n, K, M, S, instantiate sweeps (0: one trace sweep), extra env
    (14, 300, 64, 1, 0, {}),
    (14, 300, 64, 1, 3, {}),
    (14, 300, 64, 1, 3, {}),
    (14, 300, 32, 2, 3, {}),
    (12, 150, 32, 16, 3, {}),
    (12, 150, 64, 16, 3, {}),
]


def main():
    to = float(sys.argv[1]) if len(sys.argv) > 1 else 60
    for n, k, m, s, inst, env in CASES:
        e = dict(os.environ, **env)
        try:
            r = subprocess.run([sys.executable, "-c", CASE, ROOT, str(n), str(k), str(m), str(s), str(inst)], env=e,
                               capture_output=True, text=True, timeout=to)
            out = (r.stdout.strip().splitlines() or ["?"])[-1]
            print(f"n={n} K={k} M={m} S={s} inst={inst} {env}: rc={r.returncode} {out} {r.stderr.strip()[-300:]}", flush=True)
        except subprocess.TimeoutExpired:
            print(f"n={n} K={k} M={m} S={s} inst={inst} {env}: HANG (> {to} s)", flush=True)


if __name__ == "__main__":
    main()
