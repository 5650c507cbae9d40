"""Brute-force dense helpers for the oracle pins (tests only, n <= ~5).

Independent of the oracle's bit-insertion loops and of the harness's tensordot
simulator: a gate on (p0, p1) is embedded as Pi^T (I (x) G) Pi, where Pi is the
qubit-relabelling permutation matrix that moves qubit p0 to position 0 and p1 to
position 1 (built by transposing the axes of the identity reshaped to a
(2,)*n tensor), and (I (x) G) is np.kron.  Little-endian indices: the C-order
axis of qubit q in a (2,)*n reshape is n-1-q.
"""
import numpy as np


def _perm_matrix(n, order):
    """Matrix P with (P psi) having qubit order[j] moved to position j."""
    N = 1 << n
    eye = np.eye(N, dtype=np.complex128)
    cols = eye.reshape((N,) + (2,) * n)
    # new axis for position j (C-order axis n-1-j) takes old axis of qubit order[j]
    src_axes = [1 + (n - 1 - order[n - 1 - a]) for a in range(n)]
    moved = np.transpose(cols, [0] + src_axes)
    return moved.reshape(N, N).T


def embed(n, p0, p1, g):
    """Dense 2^n x 2^n matrix of a 4x4 gate g[l_out][l_in] on the ordered pair (p0, p1)."""
    rest = [q for q in range(n) if q not in (p0, p1)]
    order = [p0, p1] + rest
    P = _perm_matrix(n, order)
    big = np.kron(np.eye(1 << (n - 2)), np.asarray(g, dtype=np.complex128))
    return P.T @ big @ P


def circuit_matrix(n, pairs, gates):
    """Dense C = G_{K-1} ... G_0."""
    C = np.eye(1 << n, dtype=np.complex128)
    for (p0, p1), g in zip(pairs, gates):
        C = embed(n, int(p0), int(p1), g) @ C
    return C


def random_unitary(rng, d=4):
    z = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))[None, :]


def random_complex(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
