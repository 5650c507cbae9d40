"""Seeded synthetic inputs for QFactor-Sample instantiation (harness side).

This module is the ONLY code shared by the CUDA path's tests/bench and the CPU
oracle's tests.  It draws random numbers and builds the problem the method is
asked to solve; it holds none of the method's arithmetic (no environment, no
SVD/polar update, no sweep, no cost).  Everything here is numpy.

What it builds (SURVEY.md §8(d) "Concrete inputs"; DESIGN.md §3 "Input recipe"):

* Haar-random 4x4 blocks: QR of a complex Gaussian, columns times the phases
  of diag(R) ("columns of a random unitary matrix"; SPEC.md
  S:82 construction).
* Training / validation states: the columns of a thin QR of an N x M complex
  Gaussian with the same phase fix, stored as rows ``[M][N]``
  ("randomly selecting M mutually orthogonal states", P:112
  "sampled from the Haar random distribution").
* Circuit structures of the BASELINE.json configs (C1..C5, C5b, C5c).
* Targets ``y = U x`` with U the product of the target blocks on the same
  structure (PAPER.md P:198 re-instantiate flow: "calculate its unitary, and
  ask QFactor-Sample to instantiate that unitary using the original partition
  circuit structure").  The harness applies U with a tensor-leg contraction
  (numpy tensordot over the reshaped ``(M, 2, ..., 2)`` state), a formulation
  independent of both the oracle's bit-insertion loops and the CUDA kernels;
  the method receives y as data (the A tensor of P:127), it never computes it.
* Initial gates: R = Haar blocks per start ("various initial gate
  unitaries"); W = warm start exp(i*eps*H) T_k.

Conventions (DESIGN.md §2 readings 1-4): little-endian amplitude index (bit q
of the index is qubit q); a gate on the ordered pair (p0, p1) acts on the local
index l = b(p0) + 2*b(p1); gate matrices are row-major ``[l_out][l_in]``.

Seeds: ``numpy.random.default_rng(SeedSequence([cfg, stream, idx]))`` with
stream 0 target blocks (idx = gate), 1 training pool, 2 validation set,
3 initial gates (idx = start), 4 random pairs.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "rng_for", "haar_unitary", "haar_states", "brick_pairs", "c4_pairs",
    "apply_circuit_tensor", "warm_gate", "Problem", "make_problem", "CONFIGS",
    "GATE_VAR2", "GATE_FIXED", "GATE_VAR1", "CNOT", "u3_cnot_template", "u3_cnot_problem",
]


def rng_for(cfg: int, stream: int, idx: int = 0) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(cfg), int(stream), int(idx)]))


def _complex_gaussian(rng: np.random.Generator, shape) -> np.ndarray:
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / math.sqrt(2.0)


def haar_unitary(rng: np.random.Generator, d: int = 4) -> np.ndarray:
    """Haar-random d x d unitary: QR of a complex Gaussian with phase-fixed R."""
    z = _complex_gaussian(rng, (d, d))
    q, r = np.linalg.qr(z)
    ph = np.diagonal(r) / np.abs(np.diagonal(r))
    return np.ascontiguousarray(q * ph[None, :])


def haar_states(rng: np.random.Generator, n: int, m: int) -> np.ndarray:
    """m mutually orthonormal Haar states on n qubits, as rows ``[m][2^n]``.

    The first m columns of a Haar unitary: thin QR of a 2^n x m complex
    Gaussian with the columns multiplied by the phases of diag(R).
    """
    N = 1 << n
    if m > N or m < 1:
        raise ValueError(f"need 1 <= m <= 2^n, got m={m}, n={n}")
    z = _complex_gaussian(rng, (N, m))
    q, r = np.linalg.qr(z, mode="reduced")
    ph = np.diagonal(r) / np.abs(np.diagonal(r))
    return np.ascontiguousarray((q * ph[None, :]).T)


def basis_states(rng: np.random.Generator, n: int, m: int) -> np.ndarray:
    """m distinct computational basis states (App. D)."""
    N = 1 << n
    idx = rng.choice(N, size=m, replace=False)
    out = np.zeros((m, N), dtype=np.complex128)
    out[np.arange(m), idx] = 1.0
    return out


def brick_pairs(n: int, k: int) -> np.ndarray:
    """Brick-wall layout of adjacent pairs (SURVEY.md §8(c) reading 20).

    Layer l has the pairs (q, q+1) for q = l mod 2, l mod 2 + 2, ... < n-1;
    layers are concatenated and the stream is truncated to k gates.
    """
    out = []
    layer = 0
    while len(out) < k:
        for q in range(layer % 2, n - 1, 2):
            out.append((q, q + 1))
        layer += 1
    return np.asarray(out[:k], dtype=np.int32)


def c4_pairs(n: int, k: int, rng: np.random.Generator) -> np.ndarray:
    """Brick wall plus seeded random non-adjacent pairs (reading 20).

    Slot j with j mod 5 == 4 takes a random pair (a, b), a < b, b - a >= 2;
    the other slots take the brick stream in order.
    """
    n_rand = sum(1 for j in range(k) if j % 5 == 4)
    brick = list(map(tuple, brick_pairs(n, k - n_rand)))
    out = []
    bi = 0
    for j in range(k):
        if j % 5 == 4:
            while True:
                a, b = sorted(int(v) for v in rng.choice(n, size=2, replace=False))
                if b - a >= 2:
                    break
            out.append((a, b))
        else:
            out.append(brick[bi])
            bi += 1
    return np.asarray(out, dtype=np.int32)


def apply_circuit_tensor(n: int, pairs: np.ndarray, gates: np.ndarray, states: np.ndarray) -> np.ndarray:
    """Harness simulator: returns C states (rows), C = G_{K-1} ... G_0.

    States are reshaped to ``(M, 2, ..., 2)``; with little-endian indices the
    C-order axis of qubit q is ``1 + (n - 1 - q)``.  A gate matrix G[l_out][l_in]
    with l = b(p0) + 2 b(p1) is the tensor ``G4[o1, o0, i1, i0]``.
    """
    m = states.shape[0]
    psi = np.asarray(states, dtype=np.complex128).reshape((m,) + (2,) * n)
    for (p0, p1), g in zip(np.asarray(pairs), np.asarray(gates)):
        a0, a1 = 1 + (n - 1 - int(p0)), 1 + (n - 1 - int(p1))
        g4 = np.asarray(g, dtype=np.complex128).reshape(2, 2, 2, 2)
        res = np.tensordot(psi, g4, axes=([a1, a0], [2, 3]))
        psi = np.moveaxis(res, [-2, -1], [a1, a0])
    return np.ascontiguousarray(psi.reshape(m, 1 << n))


def warm_gate(rng: np.random.Generator, target: np.ndarray, eps: float) -> np.ndarray:
    """exp(i*eps*H) @ target with H = (A + A^dag)/2 scaled to spectral norm 1."""
    a = _complex_gaussian(rng, (4, 4))
    h = 0.5 * (a + a.conj().T)
    w, v = np.linalg.eigh(h)
    w = w / np.max(np.abs(w))
    ex = (v * np.exp(1j * eps * w)[None, :]) @ v.conj().T
    return ex @ target


@dataclasses.dataclass
class Problem:
    """One synthetic instantiation problem (all arrays complex128, C-contiguous)."""
    name: str
    n: int
    pairs: np.ndarray          # int32 [K][2]
    target: np.ndarray         # [K][4][4] target blocks (harness only)
    x: np.ndarray              # [m_pool][N] training pool
    y: np.ndarray              # [m_pool][N] = U x
    xv: np.ndarray             # [V][N] validation inputs
    yv: np.ndarray             # [V][N] = U xv
    init: np.ndarray           # [S][K][4][4] initial gates
    m_init: int
    params: dict

    @property
    def k(self) -> int:
        return int(self.pairs.shape[0])

    @property
    def s(self) -> int:
        return int(self.init.shape[0])


# BASELINE.json configs, concretised in SURVEY.md §8(d).  Fields:
# n, K, structure, m_init, m_pool, V, S, otr, window, max_iter.
CONFIGS = {
    "c1": dict(cfg=1, n=3, k=4, structure="c1", m_init=4, m_pool=4, v=0, s=1,
               otr=math.inf, window=0, max_iter=500),
    "c2": dict(cfg=2, n=6, k=20, structure="brick", m_init=8, m_pool=64, v=16, s=32,
               otr=0.1, window=5, max_iter=2000),
    "c3": dict(cfg=3, n=9, k=60, structure="brick", m_init=16, m_pool=512, v=16, s=64,
               otr=0.1, window=5, max_iter=2000),
    "c4": dict(cfg=4, n=12, k=150, structure="c4", m_init=32, m_pool=256, v=16, s=16,
               otr=0.1, window=5, max_iter=2000),
    "c5": dict(cfg=5, n=14, k=300, structure="brick", m_init=64, m_pool=64, v=16, s=1,
               otr=math.inf, window=5, max_iter=2000, w_eps=0.1),
    "c5b": dict(cfg=6, n=10, k=100, structure="brick", m_init=16, m_pool=128, v=16, s=1,
                otr=0.1, window=5, max_iter=2000),
    "c5c": dict(cfg=7, n=10, k=100, structure="brick", m_init=16, m_pool=128, v=16, s=64,
                otr=0.1, window=5, max_iter=2000),
}


def make_problem(name: str, init: str = "R", s: int | None = None, m_pool: int | None = None,
                 v: int | None = None, k: int | None = None, eps: float | None = None,
                 m_init: int | None = None) -> Problem:
    """Build config ``name`` (optionally reduced: fewer starts / gates / pool rows).

    W init strength: eps = 0.3 by default; C5 (K = 300) uses 0.1, since the
    per-gate perturbations compound over 300 blocks (eps = 0.3 starts at a
    near-random cost of 1.93 and plateaus)."""
    c = dict(CONFIGS[name])
    if eps is None:
        eps = c.get("w_eps", 0.3)
    cfg, n = c["cfg"], c["n"]
    kk = c["k"] if k is None else int(k)
    if c["structure"] == "c1":
        pairs = np.asarray([(0, 1), (1, 2), (0, 1), (1, 2)], dtype=np.int32)[:kk]
    elif c["structure"] == "brick":
        pairs = brick_pairs(n, kk)
    else:
        pairs = c4_pairs(n, kk, rng_for(cfg, 4, 0))
    target = np.stack([haar_unitary(rng_for(cfg, 0, j)) for j in range(kk)])
    mp = c["m_pool"] if m_pool is None else int(m_pool)
    vv = c["v"] if v is None else int(v)
    x = haar_states(rng_for(cfg, 1, 0), n, mp)
    y = apply_circuit_tensor(n, pairs, target, x)
    if vv > 0:
        xv = haar_states(rng_for(cfg, 2, 0), n, vv)
        yv = apply_circuit_tensor(n, pairs, target, xv)
    else:
        xv = np.zeros((0, 1 << n), dtype=np.complex128)
        yv = np.zeros((0, 1 << n), dtype=np.complex128)
    ss = c["s"] if s is None else int(s)
    gates = np.empty((ss, kk, 4, 4), dtype=np.complex128)
    for st in range(ss):
        rng = rng_for(cfg, 3, st)
        for j in range(kk):
            if init == "R":
                gates[st, j] = haar_unitary(rng)
            elif init == "W":
                gates[st, j] = warm_gate(rng, target[j], eps)
            elif init == "T":        # exact initialisation (fixed-point tests)
                gates[st, j] = target[j]
            else:
                raise ValueError(init)
    mi = min(c["m_init"], mp) if m_init is None else int(m_init)
    params = dict(dist_tol=1e-8, diff_tol_r=1e-3, plateau_window=c["window"], min_iter=6,
                  max_iter=c["max_iter"], m_init=mi, overtrain_ratio=c["otr"], beta=0.0,
                  stop_on_first=1)
    return Problem(name=name, n=n, pairs=pairs, target=target, x=x, y=y, xv=xv, yv=yv,
                   init=gates, m_init=mi, params=params)


# ------------------------------------------------ U3 + CNOT templates (NEXT-3) --
# Gate kinds of qfs_set_gate_kinds / the oracle's *_kinds entry points: a
# two-qubit variable block, a fixed gate, and a one-qubit variable gate u on the
# pair's first qubit stored as the block u (x) I (readings R24-R25).
GATE_VAR2, GATE_FIXED, GATE_VAR1 = 0, 1, 2

# CNOT with control p0 and target p1 in the local index l = b(p0) + 2 b(p1):
# |b0 b1> -> |b0, b1 xor b0>, i.e. l: 0->0, 1->3, 2->2, 3->1; G[l_out][l_in].
CNOT = np.zeros((4, 4), dtype=np.complex128)
for _li, _lo in ((0, 0), (1, 3), (2, 2), (3, 1)):
    CNOT[_lo, _li] = 1.0


def u3_cnot_template(n: int, layers: int):
    """The paper's circuit template (Table 1: U3 + CNOT): on every brick-wall
    pair (q, q+1) of every layer, a one-qubit variable gate on q, one on q+1,
    then a fixed CNOT(q -> q+1).  Returns (pairs [K][2], kinds [K])."""
    pairs, kinds = [], []
    for layer in range(layers):
        for q in range(layer % 2, n - 1, 2):
            pairs += [(q, q + 1), (q + 1, q), (q, q + 1)]
            kinds += [GATE_VAR1, GATE_VAR1, GATE_FIXED]
    return np.asarray(pairs, dtype=np.int32), np.asarray(kinds, dtype=np.int32)


def _embed1(u: np.ndarray) -> np.ndarray:
    """u (x) I in the block's local index l = b(p0) + 2 b(p1)."""
    g = np.zeros((4, 4), dtype=np.complex128)
    for lo in range(4):
        for li in range(4):
            if lo >> 1 == li >> 1:
                g[lo, li] = u[lo & 1, li & 1]
    return g


def u3_cnot_problem(n: int, layers: int, s: int, m_pool: int, v: int, init: str = "W",
                    eps: float = 0.3, seed: int = 11) -> tuple:
    """Solvable U3 + CNOT instance: target = the template with seeded Haar 2x2
    gates; W initial gates = exp(i eps H) u_target (2x2) per one-qubit slot, the
    CNOTs as given.  Returns (pairs, kinds, target [K][4][4], x, y, xv, yv, init)."""
    pairs, kinds = u3_cnot_template(n, layers)
    k = len(kinds)
    target = np.stack([_embed1(haar_unitary(rng_for(seed, 0, j), 2)) if kinds[j] == GATE_VAR1 else CNOT
                       for j in range(k)])
    x = haar_states(rng_for(seed, 1, 0), n, m_pool)
    y = apply_circuit_tensor(n, pairs, target, x)
    xv = haar_states(rng_for(seed, 2, 0), n, v) if v else np.zeros((0, 1 << n), np.complex128)
    yv = apply_circuit_tensor(n, pairs, target, xv) if v else xv.copy()
    gates = np.empty((s, k, 4, 4), dtype=np.complex128)
    for st in range(s):
        rng = rng_for(seed, 3, st)
        for j in range(k):
            if kinds[j] != GATE_VAR1:
                gates[st, j] = target[j]
            elif init == "W":
                a = _complex_gaussian(rng, (2, 2))
                h = 0.5 * (a + a.conj().T)
                w, vv = np.linalg.eigh(h)
                w = w / np.max(np.abs(w))
                gates[st, j] = _embed1((vv * np.exp(1j * eps * w)[None, :]) @ vv.conj().T @ target[j][:2, :2])
            else:
                gates[st, j] = _embed1(haar_unitary(rng, 2))
    return pairs, kinds, target, x, y, xv, yv, gates


# ------------------------------------------------------- multi-qubit blocks --
# Circuits of 2- and 3-qubit blocks ("possibly
# multi-qubit" gates).  Gate k acts on qubits[k][:arity[k]] (local index
# l = sum_j b(q_j) 2^j, first listed qubit least significant) with a d x d
# matrix, d = 2^arity; a circuit's gates are stored PACKED: gate k at complex
# offset off_k = sum_{j<k} d_j^2 (the layout of qfs_create_blocks and the
# oracle's *_blocks functions).  Layout helpers and the harness simulator only.

def gate_offsets(arity) -> np.ndarray:
    d2 = [1 << (2 * int(a)) for a in np.asarray(arity).reshape(-1)]
    return np.concatenate([[0], np.cumsum(d2)]).astype(np.int64)


def pack_gates(mats) -> np.ndarray:
    return np.concatenate([np.asarray(g, dtype=np.complex128).reshape(-1) for g in mats])


def unpack_gates(vec, arity) -> list:
    off = gate_offsets(arity)
    out = []
    for k, a in enumerate(np.asarray(arity).reshape(-1)):
        d = 1 << int(a)
        out.append(np.asarray(vec[off[k]:off[k + 1]]).reshape(d, d))
    return out


def apply_blocks_tensor(n: int, qubits, arity, packed, states: np.ndarray) -> np.ndarray:
    """Harness simulator for block circuits (tensordot, like apply_circuit_tensor):
    a gate on (q_0, .., q_{a-1}) with l = sum_j b(q_j) 2^j is the tensor
    G[o_{a-1}, .., o_0, i_{a-1}, .., i_0]."""
    m = states.shape[0]
    psi = np.asarray(states, dtype=np.complex128).reshape((m,) + (2,) * n)
    for q, a, g in zip(np.asarray(qubits).reshape(-1, 3), np.asarray(arity).reshape(-1),
                       unpack_gates(packed, arity)):
        a = int(a)
        axes = [1 + (n - 1 - int(q[j])) for j in range(a)][::-1]  # tensor order: q_{a-1} .. q_0
        ga = g.reshape((2,) * (2 * a))
        res = np.tensordot(psi, ga, axes=(axes, list(range(a, 2 * a))))
        psi = np.moveaxis(res, list(range(-a, 0)), axes)
    return np.ascontiguousarray(psi.reshape(m, 1 << n))


def block_structure(n: int, k: int, seed: int = 0):
    """Synthetic mixed circuit: every third slot a two-qubit block on an
    adjacent pair, the others three-qubit blocks on (q, q+1, q+2) sliding by
    two, each block's qubit list in a seeded order.  Returns (qubits [k][3]
    int32, arity [k] int32)."""
    if n < 3:
        raise ValueError("three-qubit blocks need n >= 3")
    rng = rng_for(seed, 4, 0)
    qubits = np.zeros((k, 3), np.int32)
    arity = np.zeros(k, np.int32)
    for j in range(k):
        if j % 3 == 2:
            q = (j * 3 + 1) % (n - 1)
            qs = [q, q + 1]
        else:
            q = (2 * j) % (n - 2)
            qs = [q, q + 1, q + 2]
        qs = list(rng.permutation(qs))
        arity[j] = len(qs)
        qubits[j, :len(qs)] = qs
    return qubits, arity


def warm_gate_d(rng: np.random.Generator, target: np.ndarray, eps: float) -> np.ndarray:
    """exp(i*eps*H) @ target (any d) with H = (A + A^dag)/2 scaled to spectral norm 1."""
    d = target.shape[0]
    a = _complex_gaussian(rng, (d, d))
    h = 0.5 * (a + a.conj().T)
    w, v = np.linalg.eigh(h)
    w = w / np.max(np.abs(w))
    return (v * np.exp(1j * eps * w)[None, :]) @ v.conj().T @ target


def block_problem(n: int, k: int, s: int, m_pool: int, v: int = 16, init: str = "W", eps: float = 0.3,
                  seed: int = 21):
    """Solvable block-circuit instance: target = seeded Haar blocks on
    block_structure(n, k); W initial gates = exp(i eps H) target per block, R =
    Haar.  Returns (qubits, arity, target packed [G], x, y, xv, yv, init [s][G])."""
    qubits, arity = block_structure(n, k, seed)
    target = pack_gates([haar_unitary(rng_for(seed, 0, j), 1 << int(a)) for j, a in enumerate(arity)])
    x = haar_states(rng_for(seed, 1, 0), n, m_pool)
    y = apply_blocks_tensor(n, qubits, arity, target, x)
    xv = haar_states(rng_for(seed, 2, 0), n, v) if v else np.zeros((0, 1 << n), np.complex128)
    yv = apply_blocks_tensor(n, qubits, arity, target, xv) if v else xv.copy()
    tg = unpack_gates(target, arity)
    gates = []
    for st in range(s):
        rng = rng_for(seed, 3, st)
        if init == "W":
            gates.append(pack_gates([warm_gate_d(rng, t, eps) for t in tg]))
        else:
            gates.append(pack_gates([haar_unitary(rng, t.shape[0]) for t in tg]))
    return qubits, arity, target, x, y, xv, yv, np.stack(gates)
