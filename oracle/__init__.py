"""CPU oracle for QFactor-Sample instantiation — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA product path (``paper_2405_12866_b200``); it loads its own plain C++17
library ``oracle/libqfs_oracle.so`` built from ``oracle/qfso.cpp``.

Pin of each function (DESIGN.md §6 lists them; every pin compares with
something other than the oracle itself):
  apply_gate        dense Kronecker embeddings (n <= 4, all ordered pairs), CNOT / X
                    truth tables (tests/golden), SWAP identity, norm, inverse
  circuit_forward   dense product of embedded gates; the tensordot harness
  environment       brute-force d^2 probe circuits; K=1 full-basis closed form E = U^dag;
                    Tr(E I) = M at the perfect match
  svd4 / polar_update / newton_polar
                    LAPACK singular values and polar factor, von Neumann optimality vs
                    1000 random unitaries, beta = 1 -> no update, golden svd_known.json
  distance          closed forms (CNOT vs identity golden cost; M = 2^n Hilbert-Schmidt
                    identity eq:qfactor_cost_func <-> eq:qfactor_sample_cost_function)
  trace_sweeps      chain invariant, per-gate monotone cost, exact-initialisation
                    fixed point, one-sweep solutions, g-shard emulation
  instantiate       controller replays (PLATEAU at sweep 6, restart geometry,
                    POOL_EXHAUSTED, MAX_ITER), winner rule (earliest, then lowest
                    index, min c_train) on constructed multistarts, c_train and the
                    validation cost (validation_cost: post-sweep gates, / V) against a
                    dense U and C (n = 5), warm convergence, generalisation statistic
  *_block / *_blocks  (multi-qubit blocks) tests/test_blocks_oracle.py: dense
                    embeddings from the index definition, probe circuits, LAPACK, the
                    pair oracle; validation_cost_blocks against a dense U and C
  Long-run trajectories beyond the first sweeps on hard landscapes: parity
  unpinned (same termination class + final-cost tolerance only).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqfs_oracle.so")
SRC = os.path.join(_HERE, "qfso.cpp")

TERM_NAMES = {0: "CONVERGED", 1: "PLATEAU", 2: "MAX_ITER", 3: "POOL_EXHAUSTED", 4: "STOPPED"}


def build(force: bool = False) -> str:
    """Compile the oracle (plain C++17, -O2, no -ffast-math, OpenMP over starts)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(_HERE, "qfso.h"))):
        tmp = f"{LIB_PATH}.tmp{os.getpid()}"
        cmd = ["g++", "-std=c++17", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wall",
               "-o", tmp, SRC]
        subprocess.run(cmd, check=True, cwd=_HERE)
        os.replace(tmp, LIB_PATH)  # atomic for concurrent test processes
    return LIB_PATH


class _Params(ctypes.Structure):
    _fields_ = [("dist_tol", ctypes.c_double), ("diff_tol_r", ctypes.c_double),
                ("plateau_window", ctypes.c_int), ("min_iter", ctypes.c_int),
                ("max_iter", ctypes.c_int), ("m_init", ctypes.c_int),
                ("overtrain_ratio", ctypes.c_double), ("beta", ctypes.c_double),
                ("stop_on_first", ctypes.c_int)]


class _Result(ctypes.Structure):
    _fields_ = [("c_train", ctypes.c_double), ("c_val", ctypes.c_double),
                ("sweeps", ctypes.c_int), ("restarts", ctypes.c_int),
                ("final_m", ctypes.c_int), ("term", ctypes.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.qfso_distance.restype = ctypes.c_double
    return _lib


def _c(a, dtype=np.complex128):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(ctypes.c_void_p)


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what} failed (rc={rc})")


def apply_gate(n, p0, p1, g, states, dagger=False):
    psi, pp = _c(np.array(states, dtype=np.complex128, copy=True))
    gg, gp = _c(g)
    _check(lib().qfso_apply_gate(n, p0, p1, gp, int(dagger), psi.shape[0], pp), "apply_gate")
    return psi


def circuit_forward(n, pairs, gates, states):
    psi, pp = _c(np.array(states, dtype=np.complex128, copy=True))
    pr, prp = _c(pairs, np.int32)
    gg, gp = _c(gates)
    _check(lib().qfso_circuit_forward(n, pr.shape[0], prp, gp, psi.shape[0], pp), "forward")
    return psi


def environment(n, p0, p1, phi, chi):
    f, fp = _c(phi)
    c, cp = _c(chi)
    e = np.zeros((4, 4), dtype=np.complex128)
    _check(lib().qfso_environment(n, p0, p1, f.shape[0], fp, cp, e.ctypes.data_as(ctypes.c_void_p)), "env")
    return e


def svd4(a):
    aa, ap = _c(a)
    x = np.zeros((4, 4), np.complex128)
    y = np.zeros((4, 4), np.complex128)
    s = np.zeros(4)
    sw = ctypes.c_int(0)
    _check(lib().qfso_svd4(ap, x.ctypes.data_as(ctypes.c_void_p), s.ctypes.data_as(ctypes.c_void_p),
                           y.ctypes.data_as(ctypes.c_void_p), ctypes.byref(sw)), "svd4")
    return x, s, y, sw.value


def polar_update(env, g_old, beta=0.0):
    e, ep = _c(env)
    go, gop = _c(g_old)
    gn = np.zeros((4, 4), np.complex128)
    ss = ctypes.c_double(0)
    _check(lib().qfso_polar_update(ep, gop, ctypes.c_double(beta), gn.ctypes.data_as(ctypes.c_void_p),
                                   ctypes.byref(ss)), "polar")
    return gn, ss.value


def newton_polar(a):
    aa, ap = _c(a)
    w = np.zeros((4, 4), np.complex128)
    it = ctypes.c_int(0)
    _check(lib().qfso_newton_polar(ap, w.ctypes.data_as(ctypes.c_void_p), ctypes.byref(it)), "newton")
    return w, it.value


def distance(a, b):
    aa, ap = _c(a)
    bb, bp = _c(b)
    n = int(np.log2(aa.shape[1]))
    return lib().qfso_distance(n, aa.shape[0], ap, bp)


def _kinds(kinds, k):
    if kinds is None:
        return None, None
    kk, kp = _c(np.asarray(kinds).reshape(k), np.int32)
    return kk, kp


def trace_sweeps(n, pairs, init_gates, x, y, m, n_sweeps, beta=0.0, g=1, threads=0, kinds=None):
    """Fixed-M sweeps without controller.  Returns dict of traces (see qfso.h).
    kinds: per-gate kind (0 two-qubit variable, 1 fixed, 2 one-qubit variable)."""
    pr, prp = _c(pairs, np.int32)
    k = pr.shape[0]
    ig, igp = _c(init_gates)
    s = ig.shape[0]
    xx, xp = _c(x[:m])
    yy, yp = _c(y[:m])
    env = np.zeros((n_sweeps, k, s, 4, 4), np.complex128)
    gates = np.zeros((n_sweeps, s, k, 4, 4), np.complex128)
    cost = np.zeros((n_sweeps, s))
    sig = np.zeros((n_sweeps, k, s))
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    kk, kp = _kinds(kinds, k)
    _check(lib().qfso_trace_sweeps_kinds(n, k, prp, kp, s, igp, m, xp, yp, ctypes.c_double(beta), n_sweeps, g,
                                         vp(env), vp(gates), vp(cost), vp(sig), threads), "trace_sweeps")
    return dict(env=env, gates=gates, cost=cost, sigma=sig)


def instantiate(n, pairs, x, y, xv, yv, init_gates, params: dict, threads=0, kinds=None):
    pr, prp = _c(pairs, np.int32)
    k = pr.shape[0]
    ig, igp = _c(init_gates)
    s = ig.shape[0]
    xx, xp = _c(x)
    yy, yp = _c(y)
    v = 0 if xv is None else int(np.asarray(xv).shape[0])
    if v:
        xvv, xvp = _c(xv)
        yvv, yvp = _c(yv)
    else:
        xvp = yvp = None
    p = _Params(**{f: params[f] for f, _ in _Params._fields_})
    out_g = np.zeros((s, k, 4, 4), np.complex128)
    res = (_Result * s)()
    win = ctypes.c_int(-1)
    kk, kp = _kinds(kinds, k)
    _check(lib().qfso_instantiate_kinds(n, k, prp, kp, xx.shape[0], xp, yp, v, xvp, yvp, s, igp, ctypes.byref(p),
                                        out_g.ctypes.data_as(ctypes.c_void_p), res, ctypes.byref(win), threads),
           "instantiate")
    results = [dict(c_train=r.c_train, c_val=r.c_val, sweeps=r.sweeps, restarts=r.restarts,
                    final_m=r.final_m, term=TERM_NAMES.get(r.term, str(r.term))) for r in res]
    return out_g, results, win.value


def bench_sweeps(n, pairs, init_gates, x, y, m, n_sweeps, threads=0):
    pr, prp = _c(pairs, np.int32)
    ig, igp = _c(init_gates)
    xx, xp = _c(x[:m])
    yy, yp = _c(y[:m])
    sec = ctypes.c_double(0)
    _check(lib().qfso_bench_sweeps(n, pr.shape[0], prp, ig.shape[0], igp, m, xp, yp, n_sweeps, threads,
                                   ctypes.byref(sec)), "bench")
    return sec.value


# ------------------------------------------------------------------ blocks --
# Multi-qubit blocks (qfso.h: arity 2 or 3, packed d x d gates).

def _blocks(qubits, arity):
    qq, qp = _c(np.asarray(qubits).reshape(-1, 3), np.int32)
    aa, ap = _c(np.asarray(arity).reshape(-1), np.int32)
    return qq, qp, aa, ap


def apply_block(n, arity, q, g, states, dagger=False):
    psi, pp = _c(np.array(states, dtype=np.complex128, copy=True))
    qq, qp = _c(list(q) + [0] * (3 - len(q)), np.int32)
    gg, gp = _c(g)
    _check(lib().qfso_apply_block(n, arity, qp, gp, int(dagger), psi.shape[0], pp), "apply_block")
    return psi


def environment_block(n, arity, q, phi, chi):
    f, fp = _c(phi)
    c, cp = _c(chi)
    qq, qp = _c(list(q) + [0] * (3 - len(q)), np.int32)
    d = 1 << arity
    e = np.zeros((d, d), dtype=np.complex128)
    _check(lib().qfso_environment_block(n, arity, qp, f.shape[0], fp, cp, e.ctypes.data_as(ctypes.c_void_p)),
           "environment_block")
    return e


def polar_update_block(env, g_old, beta=0.0):
    e, ep = _c(env)
    go, gop = _c(g_old)
    d = e.shape[0]
    gn = np.zeros((d, d), np.complex128)
    ss = ctypes.c_double(0)
    _check(lib().qfso_polar_update_block(d, ep, gop, ctypes.c_double(beta), gn.ctypes.data_as(ctypes.c_void_p),
                                         ctypes.byref(ss)), "polar_update_block")
    return gn, ss.value


def trace_sweeps_blocks(n, qubits, arity, init_gates, x, y, m, n_sweeps, beta=0.0, threads=0, kinds=None):
    """Fixed-M sweeps of a block circuit; init_gates packed [s][G] (inputs.pack_gates).
    Returns env [t][s*G] (gate-major, qfso.h), gates [t][s][G], cost [t][s], sigma [t][k][s]."""
    qq, qp, aa, ap = _blocks(qubits, arity)
    k = aa.shape[0]
    ig, igp = _c(init_gates)
    s, gsz = ig.shape
    xx, xp = _c(x[:m])
    yy, yp = _c(y[:m])
    env = np.zeros((n_sweeps, s * gsz), np.complex128)
    gates = np.zeros((n_sweeps, s, gsz), np.complex128)
    cost = np.zeros((n_sweeps, s))
    sig = np.zeros((n_sweeps, k, s))
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    kk, kp = _kinds(kinds, k)
    _check(lib().qfso_trace_sweeps_blocks(n, k, qp, ap, kp, s, igp, m, xp, yp, ctypes.c_double(beta), n_sweeps,
                                          vp(env), vp(gates), vp(cost), vp(sig), threads), "trace_sweeps_blocks")
    return dict(env=env, gates=gates, cost=cost, sigma=sig)


def instantiate_blocks(n, qubits, arity, x, y, xv, yv, init_gates, params: dict, threads=0, kinds=None):
    qq, qp, aa, ap = _blocks(qubits, arity)
    k = aa.shape[0]
    ig, igp = _c(init_gates)
    s, gsz = ig.shape
    xx, xp = _c(x)
    yy, yp = _c(y)
    v = 0 if xv is None else int(np.asarray(xv).shape[0])
    if v:
        xvv, xvp = _c(xv)
        yvv, yvp = _c(yv)
    else:
        xvp = yvp = None
    p = _Params(**{f: params[f] for f, _ in _Params._fields_})
    out_g = np.zeros((s, gsz), np.complex128)
    res = (_Result * s)()
    win = ctypes.c_int(-1)
    kk, kp = _kinds(kinds, k)
    _check(lib().qfso_instantiate_blocks(n, k, qp, ap, kp, xx.shape[0], xp, yp, v, xvp, yvp, s, igp,
                                         ctypes.byref(p), out_g.ctypes.data_as(ctypes.c_void_p), res,
                                         ctypes.byref(win), threads), "instantiate_blocks")
    results = [dict(c_train=r.c_train, c_val=r.c_val, sweeps=r.sweeps, restarts=r.restarts,
                    final_m=r.final_m, term=TERM_NAMES.get(r.term, str(r.term))) for r in res]
    return out_g, results, win.value
