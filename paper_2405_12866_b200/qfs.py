"""Thin ctypes binding of libqfs.so (include/qfs.h) — argument marshalling only.

Every step of the sweep runs in the CUDA kernels behind the C ABI; this module
only converts numpy / torch buffers to pointers and status codes to
exceptions.  There is no CPU fallback: if ``libqfs.so`` is missing or fails to
load, importing the binding raises.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# QFS_LIB=debug selects libqfs_debug.so (build.py --debug: device bounds checks); QFS_LIB=<path>.so
# an A/B build of the same sources (tools/); same ABI
_sel = os.environ.get("QFS_LIB", "")
LIB_PATH = (os.path.join(_HERE, "libqfs_debug.so") if _sel == "debug" else
            os.path.abspath(_sel) if _sel.endswith(".so") else os.path.join(_HERE, "libqfs.so"))

STATUS = {0: "QFS_OK", 1: "QFS_ERR_ARG", 2: "QFS_ERR_CAPACITY", 3: "QFS_ERR_NUMERIC",
          4: "QFS_ERR_DEVICE", 5: "QFS_ERR_STATE"}
TERM_NAMES = {0: "CONVERGED", 1: "PLATEAU", 2: "MAX_ITER", 3: "POOL_EXHAUSTED", 4: "STOPPED"}
SYMBOLS = ["qfs_create", "qfs_create_blocks", "qfs_create_emulated", "qfs_set_exchange", "qfs_set_samples_basis", "qfs_set_structure", "qfs_create_dist", "qfs_nccl_unique_id", "qfs_create_nccl", "qfs_set_samples", "qfs_set_samples_async", "qfs_set_samples_device",
           "qfs_instantiate", "qfs_trace_sweeps", "qfs_bench_sweeps", "qfs_op_apply",
           "qfs_op_environment", "qfs_op_polar", "qfs_profile_enable", "qfs_profile_read", "qfs_set_path", "qfs_set_gate_kinds",
           "qfs_launch_count", "qfs_stream", "qfs_last_error", "qfs_destroy"]


class QfsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Params(ctypes.Structure):
    _fields_ = [("dist_tol", ctypes.c_double), ("diff_tol_r", ctypes.c_double),
                ("plateau_window", ctypes.c_int), ("min_iter", ctypes.c_int),
                ("max_iter", ctypes.c_int), ("m_init", ctypes.c_int),
                ("overtrain_ratio", ctypes.c_double), ("beta", ctypes.c_double),
                ("stop_on_first", ctypes.c_int)]


class Result(ctypes.Structure):
    _fields_ = [("c_train", ctypes.c_double), ("c_val", ctypes.c_double),
                ("sweeps", ctypes.c_int), ("restarts", ctypes.c_int),
                ("final_m", ctypes.c_int), ("term", ctypes.c_int)]


_lib = None


def load(path: str = LIB_PATH):
    """Load libqfs.so (raises if absent: the product has no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} not built (run paper_2405_12866_b200.build.build())")
        lib = ctypes.CDLL(path)
        vp, ip, dp = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        lib.qfs_last_error.restype = ctypes.c_char_p
        lib.qfs_last_error.argtypes = [vp]
        lib.qfs_launch_count.restype = ctypes.c_longlong
        lib.qfs_launch_count.argtypes = [vp]
        lib.qfs_stream.restype = vp
        lib.qfs_stream.argtypes = [vp]
        lib.qfs_destroy.argtypes = [vp]
        lib.qfs_destroy.restype = None
        lib.qfs_create.argtypes = [ip, ip, vp, ip, ctypes.POINTER(vp)]
        lib.qfs_create_blocks.argtypes = [ip, ip, vp, vp, ip, ctypes.POINTER(vp)]
        lib.qfs_set_structure.argtypes = [vp, ip, vp]
        lib.qfs_create_dist.argtypes = [ip, ip, vp, ip, vp, ip, ip, ip, ctypes.POINTER(vp)]
        lib.qfs_nccl_unique_id.argtypes = [vp]
        lib.qfs_create_emulated.argtypes = [ip, ip, vp, ip, ip, ctypes.POINTER(vp)]
        lib.qfs_set_exchange.argtypes = [vp, ip]
        lib.qfs_set_samples_basis.argtypes = [vp, ip, vp, ip, vp, vp]
        lib.qfs_create_nccl.argtypes = [ip, ip, vp, ip, vp, ip, ip, ip, ctypes.POINTER(vp)]
        lib.qfs_set_samples.argtypes = [vp, ip, vp, vp, ip, vp, vp]
        lib.qfs_set_samples_async.argtypes = [vp, ip, vp, vp, ip, vp, vp]
        lib.qfs_set_samples_device.argtypes = [vp, ip, vp, vp, ip, vp, vp, vp]
        lib.qfs_instantiate.argtypes = [vp, ip, vp, ctypes.POINTER(Params), vp, vp, ctypes.POINTER(ip)]
        lib.qfs_trace_sweeps.argtypes = [vp, ip, vp, ip, dp, ip, vp, vp, vp, vp]
        lib.qfs_bench_sweeps.argtypes = [vp, ip, vp, ip, ip, ctypes.POINTER(dp)]
        lib.qfs_op_apply.argtypes = [vp, ip, ip, vp, ip, ip, vp]
        lib.qfs_op_environment.argtypes = [vp, ip, ip, ip, vp, vp, vp]
        lib.qfs_op_polar.argtypes = [vp, ip, vp, vp, dp, vp, vp]
        lib.qfs_profile_enable.argtypes = [vp, ip]
        lib.qfs_set_path.argtypes = [vp, ip]
        lib.qfs_set_gate_kinds.argtypes = [vp, vp]
        lib.qfs_profile_read.argtypes = [vp, ip, vp, vp, vp, vp, vp, ctypes.POINTER(ip)]
        for name in SYMBOLS:
            if name not in ("qfs_last_error", "qfs_launch_count", "qfs_stream", "qfs_destroy"):
                getattr(lib, name).restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def make_params(d: dict) -> Params:
    return Params(**{f: d[f] for f, _ in Params._fields_})


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0), to be broadcast to the other ranks."""
    buf = ctypes.create_string_buffer(128)
    rc = load().qfs_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p))
    if rc != 0:
        raise QfsError(rc, "ncclGetUniqueId failed")
    return buf.raw


class Context:
    """One qfs_ctx: a circuit structure on one device (qfs_create / qfs_create_dist /
    qfs_create_nccl when ``nccl_id`` is given)."""

    def __init__(self, n, pairs, device=0, nccl_comm=None, rank=0, world=1, shard_mode=0, nccl_id=None,
                 emulated_ranks=0):
        self.lib = load()
        self.n = int(n)
        self.pairs = np.ascontiguousarray(pairs, dtype=np.int32)
        self.k = int(self.pairs.shape[0])
        h = ctypes.c_void_p()
        if emulated_ranks:
            rc = self.lib.qfs_create_emulated(self.n, self.k, _ptr(self.pairs), int(device), int(emulated_ranks),
                                              ctypes.byref(h))
        elif nccl_id is not None:
            idb = ctypes.create_string_buffer(bytes(nccl_id), 128)
            rc = self.lib.qfs_create_nccl(self.n, self.k, _ptr(self.pairs), int(device),
                                          ctypes.cast(idb, ctypes.c_void_p), int(rank), int(world),
                                          int(shard_mode), ctypes.byref(h))
        elif nccl_comm is None and world == 1:
            rc = self.lib.qfs_create(self.n, self.k, _ptr(self.pairs), int(device), ctypes.byref(h))
        else:
            rc = self.lib.qfs_create_dist(self.n, self.k, _ptr(self.pairs), int(device),
                                          ctypes.c_void_p(nccl_comm or 0), int(rank), int(world),
                                          int(shard_mode), ctypes.byref(h))
        self.h = h
        if rc != 0:
            msg = self.lib.qfs_last_error(h).decode() if h.value else "invalid arguments"
            if h.value:
                self.lib.qfs_destroy(h)
            self.h = None
            raise QfsError(rc, msg)
        self.world = int(world)
        self.shard_mode = int(shard_mode)

    def _check(self, rc):
        if rc != 0:
            raise QfsError(rc, self.lib.qfs_last_error(self.h).decode())

    def close(self):
        if self.h is not None and self.h.value:
            self.lib.qfs_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- samples ---------------------------------------------------------
    def set_samples(self, x, y, xv=None, yv=None):
        """Host arrays (numpy complex128 [rows][2^n]; or any object exposing a
        host pointer via .ctypes / data_ptr())."""
        x, y = _c128(x), _c128(y)
        v = 0 if xv is None else int(np.asarray(xv).shape[0])
        xv = _c128(xv) if v else None
        yv = _c128(yv) if v else None
        self._keep = (x, y, xv, yv)
        self._check(self.lib.qfs_set_samples(self.h, x.shape[0], _ptr(x), _ptr(y), v, _ptr(xv), _ptr(yv)))

    def set_samples_basis(self, y, xv=None, yv=None):
        """qfs_set_samples_basis: training inputs x_m = e_m (implicit, never stored),
        y [m_pool][2^n] their images (the first m_pool columns of U, as rows)."""
        y = _c128(y)
        v = 0 if xv is None else int(np.asarray(xv).shape[0])
        xv = _c128(xv) if v else None
        yv = _c128(yv) if v else None
        self._keep = (y, xv, yv)
        self._check(self.lib.qfs_set_samples_basis(self.h, y.shape[0], _ptr(y), v, _ptr(xv), _ptr(yv)))

    def set_samples_host_ptr(self, m_pool, px, py, v, pxv, pyv):
        """Raw host pointers (e.g. pinned torch tensors' data_ptr())."""
        self._check(self.lib.qfs_set_samples(self.h, int(m_pool), ctypes.c_void_p(px), ctypes.c_void_p(py),
                                             int(v), ctypes.c_void_p(pxv or 0), ctypes.c_void_p(pyv or 0)))

    def set_samples_async_host_ptr(self, m_pool, px, py, v, pxv, pyv):
        """qfs_set_samples_async: queue a sample set (raw host pointers, ideally
        pinned); the next instantiate / trace call consumes it.  The buffers
        must stay alive and unchanged until then."""
        self._check(self.lib.qfs_set_samples_async(self.h, int(m_pool), ctypes.c_void_p(px), ctypes.c_void_p(py),
                                                   int(v), ctypes.c_void_p(pxv or 0), ctypes.c_void_p(pyv or 0)))

    def set_samples_device(self, dx, dy, dxv=None, dyv=None, stream=None):
        """torch CUDA tensors (complex128, contiguous) on the context's device."""
        v = 0 if dxv is None else int(dxv.shape[0])
        st = ctypes.c_void_p(stream.cuda_stream if stream is not None else 0)
        self._check(self.lib.qfs_set_samples_device(
            self.h, int(dx.shape[0]), ctypes.c_void_p(dx.data_ptr()), ctypes.c_void_p(dy.data_ptr()), v,
            ctypes.c_void_p(dxv.data_ptr() if v else 0), ctypes.c_void_p(dyv.data_ptr() if v else 0), st))

    # -- instantiation -----------------------------------------------------
    def instantiate(self, init_gates, params: dict, out=None):
        """qfs_instantiate.  ``out``: optional caller-owned complex128 array of the
        gates' shape to receive the result (the C ABI's out_gates), e.g. reused
        across calls to avoid allocating (and page-faulting) a fresh array."""
        g = _c128(init_gates)
        s = g.shape[0]
        if out is None:
            out = np.empty_like(g)  # filled by qfs_instantiate (no zeroing pass)
        elif out.shape != g.shape or out.dtype != np.complex128 or not out.flags.c_contiguous or out is g:
            raise ValueError("out must be a distinct C-contiguous complex128 array of the gates' shape")
        res = (Result * s)()
        win = ctypes.c_int(-1)
        p = make_params(params)
        self._check(self.lib.qfs_instantiate(self.h, s, _ptr(g), ctypes.byref(p), _ptr(out),
                                             ctypes.cast(res, ctypes.c_void_p), ctypes.byref(win)))
        results = [dict(c_train=r.c_train, c_val=r.c_val, sweeps=r.sweeps, restarts=r.restarts,
                        final_m=r.final_m, term=TERM_NAMES.get(r.term, str(r.term))) for r in res]
        return out, results, win.value

    def trace_sweeps(self, init_gates, m, n_sweeps, beta=0.0, env=True, gates=True, cost=True, sigma=True):
        g = _c128(init_gates)
        s, k = g.shape[0], self.k
        e = np.zeros((n_sweeps, k, s, 4, 4), np.complex128) if env else None
        gt = np.zeros((n_sweeps, s, k, 4, 4), np.complex128) if gates else None
        ct = np.zeros((n_sweeps, s)) if cost else None
        sg = np.zeros((n_sweeps, k, s)) if sigma else None
        self._check(self.lib.qfs_trace_sweeps(self.h, s, _ptr(g), int(m), float(beta), int(n_sweeps),
                                              _ptr(e), _ptr(gt), _ptr(ct), _ptr(sg)))
        return dict(env=e, gates=gt, cost=ct, sigma=sg)

    def bench_sweeps(self, init_gates, m, n_sweeps):
        g = _c128(init_gates)
        sec = ctypes.c_double(0)
        self._check(self.lib.qfs_bench_sweeps(self.h, g.shape[0], _ptr(g), int(m), int(n_sweeps),
                                              ctypes.byref(sec)))
        return sec.value

    # -- kernel-level ops ----------------------------------------------------
    def op_apply(self, p0, p1, g, psi, dagger=False):
        out = np.array(psi, dtype=np.complex128, copy=True, order="C")
        gg = _c128(g)
        self._check(self.lib.qfs_op_apply(self.h, int(p0), int(p1), _ptr(gg), int(dagger), out.shape[0], _ptr(out)))
        return out

    def op_environment(self, p0, p1, phi, chi):
        f, c = _c128(phi), _c128(chi)
        e = np.zeros((4, 4), np.complex128)
        self._check(self.lib.qfs_op_environment(self.h, int(p0), int(p1), f.shape[0], _ptr(f), _ptr(c), _ptr(e)))
        return e

    def op_polar(self, env, g_old, beta=0.0):
        e, go = _c128(env), _c128(g_old)
        cnt = e.shape[0]
        gn = np.zeros_like(e)
        ss = np.zeros(cnt)
        self._check(self.lib.qfs_op_polar(self.h, cnt, _ptr(e), _ptr(go), float(beta), _ptr(gn), _ptr(ss)))
        return gn, ss

    # -- profiling -------------------------------------------------------------
    def profile_enable(self, on=True):
        self._check(self.lib.qfs_profile_enable(self.h, int(on)))

    def profile_read(self):
        cap = 16
        names = (ctypes.c_char_p * cap)()
        la = np.zeros(cap, np.int64)
        ms = np.zeros(cap)
        by = np.zeros(cap)
        fl = np.zeros(cap)
        cnt = ctypes.c_int(0)
        self._check(self.lib.qfs_profile_read(self.h, cap, ctypes.cast(names, ctypes.c_void_p), _ptr(la), _ptr(ms),
                                              _ptr(by), _ptr(fl), ctypes.byref(cnt)))
        return {names[i].decode(): dict(launches=int(la[i]), ms=float(ms[i]), bytes=float(by[i]),
                                        flops=float(fl[i])) for i in range(cnt.value)}

    def set_gate_kinds(self, kinds=None):
        """Per-gate kinds: 0 two-qubit variable, 1 fixed, 2 one-qubit variable (u (x) I)."""
        if kinds is None:
            self._check(self.lib.qfs_set_gate_kinds(self.h, None))
            return
        k = np.ascontiguousarray(np.asarray(kinds, dtype=np.int32))
        self._check(self.lib.qfs_set_gate_kinds(self.h, _ptr(k)))

    def set_structure(self, pairs):
        """qfs_set_structure: a new circuit structure (same n) on this context."""
        pr = np.ascontiguousarray(pairs, dtype=np.int32)
        self._check(self.lib.qfs_set_structure(self.h, int(pr.shape[0]), _ptr(pr)))
        self.pairs = pr
        self.k = int(pr.shape[0])

    def set_exchange(self, mode):
        """Sample mode: 0 / "nccl" host NCCL all-reduce per gate, 1 / "device" device-initiated exchange."""
        m = {"nccl": 0, "device": 1}.get(mode, mode)
        self._check(self.lib.qfs_set_exchange(self.h, int(m)))

    def set_path(self, path):
        """'auto' | 'streamed' | 'resident' (qfs_set_path)."""
        code = {"auto": 0, "streamed": 1, "resident": 2}[path] if isinstance(path, str) else int(path)
        self._check(self.lib.qfs_set_path(self.h, code))

    def launch_count(self):
        return int(self.lib.qfs_launch_count(self.h))

    def stream_ptr(self):
        return self.lib.qfs_stream(self.h)



class BlockContext(Context):
    """qfs_create_blocks: a circuit of 2- and 3-qubit blocks (qubits [k][3],
    arity [k]); gates are PACKED per start ([s][G] complex128, see
    inputs.pack_gates and include/qfs.h)."""

    def __init__(self, n, qubits, arity, device=0):
        self.lib = load()
        self.n = int(n)
        self.qubits = np.ascontiguousarray(np.asarray(qubits).reshape(-1, 3), dtype=np.int32)
        self.arity = np.ascontiguousarray(np.asarray(arity).reshape(-1), dtype=np.int32)
        self.k = int(self.arity.shape[0])
        self.gsz = int(sum(1 << (2 * int(a)) for a in self.arity))
        self.pairs = np.ascontiguousarray(self.qubits[:, :2])
        h = ctypes.c_void_p()
        rc = self.lib.qfs_create_blocks(self.n, self.k, _ptr(self.qubits), _ptr(self.arity), int(device),
                                        ctypes.byref(h))
        self.h = h
        if rc != 0:
            msg = self.lib.qfs_last_error(h).decode() if h.value else "invalid arguments"
            if h.value:
                self.lib.qfs_destroy(h)
            self.h = None
            raise QfsError(rc, msg)
        self.world = 1
        self.shard_mode = 0

    def trace_sweeps(self, init_gates, m, n_sweeps, beta=0.0, env=True, gates=True, cost=True, sigma=True):
        g = _c128(np.asarray(init_gates).reshape(-1, self.gsz))
        s, k = g.shape[0], self.k
        e = np.zeros((n_sweeps, s * self.gsz), np.complex128) if env else None
        gt = np.zeros((n_sweeps, s, self.gsz), np.complex128) if gates else None
        ct = np.zeros((n_sweeps, s)) if cost else None
        sg = np.zeros((n_sweeps, k, s)) if sigma else None
        self._check(self.lib.qfs_trace_sweeps(self.h, s, _ptr(g), int(m), float(beta), int(n_sweeps),
                                              _ptr(e), _ptr(gt), _ptr(ct), _ptr(sg)))
        return dict(env=e, gates=gt, cost=ct, sigma=sg)

def default_params(**kw) -> dict:
    d = dict(dist_tol=1e-8, diff_tol_r=1e-3, plateau_window=5, min_iter=6, max_iter=1000,
             m_init=2, overtrain_ratio=0.1, beta=0.0, stop_on_first=1)
    d.update(kw)
    if d["overtrain_ratio"] is None:
        d["overtrain_ratio"] = math.inf
    return d
