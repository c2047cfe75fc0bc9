"""ctypes binding of the CPU oracle (oracle/shiftk_oracle.c) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs
may import this package.  The product package (paper_2001_08707_b200) never imports it, and
the oracle never imports the product package; both take their inputs from ``synth``.

Parity status of each oracle function:
  or_heisenberg_apply  pinned: Table 3 eigenvalues, ferromagnet, one-magnon waves
  or_csr_*_apply       pinned: scipy.sparse product on the same CSR arrays
  or_heisenberg_sz_*   pinned: restriction of or_heisenberg_apply to the sector, dimension 924
                       (P:L761), Table 3 from the sector alone; rank/unrank vs enumeration
  or_update (COCG)     pinned: dense solves, Lanczos continued fraction, pi = chi ratio,
                       collinearity, b^dagger r_n = 0, exact termination, sum rule
  or_update (BiCG)     pinned: dense solves, bi-orthogonality, BiCG == COCG on real H
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "shiftk_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_LIB_OMP_PATH = os.path.join(_HERE, "liboracle_omp.so")

COCG, BICG = 0, 1
ITERATING, CONVERGED, MAXITER, BREAKDOWN = 0, 1, 2, 3
FLAG_REVERSE, FLAG_NO_SWITCH = 1, 2
STATUS_NAMES = {0: "iterating", 1: "converged", 2: "maxiter", 3: "breakdown"}


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no fast-math, no BLAS): liboracle.so (one thread) and
    liboracle_omp.so (-fopenmp; the same order of every floating-point operation, so the same
    bits — see the header of shiftk_oracle.c)."""
    for path, extra in ((_LIB_PATH, []), (_LIB_OMP_PATH, ["-fopenmp"])):
        if force or not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(_SRC):
            tmp = path + ".tmp"
            subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-fno-fast-math",
                                   "-ffp-contract=off"] + extra + ["-o", tmp, _SRC, "-lm"])
            os.replace(tmp, path)
    return _LIB_PATH


_libs = {}
_c128p = ctypes.c_void_p
# default build for the module-level functions and Oracle(): ORACLE_OMP=1 selects the OpenMP one
_DEFAULT_OMP = os.environ.get("ORACLE_OMP", "0") == "1"


def threads() -> int:
    """Threads the OpenMP build uses (OMP_NUM_THREADS, else the host's cores)."""
    n = os.environ.get("OMP_NUM_THREADS")
    return int(n) if n else (os.cpu_count() or 1)


def lib(omp: Optional[bool] = None):
    omp = _DEFAULT_OMP if omp is None else bool(omp)
    if omp not in _libs:
        build()
        _libs[omp] = ctypes.CDLL(_LIB_OMP_PATH if omp else _LIB_PATH)
        L = _libs[omp]
        L.or_create.restype = ctypes.c_void_p
        L.or_create.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _c128p, _c128p,
                                ctypes.c_int64, _c128p, ctypes.c_int, ctypes.c_double,
                                ctypes.c_int64, ctypes.c_int]
        L.or_create_subset.restype = ctypes.c_void_p
        L.or_create_subset.argtypes = L.or_create.argtypes + [ctypes.c_void_p]
        class _C(ctypes.Structure):
            _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]
        L._C = _C
        L.or_heisenberg_row.restype = _C
        L.or_heisenberg_row.argtypes = [ctypes.c_int, ctypes.c_double, _c128p, ctypes.c_int64]
        L.or_csr_real_row.restype = _C
        L.or_csr_real_row.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64]
        L.or_csr_cplx_row.restype = _C
        L.or_csr_cplx_row.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64]
        L.or_destroy.argtypes = [ctypes.c_void_p]
        L.or_update.restype = ctypes.c_int
        L.or_update.argtypes = [ctypes.c_void_p, _c128p, _c128p]
        L.or_heisenberg_apply.argtypes = [ctypes.c_int, ctypes.c_double, _c128p, _c128p]
        L.or_csr_real_apply.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, _c128p, _c128p]
        L.or_csr_cplx_apply.argtypes = L.or_csr_real_apply.argtypes
        for name, rt in [("or_status", ctypes.c_int), ("or_iterations", ctypes.c_int64),
                         ("or_switches", ctypes.c_int64), ("or_spmv_count", ctypes.c_int64),
                         ("or_seed_index", ctypes.c_int64), ("or_r", ctypes.c_void_p),
                         ("or_r_old", ctypes.c_void_p), ("or_t", ctypes.c_void_p),
                         ("or_pi", ctypes.c_void_p), ("or_pi_old", ctypes.c_void_p),
                         ("or_res", ctypes.c_void_p), ("or_active", ctypes.c_void_p),
                         ("or_retired_at", ctypes.c_void_p), ("or_y", ctypes.c_void_p)]:
            getattr(L, name).restype = rt
            getattr(L, name).argtypes = [ctypes.c_void_p]
        L.or_recalc.argtypes = [ctypes.c_void_p, ctypes.c_int64, _c128p, ctypes.c_double, _c128p, ctypes.c_void_p]
        L.or_log_length.restype = ctypes.c_int64
        L.or_log_length.argtypes = [ctypes.c_void_p]
        L.or_x.restype = ctypes.c_void_p
        L.or_x.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        L.or_scalars.argtypes = [ctypes.c_void_p, _c128p]
        L.or_sz_dim.restype = ctypes.c_int64
        L.or_sz_dim.argtypes = [ctypes.c_int, ctypes.c_int]
        L.or_sz_states.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.or_heisenberg_sz_apply.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_void_p,
                                             ctypes.c_int64, _c128p, _c128p]
        L.or_sz_rank.restype = ctypes.c_int64
        L.or_sz_rank.argtypes = [ctypes.c_int, ctypes.c_int64]
        L.or_sz_unrank.restype = ctypes.c_int64
        L.or_sz_unrank.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64]
        L.or_heisenberg_sz_row.restype = _C
        L.or_heisenberg_sz_row.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, _c128p,
                                           ctypes.c_int64]
    return _libs[omp]


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _view(addr: int, n: int, dtype, copy: bool = True) -> np.ndarray:
    """n elements of dtype at a C pointer: a copy, or (copy=False) a view valid until the
    oracle's next call that moves the buffer."""
    dt = np.dtype(dtype)
    buf = (ctypes.c_char * (n * dt.itemsize)).from_address(addr)
    a = np.frombuffer(buf, dtype=dt, count=n)
    return a.copy() if copy else a


# ------------------------------------------------------------------------------- operators

def heisenberg_apply(L: int, J: float, r: np.ndarray, out: Optional[np.ndarray] = None,
                     omp: Optional[bool] = None) -> np.ndarray:
    r = np.ascontiguousarray(r, dtype=np.complex128)
    q = np.empty_like(r) if out is None else out
    lib(omp).or_heisenberg_apply(L, J, _ptr(r), _ptr(q))
    return q


def sz_dim(L: int, n: int) -> int:
    return int(lib().or_sz_dim(L, n))


def sz_states(L: int, n: int) -> np.ndarray:
    """The sector basis: L-bit states with n up spins, ascending (R28)."""
    out = np.empty(sz_dim(L, n), dtype=np.int64)
    lib().or_sz_states(L, n, _ptr(out))
    return out


def sz_rank(L: int, s: int) -> int:
    return int(lib().or_sz_rank(L, int(s)))


def sz_unrank(L: int, n: int, rank: int) -> int:
    return int(lib().or_sz_unrank(L, n, int(rank)))


def heisenberg_sz_apply(L: int, n: int, J: float, r: np.ndarray) -> np.ndarray:
    r = np.ascontiguousarray(r, dtype=np.complex128)
    st = sz_states(L, n)
    assert r.shape[0] == st.shape[0]
    q = np.empty_like(r)
    lib().or_heisenberg_sz_apply(L, J, _ptr(st), st.shape[0], _ptr(r), _ptr(q))
    return q


def csr_apply(op: dict, r: np.ndarray, out: Optional[np.ndarray] = None,
              omp: Optional[bool] = None) -> np.ndarray:
    r = np.ascontiguousarray(r, dtype=np.complex128)
    q = np.empty_like(r) if out is None else out
    M = op["row_ptr"].shape[0] - 1
    fn = lib(omp).or_csr_real_apply if op["kind"] == "csr_real" else lib(omp).or_csr_cplx_apply
    fn(M, _ptr(op["row_ptr"]), _ptr(op["col"]), _ptr(op["val"]), _ptr(r), _ptr(q))
    return q


def apply_rows(op: dict, r: np.ndarray, rows) -> np.ndarray:
    """q_s = (H r)_s for the listed rows only (same arithmetic as apply_op)."""
    r = np.ascontiguousarray(r, dtype=np.complex128)
    out = np.empty(len(rows), dtype=np.complex128)
    L_ = lib()
    for j, s in enumerate(rows):
        if op["kind"] == "heisenberg":
            v = L_.or_heisenberg_row(op["L"], op["J"], _ptr(r), int(s))
        elif op["kind"] == "heisenberg_sz":
            v = L_.or_heisenberg_sz_row(op["L"], op["n_up"], op["J"], _ptr(r), int(s))
        elif op["kind"] == "csr_real":
            v = L_.or_csr_real_row(_ptr(op["row_ptr"]), _ptr(op["col"]), _ptr(op["val"]), _ptr(r), int(s))
        else:
            v = L_.or_csr_cplx_row(_ptr(op["row_ptr"]), _ptr(op["col"]), _ptr(op["val"]), _ptr(r), int(s))
        out[j] = complex(v.re, v.im)
    return out


def heisenberg_sz_row_fn(L: int, n: int, J: float, rfun, a: int) -> complex:
    """(H r)_a on the sector with r given as a function of the row index (for vectors too large
    to hold on the host): the sum over the L bonds (i, i+1 mod L) of J S_i.S_j, P:L1048-1054 —
    +J/4 r_a if the spins are parallel, else -J/4 r_a + J/2 r_{rank(s with both flipped)} — in
    the same order as or_heisenberg_sz_row (pinned against it in tests/test_oracle_pins.py)."""
    s = sz_unrank(L, n, a)
    acc = 0j
    for i in range(L):
        j = (i + 1) % L
        if ((s >> i) & 1) == ((s >> j) & 1):
            acc += 0.25 * J * rfun(a)
        else:
            acc += -0.25 * J * rfun(a)
            acc += 0.5 * J * rfun(sz_rank(L, s ^ ((1 << i) | (1 << j))))
    return acc


def apply_op(op: dict, r: np.ndarray, out: Optional[np.ndarray] = None,
             omp: Optional[bool] = None) -> np.ndarray:
    """q = H r with the oracle's own operator code (into ``out`` when given)."""
    if op["kind"] == "heisenberg":
        return heisenberg_apply(op["L"], op["J"], r, out, omp)
    if op["kind"] == "heisenberg_sz":
        q = heisenberg_sz_apply(op["L"], op["n_up"], op["J"], r)
        if out is not None:
            out[...] = q
            return out
        return q
    return csr_apply(op, r, out, omp)


# ------------------------------------------------------------------------------- solver

class Oracle:
    """Reverse-communication shifted COCG/BiCG state machine (init/update/get/finalize,
    P:L517-523, Alg. 1)."""

    def __init__(self, method: str, b: np.ndarray, z: np.ndarray, *, left: Optional[np.ndarray] = None,
                 full_x: bool = False, tol: float = 1e-10, itermax: int = 10000, flags: int = 0,
                 keep: Optional[np.ndarray] = None, omp: Optional[bool] = None):
        """b and left are borrowed by the C state: this object keeps references to them.
        omp selects the OpenMP build (bit-identical results; default: ORACLE_OMP env)."""
        self._h = None
        self.omp = _DEFAULT_OMP if omp is None else bool(omp)
        self._q = self._qt = None   # reused H r / H t buffers of step()
        self.method = COCG if method == "cocg" else BICG
        self.b = np.ascontiguousarray(b, dtype=np.complex128)
        self.z = np.ascontiguousarray(z, dtype=np.complex128)
        self.M, self.nz = self.b.shape[0], self.z.shape[0]
        self.left = None if left is None else np.ascontiguousarray(left, dtype=np.complex128)
        self.nleft = 1 if left is None else self.left.shape[0]
        self.full_x = bool(full_x)
        self._keep = None if keep is None else np.ascontiguousarray(keep, dtype=np.uint8)
        self.tol = tol
        self._h = self._lib().or_create_subset(self.method, self.M, self.nz, _ptr(self.z), _ptr(self.b),
                                         self.nleft, 0 if self.left is None else _ptr(self.left),
                                         int(self.full_x), float(tol), int(itermax), int(flags),
                                         0 if self._keep is None else _ptr(self._keep))
        if not self._h:
            raise ValueError("oracle init rejected its arguments")

    def _lib(self):
        return lib(self.omp)

    def close(self):
        if self._h:
            self._lib().or_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    # reverse communication -----------------------------------------------------------
    def r(self) -> np.ndarray:
        return _view(self._lib().or_r(self._h), self.M, np.complex128)

    def r_old(self) -> np.ndarray:
        return _view(self._lib().or_r_old(self._h), self.M, np.complex128)

    def t(self) -> np.ndarray:
        return _view(self._lib().or_t(self._h), self.M, np.complex128)

    def update(self, q: np.ndarray, qt: Optional[np.ndarray] = None) -> int:
        """Reverse communication: the caller supplies q = H r (and qt = H t for BiCG)."""
        q = np.ascontiguousarray(q, dtype=np.complex128)
        qt_p = 0
        if self.method == BICG:
            qt = np.ascontiguousarray(qt, dtype=np.complex128)
            qt_p = _ptr(qt)
        return self._lib().or_update(self._h, _ptr(q), qt_p)

    def step(self, op: dict) -> int:
        """One iteration with the oracle's own operator: q = H r (and H t for BiCG), update.
        r is read in place and q lives in a buffer reused from step to step (no M-vector copy)."""
        if self.status != ITERATING:
            return self.status
        if self._q is None:
            self._q = np.empty(self.M, dtype=np.complex128)
        L_ = self._lib()
        apply_op(op, _view(L_.or_r(self._h), self.M, np.complex128, copy=False), self._q, self.omp)
        qt = None
        if self.method == BICG:
            if self._qt is None:
                self._qt = np.empty(self.M, dtype=np.complex128)
            qt = apply_op(op, _view(L_.or_t(self._h), self.M, np.complex128, copy=False), self._qt, self.omp)
        return self.update(self._q, qt)

    def run(self, op: dict, max_iters: int) -> int:
        st = self.status
        for _ in range(max_iters):
            st = self.step(op)
            if st != ITERATING:
                break
        return st

    # getters -------------------------------------------------------------------------
    @property
    def status(self) -> int:
        return self._lib().or_status(self._h)

    @property
    def iterations(self) -> int:
        return self._lib().or_iterations(self._h)

    @property
    def switches(self) -> int:
        return self._lib().or_switches(self._h)

    @property
    def spmv_count(self) -> int:
        return self._lib().or_spmv_count(self._h)

    @property
    def seed_index(self) -> int:
        return self._lib().or_seed_index(self._h)

    def residuals(self) -> np.ndarray:
        return _view(self._lib().or_res(self._h), self.nz, np.float64)

    def active(self) -> np.ndarray:
        return _view(self._lib().or_active(self._h), self.nz, np.uint8).astype(bool)

    def retired_at(self) -> np.ndarray:
        return _view(self._lib().or_retired_at(self._h), self.nz, np.int64)

    def pi(self) -> np.ndarray:
        return _view(self._lib().or_pi(self._h), self.nz, np.complex128)

    def pi_old(self) -> np.ndarray:
        return _view(self._lib().or_pi_old(self._h), self.nz, np.complex128)

    def projections(self) -> np.ndarray:
        """y[k, l] = a_l^dagger x^(k) from the projected recurrences."""
        return _view(self._lib().or_y(self._h), self.nz * self.nleft, np.complex128).reshape(self.nz, self.nleft)

    def solution(self, k: int) -> np.ndarray:
        if not self.full_x:
            raise ValueError("full x not stored")
        addr = self._lib().or_x(self._h, k)
        if not addr:
            raise ValueError(f"x of shift {k} not carried (keep mask)")
        return _view(addr, self.M, np.complex128)

    def recalc(self, z_new, tol: Optional[float] = None):
        """Projections at new shifts from the coefficient log, no operator use."""
        z_new = np.ascontiguousarray(z_new, dtype=np.complex128)
        y = np.zeros((z_new.shape[0], self.nleft), dtype=np.complex128)
        res = np.zeros(z_new.shape[0], dtype=np.float64)
        self._lib().or_recalc(self._h, z_new.shape[0], _ptr(z_new), float(self.tol if tol is None else tol),
                        _ptr(y), res.ctypes.data)
        return y, res

    @property
    def log_length(self) -> int:
        return self._lib().or_log_length(self._h)

    def scalars(self) -> dict:
        out = np.zeros(6, dtype=np.complex128)
        self._lib().or_scalars(self._h, _ptr(out))
        return dict(alpha=out[0], beta=out[1], rho=out[2], w=out[3], z_seed=out[4], alpha_prev=out[5])


def solve(problem, max_iters: Optional[int] = None, flags: int = 0) -> Oracle:
    """Run the oracle on a synth.Problem until convergence / max_iters."""
    o = Oracle(problem.method, problem.b, problem.z, left=problem.left, full_x=problem.full_x,
               tol=problem.tol, itermax=problem.itermax, flags=flags)
    o.run(problem.op, problem.itermax if max_iters is None else max_iters)
    return o
