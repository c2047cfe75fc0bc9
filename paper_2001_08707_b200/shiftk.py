"""Thin ctypes binding of libshiftk.so (include/shiftk.h).  Argument marshalling only: every
step of the method runs in the library's sm_100a kernels.  There is no CPU fallback: if the
library or a CUDA device is missing, loading fails loudly.

Names follow the C-ABI (sk_init / sk_update / sk_run / sk_get_* / sk_finalize), which follows
the paper's init / update / getresidual / finalize flow (Alg. 1
P:L529-552).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SHIFTK_LIB") or os.path.join(_HERE, "libshiftk.so")   # (override: experiments)

COCG, BICG = 0, 1
OP_HEISENBERG, OP_CSR_REAL, OP_CSR_CPLX, OP_RC, OP_HEISENBERG_SZ = 0, 1, 2, 3, 4
ITERATING, CONVERGED, MAXITER, BREAKDOWN = 0, 1, 2, 3
STATUS_NAMES = {0: "iterating", 1: "converged", 2: "maxiter", 3: "breakdown"}
MEM_HOST, MEM_DEVICE = 0, 1
FLAG_NO_SWITCH = 1
FLAG_LOG = 2
ERRORS = {0: "SK_OK", -1: "SK_EINVAL", -2: "SK_ENOMEM", -3: "SK_ECUDA", -4: "SK_ENCCL",
          -5: "SK_ESTATE", -6: "SK_EUNSUPPORTED"}
EXPORTS = ["sk_init", "sk_update", "sk_update_rc", "sk_get_seed_vectors", "sk_run", "sk_enqueue",
           "sk_get_residual", "sk_get_projection", "sk_get_solution", "sk_get_shift_state",
           "sk_get_coefficients", "sk_finalize", "sk_apply_operator", "sk_last_error", "sk_version",
           "sk_profile_enable", "sk_get_profile", "sk_copy_solution", "sk_debug_timestamps",
           "sk_ipc_handle", "sk_nccl_unique_id", "sk_connect", "sk_group_create", "sk_group_connect",
           "sk_group_update", "sk_group_run", "sk_group_destroy", "sk_recalc", "sk_checkpoint",
           "sk_restore", "sk_combine", "sk_gram", "sk_get_info", "sk_connect_host", "sk_nccl_selftest"]


class ShiftkError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn} -> {ERRORS.get(code, code)}: {msg}")
        self.code = code


class sk_cplx(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class sk_operator(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("L", ctypes.c_int32), ("J", ctypes.c_double),
                ("M", ctypes.c_int64), ("M_local", ctypes.c_int64), ("row_begin", ctypes.c_int64),
                ("nnz", ctypes.c_int64), ("row_ptr", ctypes.c_void_p), ("col", ctypes.c_void_p),
                ("val", ctypes.c_void_p), ("n_up", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class sk_params(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int32), ("flags", ctypes.c_int32), ("n_shift", ctypes.c_int64),
                ("z", ctypes.c_void_p), ("b", ctypes.c_void_p), ("b_mem", ctypes.c_int32),
                ("left_mem", ctypes.c_int32), ("n_left", ctypes.c_int64), ("left", ctypes.c_void_p),
                ("full_x", ctypes.c_int32), ("tol", ctypes.c_double), ("itermax", ctypes.c_int64)]


class sk_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("nccl_id", ctypes.c_void_p), ("stream", ctypes.c_void_p),
                ("group", ctypes.c_void_p)]


class sk_coeffs(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("seed_index", ctypes.c_int64),
                ("switches", ctypes.c_int64), ("spmv_count", ctypes.c_int64),
                ("n_active", ctypes.c_int64), ("status", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("z_seed", sk_cplx), ("alpha", sk_cplx), ("rho", sk_cplx), ("beta", sk_cplx),
                ("seed_residual", ctypes.c_double)]


class sk_info(ctypes.Structure):
    _fields_ = [("split_ahi", ctypes.c_int32), ("spmv_ctas", ctypes.c_int32),
                ("update_ctas", ctypes.c_int32), ("shift_agents", ctypes.c_int32),
                ("arena_bytes", ctypes.c_int64), ("split_fuse", ctypes.c_int32),
                ("left_real", ctypes.c_int32), ("csr_col_blocks", ctypes.c_int32),
                ("csr_block_shift", ctypes.c_int32)]


class sk_profile(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("launches", ctypes.c_int64),
                ("ms_spmv", ctypes.c_double), ("ms_scalar", ctypes.c_double),
                ("ms_update", ctypes.c_double)]


_lib = None

# sk_allreduce_fn: int (*)(void *user, const double *send, double *recv, int64_t n)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double), ctypes.c_int64)


def load(path: str = LIB_PATH):
    """Load libshiftk.so (no fallback: raises if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path)
    P, I64, I32, VP = ctypes.POINTER, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    sig = {
        "sk_init": [P(VP), P(sk_operator), P(sk_params), P(sk_dist)],
        "sk_update": [VP, P(I32)],
        "sk_update_rc": [VP, VP, VP, P(I32)],
        "sk_get_seed_vectors": [VP, P(VP), P(VP)],
        "sk_run": [VP, I64, I32, P(I32)],
        "sk_enqueue": [VP, I64],
        "sk_get_residual": [VP, VP],
        "sk_get_projection": [VP, VP],
        "sk_get_solution": [VP, I64, P(VP)],
        "sk_get_shift_state": [VP, VP, VP, VP],
        "sk_get_coefficients": [VP, P(sk_coeffs)],
        "sk_finalize": [P(VP)],
        "sk_apply_operator": [P(sk_operator), VP, VP, VP],
        "sk_combine": [VP, I64, I64, I64, VP, I64, VP, VP],
        "sk_gram": [VP, I64, VP, I64, I64, VP, VP],
        "sk_profile_enable": [VP, I32],
        "sk_copy_solution": [VP, I64, VP, I32],
        "sk_debug_timestamps": [VP, VP],
        "sk_ipc_handle": [VP, VP],
        "sk_nccl_unique_id": [VP],
        "sk_nccl_selftest": [I32, I64, VP, VP, VP],
        "sk_connect": [VP, VP, VP],
        "sk_group_create": [P(VP), I32, I32],
        "sk_group_connect": [VP],
        "sk_group_update": [VP, P(I32)],
        "sk_group_run": [VP, I64, P(I32)],
        "sk_group_destroy": [P(VP)],
        "sk_recalc": [VP, I64, VP, VP, VP],
        "sk_checkpoint": [VP, VP, P(ctypes.c_size_t)],
        "sk_restore": [VP, VP, ctypes.c_size_t],
        "sk_get_profile": [VP, P(sk_profile), I32],
        "sk_get_info": [VP, P(sk_info)],
        "sk_connect_host": [VP, VP, ALLREDUCE_FN, VP],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.sk_last_error.restype = ctypes.c_char_p
    L.sk_version.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(code: int, fn: str):
    if code != 0:
        raise ShiftkError(code, fn, load().sk_last_error().decode())


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _ptr_mem(a):
    """(pointer, sk_mem) of a numpy array (host) or a torch tensor (host or cuda)."""
    if a is None:
        return None, MEM_HOST
    if _is_torch(a):
        assert a.is_contiguous()
        return a.data_ptr(), (MEM_DEVICE if a.is_cuda else MEM_HOST)
    assert isinstance(a, np.ndarray) and a.flags.c_contiguous
    return a.ctypes.data, MEM_HOST


def make_operator(op: dict, M: int, dev_arrays: Optional[dict] = None, *, M_local: Optional[int] = None,
                  row_begin: int = 0) -> sk_operator:
    """Build sk_operator from a synth op dict; CSR arrays must be given as device tensors in
    ``dev_arrays`` (row_ptr int64, col int32, val float64/complex128) holding this rank's rows
    [row_begin, row_begin + M_local) of the global M x M matrix."""
    o = sk_operator()
    o.M = M
    o.M_local = M if M_local is None else M_local
    o.row_begin = row_begin
    if op["kind"] == "heisenberg":
        o.kind, o.L, o.J = OP_HEISENBERG, int(op["L"]), float(op["J"])
    elif op["kind"] in ("csr_real", "csr_cplx"):
        o.kind = OP_CSR_REAL if op["kind"] == "csr_real" else OP_CSR_CPLX
        d = dev_arrays
        o.row_ptr, o.col, o.val = d["row_ptr"].data_ptr(), d["col"].data_ptr(), d["val"].data_ptr()
        o.nnz = int(d["col"].numel())
    elif op["kind"] == "heisenberg_sz":
        o.kind, o.L, o.J, o.n_up = OP_HEISENBERG_SZ, int(op["L"]), float(op["J"]), int(op["n_up"])
    elif op["kind"] == "rc":
        o.kind = OP_RC
    else:
        raise ValueError(op["kind"])
    return o


class _CudaView:
    """__cuda_array_interface__ wrapper so torch.as_tensor can view a library-owned buffer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<c16", "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_view(ptr: int, n: int):
    """torch complex128 view (no copy) of n elements at a library device pointer."""
    import torch
    return torch.as_tensor(_CudaView(ptr, n), device="cuda")


def apply_operator(op: sk_operator, r_dev, q_dev, stream: int = 0):
    """q = H r on device tensors (complex128)."""
    _check(load().sk_apply_operator(ctypes.byref(op), r_dev.data_ptr(), q_dev.data_ptr(),
                                    ctypes.c_void_p(stream)), "sk_apply_operator")


def combine(X_ptr: int, n_in: int, ld_x: int, M: int, W: np.ndarray, out_dev, stream: int = 0):
    """out[c] = sum_j W[j, c] X[j] (device rows of stride ld_x; W host [n_in, n_out])."""
    W = np.ascontiguousarray(W, dtype=np.complex128)
    assert W.shape[0] == n_in
    _check(load().sk_combine(X_ptr, n_in, ld_x, M, W.ctypes.data, W.shape[1], out_dev.data_ptr(),
                             ctypes.c_void_p(stream)), "sk_combine")


def gram(A_dev, B_dev, stream: int = 0) -> np.ndarray:
    """A^dagger B for device row blocks A [na, M], B [nb, M] (host result [na, nb])."""
    na, M = A_dev.shape
    nb = B_dev.shape[0]
    G = np.empty((na, nb), dtype=np.complex128)
    _check(load().sk_gram(A_dev.data_ptr(), na, B_dev.data_ptr(), nb, M, G.ctypes.data,
                          ctypes.c_void_p(stream)), "sk_gram")
    return G


class Group:
    """Loopback group: ``world`` virtual ranks on one GPU (sk_group_*)."""

    def __init__(self, world: int, device: int = 0):
        self._h = ctypes.c_void_p()
        self.world = world
        _check(load().sk_group_create(ctypes.byref(self._h), world, device), "sk_group_create")
        self.members = []

    def connect(self):
        _check(load().sk_group_connect(self._h), "sk_group_connect")

    def update(self) -> int:
        st = ctypes.c_int32()
        _check(load().sk_group_update(self._h, ctypes.byref(st)), "sk_group_update")
        return st.value

    def run(self, max_iters: int) -> int:
        st = ctypes.c_int32()
        _check(load().sk_group_run(self._h, max_iters, ctypes.byref(st)), "sk_group_run")
        return st.value

    def close(self):
        for m in self.members:
            m.finalize()
        self.members = []
        if self._h and self._h.value:
            _check(load().sk_group_destroy(ctypes.byref(self._h)), "sk_group_destroy")


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_char * 128)()
    _check(load().sk_nccl_unique_id(buf), "sk_nccl_unique_id")
    return bytes(buf)


def nccl_selftest(x: np.ndarray, device: int = 0):
    """sk_nccl_selftest: all-reduce ``x`` (float64) over a one-rank communicator, directly and
    from a captured graph; returns both results."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    o1, o2 = np.empty_like(x), np.empty_like(x)
    _check(load().sk_nccl_selftest(device, x.size, x.ctypes.data, o1.ctypes.data, o2.ctypes.data), "sk_nccl_selftest")
    return o1, o2


class Solver:
    """One sk_ctx.  ``b``/``left`` may be numpy arrays (host; copied) or torch tensors (device:
    b copied, left borrowed).  ``op`` is an sk_operator (keep its device arrays alive).
    Multi-rank: ``rank``/``world`` with either ``group`` (loopback) or, for one process per
    GPU, a later :meth:`connect`."""

    def __init__(self, op: sk_operator, method: str, b, z: np.ndarray, *, left=None,
                 full_x: bool = False, tol: float = 1e-10, itermax: int = 10000, flags: int = 0,
                 device: int = 0, stream: int = 0, rank: int = 0, world: int = 1,
                 group: Optional[Group] = None):
        L = load()
        self._keep = [op, b, left]
        self.z = np.ascontiguousarray(z, dtype=np.complex128)
        self.nz = int(self.z.shape[0])
        self.nl = 1 if left is None else int(left.shape[0])
        self.full_x = bool(full_x)
        p = sk_params()
        p.method = COCG if method == "cocg" else BICG
        p.flags = flags
        p.n_shift = self.nz
        p.z = self.z.ctypes.data
        p.b, p.b_mem = _ptr_mem(b)
        if left is None:
            p.n_left, p.left, p.left_mem = 0, None, MEM_HOST
        else:
            p.left, p.left_mem = _ptr_mem(left)
            p.n_left = self.nl
        p.full_x = int(full_x)
        p.tol = tol
        p.itermax = itermax
        d = sk_dist()
        d.rank, d.world, d.device = rank, world, device
        d.nccl_id, d.stream = None, stream or None
        d.group = group._h.value if group is not None else None
        self._h = ctypes.c_void_p()
        _check(L.sk_init(ctypes.byref(self._h), ctypes.byref(op), ctypes.byref(p), ctypes.byref(d)),
               "sk_init")
        self.M = int(op.M_local)
        if group is not None:
            group.members.append(self)

    # -- multi-rank (one process per GPU) ---------------------------------------------------
    def ipc_handle(self) -> bytes:
        buf = (ctypes.c_char * 64)()
        _check(load().sk_ipc_handle(self._h, buf), "sk_ipc_handle")
        return bytes(buf)

    def connect(self, handles: bytes, nccl_id: bytes):
        _check(load().sk_connect(self._h, handles, nccl_id), "sk_connect")

    def connect_host(self, handles: bytes, allreduce):
        """sk_connect_host: `allreduce(send: np.ndarray, recv: np.ndarray)` sums `send` (float64,
        host) over the ranks into `recv` (marshalling only: the arithmetic of the method stays
        in the kernels; this is the collective the caller owns, e.g. MPI or gloo)."""
        import numpy as _np

        def cb(user, send, recv, n):
            try:
                allreduce(_np.ctypeslib.as_array(send, shape=(n,)), _np.ctypeslib.as_array(recv, shape=(n,)))
                return 0
            except Exception:   # reported to the library as a failed collective (SK_ENCCL)
                return 1
        self._allreduce_cb = ALLREDUCE_FN(cb)   # kept alive as long as the context
        _check(load().sk_connect_host(self._h, handles, self._allreduce_cb, None), "sk_connect_host")

    # -- iteration ---------------------------------------------------------------------
    def update(self) -> int:
        st = ctypes.c_int32()
        _check(load().sk_update(self._h, ctypes.byref(st)), "sk_update")
        return st.value

    def update_rc(self, q_dev, qt_dev=None) -> int:
        st = ctypes.c_int32()
        _check(load().sk_update_rc(self._h, q_dev.data_ptr(),
                                   None if qt_dev is None else qt_dev.data_ptr(), ctypes.byref(st)),
               "sk_update_rc")
        return st.value

    def seed_vectors(self):
        r, t = ctypes.c_void_p(), ctypes.c_void_p()
        _check(load().sk_get_seed_vectors(self._h, ctypes.byref(r), ctypes.byref(t)), "sk_get_seed_vectors")
        return r.value, t.value

    def run(self, max_iters: int, poll_every: int = 64) -> int:
        st = ctypes.c_int32()
        _check(load().sk_run(self._h, max_iters, poll_every, ctypes.byref(st)), "sk_run")
        return st.value

    def enqueue(self, iters: int):
        _check(load().sk_enqueue(self._h, iters), "sk_enqueue")

    # -- results -------------------------------------------------------------------------
    def residuals(self) -> np.ndarray:
        out = np.empty(self.nz, dtype=np.float64)
        _check(load().sk_get_residual(self._h, out.ctypes.data), "sk_get_residual")
        return out

    def projections(self) -> np.ndarray:
        out = np.empty((self.nz, self.nl), dtype=np.complex128)
        _check(load().sk_get_projection(self._h, out.ctypes.data), "sk_get_projection")
        return out

    def solution_ptr(self, k: int) -> int:
        x = ctypes.c_void_p()
        _check(load().sk_get_solution(self._h, k, ctypes.byref(x)), "sk_get_solution")
        return x.value

    def solution(self, k: int) -> np.ndarray:
        """x^(k) copied to host (full mode)."""
        out = np.empty(self.M, dtype=np.complex128)
        _check(load().sk_copy_solution(self._h, k, out.ctypes.data, MEM_HOST), "sk_copy_solution")
        return out

    def recalc(self, z_new):
        """Projections (and residuals) at new shifts from the coefficient log (SK_FLAG_LOG)."""
        z_new = np.ascontiguousarray(z_new, dtype=np.complex128)
        y = np.empty((z_new.shape[0], self.nl), dtype=np.complex128)
        res = np.empty(z_new.shape[0], dtype=np.float64)
        _check(load().sk_recalc(self._h, z_new.shape[0], z_new.ctypes.data, y.ctypes.data, res.ctypes.data),
               "sk_recalc")
        return y, res

    def checkpoint(self) -> bytes:
        """Complete solver state (restart: P:L520)."""
        n = ctypes.c_size_t(0)
        _check(load().sk_checkpoint(self._h, None, ctypes.byref(n)), "sk_checkpoint")
        buf = ctypes.create_string_buffer(n.value)
        _check(load().sk_checkpoint(self._h, buf, ctypes.byref(n)), "sk_checkpoint")
        return buf.raw[:n.value]

    def restore(self, blob: bytes):
        _check(load().sk_restore(self._h, blob, len(blob)), "sk_restore")

    def shift_state(self):
        pi = np.empty(self.nz, dtype=np.complex128)
        act = np.empty(self.nz, dtype=np.uint8)
        ret = np.empty(self.nz, dtype=np.int64)
        _check(load().sk_get_shift_state(self._h, pi.ctypes.data, act.ctypes.data, ret.ctypes.data),
               "sk_get_shift_state")
        return pi, act.astype(bool), ret

    def coefficients(self) -> dict:
        c = sk_coeffs()
        _check(load().sk_get_coefficients(self._h, ctypes.byref(c)), "sk_get_coefficients")
        cz = lambda v: complex(v.re, v.im)
        return dict(iterations=c.iterations, seed_index=c.seed_index, switches=c.switches,
                    spmv_count=c.spmv_count, n_active=c.n_active, status=c.status,
                    z_seed=cz(c.z_seed), alpha=cz(c.alpha), rho=cz(c.rho), beta=cz(c.beta),
                    seed_residual=c.seed_residual)

    def info(self) -> dict:
        """The execution plan sk_init chose (sk_get_info): bond split, CTA counts, arena size."""
        i = sk_info()
        _check(load().sk_get_info(self._h, ctypes.byref(i)), "sk_get_info")
        return dict(split_ahi=i.split_ahi, spmv_ctas=i.spmv_ctas, update_ctas=i.update_ctas,
                    shift_agents=i.shift_agents, arena_bytes=i.arena_bytes,
                    split_fuse=i.split_fuse, left_real=i.left_real,
                    csr_col_blocks=i.csr_col_blocks, csr_block_shift=i.csr_block_shift)

    def debug_timestamps(self) -> np.ndarray:
        out = np.zeros(16, dtype=np.int64)
        _check(load().sk_debug_timestamps(self._h, out.ctypes.data), "sk_debug_timestamps")
        return out

    def profile_enable(self, on: bool = True):
        _check(load().sk_profile_enable(self._h, int(on)), "sk_profile_enable")

    def profile(self, reset: bool = False) -> dict:
        p = sk_profile()
        _check(load().sk_get_profile(self._h, ctypes.byref(p), int(reset)), "sk_get_profile")
        return dict(iterations=p.iterations, launches=p.launches, ms_spmv=p.ms_spmv,
                    ms_scalar=p.ms_scalar, ms_update=p.ms_update)

    @property
    def iterations(self) -> int:
        return self.coefficients()["iterations"]

    def finalize(self):
        if self._h and self._h.value:
            _check(load().sk_finalize(ctypes.byref(self._h)), "sk_finalize")
        self._keep = []

    def __del__(self):
        try:
            self.finalize()
        except Exception:
            pass
