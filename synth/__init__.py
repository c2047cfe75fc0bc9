"""Seeded synthetic inputs for the shifted-Krylov hot path (configs C1-C5 and scaled variants).

This module is the ONE place shared by the oracle side (tests/, bench.py cpu_baseline) and the
CUDA side (paper_2001_08707_b200).  It holds no arithmetic of the method: it only draws the
shifts z_k, the right-hand side b, the left vectors a_l and the operator H (a Heisenberg chain
descriptor or a CSR matrix) from numpy ``Generator(PCG64(seed))`` streams, in the draw order
fixed by DESIGN.md "Input recipe".

Paper anchors (PAPER.md = /root/reference/PAPER.md, cited as P:Lnnn):
  * spectrum shifts  omega_i = omega_min + i (omega_max - omega_min)/N, i < N
  * contour points   z_j = gamma + rho exp(2 pi i (j + 1/2)/N_z)
  * Heisenberg chain H = J sum_i S_i . S_{i+1}, periodic, S = 1/2
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = ["Problem", "CONFIGS", "make_problem", "spectrum_shifts", "contour_shifts",
           "heisenberg_problem", "heisenberg_sz_problem", "ss_inputs", "csr_real_problem", "lattice_problem"]


@dataclasses.dataclass
class Problem:
    """One seeded instance of (z_k I - H) x^(k) = b with optional left vectors a_l.

    op:    {"kind": "heisenberg", "L": int, "J": float}
           {"kind": "csr_real", "row_ptr": int64[M+1], "col": int32[nnz], "val": float64[nnz]}
           {"kind": "csr_cplx", "row_ptr": int64[M+1], "col": int32[nnz], "val": complex128[nnz]}
    b:     complex128[M] (normalised, ||b||_2 = 1)
    z:     complex128[N_z]
    left:  complex128[N_left, M] or None (None = projection onto b itself, "a = b")
    """
    name: str
    M: int
    op: dict
    b: np.ndarray
    z: np.ndarray
    left: Optional[np.ndarray]
    method: str          # "cocg" | "bicg"   (Table 1)
    full_x: bool         # store x^(k) (P = I)
    tol: float
    itermax: int
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def n_shift(self) -> int:
        return int(self.z.shape[0])

    @property
    def n_left(self) -> int:
        return 1 if self.left is None else int(self.left.shape[0])


def spectrum_shifts(n: int, wmin: float, wmax: float, delta: float) -> np.ndarray:
    """omega_i = wmin + i (wmax - wmin)/n (right end excluded) plus i*delta."""
    i = np.arange(n, dtype=np.float64)
    return (wmin + i * (wmax - wmin) / n + 1j * delta).astype(np.complex128)


def contour_shifts(n: int, gamma: float, rho: float) -> np.ndarray:
    """z_j = gamma + rho exp(2 pi i (j + 1/2)/n)."""
    j = np.arange(n, dtype=np.float64)
    return (gamma + rho * np.exp(2j * np.pi * (j + 0.5) / n)).astype(np.complex128)


def _normalise(v: np.ndarray) -> np.ndarray:
    nrm = math.sqrt(float(np.vdot(v, v).real))
    return v / nrm


def heisenberg_problem(name: str, L: int, seed: int, z: np.ndarray, *, J: float = 1.0,
                       full_x: bool = False, tol: float = 1e-10, itermax: int = 20000) -> Problem:
    """Heisenberg chain, full 2^L space, b = normalised PCG64(seed).standard_normal(2^L), a = b."""
    M = 1 << L
    rng = np.random.Generator(np.random.PCG64(seed))
    b = _normalise(rng.standard_normal(M)).astype(np.complex128)
    return Problem(name=name, M=M, op={"kind": "heisenberg", "L": L, "J": float(J)}, b=b, z=z,
                   left=None, method="cocg", full_x=full_x, tol=tol, itermax=itermax,
                   meta={"L": L, "seed": seed})


def heisenberg_sz_problem(name: str, L: int, n_up: int, seed: int, z: np.ndarray, *, J: float = 1.0,
                          full_x: bool = False, tol: float = 1e-10, itermax: int = 20000) -> Problem:
    """Heisenberg chain restricted to the sector of n_up up spins (rows = the
    L-bit states with popcount n_up in ascending order, R28); b = normalised
    PCG64(seed).standard_normal(C(L, n_up)), a = b."""
    M = math.comb(L, n_up)
    rng = np.random.Generator(np.random.PCG64(seed))
    b = _normalise(rng.standard_normal(M)).astype(np.complex128)
    return Problem(name=name, M=M, op={"kind": "heisenberg_sz", "L": L, "J": float(J), "n_up": n_up},
                   b=b, z=z, left=None, method="cocg", full_x=full_x, tol=tol, itermax=itermax,
                   meta={"L": L, "n_up": n_up, "seed": seed})


def ss_inputs(L: int = 12, n_up: int = 6, n_l: int = 5, seed: int = 7, gamma: float = -5.0,
              rho: float = 0.8, n_z: int = 100):
    """Inputs of the contour-integral example (Table 3): the
    sector operator, N_l source vectors phi_l with i.i.d. standard normal entries (drawn from
    PCG64(seed) as one [n_l, C(L, n_up)] array; R29), and the contour points."""
    D = math.comb(L, n_up)
    rng = np.random.Generator(np.random.PCG64(seed))
    phis = rng.standard_normal((n_l, D)).astype(np.complex128)
    op = {"kind": "heisenberg_sz", "L": L, "J": 1.0, "n_up": n_up}
    return op, phis, contour_shifts(n_z, gamma, rho)


def csr_real_problem(name: str, M: int, seed: int, z: np.ndarray, *, n_match: int = 11,
                     full_x: bool = True, tol: float = 1e-10, itermax: int = 20000) -> Problem:
    """C3 recipe: circulant band (i, i+-1, i+-2 mod M) plus ``n_match``
    random perfect matchings (a permutation split into consecutive pairs); symmetric values,
    off-diagonal U[-1,1], diagonal U[-4,4]; collisions merged by summing.

    Draw order from PCG64(seed): b (M normals); n_match permutations; diagonal (M);
    band+1 values (M); band+2 values (M); one value per matched pair per matching (M/2 each).
    """
    assert M >= 8 and M % 2 == 0
    rng = np.random.Generator(np.random.PCG64(seed))
    b = _normalise(rng.standard_normal(M)).astype(np.complex128)
    perms = [rng.permutation(M) for _ in range(n_match)]
    diag = rng.uniform(-4.0, 4.0, M)
    v1 = rng.uniform(-1.0, 1.0, M)   # bond (i, i+1 mod M)
    v2 = rng.uniform(-1.0, 1.0, M)   # bond (i, i+2 mod M)
    width = 5 + n_match
    cols = np.empty((M, width), dtype=np.int64)
    vals = np.empty((M, width), dtype=np.float64)
    i = np.arange(M, dtype=np.int64)
    cols[:, 0] = i;            vals[:, 0] = diag
    cols[:, 1] = (i + 1) % M;  vals[:, 1] = v1
    cols[:, 2] = (i - 1) % M;  vals[:, 2] = v1[(i - 1) % M]
    cols[:, 3] = (i + 2) % M;  vals[:, 3] = v2
    cols[:, 4] = (i - 2) % M;  vals[:, 4] = v2[(i - 2) % M]
    for m, perm in enumerate(perms):
        pv = rng.uniform(-1.0, 1.0, M // 2)
        a, c = perm[0::2], perm[1::2]
        cols[a, 5 + m] = c; vals[a, 5 + m] = pv
        cols[c, 5 + m] = a; vals[c, 5 + m] = pv
    del perms
    row_ptr, col, val = _rows_to_csr(cols, vals)
    return Problem(name=name, M=M, op={"kind": "csr_real", "row_ptr": row_ptr, "col": col,
                                        "val": val},
                   b=b, z=z, left=None, method="cocg", full_x=full_x, tol=tol, itermax=itermax,
                   meta={"seed": seed, "n_match": n_match, "nnz": int(col.shape[0])})


def lattice_problem(name: str, W: int, seed: int, z: np.ndarray, n_left: int, *,
                    tol: float = 1e-10, itermax: int = 50000, full_x: bool = False) -> Problem:
    """C4 recipe: periodic W x W torus, site i = y W + x, hopping
    H[i, i+x] = exp(i theta_x[i]), H[i, i+y] = exp(i theta_y[i]) (Hermitian partners conjugated),
    theta ~ U[0, 2 pi), on-site U[-1,1].  b real Gaussian; left vectors complex Gaussian with
    re, im ~ N(0, 1/2).

    Draw order from PCG64(seed): b (M); per left vector re (M) then im (M); on-site (M);
    theta_x (M); theta_y (M).
    """
    assert W >= 3
    M = W * W
    rng = np.random.Generator(np.random.PCG64(seed))
    b = _normalise(rng.standard_normal(M)).astype(np.complex128)
    left = np.empty((n_left, M), dtype=np.complex128)
    s = math.sqrt(0.5)
    for l in range(n_left):
        left[l].real = rng.standard_normal(M) * s
        left[l].imag = rng.standard_normal(M) * s
    onsite = rng.uniform(-1.0, 1.0, M)
    tx = rng.uniform(0.0, 2.0 * math.pi, M)
    ty = rng.uniform(0.0, 2.0 * math.pi, M)
    i = np.arange(M, dtype=np.int64)
    x, y = i % W, i // W
    right = y * W + (x + 1) % W
    lft = y * W + (x - 1) % W
    up = ((y + 1) % W) * W + x
    down = ((y - 1) % W) * W + x
    cols = np.stack([i, right, lft, up, down], axis=1)
    vals = np.empty((M, 5), dtype=np.complex128)
    vals[:, 0] = onsite
    vals[:, 1] = np.exp(1j * tx)           # H[i, i+x]
    vals[:, 2] = np.exp(-1j * tx[lft])     # H[i, i-x] = conj(H[i-x, i])
    vals[:, 3] = np.exp(1j * ty)           # H[i, i+y]
    vals[:, 4] = np.exp(-1j * ty[down])    # H[i, i-y]
    row_ptr, col, val = _rows_to_csr(cols, vals)
    return Problem(name=name, M=M, op={"kind": "csr_cplx", "row_ptr": row_ptr, "col": col,
                                        "val": val},
                   b=b, z=z, left=left, method="bicg", full_x=full_x, tol=tol, itermax=itermax,
                   meta={"seed": seed, "W": W, "nnz": int(col.shape[0])})


def _rows_to_csr(cols: np.ndarray, vals: np.ndarray):
    """Fixed-width per-row (col, val) lists -> CSR with sorted columns; equal columns in one
    row are merged by summing their values."""
    M, width = cols.shape
    order = np.argsort(cols, axis=1, kind="stable")
    cols = np.take_along_axis(cols, order, axis=1)
    vals = np.take_along_axis(vals, order, axis=1)
    dup = np.zeros((M, width), dtype=bool)
    dup[:, 1:] = cols[:, 1:] == cols[:, :-1]
    if dup.any():
        # fold duplicates into the first occurrence (rows with >2 equal columns handled by loop)
        r, c = np.nonzero(dup)
        for rr, cc in zip(r.tolist(), c.tolist()):
            k = cc - 1
            while dup[rr, k]:
                k -= 1
            vals[rr, k] += vals[rr, cc]
        keep = ~dup
        counts = keep.sum(axis=1)
        row_ptr = np.zeros(M + 1, dtype=np.int64)
        np.cumsum(counts, out=row_ptr[1:])
        col = cols[keep].astype(np.int32)
        val = vals[keep]
    else:
        row_ptr = np.arange(0, (M + 1) * width, width, dtype=np.int64)
        col = cols.reshape(-1).astype(np.int32)
        val = vals.reshape(-1)
    return row_ptr, col, np.ascontiguousarray(val)


# ---------------------------------------------------------------------------------------------
# The five BASELINE.json configs; ``scale`` shrinks them for parity tests.
# ---------------------------------------------------------------------------------------------

CONFIGS = {
    "c1": dict(desc="Heisenberg L=12, 16 shifts w+0.1i in [-6,2), COCG, full x", L=12, seed=0,
               nz=16, w=(-6.0, 2.0), delta=0.1, full_x=True, tol=1e-10, itermax=2000),
    "c2": dict(desc="Heisenberg L=20, 1024 shifts w+0.05i in [-10,4), COCG, a=b", L=20, seed=1,
               nz=1024, w=(-10.0, 4.0), delta=0.05, full_x=False, tol=1e-10, itermax=20000),
    "c3": dict(desc="real-symmetric CSR M=2^24 x16 nnz, 128 shifts w+0.02i in [-6,6), COCG, full x",
               M=1 << 24, seed=2, nz=128, w=(-6.0, 6.0), delta=0.02, full_x=True, tol=1e-10,
               itermax=20000),
    "c4": dict(desc="Hermitian Peierls lattice 8192^2, 64 contour points, 32 left vectors, BiCG",
               W=8192, seed=3, nz=64, gamma=0.5, rho=0.25, n_left=32, tol=1e-10, itermax=50000),
    "c5": dict(desc="Heisenberg L=30, 512 shifts w+0.05i in [-16,4), COCG, a=b", L=30, seed=4,
               nz=512, w=(-16.0, 4.0), delta=0.05, full_x=False, tol=1e-10, itermax=20000),
    # C5's chain in its largest sector (2Sz = 0, C(30,15) = 1.55e8 rows)
    "c5sz": dict(desc="Heisenberg L=30 Sz=0 sector, 512 shifts w+0.05i in [-16,4), COCG, a=b",
                 L=30, n_up=15, seed=4, nz=512, w=(-16.0, 4.0), delta=0.05, full_x=False,
                 tol=1e-10, itermax=20000),
}


def make_problem(name: str, **override) -> Problem:
    """Build config ``name`` (c1..c5); keyword overrides (L, M, W, nz, n_left, tol, itermax,
    full_x, seed) give the scaled-down parity variants.  The shift geometry keeps the config's
    window and broadening."""
    cfg = dict(CONFIGS[name])
    cfg.update(override)
    tag = name if not override else name + "[" + ",".join(f"{k}={v}" for k, v in
                                                         sorted(override.items())) + "]"
    if name in ("c1", "c2", "c5"):
        z = spectrum_shifts(cfg["nz"], cfg["w"][0], cfg["w"][1], cfg["delta"])
        return heisenberg_problem(tag, cfg["L"], cfg["seed"], z, full_x=cfg["full_x"],
                                  tol=cfg["tol"], itermax=cfg["itermax"])
    if name == "c5sz":
        z = spectrum_shifts(cfg["nz"], cfg["w"][0], cfg["w"][1], cfg["delta"])
        n_up = cfg["n_up"] if "n_up" in override else cfg["L"] // 2
        return heisenberg_sz_problem(tag, cfg["L"], n_up, cfg["seed"], z, full_x=cfg["full_x"],
                                     tol=cfg["tol"], itermax=cfg["itermax"])
    if name == "c3":
        z = spectrum_shifts(cfg["nz"], cfg["w"][0], cfg["w"][1], cfg["delta"])
        return csr_real_problem(tag, cfg["M"], cfg["seed"], z, full_x=cfg["full_x"],
                                tol=cfg["tol"], itermax=cfg["itermax"])
    if name == "c4":
        z = contour_shifts(cfg["nz"], cfg["gamma"], cfg["rho"])
        return lattice_problem(tag, cfg["W"], cfg["seed"], z, cfg["n_left"], tol=cfg["tol"],
                               itermax=cfg["itermax"])
    raise KeyError(name)
