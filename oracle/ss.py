"""Contour-integral (Sakurai-Sugiura) eigenvalues from the shifted solver's solutions (SURVEY
§8(f) f-2; PAPER.md "Calculation of internal eigenpairs") — TEST INFRASTRUCTURE
ONLY (same rules as oracle/__init__.py).  Plain numpy, the paper's steps in its order:

  x_{j,l} = (z_j I - H)^{-1} phi_l            the shifted solver, P:L700-704 (phi'_0); run on
            phi_l/||phi_l|| (R18) and scaled back by ||phi_l|| (linear)
  s_{k,l} = 1/(2 pi i) oint (z - z0)^k x(z) dz  P:L708-712, trapezoidal rule on the circle
            z_j = gamma + rho e^{2 pi i (j + 1/2)/N_z}: dz = i (z_j - gamma) dtheta,
            dtheta = 2 pi / N_z, so s_{k,l} = sum_j (z_j - gamma)/N_z (z_j - z0)^k x_{j,l};
            z0 = gamma (the paper leaves z0 free; R29)
  S = (s_{0,0} .. s_{Nk-1,0}, s_{0,1}, .., s_{Nk-1,Nl-1})
  S = U Sigma V^dagger; keep singular values >= 1e-3       P:L735-745, Table 3 caption (R29:
            absolute, with phi_l of i.i.d. standard normal entries — the reading that
            reproduces all three SS columns of Table 3)
  H~ = U~^dagger H U~, eigenvalues of H~
Parity status: pinned by Table 3, columns SS(10,1), SS(10,2), SS(10,5).
"""
from __future__ import annotations

import numpy as np

from . import CONVERGED, Oracle, apply_op


def contour_solutions(op: dict, phis: np.ndarray, z: np.ndarray, *, tol: float = 1e-10,
                      itermax: int = 20000) -> np.ndarray:
    """X[l, j, :] = (z_j - H)^{-1} phi_l by the oracle's shifted COCG (one run per phi_l)."""
    n_l, M = phis.shape
    X = np.empty((n_l, z.shape[0], M), dtype=np.complex128)
    for l in range(n_l):
        nrm = np.sqrt(np.vdot(phis[l], phis[l]).real)
        o = Oracle("cocg", phis[l] / nrm, z, full_x=True, tol=tol, itermax=itermax)
        assert o.run(op, itermax) == CONVERGED
        for j in range(z.shape[0]):
            X[l, j] = nrm * o.solution(j)
    return X


def moments(X: np.ndarray, z: np.ndarray, gamma: complex, n_k: int) -> np.ndarray:
    """S columns s_{k,l} (column index l * n_k + k), trapezoidal rule, z0 = gamma."""
    n_l, n_z, M = X.shape
    S = np.empty((M, n_l * n_k), dtype=np.complex128)
    for l in range(n_l):
        for k in range(n_k):
            s = np.zeros(M, dtype=np.complex128)
            for j in range(n_z):
                s += (z[j] - gamma) / n_z * (z[j] - gamma) ** k * X[l, j]
            S[:, l * n_k + k] = s
    return S


def rayleigh_ritz(op: dict, S: np.ndarray, sv_tol: float = 1e-3):
    """SVD of S, the kept left singular vectors U~, and the eigenvalues of U~^dagger H U~."""
    U, sig, _ = np.linalg.svd(S, full_matrices=False)
    keep = sig >= sv_tol
    Ut = U[:, keep]
    HU = np.stack([apply_op(op, np.ascontiguousarray(Ut[:, c])) for c in range(Ut.shape[1])], axis=1)
    Ht = Ut.conj().T @ HU
    return np.sort(np.linalg.eigvals(Ht).real), sig


def ss_eigenvalues(op: dict, phis: np.ndarray, gamma: float, rho: float, n_z: int, n_k: int,
                   *, sv_tol: float = 1e-3, tol: float = 1e-10):
    """Eigenvalues inside the circle |z - gamma| < rho (ascending) and the singular values."""
    j = np.arange(n_z, dtype=np.float64)
    z = (gamma + rho * np.exp(2j * np.pi * (j + 0.5) / n_z)).astype(np.complex128)
    X = contour_solutions(op, phis, z, tol=tol)
    S = moments(X, z, gamma, n_k)
    ev, sig = rayleigh_ritz(op, S, sv_tol)
    return ev[np.abs(ev - gamma) < rho], sig
