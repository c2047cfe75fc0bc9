"""Contour-integral (Sakurai-Sugiura) eigenvalues inside a circle, on the shifted solver
(PAPER.md "Calculation of internal eigenpairs", Table 3).

Device work goes through libshiftk: one full-mode solver run per source vector phi_l on the
contour points z_j = gamma + rho e^{2 pi i (j + 1/2)/N_z}, the moments
s_{k,l} = sum_j (z_j - gamma)/N_z (z_j - gamma)^k ||phi_l|| x^(j) (trapezoidal rule for
P:L708-712, z0 = gamma; the solver runs on phi_l/||phi_l||, R18/R29) by sk_combine,
the Gram matrices by sk_gram, H U~ by sk_apply_operator.  The SVD of the tall S is taken
through its Gram matrix S^dagger S = V Sigma^2 V^dagger; singular values below `sv_tol`
(absolute, Table 3 caption) are dropped; the Ritz values solve the M_nz x M_nz generalised
problem (U~^dagger H U~) v = lambda (U~^dagger U~) v on the host.
"""
from __future__ import annotations

import numpy as np

from . import shiftk


def contour_points(n_z: int, gamma: float, rho: float) -> np.ndarray:
    j = np.arange(n_z, dtype=np.float64)
    return (gamma + rho * np.exp(2j * np.pi * (j + 0.5) / n_z)).astype(np.complex128)


def ss_eigenvalues(op: dict, phis: np.ndarray, gamma: float, rho: float, n_z: int, n_k: int, *,
                   sv_tol: float = 1e-3, tol: float = 1e-10, itermax: int = 20000,
                   device: str = "cuda:0", dev_arrays=None, return_details: bool = False):
    """Eigenvalues of H inside |z - gamma| < rho (ascending) from n_l = len(phis) sources.
    CSR operators need their device arrays (`dev_arrays`); a complex Hermitian H is solved
    with BiCG, a real-symmetric one with COCG (Table 1)."""
    import torch
    dev = torch.device(device)
    n_l, M = phis.shape
    z = contour_points(n_z, gamma, rho)
    hop = shiftk.make_operator(op, M, dev_arrays)
    method = "bicg" if op["kind"] == "csr_cplx" else "cocg"
    S = torch.empty((n_l * n_k, M), dtype=torch.complex128, device=dev)
    iters = []
    for l in range(n_l):
        nrm = float(np.sqrt(np.vdot(phis[l], phis[l]).real))
        b = torch.from_numpy(np.ascontiguousarray(phis[l] / nrm)).to(dev)
        sol = shiftk.Solver(hop, method, b, z, full_x=True, tol=tol, itermax=itermax)
        st = sol.run(itermax)
        if st != shiftk.CONVERGED:
            raise RuntimeError(f"contour solve {l}: status {st}")
        iters.append(sol.coefficients()["iterations"])
        x0 = sol.solution_ptr(0)
        ld = (sol.solution_ptr(1) - x0) // 16 if n_z > 1 else M
        w = (z - gamma) / n_z * nrm
        W = np.stack([w * (z - gamma) ** k for k in range(n_k)], axis=1)   # [n_z, n_k]
        shiftk.combine(x0, n_z, ld, M, W, S[l * n_k:(l + 1) * n_k])
        sol.finalize()
    G = shiftk.gram(S, S)
    lam, V = np.linalg.eigh(G)                       # S^dagger S = V Sigma^2 V^dagger
    sig = np.sqrt(np.clip(lam[::-1], 0.0, None))
    V = V[:, ::-1]
    keep = sig >= sv_tol
    Wu = V[:, keep] / sig[keep]                        # U~ = S V Sigma^{-1}
    r = int(keep.sum())
    U = torch.empty((r, M), dtype=torch.complex128, device=dev)
    shiftk.combine(S.data_ptr(), S.shape[0], M, M, Wu, U)
    HU = torch.empty_like(U)
    for c in range(r):
        shiftk.apply_operator(hop, U[c], HU[c])
    A = shiftk.gram(U, HU)
    B = shiftk.gram(U, U)
    ev = np.sort(np.linalg.eigvals(np.linalg.solve(B, A)).real)
    inside = ev[np.abs(ev - gamma) < rho]
    if return_details:
        return inside, {"singular_values": sig, "rank": r, "iterations": iters, "all_ritz": ev}
    return inside
