"""Contour-integral eigensolver on the GPU: the building blocks sk_combine /
sk_gram against numpy, and the whole Sakurai-Sugiura pipeline (full-mode shifted COCG on the
Sz = 0 sector, moments, Gram-matrix SVD, Rayleigh-Ritz) against Table 3 and the
oracle's implementation (oracle/ss.py)."""
import os

import numpy as np
import pytest

import oracle
import oracle.ss as oss
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2001_08707_b200 import contour, shiftk  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_combine_matches_numpy():
    rng = np.random.default_rng(1)
    n_in, M, n_out, ld = 37, 5001, 13, 5003
    X = rng.standard_normal((n_in, ld)) + 1j * rng.standard_normal((n_in, ld))
    W = rng.standard_normal((n_in, n_out)) + 1j * rng.standard_normal((n_in, n_out))
    Xd = torch.from_numpy(X).cuda()
    out = torch.empty((n_out, M), dtype=torch.complex128, device="cuda")
    shiftk.combine(Xd.data_ptr(), n_in, ld, M, W, out)
    want = W.T @ X[:, :M]
    assert np.max(np.abs(out.cpu().numpy() - want)) <= 1e-13 * np.max(np.abs(want))


def test_gram_matches_numpy_and_is_deterministic():
    rng = np.random.default_rng(2)
    na, nb, M = 50, 7, 12345
    A = rng.standard_normal((na, M)) + 1j * rng.standard_normal((na, M))
    B = rng.standard_normal((nb, M)) + 1j * rng.standard_normal((nb, M))
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    G = shiftk.gram(Ad, Bd)
    want = A.conj() @ B.T
    assert np.max(np.abs(G - want)) <= 1e-12 * np.max(np.abs(want))
    assert np.array_equal(G, shiftk.gram(Ad, Bd))


@pytest.mark.parametrize("col,n_l", [(1, 1), (2, 2), (3, 5)])
def test_ss_pipeline_reproduces_table3(col, n_l):
    tab = np.loadtxt(os.path.join(GOLDEN, "table3_ss.txt"))
    want = tab[:, col][~np.isnan(tab[:, col])]
    op, phis, z = synth.ss_inputs()
    ev, info = contour.ss_eigenvalues(op, phis[:n_l], -5.0, 0.8, 100, 10, return_details=True)
    assert ev.size == want.size, info["singular_values"][:10]
    assert np.max(np.abs(ev - want)) < 1e-6
    eo, sig_o = oss.ss_eigenvalues(op, phis[:n_l], -5.0, 0.8, 100, 10)
    assert np.max(np.abs(ev - eo)) < 1e-9
    k = min(info["rank"] + 1, sig_o.size)
    assert np.allclose(info["singular_values"][:info["rank"]], sig_o[:info["rank"]], rtol=1e-7)
    assert np.all(info["singular_values"][info["rank"]:k] < 1e-3)


def test_ss_on_the_complex_lattice_matches_dense_eigenvalues():
    """The contour-integral path on a complex Hermitian CSR operator (BiCG, Table 1): the C4
    Peierls lattice at 8 x 8 sites, eigenvalues inside a circle against a dense eigensolve."""
    p = synth.make_problem("c4", W=8, nz=4, n_left=1)
    M = p.M
    H = np.zeros((M, M), dtype=np.complex128)
    e = np.zeros(M, dtype=np.complex128)
    for j in range(M):
        e[:] = 0
        e[j] = 1
        H[:, j] = oracle.apply_op(p.op, e)
    lam = np.linalg.eigvalsh(H)
    gaps = np.diff(lam)
    k = int(np.argmax(gaps[M // 2:M // 2 + 20])) + M // 2   # a well separated window edge
    gamma = 0.5 * (lam[k - 5] + lam[k])
    rho = 0.5 * (lam[k] - lam[k - 5]) + 0.5 * gaps[k]
    want = lam[np.abs(lam - gamma) < rho]
    rng = np.random.Generator(np.random.PCG64(11))
    phis = rng.standard_normal((6, M)) + 1j * rng.standard_normal((6, M))
    arrays = {kk: torch.from_numpy(p.op[kk]).cuda() for kk in ("row_ptr", "col", "val")}
    ev = contour.ss_eigenvalues(p.op, phis, gamma, rho, 128, 8, dev_arrays=arrays, sv_tol=1e-6)
    assert ev.size == want.size
    assert np.max(np.abs(ev - want)) < 1e-7
