"""GPU parity at BASELINE.json's FULL sizes (C3, C4, C5), in the launch configuration bench.py
times, on what the oracle can afford there:

* C3 (M = 2^24, 128 shifts, full x): the first n_w iterations against the oracle, all residuals
  and projections compared, x^(k) compared for two carried shifts (the oracle's keep mask: its
  scalar recurrences and seed switching still run over all 128 shifts);
* C4 (8192^2 lattice, 64 contour points, 32 left vectors, BiCG): first n_w iterations, all
  64 x 32 projections and residuals;
* C5 (L = 30, 2^30 states, 512 shifts, a = b): the first iterations against the oracle (all
  512 residuals and projections), sampled rows of H r against the oracle's row routine, the
  ferromagnet H 1 = (L/4) 1 bit-exactly, and exact termination after 3 iterations for a
  right-hand side with 3 distinct energies (closed-form G(z)) — properties that hold at any size;
  its Sz = 0 sector (f-3): sampled rows.

Window length: n_w = min(cap, self-divergence horizon), the horizon measured
on a scaled instance of the same geometry (tests/horizon.py; two oracle runs at full size would
double the cost).  The oracle runs its OpenMP build here (bit-identical to the one-thread build,
tests/test_oracle_pins.py::test_openmp_build_is_bit_identical) on the host's cores.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from horizon import horizon_of

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2001_08707_b200 import shiftk  # noqa: E402
from paper_2001_08707_b200.device import make_solver, to_device  # noqa: E402

REL = 1e-9


def proj_err(a, b):
    return np.max(np.abs(a - b), axis=1) / np.maximum(np.max(np.abs(b), axis=1), 1e-300)


def window(p, n_w, keep=None, check_x=()):
    dp = to_device(p)
    g = make_solver(dp)
    o = oracle.Oracle(p.method, p.b, p.z, left=p.left, full_x=p.full_x, tol=p.tol,
                      itermax=p.itermax, keep=keep, omp=True)
    for n in range(n_w):
        assert g.update() == o.step(p.op) == shiftk.ITERATING
        rg, ro = g.residuals(), o.residuals()
        assert np.all(np.abs(rg - ro) <= REL * ro), (n, np.max(np.abs(rg - ro) / ro))
        assert np.all(proj_err(g.projections(), o.projections()) <= REL), n
        for k in check_x:
            xo = o.solution(k)
            assert np.linalg.norm(g.solution(k) - xo) <= REL * np.linalg.norm(xo), (n, k)
    return dp, g


def sampled_rows(p, dp, r, rows):
    rd = torch.from_numpy(r).cuda()
    qd = torch.empty_like(rd)
    shiftk.apply_operator(dp.op, rd, qd)
    torch.cuda.synchronize()
    qg = qd[torch.as_tensor(rows, device="cuda")].cpu().numpy()
    qo = oracle.apply_rows(p.op, r, rows)
    assert np.max(np.abs(qg - qo)) <= 1e-14 * np.max(np.abs(qo))


def test_c3_full_size():
    n_w = min(20, horizon_of("c3", 20, M=1 << 14))
    assert n_w >= 10, n_w
    p = synth.make_problem("c3")
    keep = np.zeros(p.n_shift, dtype=np.uint8)
    keep[[5, 77]] = 1
    dp, g = window(p, n_w, keep=keep, check_x=(5, 77))
    rows = np.random.default_rng(7).integers(0, p.M, 64)
    sampled_rows(p, dp, p.b, rows)


def test_c4_full_size():
    n_w = min(12, horizon_of("c4", 12, W=64))
    assert n_w >= 8, n_w
    p = synth.make_problem("c4")
    dp, g = window(p, n_w)
    c = g.coefficients()
    assert c["spmv_count"] == 2 * c["iterations"] == 2 * n_w
    rows = np.random.default_rng(8).integers(0, p.M, 64)
    sampled_rows(p, dp, p.left[3], rows)


def test_c5_full_size_window():
    """C5 exactly as bench.py times it (L = 30, M = 2^30, 512 shifts w + 0.05i in [-16, 4), a = b,
    the single-GPU pair / split SpMV and the fused update): the first iterations against the
    oracle on all 512 shifts, 1e-9 on residuals and projections."""
    n_w = min(5, horizon_of("c5", 5, L=18))
    assert n_w == 5
    p = synth.make_problem("c5")
    dp, g = window(p, n_w)
    assert g.coefficients()["iterations"] == n_w
    del dp, g, p
    torch.cuda.empty_cache()


def _popcount(a):
    return np.bitwise_count(a)


def test_c5_full_size_operator_and_exact_termination():
    L = 30
    M = 1 << L
    op = shiftk.make_operator({"kind": "heisenberg", "L": L, "J": 1.0}, M)
    # (1) ferromagnet, bit-exact, every cross-shard bond exercised
    one = torch.ones(M, dtype=torch.complex128, device="cuda")
    q = torch.empty_like(one)
    shiftk.apply_operator(op, one, q)
    assert torch.equal(q, torch.full_like(one, L / 4))
    del one, q
    torch.cuda.empty_cache()
    # (2) sampled rows of H b for the C5 right-hand side
    p = synth.make_problem("c5")
    dp = to_device(p)
    rows = np.concatenate([[0, 1, M - 1, M // 2 + 12345], np.random.default_rng(9).integers(0, M, 60)])
    sampled_rows(p, dp, p.b, rows)
    del dp, p
    torch.cuda.empty_cache()
    # (3) exact termination: b = product state + two real one-magnon standing waves, energies
    #     L/4, J(L/4 - 1 + cos k): COCG stops after 3 iterations with G(z) = sum_j w_j/(z - E_j)
    th = 0.9
    s = np.arange(M, dtype=np.uint32)
    pc = _popcount(s).astype(np.float64)
    del s
    psiF = np.cos(th / 2) ** pc * np.sin(th / 2) ** (L - pc)
    del pc
    psiF *= 0.6 / np.linalg.norm(psiF)
    b = psiF.astype(np.complex128)
    wF = float(np.vdot(psiF, psiF).real)
    del psiF
    comps_w, energies = [wF], [L / 4]
    for m, cnorm in [(2, 0.5), (7, 0.62)]:
        k = 2 * math.pi * m / L
        w = np.array([math.cos(k * j) for j in range(L)])
        w *= cnorm / np.linalg.norm(w)
        for j in range(L):
            b[1 << j] += w[j]
        comps_w.append(float(np.dot(w, w)))
        energies.append(L / 4 - 1 + math.cos(k))
    z = synth.spectrum_shifts(24, -16.0, 4.0, 0.05)
    bd = torch.from_numpy(b).cuda()
    del b
    g = shiftk.Solver(op, "cocg", bd, z, tol=1e-10, itermax=50)
    st = g.run(50)
    assert st == shiftk.CONVERGED and g.iterations == 3
    Gex = np.array([sum(wj / (zz - e) for wj, e in zip(comps_w, energies)) for zz in z])
    res = g.residuals()
    assert np.max(res) < 1e-10
    # rigorous bound |G_n - G| <= ||r^(k)|| / |Im z| (rounding of psi_F dominates at L = 30)
    assert np.all(np.abs(g.projections()[:, 0] - Gex) <= res / 0.05 + 1e-13)


def test_c5sz_full_size_sector_operator_sampled_rows():
    """The L = 30 chain in its Sz = 0 sector (f-3, C(30,15) = 155,117,520 rows): sampled rows of
    H r (GPU combinatorial ranking) against the oracle's counting-rank row routine, including
    the first and last rows and rows whose periodic bond is active."""
    L, n = 30, 15
    D = math.comb(L, n)
    rng = np.random.default_rng(30)
    r = rng.standard_normal(D) + 1j * rng.standard_normal(D)
    op = shiftk.make_operator({"kind": "heisenberg_sz", "L": L, "J": 1.0, "n_up": n}, D)
    rd = torch.from_numpy(r).cuda()
    qd = torch.empty_like(rd)
    shiftk.apply_operator(op, rd, qd)
    torch.cuda.synchronize()
    rows = [0, 1, 2, D // 3, D // 2, D - 2, D - 1] + list(rng.integers(0, D, 40))
    q_rows = qd[torch.tensor(rows, device="cuda")].cpu().numpy()
    del qd, rd
    qo = oracle.apply_rows({"kind": "heisenberg_sz", "L": L, "n_up": n, "J": 1.0}, r, rows)
    assert np.max(np.abs(q_rows - qo) / np.maximum(np.abs(qo), 1e-300)) <= 1e-13


def _hash_vec_np(k):
    """r_k from an integer hash of the row index (20-bit fractions: exact in fp64 on both sides)."""
    k = np.asarray(k, dtype=np.int64)
    re = ((k * 2654435761) & 0xFFFFF).astype(np.float64) / 1048576.0 - 0.5
    im = (((k * 40503 + 12345) >> 3) & 0xFFFFF).astype(np.float64) / 1048576.0 - 0.5
    return re + 1j * im


def test_sector_operator_beyond_2_31_rows_sampled():
    """L = 34, Sz = 0: C(34,17) = 2,333,606,220 rows (> 2^31; 37 GB per vector), the block
    kernel's 64-bit row and block offsets.  r_k is an integer hash of k, generated on the GPU in
    chunks and evaluated by the oracle's row routine as a function (the vector does not fit on
    the host); sampled rows incl. the first, last and around 2^31."""
    L, n = 34, 17
    D = math.comb(L, n)
    rd = torch.empty(D, dtype=torch.complex128, device="cuda")
    ch = 1 << 27
    for k0 in range(0, D, ch):
        k = torch.arange(k0, min(D, k0 + ch), dtype=torch.int64, device="cuda")
        re = ((k * 2654435761) & 0xFFFFF).to(torch.float64) / 1048576.0 - 0.5
        im = (((k * 40503 + 12345) >> 3) & 0xFFFFF).to(torch.float64) / 1048576.0 - 0.5
        rd[k0:k0 + k.shape[0]] = torch.complex(re, im)
        del k, re, im
    qd = torch.empty_like(rd)
    op = shiftk.make_operator({"kind": "heisenberg_sz", "L": L, "J": 1.0, "n_up": n}, D)
    shiftk.apply_operator(op, rd, qd)
    torch.cuda.synchronize()
    rng = np.random.default_rng(34)
    rows = [0, 1, (1 << 31) - 1, 1 << 31, (1 << 31) + 1, D // 2, D - 2, D - 1] + list(rng.integers(0, D, 24))
    q_rows = qd[torch.tensor(rows, device="cuda")].cpu().numpy()
    assert np.array_equal(rd[torch.tensor(rows[:4], device="cuda")].cpu().numpy(), _hash_vec_np(rows[:4]))
    del qd, rd
    torch.cuda.empty_cache()
    qo = np.array([oracle.heisenberg_sz_row_fn(L, n, 1.0, lambda k: complex(_hash_vec_np(k)), a) for a in rows])
    # |q_a| <= (L/4 + L/2) max|r|; rounding of a 35-term sum is ~1e-15 of that
    assert np.max(np.abs(q_rows - qo)) <= 1e-13
