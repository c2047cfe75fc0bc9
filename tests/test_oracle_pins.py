"""Pins of the CPU oracle (oracle/) against what the paper and the mathematics fix.

None of these compare the oracle with itself: each checks it against a printed value of the
paper, a closed form, an independent textbook routine (Lanczos with full reorthogonalisation,
numpy/scipy dense solves), or an identity that a dropped term / wrong sign / wrong index would
break.  PAPER.md lines are cited as P:Lnnn.
"""
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def popcount(a):
    a = np.asarray(a, dtype=np.int64)
    c = np.zeros_like(a)
    for i in range(62):
        c += (a >> i) & 1
    return c


def dense_heisenberg(L, J=1.0, sector=None):
    """Dense H assembled column by column from the oracle's H.v on unit vectors."""
    M = 1 << L
    states = np.arange(M) if sector is None else np.nonzero(popcount(np.arange(M)) == sector)[0]
    H = np.zeros((states.size, states.size))
    e = np.zeros(M, dtype=np.complex128)
    for c, s in enumerate(states):
        e[s] = 1.0
        H[:, c] = oracle.heisenberg_apply(L, J, e)[states].real
        e[s] = 0.0
    return H, states


def dense_csr(op):
    M = op["row_ptr"].shape[0] - 1
    return sp.csr_matrix((op["val"], op["col"], op["row_ptr"]), shape=(M, M)).toarray()


# ----------------------------------------------------------------------------- operator pins

def test_heisenberg_table3_eigenvalues():
    """P:L785-791 (Table 3, H-Phi column), P:L761 (dim 924), P:L861 (E_0 = -5.387)."""
    want = np.loadtxt(os.path.join(GOLDEN, "table3_heisenberg_L12.txt"))
    H, states = dense_heisenberg(12, sector=6)
    assert states.size == 924
    assert np.allclose(H, H.T, atol=0)
    ev = np.linalg.eigvalsh(H)[:7]
    assert np.max(np.abs(ev - want)) < 1e-6
    assert abs(ev[0] - (-5.387)) < 5e-4


@pytest.mark.parametrize("L", [4, 12, 16])
def test_heisenberg_ferromagnet_bit_exact(L):
    """All-ones vector = ferromagnetic product state: H 1 = (J L/4) 1 exactly (multiples of 1/4)."""
    q = oracle.heisenberg_apply(L, 1.0, np.ones(1 << L, dtype=np.complex128))
    assert np.array_equal(q, np.full(1 << L, L / 4.0, dtype=np.complex128))


def test_heisenberg_product_state_eigenvector():
    """psi_s = cos(th/2)^popc(s) sin(th/2)^(L-popc(s)) is in the ferromagnetic multiplet, E = JL/4."""
    L, th = 12, 0.7
    pc = popcount(np.arange(1 << L))
    psi = (math.cos(th / 2) ** pc * math.sin(th / 2) ** (L - pc)).astype(np.complex128)
    q = oracle.heisenberg_apply(L, 1.0, psi)
    assert np.linalg.norm(q - (L / 4) * psi) / np.linalg.norm(psi) < 1e-14


@pytest.mark.parametrize("L", [8, 12])
def test_heisenberg_one_magnon_dispersion(L):
    """One up spin in a down background, plane wave e^{ikj}: E(k) = J(L/4 - 1 + cos k)."""
    for m in range(L):
        k = 2 * math.pi * m / L
        psi = np.zeros(1 << L, dtype=np.complex128)
        for j in range(L):
            psi[1 << j] = np.exp(1j * k * j)
        q = oracle.heisenberg_apply(L, 1.0, psi)
        E = L / 4 - 1 + math.cos(k)
        assert np.linalg.norm(q - E * psi) < 1e-13


def test_heisenberg_symmetric_and_sz_conserving():
    L = 8
    H, _ = dense_heisenberg(L)
    assert np.array_equal(H, H.T)
    pc = popcount(np.arange(1 << L))
    nz = np.nonzero(H)
    assert np.all(pc[nz[0]] == pc[nz[1]])


def test_heisenberg_L2_double_counted_bond():
    """L=2 periodic counts bond (0,1) twice: spectrum 2 x {-3/4, 1/4 x3}."""
    H, _ = dense_heisenberg(2)
    assert np.allclose(np.linalg.eigvalsh(H), [-1.5, 0.5, 0.5, 0.5])


@pytest.mark.parametrize("kind", ["c3", "c4"])
def test_csr_apply_matches_scipy(kind):
    p = synth.make_problem("c3", M=1 << 12) if kind == "c3" else synth.make_problem("c4", W=24, n_left=2)
    rng = np.random.default_rng(5)
    r = rng.standard_normal(p.M) + 1j * rng.standard_normal(p.M)
    A = sp.csr_matrix((p.op["val"], p.op["col"], p.op["row_ptr"]), shape=(p.M, p.M))
    want = A @ r
    got = oracle.csr_apply(p.op, r)
    assert np.max(np.abs(got - want)) <= 1e-14 * np.max(np.abs(want))
    # structure: symmetric (C3) / Hermitian (C4) as the recipe says
    D = A.toarray()
    assert np.allclose(D, D.conj().T, atol=0)


# ----------------------------------------------------------------------------- solver pins

def _dense_bound(a_norm, tol, imz):
    # |a^dag (x_n - x)| = |a^dag G(z) r^(k)| <= ||a|| ||r^(k)|| / |Im z|  (H Hermitian)
    return a_norm * (tol + 1e-12) / abs(imz)


def test_cocg_c1_matches_dense_solves():
    """C1 exactly (L=12, 16 shifts): converged x^(k) and b^dag x^(k) vs numpy dense solves."""
    p = synth.make_problem("c1")
    o = oracle.solve(p)
    assert o.status == oracle.CONVERGED
    H, _ = dense_heisenberg(12)
    lam, U = np.linalg.eigh(H)           # x = U (z - lam)^{-1} U^T b  (dense direct solve)
    Ub = U.T @ p.b
    y = o.projections()
    for k, z in enumerate(p.z):
        x = U @ (Ub / (z - lam))
        assert abs(y[k, 0] - np.vdot(p.b, x)) <= _dense_bound(1.0, p.tol, z.imag)
        assert np.linalg.norm(o.solution(k) - x) <= (p.tol + 1e-12) / abs(z.imag)
        # projected recurrence (EQ-SHIFTEDCG-y/u) == projection of the full recurrence
        assert abs(y[k, 0] - np.vdot(p.b, o.solution(k))) < 1e-12
    assert np.all(o.residuals() < p.tol)


def test_bicg_lattice_matches_dense_solves():
    """C4 recipe at W=8 (64 sites), 16 contour points, 3 complex left vectors: BiCG y vs dense."""
    p = synth.make_problem("c4", W=8, nz=16, n_left=3)
    o = oracle.solve(p)
    assert o.status == oracle.CONVERGED
    H = dense_csr(p.op)
    y = o.projections()
    for k, z in enumerate(p.z):
        x = np.linalg.solve(z * np.eye(p.M) - H, p.b)
        for l in range(3):
            want = np.vdot(p.left[l], x)
            assert abs(y[k, l] - want) <= _dense_bound(np.linalg.norm(p.left[l]), p.tol, z.imag)


def test_bicg_full_x_matches_dense():
    p = synth.make_problem("c4", W=6, nz=8, n_left=2)
    o = oracle.Oracle("bicg", p.b, p.z, left=p.left, full_x=True, tol=1e-11, itermax=500)
    assert o.run(p.op, 500) == oracle.CONVERGED
    H = dense_csr(p.op)
    for k, z in enumerate(p.z):
        x = np.linalg.solve(z * np.eye(p.M) - H, p.b)
        assert np.linalg.norm(o.solution(k) - x) <= (1e-11 + 1e-12) / abs(z.imag)


def test_cocg_csr_real_matches_dense():
    p = synth.make_problem("c3", M=512, nz=12)
    o = oracle.Oracle("cocg", p.b, p.z, full_x=True, tol=1e-10, itermax=5000)
    assert o.run(p.op, 5000) == oracle.CONVERGED
    H = dense_csr(p.op)
    for k, z in enumerate(p.z):
        x = np.linalg.solve(z * np.eye(p.M) - H, p.b)
        assert np.linalg.norm(o.solution(k) - x) <= (1e-10 + 1e-12) / abs(z.imag)


def _lanczos(Hmul, b, n):
    """Textbook Lanczos with full reorthogonalisation (independent of the oracle's recurrences):
    returns alpha[0..n), beta[0..n] (beta[j] couples v_j and v_{j+1})."""
    V = [b / np.linalg.norm(b)]
    al, be = [], []
    for j in range(n):
        w = Hmul(V[j])
        a = np.vdot(V[j], w).real
        w = w - a * V[j] - (be[-1] * V[j - 1] if j > 0 else 0)
        for v in V:  # full reorthogonalisation (twice)
            w = w - np.vdot(v, w) * v
        for v in V:
            w = w - np.vdot(v, w) * v
        bnext = np.linalg.norm(w)
        al.append(a)
        be.append(bnext)
        V.append(w / bnext)
    return np.array(al), np.array(be)


@pytest.mark.parametrize("L", [10, 17])
def test_cocg_is_lanczos_fom(L):
    """COCG with real-symmetric H, real b is Lanczos-FOM (SURVEY §0 finding 3):
    b^T x_n(z) = ||b||^2 [(z - T_n)^{-1}]_{11};  pi_n^k = chi_n(z_k)/chi_n(z_seed);
    ||r_n^(k)|| = ||b|| prod_{j<=n} beta_j / |chi_n(z_k)|, chi_n(z) = det(z - T_n).
    L = 17 (2^17 rows) spans four reduction chunks of the oracle (OR_CHUNK = 2^15)."""
    p = synth.make_problem("c2", L=L, nz=24)
    Hmul = lambda v: oracle.heisenberg_apply(L, 1.0, v)
    al, be = _lanczos(Hmul, p.b, 26)
    o = oracle.Oracle("cocg", p.b, p.z, tol=1e-300, itermax=100)
    for n in range(1, 26):
        assert o.step(p.op) == oracle.ITERATING
        T = np.diag(al[:n]) + np.diag(be[:n - 1], 1) + np.diag(be[:n - 1], -1)
        y = o.projections()[:, 0]
        chi = np.array([np.linalg.det(z * np.eye(n) - T) for z in p.z])
        zs = o.scalars()["z_seed"]
        chi_s = np.linalg.det(zs * np.eye(n) - T)
        res_cf = np.prod(be[:n]) / np.abs(chi)
        for k, z in enumerate(p.z):
            e1 = np.zeros(n); e1[0] = 1
            g = np.linalg.solve(z * np.eye(n) - T, e1)[0]
            assert abs(y[k] - g) <= 1e-10 * max(1.0, abs(g))
        assert np.max(np.abs(o.pi() - chi / chi_s) / np.abs(chi / chi_s)) < 1e-11
        assert np.max(np.abs(o.residuals() - res_cf) / res_cf) < 1e-11


def test_cocg_orthogonality_and_projection_zero():
    """App. A: r_i^T r_j = 0 (i != j); real b: b^dagger r_n = 0 for n >= 1."""
    p = synth.make_problem("c2", L=10, nz=8)
    o = oracle.Oracle("cocg", p.b, p.z, tol=1e-300, itermax=100)
    rs = [o.r()]
    # finite precision: orthogonality decays geometrically once Ritz values converge (classic
    # Lanczos behaviour, ~1e-15 -> 1e-9 over n = 10..27 here), so the pin window is n <= 18.
    for _ in range(18):
        o.step(p.op)
        rs.append(o.r())
    for i in range(len(rs)):
        for j in range(i):
            v = abs(np.dot(rs[i], rs[j])) / (np.linalg.norm(rs[i]) * np.linalg.norm(rs[j]))
            assert v < 1e-12
        if i > 0:
            assert abs(np.vdot(p.b, rs[i])) / np.linalg.norm(rs[i]) < 1e-12


@pytest.mark.parametrize("W", [10, 200])
def test_bicg_biorthogonality(W):
    """App. B: t_i^dagger r_j = 0 (i != j), t_i^dagger r_i != 0; complex b so the
    shadow sequence is not a multiple of r.  W = 200 (40000 rows) spans two reduction chunks."""
    p = synth.make_problem("c4", W=W, nz=6, n_left=1)
    rng = np.random.default_rng(11)
    b = rng.standard_normal(p.M) + 1j * rng.standard_normal(p.M)
    b /= np.linalg.norm(b)
    o = oracle.Oracle("bicg", b, p.z, tol=1e-300, itermax=100)
    rs, ts = [o.r()], [o.t()]
    for _ in range(25):
        o.step(p.op)
        rs.append(o.r()); ts.append(o.t())
    for i in range(len(rs)):
        for j in range(len(rs)):
            v = abs(np.vdot(ts[i], rs[j])) / (np.linalg.norm(ts[i]) * np.linalg.norm(rs[j]))
            if i != j:
                assert v < 1e-8
            else:
                assert v > 1e-6


def test_bicg_equals_cocg_on_real_symmetric():
    """Table 1: on real-symmetric H with t_0 = conj(b), BiCG and COCG generate the
    same iterates; y agree inside the trajectory window, converged G agree to the tol bound."""
    p = synth.make_problem("c2", L=8, nz=12)
    a = oracle.Oracle("cocg", p.b, p.z, tol=p.tol, itermax=3000)
    b = oracle.Oracle("bicg", p.b, p.z, tol=p.tol, itermax=3000)
    for _ in range(20):
        a.step(p.op); b.step(p.op)
    assert np.max(np.abs(a.projections() - b.projections())) < 1e-12
    a.run(p.op, 3000); b.run(p.op, 3000)
    assert a.status == b.status == oracle.CONVERGED
    assert b.spmv_count == 2 * b.iterations and a.spmv_count == a.iterations
    d = np.abs(a.projections() - b.projections())[:, 0]
    assert np.all(d <= 2 * _dense_bound(1.0, p.tol, 0.05))


def test_collinear_residuals_full_mode():
    """EQ-COLLINEAR: explicit b - (z_k I - H) x_n^k equals r_n / pi_n^k."""
    L = 8
    p = synth.make_problem("c1", L=L, nz=10)
    H, _ = dense_heisenberg(L)
    o = oracle.Oracle("cocg", p.b, p.z, full_x=True, tol=1e-11, itermax=400)
    for _ in range(400):
        st = o.step(p.op)
        r, pi, act = o.r(), o.pi(), o.active()
        for k in np.nonzero(act)[0]:
            ex = p.b - (p.z[k] * o.solution(k) - H @ o.solution(k))
            ne = np.linalg.norm(ex)
            # the explicit residual itself carries ~1e-15 absolute rounding: relative 1e-10
            # above 1e-4, absolute 1e-14 below
            assert np.linalg.norm(ex - r / pi[k]) <= 1e-10 * max(ne, 1e-4)
            assert abs(np.linalg.norm(r) / abs(pi[k]) - ne) <= 1e-10 * max(ne, 1e-4)
        if st != oracle.ITERATING:
            break
    assert st == oracle.CONVERGED


def test_seed_switch_continuity_and_equivalence():
    """a switch is a pure change of representation.  (a) the residual reported at
    step 10 equals ||r||/|pi_k| recomputed after the switch; (b) switch vs no-switch runs agree
    inside the trajectory window; (c) the switching run converges."""
    p = synth.make_problem("c2", L=10, nz=32)
    a = oracle.Oracle("cocg", p.b, p.z, tol=p.tol, itermax=5000)
    b = oracle.Oracle("cocg", p.b, p.z, tol=p.tol, itermax=5000, flags=oracle.FLAG_NO_SWITCH)
    c = oracle.Oracle("cocg", p.b, p.z, tol=p.tol, itermax=5000, flags=oracle.FLAG_REVERSE)
    # trajectory window: two correct fp64 runs differing only in summation order (c) stay within
    # 1e-12 for ~22 iterations at this size (SURVEY §0 finding 4); switch/no-switch must too.
    for n in range(22):
        a.step(p.op); b.step(p.op); c.step(p.op)
        res = a.residuals()
        again = np.linalg.norm(a.r()) / np.abs(a.pi())
        act = a.active()
        assert np.max(np.abs(res[act] - again[act]) / res[act]) < 1e-12
        horizon = max(np.max(np.abs(a.projections() - c.projections())), 1e-13)
        assert np.max(np.abs(a.residuals() - b.residuals()) / b.residuals()) < 1e-11
        assert np.max(np.abs(a.projections() - b.projections())) < max(1e-11, 10 * horizon)
    assert a.switches > 0 and b.switches == 0
    # Without switching the seed z_0 = -10 + 0.05i (far below the spectrum) converges first and
    # its residual keeps shrinking until rho_n underflows the 1e-300 breakdown guard while other
    # shifts are still active -- the failure mode seed switching exists for.
    assert a.run(p.op, 5000) == oracle.CONVERGED
    assert b.run(p.op, 5000) in (oracle.CONVERGED, oracle.BREAKDOWN)


def test_sum_rule_and_ed_window():
    """-(1/pi) sum_k Im G(w_k + i delta) dw -> ||b||^2 = 1 (BASELINE north_star sum rule), and the
    same grid sum equals the exact windowed Lorentzian integral from exact diagonalisation."""
    L = 12
    p = synth.make_problem("c2", L=L)             # C2 shift set: 1024 points in [-10,4), 0.05i
    o = oracle.solve(p)
    assert o.status == oracle.CONVERGED
    G = o.projections()[:, 0]
    dw = 14.0 / 1024
    s = -np.sum(G.imag) * dw / math.pi
    assert abs(s - 1.0) < 1e-2
    H, _ = dense_heisenberg(L)
    lam, U = np.linalg.eigh(H)
    wgt = np.abs(U.T @ p.b) ** 2
    # exact grid sum from ED (closed form of each sample) and the continuous window integral
    Gex = np.array([np.sum(wgt / (z - lam)) for z in p.z])
    assert np.max(np.abs(G - Gex)) <= _dense_bound(1.0, p.tol, 0.05)
    win = np.sum(wgt * (np.arctan((4.0 - lam) / 0.05) - np.arctan((-10.0 - lam) / 0.05))) / math.pi
    assert abs(s - win) < 1e-4


def test_exact_termination_closed_form():
    """b = product-state ferromagnet + two real one-magnon standing waves: 3 distinct energies,
    so COCG terminates after 3 iterations with G(z) = sum_j w_j/(z - E_j) (closed form)."""
    L = 12
    M = 1 << L
    th = 0.9
    pc = popcount(np.arange(M))
    psiF = (math.cos(th / 2) ** pc * math.sin(th / 2) ** (L - pc))
    comps, energies = [0.6 * psiF / np.linalg.norm(psiF)], [L / 4]
    for m, c in [(2, 0.5), (5, 0.62)]:
        k = 2 * math.pi * m / L
        w = np.zeros(M)
        for j in range(L):
            w[1 << j] = math.cos(k * j)
        comps.append(c * w / np.linalg.norm(w))
        energies.append(L / 4 - 1 + math.cos(k))
    b = np.sum(comps, axis=0).astype(np.complex128)
    nb2 = np.vdot(b, b).real
    z = synth.spectrum_shifts(40, -4.0, 5.0, 0.05)
    o = oracle.Oracle("cocg", b, z, tol=1e-10, itermax=50)
    st = o.run({"kind": "heisenberg", "L": L, "J": 1.0}, 50)
    assert st == oracle.CONVERGED and o.iterations == 3
    wj = np.array([np.vdot(c, c).real for c in comps])
    assert abs(wj.sum() - nb2) < 1e-14
    Gex = np.array([np.sum(wj / (zz - np.array(energies))) for zz in z])
    # rigorous: |G_n - G| <= ||r^(k)|| / |Im z|  (res after 3 iterations ~3e-12: rounding of psi_F)
    bound = o.residuals() / 0.05 + 1e-13
    assert np.all(np.abs(o.projections()[:, 0] - Gex) <= bound)
    assert np.max(o.residuals()) < 1e-11


def test_conjugate_symmetry():
    """Hermitian H: G_bb(conj z) = conj G_bb(z)."""
    p = synth.make_problem("c1", L=10, nz=16)
    a = oracle.Oracle("cocg", p.b, p.z, tol=1e-11, itermax=4000)
    b = oracle.Oracle("cocg", p.b, np.conj(p.z), tol=1e-11, itermax=4000)
    a.run(p.op, 4000); b.run(p.op, 4000)
    d = np.abs(a.projections() - np.conj(b.projections()))
    assert np.all(d <= 2 * _dense_bound(1, 1e-11, 0.1))


def test_spmv_count_independent_of_nz():
    """Table 2: SpMV per iteration is 1 (COCG) / 2 (BiCG) independent of N_eq."""
    for nz in (1, 10, 100):
        p = synth.make_problem("c2", L=8, nz=nz)
        o = oracle.Oracle("cocg", p.b, p.z, tol=1e-10, itermax=37)
        o.run(p.op, 37)
        assert o.spmv_count == o.iterations == 37 or o.status == oracle.CONVERGED
        q = synth.make_problem("c4", W=6, nz=nz, n_left=1)
        o = oracle.Oracle("bicg", q.b, q.z, left=q.left, tol=1e-10, itermax=15)
        o.run(q.op, 15)
        assert o.spmv_count == 2 * o.iterations


# ----------------------------------------------------------------------------- edge cases

def test_edge_breakdown_rho_zero():
    """COCG with b^T b = 0 (b = (e_0 + i e_1)/sqrt 2): rho_0 = 0 -> BREAKDOWN (R12)."""
    b = np.zeros(16, dtype=np.complex128)
    b[0], b[1] = 1 / math.sqrt(2), 1j / math.sqrt(2)
    o = oracle.Oracle("cocg", b, np.array([0.3 + 0.1j]), tol=1e-10, itermax=10)
    assert o.step({"kind": "heisenberg", "L": 4, "J": 1.0}) == oracle.BREAKDOWN


def test_edge_eigenvector_rhs_terminates_in_one():
    """b = all-ones/||.|| (an eigenvector, E = L/4): r_1 = 0, every shift retires at n = 1 and the
    solution is b/(z - E) exactly (no 0/0: retirement precedes the next division)."""
    L = 6
    b = np.ones(1 << L, dtype=np.complex128) / math.sqrt(1 << L)
    z = synth.spectrum_shifts(5, -3, 2, 0.1)
    o = oracle.Oracle("cocg", b, z, full_x=True, tol=1e-12, itermax=10)
    assert o.run({"kind": "heisenberg", "L": L, "J": 1.0}, 10) == oracle.CONVERGED
    assert o.iterations == 1
    for k in range(5):
        assert np.allclose(o.solution(k), b / (z[k] - L / 4), rtol=1e-14, atol=0)


def test_edge_maxiter_and_single_shift():
    p = synth.make_problem("c2", L=8, nz=1)
    o = oracle.Oracle("cocg", p.b, p.z, tol=1e-10, itermax=3)
    assert o.run(p.op, 100) == oracle.MAXITER and o.iterations == 3
    assert o.switches == 0
    # after init, the residual of every shift is ||b|| (pi_0 = 1)
    o2 = oracle.Oracle("cocg", p.b, synth.spectrum_shifts(4, -1, 1, 0.1), tol=1e-10, itermax=3)
    assert np.allclose(o2.residuals(), 1.0, rtol=1e-15)


def test_edge_invalid_arguments():
    b = np.ones(4, dtype=np.complex128)
    with pytest.raises(ValueError):
        oracle.Oracle("cocg", b, np.array([0.1j]), tol=0.0)
    with pytest.raises(ValueError):
        oracle.Oracle("cocg", b, np.array([0.1j]), itermax=0)


def test_recalc_identity_and_new_shifts_vs_dense():
    """Recalculation from the coefficient log: replaying the logged recurrences at
    the original shifts reproduces the run's projections; at new shifts between
    them it matches a dense solve within the replayed residual's bound."""
    L = 10
    p = synth.make_problem("c2", L=L, nz=32)
    o = oracle.solve(p)
    assert o.status == oracle.CONVERGED and o.log_length == o.iterations
    y, res = o.recalc(p.z)
    assert np.max(np.abs(y - o.projections())) <= 1e-12 * np.max(np.abs(o.projections()))
    assert np.all(res < p.tol)
    H, _ = dense_heisenberg(L)
    lam, U = np.linalg.eigh(H)
    Ub = U.T @ p.b
    z_new = synth.spectrum_shifts(31, -10.0 + 14.0 / 64, 4.0 + 14.0 / 64, 0.05)   # midpoints
    y2, res2 = o.recalc(z_new)
    for k, z in enumerate(z_new):
        exact = np.vdot(p.b, U @ (Ub / (z - lam)))
        assert abs(y2[k, 0] - exact) <= (res2[k] + 1e-12) / 0.05
    assert o.spmv_count == o.iterations     # recalc used no operator application


# ------------------------------------------------------------------------------- Sz sector (f-3)

def test_sz_sector_dimension():
    """the L=12, Sz=0 sector has 924 states; the oracle's basis is the ascending list."""
    assert oracle.sz_dim(12, 6) == 924
    st = oracle.sz_states(12, 6)
    assert st.size == 924 and np.all(np.diff(st) > 0)
    assert np.all(popcount(st) == 6)
    assert oracle.sz_dim(30, 15) == math.comb(30, 15)


@pytest.mark.parametrize("L,n", [(10, 0), (10, 3), (10, 5), (11, 7), (12, 12)])
def test_sz_rank_unrank_match_enumeration(L, n):
    """The counting rank / unrank (used for sampled rows at large L) against brute-force order."""
    st = oracle.sz_states(L, n)
    for i, s in enumerate(st):
        assert oracle.sz_rank(L, s) == i
        assert oracle.sz_unrank(L, n, i) == s


@pytest.mark.parametrize("L,n", [(10, 5), (10, 3), (11, 6), (9, 1)])
def test_sz_apply_is_the_restriction_of_the_full_operator(L, n):
    """H conserves S^z: the full-space product of a vector supported on the sector stays in the
    sector and equals the sector product there (same per-row arithmetic: bit-exact)."""
    rng = np.random.default_rng(L * 100 + n)
    st = oracle.sz_states(L, n)
    r = rng.standard_normal(st.size) + 1j * rng.standard_normal(st.size)
    full = np.zeros(1 << L, dtype=np.complex128)
    full[st] = r
    qf = oracle.heisenberg_apply(L, 1.0, full)
    qs = oracle.heisenberg_sz_apply(L, n, 1.0, r)
    assert np.array_equal(qf[st], qs)
    mask = np.ones(1 << L, dtype=bool)
    mask[st] = False
    assert np.all(qf[mask] == 0)


def test_sz_sector_table3_from_the_sector_alone():
    """Table 3 from the 924 x 924 sector operator built column by column."""
    want = np.loadtxt(os.path.join(GOLDEN, "table3_heisenberg_L12.txt"))
    D = oracle.sz_dim(12, 6)
    H = np.empty((D, D))
    e = np.zeros(D, dtype=np.complex128)
    for j in range(D):
        e[:] = 0
        e[j] = 1
        H[:, j] = oracle.heisenberg_sz_apply(12, 6, 1.0, e).real
    assert np.array_equal(H, H.T)
    ev = np.linalg.eigvalsh(H)[:7]
    assert np.max(np.abs(ev - want)) < 1e-6


def test_sz_sampled_rows_match_the_full_product():
    """or_heisenberg_sz_row (counting rank, no list) = the list-based product, row by row."""
    L, n = 12, 5
    rng = np.random.default_rng(5)
    D = oracle.sz_dim(L, n)
    r = rng.standard_normal(D) + 1j * rng.standard_normal(D)
    q = oracle.heisenberg_sz_apply(L, n, 1.0, r)
    op = {"kind": "heisenberg_sz", "L": L, "n_up": n, "J": 1.0}
    rows = [0, 1, 17, D // 2, D - 1]
    assert np.array_equal(oracle.apply_rows(op, r, rows), q[rows])


def test_sz_row_fn_matches_the_full_product():
    """heisenberg_sz_row_fn (r as a function of the row) = the list-based product, row by row
    (it serves the L = 34 GPU check, whose vector does not fit on the host)."""
    L, n = 13, 6
    rng = np.random.default_rng(13)
    D = oracle.sz_dim(L, n)
    r = rng.standard_normal(D) + 1j * rng.standard_normal(D)
    q = oracle.heisenberg_sz_apply(L, n, 0.7, r)
    rows = [0, 1, 2, 100, D // 2, D - 2, D - 1]
    got = np.array([oracle.heisenberg_sz_row_fn(L, n, 0.7, lambda k: r[k], a) for a in rows])
    assert np.max(np.abs(got - q[rows])) <= 1e-14 * np.max(np.abs(q))


def test_sz_sector_solver_matches_dense_solve():
    """Shifted COCG on the sector operator (the same oracle solver) converges to the dense
    sector solve: y_k = b^dagger (z_k - H_sector)^-1 b."""
    p = synth.make_problem("c5sz", L=10, nz=8)
    D = p.M
    H = np.empty((D, D))
    e = np.zeros(D, dtype=np.complex128)
    for j in range(D):
        e[:] = 0
        e[j] = 1
        H[:, j] = oracle.heisenberg_sz_apply(10, 5, 1.0, e).real
    o = oracle.solve(p)
    assert o.status == oracle.CONVERGED
    y = o.projections()[:, 0]
    for k, zk in enumerate(p.z):
        x = np.linalg.solve(zk * np.eye(D) - H, p.b)
        yd = np.vdot(p.b, x)
        assert abs(y[k] - yd) <= (p.tol + 1e-12) / abs(zk.imag)


# ------------------------------------------------------------------------------- contour integral (f-2)

@pytest.mark.parametrize("col,n_l", [(1, 1), (2, 2), (3, 5)])
def test_ss_table3_columns(col, n_l):
    """Table 3: SS(10, N_l) on the L=12 Sz=0 chain, gamma=-5, rho=0.8, N_z=100,
    singular values < 1e-3 discarded — the printed digits, including the collapsed degenerate
    pairs of SS(10,1) (one source vector sees one vector per eigenspace)."""
    import oracle.ss as ss
    tab = np.loadtxt(os.path.join(GOLDEN, "table3_ss.txt"))
    want = tab[:, col][~np.isnan(tab[:, col])]
    op, phis, z = synth.ss_inputs()
    ev, sig = ss.ss_eigenvalues(op, phis[:n_l], -5.0, 0.8, 100, 10)
    assert ev.size == want.size
    assert np.max(np.abs(ev - want)) < 1e-6


def test_ss_table3_with_complex_sources():
    """The eigenvalues do not depend on the source vectors: complex phi (real and imaginary parts
    from two of the seeded real draws) give the SS(10,5) column of Table 3 again — with complex
    S the Rayleigh-Ritz matrix needs U~^dagger, not U~^T."""
    import oracle.ss as ss
    tab = np.loadtxt(os.path.join(GOLDEN, "table3_ss.txt"))
    op, phis, z = synth.ss_inputs(n_l=10)
    cphis = phis[:5] + 1j * phis[5:]
    ev, sig = ss.ss_eigenvalues(op, cphis, -5.0, 0.8, 100, 10)
    assert ev.size == 7 and np.max(np.abs(ev - tab[:, 3])) < 1e-6


def test_ss_moments_are_the_quadrature_filter_of_the_spectrum():
    """s_{k,0} = (1/2 pi i) oint (z - gamma)^k (z - H)^{-1} phi dz by the trapezoidal
    rule on z_j is exactly Y f_k(Lambda) Y^dagger phi with the rational filter
    f_k(lam) = sum_j (z_j - gamma)/N_z (z_j - gamma)^k / (z_j - lam) — checked against the
    eigen-decomposition of the sector matrix; f_0 is ~1 inside the circle and ~0 outside
    (the spectral projector P_Gamma)."""
    import oracle.ss as ss
    op, phis, z = synth.ss_inputs(L=10, n_up=5, n_l=1, n_z=64, gamma=-4.0, rho=0.6)
    D = phis.shape[1]
    H = np.empty((D, D))
    e = np.zeros(D, dtype=np.complex128)
    for j in range(D):
        e[:] = 0
        e[j] = 1
        H[:, j] = oracle.heisenberg_sz_apply(10, 5, 1.0, e).real
    lam, Y = np.linalg.eigh(H)
    X = ss.contour_solutions(op, phis, z)
    S = ss.moments(X, z, -4.0, 3)
    c = Y.conj().T @ phis[0]
    for k in range(3):
        f = np.array([np.sum((z + 4.0) / z.size * (z + 4.0) ** k / (z - l)) for l in lam])
        want = Y @ (f * c)
        assert np.linalg.norm(S[:, k] - want) < 1e-8 * np.linalg.norm(phis[0])
    f0 = np.array([np.sum((z + 4.0) / z.size / (z - l)) for l in lam])
    inside = np.abs(lam + 4.0) < 0.6
    assert inside.sum() >= 2
    far = np.abs(np.abs(lam + 4.0) - 0.6) > 0.1
    assert np.all(np.abs(f0[inside & far] - 1) < 1e-3) and np.all(np.abs(f0[~inside & far]) < 1e-3)


# ----------------------------------------------------------------------------- row routines

@pytest.mark.parametrize("L", [12, 13])
def test_heisenberg_row_routine_matches_the_full_product(L):
    """or_heisenberg_row (the checker behind every sampled-row GPU test at L = 30) against the
    full product or_heisenberg_apply, which is pinned above by Table 3, the
    ferromagnet and the magnon dispersion: every row, a complex random vector (a wrong flip
    partner or bond would move most rows)."""
    rng = np.random.default_rng(100 + L)
    M = 1 << L
    r = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    op = {"kind": "heisenberg", "L": L, "J": 1.0}
    full = oracle.apply_op(op, r)
    rows = np.arange(M)
    assert np.array_equal(oracle.apply_rows(op, r, rows), full)
    # and directly against the bond sum of P:L831 written out for a handful of rows
    for s in (0, 1, M - 1, M // 3, 0b1011 % M):
        acc = 0j
        for i in range(L):
            j = (i + 1) % L
            if ((s >> i) & 1) == ((s >> j) & 1):
                acc += 0.25 * r[s]
            else:
                acc += -0.25 * r[s] + 0.5 * r[s ^ ((1 << i) | (1 << j))]
        assert abs(oracle.apply_rows(op, r, [s])[0] - acc) <= 1e-14 * abs(acc)


@pytest.mark.parametrize("kind,kw", [("c3", dict(M=1 << 12)), ("c4", dict(W=24, nz=4, n_left=1))])
def test_csr_row_routines_match_scipy(kind, kw):
    """or_csr_real_row / or_csr_cplx_row (the checkers of the sampled C3/C4 rows) against the
    scipy.sparse product on the same CSR arrays (an independent library routine), every row."""
    p = synth.make_problem(kind, **kw)
    rng = np.random.default_rng(7)
    r = rng.standard_normal(p.M) + 1j * rng.standard_normal(p.M)
    want = sp.csr_matrix((p.op["val"], p.op["col"], p.op["row_ptr"]), shape=(p.M, p.M)) @ r
    got = oracle.apply_rows(p.op, r, np.arange(p.M))
    assert np.max(np.abs(got - want)) <= 1e-14 * np.max(np.abs(want))


# ----------------------------------------------------------------------------- OpenMP build

@pytest.mark.parametrize("name,kw", [("c1", dict(L=16, nz=6)), ("c4", dict(W=190, nz=4, n_left=3))])
def test_openmp_build_is_bit_identical(name, kw):
    """liboracle_omp.so (the reference arm's all-core oracle) performs the same floating-point
    operations in the same order as liboracle.so: residuals, projections, r and x agree bit for
    bit after 30 iterations (sizes spanning several reduction chunks; seed switches included)."""
    p = synth.make_problem(name, **kw)
    a = oracle.Oracle(p.method, p.b, p.z, left=p.left, full_x=p.full_x, tol=p.tol, itermax=500, omp=False)
    b = oracle.Oracle(p.method, p.b, p.z, left=p.left, full_x=p.full_x, tol=p.tol, itermax=500, omp=True)
    for _ in range(30):
        assert a.step(p.op) == b.step(p.op)
    assert a.switches == b.switches > 0
    assert np.array_equal(a.residuals(), b.residuals())
    assert np.array_equal(a.projections(), b.projections())
    assert np.array_equal(a.r(), b.r())
    if p.full_x:
        assert np.array_equal(a.solution(2), b.solution(2))


# ----------------------------------------------------------------------------- horizon tool

def test_self_divergence_horizon_tool():
    """tests/horizon.py: two correct orderings of the oracle agree to 1e-11 for
    a few dozen iterations (31 for C1's geometry), then drift apart — the tool finds a finite
    horizon there, and reports the whole run for an input that terminates exactly (3 energies)."""
    from horizon import horizon
    p = synth.make_problem("c1")
    h = horizon(p, 200)
    assert 25 <= h < 200, h
    # agreement really fails right after the horizon: the two runs differ by more than 1e-12
    a = oracle.Oracle(p.method, p.b, p.z, tol=p.tol, itermax=p.itermax)
    b = oracle.Oracle(p.method, p.b, p.z, tol=p.tol, itermax=p.itermax, flags=oracle.FLAG_REVERSE)
    for _ in range(h + 1):
        a.step(p.op); b.step(p.op)
    d = max(np.max(np.abs(a.residuals() - b.residuals()) / a.residuals()),
            np.max(np.abs(a.projections() - b.projections()) / np.abs(a.projections())))
    assert d > 1e-11 or not np.array_equal(a.retired_at(), b.retired_at())
