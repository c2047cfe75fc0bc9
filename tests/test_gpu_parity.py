"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded inputs.

Protocol:
  * trajectory window: per iteration n <= n_w and per shift, |dres|/res <= 1e-9 and the
    normwise projection error max_l|dy_kl| / max_l|y_kl| <= 1e-9 (R23); the seed index and
    the retirement iterations agree.  n_w = min(cap, horizon): the self-divergence horizon of
    two correct fp64 orderings of the oracle (tests/horizon.py), measured on
    the test's own input; the cap bounds the oracle's cost.
  * converged: per-shift projection error <= 1e-9; every residual below tol on both sides.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from horizon import horizon

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2001_08707_b200 import shiftk  # noqa: E402
from paper_2001_08707_b200.device import make_solver, to_device  # noqa: E402

REL = 1e-9


def proj_err(a, b):
    """normwise per-shift relative error of projections y[k, l] (R23)."""
    num = np.max(np.abs(a - b), axis=1)
    den = np.maximum(np.max(np.abs(b), axis=1), 1e-300)
    return num / den


def run_window(problem, n_cap, *, full_check=False, flags=0, tol=None):
    n_w = horizon(problem, n_cap, flags=flags, tol=tol)
    assert n_w >= min(n_cap, 3), ("self-divergence horizon too short", n_w)
    dp = to_device(problem)
    g = make_solver(dp, flags=flags, tol=tol)
    o = oracle.Oracle(problem.method, problem.b, problem.z, left=problem.left,
                      full_x=problem.full_x, tol=problem.tol if tol is None else tol,
                      itermax=problem.itermax, flags=flags)
    worst_res = worst_y = 0.0
    for n in range(n_w):
        sg = g.update()
        so = o.step(problem.op)
        assert sg == so, (n, sg, so)
        rg, ro = g.residuals(), o.residuals()
        worst_res = max(worst_res, float(np.max(np.abs(rg - ro) / ro)))
        assert np.all(np.abs(rg - ro) <= REL * ro), (n, np.max(np.abs(rg - ro) / ro))
        e = proj_err(g.projections(), o.projections())
        worst_y = max(worst_y, float(np.max(e)))
        assert np.all(e <= REL), (n, np.max(e))
        c = g.coefficients()
        if c["seed_index"] != o.seed_index:
            # several results are correct: a (near-)tie of |pi| (e.g. conjugate contour points
            # z, conj(z) with real b and Hermitian H have equal |pi| in exact arithmetic); the
            # GPU's choice must then also be a minimiser of |pi| in the oracle's state.
            pio = np.abs(o.pi())
            assert o.active()[c["seed_index"]], n
            assert abs(pio[c["seed_index"]] / pio[o.seed_index] - 1) < 1e-9, n
        assert c["iterations"] == o.iterations == n + 1
        _, act, ret = g.shift_state()
        assert np.array_equal(act, o.active()), n
        assert np.array_equal(ret, o.retired_at()), n
        if full_check:
            for k in range(problem.n_shift):
                xg = g.solution(k)
                xo = o.solution(k)
                assert np.linalg.norm(xg - xo) <= REL * np.linalg.norm(xo), (n, k)
        if sg != shiftk.ITERATING:
            break
    return g, o, worst_res, worst_y


# ------------------------------------------------------------------------------- operators

@pytest.mark.parametrize("L", [4, 12, 17, 23, 24, 25])
def test_heisenberg_operator_parity(L):
    rng = np.random.default_rng(L)
    r = rng.standard_normal(1 << L) + 1j * rng.standard_normal(1 << L)
    op = shiftk.make_operator({"kind": "heisenberg", "L": L, "J": 1.0}, 1 << L)
    rd = torch.from_numpy(r).cuda()
    qd = torch.empty_like(rd)
    shiftk.apply_operator(op, rd, qd)
    torch.cuda.synchronize()
    qo = oracle.heisenberg_apply(L, 1.0, r)
    assert np.max(np.abs(qd.cpu().numpy() - qo)) <= 1e-14 * np.max(np.abs(qo))


@pytest.mark.parametrize("L,n", [(12, 6), (16, 8), (14, 3), (11, 0), (20, 10),
                                 # block-kernel edges: one high bit (L <= 13), tiny chains,
                                 # empty/full classes, a far-from-half sector, 22 sites
                                 (2, 1), (3, 1), (3, 2), (5, 2), (13, 6), (13, 13), (13, 0),
                                 (14, 7), (21, 4), (22, 11)])
def test_heisenberg_sz_operator_parity(L, n):
    """Sector operator (f-3): GPU combinatorial ranking vs the oracle's enumerated basis."""
    rng = np.random.default_rng(L * 7 + n)
    D = oracle.sz_dim(L, n)
    r = rng.standard_normal(D) + 1j * rng.standard_normal(D)
    op = shiftk.make_operator({"kind": "heisenberg_sz", "L": L, "J": 1.0, "n_up": n}, D)
    rd = torch.from_numpy(r).cuda()
    qd = torch.empty_like(rd)
    shiftk.apply_operator(op, rd, qd)
    torch.cuda.synchronize()
    qo = oracle.heisenberg_sz_apply(L, n, 1.0, r)
    assert np.max(np.abs(qd.cpu().numpy() - qo)) <= 1e-14 * np.max(np.abs(qo))


def test_heisenberg_sz_window():
    """Trajectory window on the Sz = 0 sector of a 16-site chain (C(16,8) = 12870 rows)."""
    run_window(synth.make_problem("c5sz", L=16, nz=64), 20)


def test_rank_stepping_sector_kernel_still_matches():
    """The earlier rank-stepping sector kernel (SHIFTK_SZ_RANK=1, read once per process, so in a
    subprocess): operator parity and a short solver window (per-CTA w partials)."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, synth, oracle\n"
        "from paper_2001_08707_b200 import shiftk\n"
        "from test_gpu_parity import run_window\n"
        "for L, n in [(16, 8), (14, 3), (13, 13)]:\n"
        "    D = oracle.sz_dim(L, n)\n"
        "    r = np.random.default_rng(L).standard_normal(D) + 0.5j\n"
        "    op = shiftk.make_operator({'kind': 'heisenberg_sz', 'L': L, 'J': 1.0, 'n_up': n}, D)\n"
        "    rd = torch.from_numpy(r).cuda(); qd = torch.empty_like(rd)\n"
        "    shiftk.apply_operator(op, rd, qd); torch.cuda.synchronize()\n"
        "    qo = oracle.heisenberg_sz_apply(L, n, 1.0, r)\n"
        "    assert np.max(np.abs(qd.cpu().numpy() - qo)) <= 1e-14 * np.max(np.abs(qo)), (L, n)\n"
        "run_window(synth.make_problem('c5sz', L=16, nz=16), 10)\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SHIFTK_SZ_RANK="1", PYTHONPATH=root + os.pathsep + os.path.join(root, "tests"))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-3000:]


def test_heisenberg_sz_window_grouped_partials():
    """26 sites, Sz = 0 (C(26,13) = 10,400,600 rows, 2^14 high-bit blocks): the block kernel's
    queue-dealt blocks and its per-block + per-group w partials (more than kStreamDirect blocks)."""
    run_window(synth.make_problem("c5sz", L=26, nz=8), 4)


def test_heisenberg_sz_queue_order_is_bitwise_irrelevant():
    """The sector SpMV deals blocks from a queue (the order differs launch to launch), but w is
    summed per block and per group in index order: sk_run == stepwise, bit for bit."""
    p = synth.make_problem("c5sz", L=26, nz=8)
    dp = to_device(p)
    a = make_solver(dp)
    b = make_solver(dp)
    for _ in range(12):
        a.update()
    b.run(12, poll_every=5)
    assert np.array_equal(a.residuals(), b.residuals())
    assert np.array_equal(a.projections(), b.projections())
    assert a.coefficients() == b.coefficients()


def test_heisenberg_ferromagnet_bit_exact_gpu():
    L = 20
    op = shiftk.make_operator({"kind": "heisenberg", "L": L, "J": 1.0}, 1 << L)
    rd = torch.ones(1 << L, dtype=torch.complex128, device="cuda")
    qd = torch.empty_like(rd)
    shiftk.apply_operator(op, rd, qd)
    assert torch.equal(qd, torch.full_like(rd, L / 4))


@pytest.mark.parametrize("kind", ["c3", "c4"])
def test_csr_operator_parity(kind):
    p = synth.make_problem("c3", M=1 << 13) if kind == "c3" else synth.make_problem("c4", W=40, n_left=1)
    dp = to_device(p)
    rng = np.random.default_rng(3)
    r = rng.standard_normal(p.M) + 1j * rng.standard_normal(p.M)
    rd = torch.from_numpy(r).cuda()
    qd = torch.empty_like(rd)
    shiftk.apply_operator(dp.op, rd, qd)
    torch.cuda.synchronize()
    qo = oracle.csr_apply(p.op, r)
    assert np.max(np.abs(qd.cpu().numpy() - qo)) <= 1e-14 * np.max(np.abs(qo))


# ------------------------------------------------------------------------------- trajectories

def test_c1_trajectory_full_x():
    p = synth.make_problem("c1")
    run_window(p, 30, full_check=True)


def test_c1_converged():
    p = synth.make_problem("c1")
    dp = to_device(p)
    g = make_solver(dp)
    st = g.run(p.itermax)
    assert st == shiftk.CONVERGED
    o = oracle.solve(p)
    assert o.status == oracle.CONVERGED
    assert np.all(proj_err(g.projections(), o.projections()) <= REL)
    assert np.all(g.residuals() < p.tol) and np.all(o.residuals() < p.tol)
    # x^(k) at convergence: both within tol/|Im z| of the exact solution
    for k in range(p.n_shift):
        xg = g.solution(k)
        xo = o.solution(k)
        assert np.linalg.norm(xg - xo) <= 2 * (p.tol + 1e-12) / 0.1


def test_c2_scaled_trajectory_and_converged():
    p = synth.make_problem("c2", L=14)
    run_window(p, 25)
    dp = to_device(p)
    g = make_solver(dp)
    assert g.run(p.itermax) == shiftk.CONVERGED
    o = oracle.solve(p)
    assert o.status == oracle.CONVERGED
    assert np.all(proj_err(g.projections(), o.projections()) <= REL)
    assert np.all(g.residuals() < p.tol)


def test_c2_full_size_window():
    """C2 at its full size (L=20, 1024 shifts), the bench workload, first 15 iterations."""
    p = synth.make_problem("c2")
    run_window(p, 15)


def test_c3_scaled_trajectory_full_x():
    p = synth.make_problem("c3", M=1 << 12, nz=32)
    run_window(p, 20, full_check=True)


def test_c4_scaled_bicg_trajectory_and_converged():
    p = synth.make_problem("c4", W=24, n_left=32)
    run_window(p, 20)
    dp = to_device(p)
    g = make_solver(dp)
    assert g.run(p.itermax) == shiftk.CONVERGED
    o = oracle.solve(p)
    assert o.status == oracle.CONVERGED
    assert np.all(proj_err(g.projections(), o.projections()) <= REL)


def test_c5_scaled_trajectory():
    p = synth.make_problem("c5", L=16)
    run_window(p, 20)


@pytest.mark.parametrize("name,kw", [("c2", dict(L=14, nz=32)), ("c2", dict(L=11, nz=16)),
                                     ("c5sz", dict(L=14, nz=32)), ("c2", dict(L=23, nz=8))])
def test_bicg_on_the_real_chain(name, kw):
    """BiCG on a real-symmetric operator (allowed; equals COCG in exact arithmetic, Table 1):
    exercises the two-right-hand-side paths of the tiled (L=14), simple (L=11), sector and
    (L=23, NRHS=2 falls back to the tiled kernel) Heisenberg SpMV kernels."""
    import dataclasses
    p = dataclasses.replace(synth.make_problem(name, **kw), method="bicg")
    run_window(p, 4 if kw.get("L", 0) >= 20 else 15)


# ------------------------------------------------------------------------------- semantics

def test_run_equals_stepwise_bitwise():
    """sk_run (graph-captured) and repeated sk_update enqueue the same kernels in the same
    order: results are bit-identical (deterministic reductions)."""
    p = synth.make_problem("c2", L=12, nz=64)
    dp = to_device(p)
    a = make_solver(dp)
    b = make_solver(dp)
    for _ in range(50):
        a.update()
    b.run(50, poll_every=7)
    assert np.array_equal(a.residuals(), b.residuals())
    assert np.array_equal(a.projections(), b.projections())
    assert a.coefficients() == b.coefficients()


def test_grouped_partials_window_and_determinism():
    """L=23: 8192 tiles, so the streaming SpMV reduces w through per-group partials summed by
    whichever CTA completes a group; the dynamic tile queue must still give bit-identical runs
    and oracle parity."""
    p = synth.make_problem("c2", L=23, nz=16)
    g, o, _, _ = run_window(p, 4)
    h = make_solver(to_device(p))
    for _ in range(4):
        h.update()
    assert np.array_equal(g.residuals(), h.residuals())
    assert g.coefficients() == h.coefficients()


def _subprocess(code: str, env_extra: dict, timeout: int = 900):
    """Run `code` in a fresh interpreter (the SHIFTK_* switches are read once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root + os.pathsep + os.path.join(root, "tests"), **env_extra)
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), (out.stdout[-2000:], out.stderr[-3000:])


def test_bond_split_default_at_l24_window_and_determinism():
    """L=24 with one left vector (a = b): the bond split is on by default — the
    streaming SpMV applies the diagonal and bonds i < 16, the update the bonds 16..22 and the
    periodic bond from its B-tiles.  Oracle window, bit-identical reruns."""
    p = synth.make_problem("c2", L=24, nz=8)
    g, o, _, _ = run_window(p, 4)
    assert g.info()["split_ahi"] == 24 - 8
    h = make_solver(to_device(p))
    for _ in range(4):
        h.update()
    assert np.array_equal(g.residuals(), h.residuals())
    assert g.coefficients() == h.coefficients()


SPLIT_FORCED = """
import numpy as np, oracle, synth
from paper_2001_08707_b200 import shiftk
from paper_2001_08707_b200.device import make_solver, to_device
from test_gpu_parity import run_window, proj_err, REL
for L in (20, 21, 22):
    p = synth.make_problem("c2", L=L, nz=64)
    g, o, wr, wy = run_window(p, 40)
    assert g.info()["split_ahi"] == L - 8, g.info()
    # graph-captured sk_run == stepwise, bit for bit (fixed-order w_A + w_B partials)
    n = g.iterations
    h = make_solver(to_device(p))
    h.run(n, poll_every=n)
    assert np.array_equal(g.residuals(), h.residuals()) and np.array_equal(g.projections(), h.projections())
    assert g.coefficients() == h.coefficients()
# restart in split mode (the w_B partials of r_n travel in the checkpoint) against the oracle
p = synth.make_problem("c2", L=20, nz=64)
dp = to_device(p)
a = make_solver(dp)
a.run(10)
blob = a.checkpoint()
a.finalize()
g = make_solver(dp)
g.restore(blob)
o = oracle.Oracle(p.method, p.b, p.z, left=p.left, tol=p.tol, itermax=p.itermax)
for _ in range(10):
    o.step(p.op)
for n in range(10, 25):
    assert g.update() == o.step(p.op)
    rg, ro = g.residuals(), o.residuals()
    assert np.all(np.abs(rg - ro) <= REL * ro), (n, np.max(np.abs(rg - ro) / ro))
    assert np.all(proj_err(g.projections(), o.projections()) <= REL), n
# converged run (C2's geometry scaled to L = 20 would take ~3000 iterations: L = 20, 16 shifts
# far from the real axis converge fast) against the oracle
import dataclasses
q = dataclasses.replace(synth.make_problem("c2", L=20, nz=16), z=synth.make_problem("c2", L=20, nz=16).z + 0.5j)
g = make_solver(to_device(q))
assert g.run(q.itermax) == shiftk.CONVERGED
o = oracle.Oracle(q.method, q.b, q.z, left=q.left, tol=q.tol, itermax=q.itermax)
assert o.run(q.op, q.itermax) == oracle.CONVERGED
assert np.all(proj_err(g.projections(), o.projections()) <= REL)
assert np.all(g.residuals() < q.tol) and np.all(o.residuals() < q.tol)
print("ok")
"""


@pytest.mark.parametrize("a_kernel", ["stream", "tiled", "tiled-lo"])
def test_bond_split_forced_at_small_l(a_kernel):
    """The bond split forced at L = 20, 21, 22 (SHIFTK_HEIS_SPLIT=1; H_A by the streaming SpMV
    (SHIFTK_HEIS_STREAM=1, per-tile w partials) or the tiled one (per-CTA partials); AHI =
    12..14, so the B-tiles cover 7 chain bonds + the periodic one and 2^8..2^10 B-tiles over 148
    CTAs): 40-iteration oracle windows on 64 shifts, graph == stepwise bitwise, restart from a
    checkpoint against the oracle, and a converged run."""
    env = {"SHIFTK_HEIS_SPLIT": "1", "SHIFTK_HEIS_STREAM": "1" if a_kernel == "stream" else "0"}
    if a_kernel == "tiled-lo":   # the piece bonds (0,1)..(2,3) in the update's H_B as well
        env["SHIFTK_SPLIT_LO"] = "1"
    _subprocess(SPLIT_FORCED, env)


SPLIT_MODES = """
import dataclasses, os
import numpy as np, oracle, synth
from paper_2001_08707_b200.device import make_solver, to_device
from test_gpu_parity import run_window
want_fuse, want_real = int(os.environ["WANT_FUSE"]), int(os.environ["WANT_REAL"])
p = synth.make_problem("c2", L=20, nz=64)
if os.environ.get("COMPLEX_LEFT"):   # one explicit complex left vector (a != b): Im a != 0
    rng = np.random.Generator(np.random.PCG64(11))
    a = rng.standard_normal(p.M) + 1j * rng.standard_normal(p.M)
    p = dataclasses.replace(p, left=(a / np.linalg.norm(a)).reshape(1, -1))
g, o, wr, wy = run_window(p, 30)
i = g.info()
assert i["split_ahi"] == 12 and i["split_fuse"] == want_fuse and i["left_real"] == want_real, i
h = make_solver(to_device(p))   # graph-captured == stepwise, bit for bit
h.run(g.iterations, poll_every=g.iterations)
assert np.array_equal(g.residuals(), h.residuals()) and np.array_equal(g.projections(), h.projections())
print("ok")
"""


@pytest.mark.parametrize("mode", ["plain", "fuse-only", "real-only", "complex-left"])
def test_bond_split_fuse_and_real_left_switches(mode):
    """The bond split's fused r_{n-1} term (u = H_A r_n - kappa r_{n-1} written by the SpMV) and
    its real left vector in B-tile order switched off one at a time
    (SHIFTK_SPLIT_FUSE=0 / SHIFTK_LEFT_REAL=0), and a complex left vector (the flag raised at
    init sends the update back to the complex stream): each a 30-iteration oracle window at
    L = 20 with the split forced; the default (both on) is test_bond_split_forced_at_small_l."""
    env = {"SHIFTK_HEIS_SPLIT": "1", "SHIFTK_HEIS_STREAM": "0"}
    fuse, real = 1, 1
    if mode in ("plain", "real-only"):
        env["SHIFTK_SPLIT_FUSE"] = "0"
        fuse = 0
    if mode in ("plain", "fuse-only"):
        env["SHIFTK_LEFT_REAL"] = "0"
        real = 0
    if mode == "complex-left":
        env["COMPLEX_LEFT"] = "1"
        real = 0
    env.update(WANT_FUSE=str(fuse), WANT_REAL=str(real))
    _subprocess(SPLIT_MODES, env)


CSR_BLOCKED = """
import os
import numpy as np, oracle, synth
from paper_2001_08707_b200.device import make_solver, to_device
from test_gpu_parity import run_window
kind = os.environ["CSR_KIND"]
p = synth.make_problem("c3", M=1 << 13, nz=16) if kind == "c3" else synth.make_problem("c4", W=64, nz=8, n_left=3)
g, o, wr, wy = run_window(p, 25, full_check=(kind == "c3"))
i = g.info()
assert i["csr_col_blocks"] == int(os.environ["WANT_BLOCKS"]), i
h = make_solver(to_device(p))   # graph-captured == stepwise, bit for bit
h.run(g.iterations, poll_every=g.iterations)
assert np.array_equal(g.residuals(), h.residuals()) and np.array_equal(g.projections(), h.projections())
assert h.profile()["launches"] >= g.iterations * (1 + i["csr_col_blocks"])
print("ok")
"""


@pytest.mark.parametrize("kind,bshift,blocks", [("c3", 11, 4), ("c3", 12, 2), ("c4", 10, 4)])
def test_csr_column_blocked_passes(kind, bshift, blocks):
    """The column-blocked CSR SpMV (chosen at full-size C3, forced here with
    SHIFTK_CSR_BLOCKED=1 and small blocks): q accumulated over 2 or 4 passes of 2^bshift
    columns each, w and the finish agent in the last — oracle windows on scaled C3 (real CSR,
    COCG, full x) and C4 (complex CSR, two right-hand sides, BiCG), graph == stepwise bitwise."""
    _subprocess(CSR_BLOCKED, {"SHIFTK_CSR_BLOCKED": "1", "SHIFTK_CSR_BSHIFT": str(bshift),
                              "CSR_KIND": kind, "WANT_BLOCKS": str(blocks)})


def test_tile_pairs_window_and_determinism():
    """L=24 with the bond split off (SHIFTK_HEIS_SPLIT=0): the streaming SpMV works on tile pairs
    across the top spin bit (each the other's periodic partner); oracle window and bit-identical
    reruns."""
    _subprocess("""
import numpy as np, synth
from paper_2001_08707_b200.device import make_solver, to_device
from test_gpu_parity import run_window
p = synth.make_problem("c2", L=24, nz=8)
g, o, _, _ = run_window(p, 3)
assert g.info()["split_ahi"] == 0
h = make_solver(to_device(p))
for _ in range(3):
    h.update()
assert np.array_equal(g.residuals(), h.residuals())
assert g.coefficients() == h.coefficients()
print("ok")
""", {"SHIFTK_HEIS_SPLIT": "0"})


def test_many_shifts_beyond_the_shared_memory_flags():
    """N_z = 5000 > 4096: the finish compacts the active flags from global memory and the update
    uses eight shift agents."""
    p = synth.make_problem("c2", L=10, nz=5000)
    run_window(p, 12)


def test_full_mode_with_several_left_vectors():
    """Full x together with N_left = 6 projections (the FULL update kernel with NLMAX = 8)."""
    import dataclasses
    p = dataclasses.replace(synth.make_problem("c4", W=12, nz=8, n_left=6), full_x=True)
    run_window(p, 12, full_check=True)


def test_run_past_convergence_equals_stepwise():
    """sk_run polls every 64 iterations, so it launches iterations past convergence; they must be
    no-ops: the same iteration count, residuals and projections as stepping until converged."""
    p = synth.make_problem("c1", L=10, nz=8)
    dp = to_device(p)
    a = make_solver(dp)
    n = 0
    while a.update() == shiftk.ITERATING:
        n += 1
    b = make_solver(dp)
    assert b.run(p.itermax, poll_every=64) == shiftk.CONVERGED
    assert a.coefficients() == b.coefficients()
    assert np.array_equal(a.residuals(), b.residuals())
    assert np.array_equal(a.projections(), b.projections())
    for k in (0, p.n_shift - 1):
        assert np.array_equal(a.solution(k), b.solution(k))


def test_rc_equals_builtin_operator():
    """Reverse communication: caller-computed q = H r gives the same iterates."""
    p = synth.make_problem("c2", L=10, nz=16)
    dp = to_device(p)
    a = make_solver(dp)
    rc_op = shiftk.make_operator({"kind": "rc"}, p.M)
    b = shiftk.Solver(rc_op, "cocg", dp.b, p.z, tol=p.tol, itermax=p.itermax)
    hop = shiftk.make_operator(p.op, p.M)
    q = torch.empty_like(dp.b)
    for _ in range(40):
        a.update()
        rptr, _ = b.seed_vectors()
        r = shiftk.device_view(rptr, p.M)
        shiftk.apply_operator(hop, r, q)
        torch.cuda.synchronize()
        b.update_rc(q)
    assert np.array_equal(a.residuals(), b.residuals())
    assert np.array_equal(a.projections(), b.projections())


def test_host_inputs_equal_device_inputs():
    p = synth.make_problem("c4", W=12, nz=8, n_left=3)
    dp = to_device(p)
    a = make_solver(dp)
    b = make_solver(dp, host_inputs=True)
    a.run(30); b.run(30)
    assert np.array_equal(a.projections(), b.projections())


def test_edge_cases():
    # itermax = 1 -> MAXITER after one iteration
    p = synth.make_problem("c2", L=8, nz=4)
    dp = to_device(p)
    g = make_solver(dp, itermax=1)
    assert g.update() == shiftk.MAXITER
    assert g.update() == shiftk.MAXITER and g.iterations == 1
    # single shift, no switching possible
    p1 = synth.make_problem("c2", L=8, nz=1)
    g1 = make_solver(to_device(p1))
    assert g1.run(5000) == shiftk.CONVERGED and g1.coefficients()["switches"] == 0
    # right-hand side = eigenvector: converged after exactly one iteration, x = b/(z - E)
    L = 6
    b = np.ones(1 << L, dtype=np.complex128) / 8.0
    z = synth.spectrum_shifts(5, -3, 2, 0.1)
    op = shiftk.make_operator({"kind": "heisenberg", "L": L, "J": 1.0}, 1 << L)
    bd = torch.from_numpy(b).cuda()
    g2 = shiftk.Solver(op, "cocg", bd, z, full_x=True, tol=1e-12, itermax=10)
    assert g2.run(10) == shiftk.CONVERGED and g2.iterations == 1
    for k in range(5):
        assert np.allclose(g2.solution(k), b / (z[k] - L / 4), rtol=1e-14, atol=0)
    # breakdown: b^T b = 0
    bb = np.zeros(16, dtype=np.complex128)
    bb[0], bb[1] = 1 / math.sqrt(2), 1j / math.sqrt(2)
    op4 = shiftk.make_operator({"kind": "heisenberg", "L": 4, "J": 1.0}, 16)
    g3 = shiftk.Solver(op4, "cocg", torch.from_numpy(bb).cuda(), np.array([0.3 + 0.1j]), tol=1e-10, itermax=10)
    assert g3.update() == shiftk.BREAKDOWN


def test_errors():
    op4 = shiftk.make_operator({"kind": "heisenberg", "L": 4, "J": 1.0}, 16)
    b = torch.ones(16, dtype=torch.complex128, device="cuda")
    z = np.array([0.1j])
    with pytest.raises(shiftk.ShiftkError) as e:
        shiftk.Solver(op4, "cocg", b, z, tol=-1.0)
    assert e.value.code == -1
    with pytest.raises(shiftk.ShiftkError) as e:
        shiftk.Solver(op4, "cocg", torch.zeros_like(b), z)
    assert e.value.code == -1
    p = synth.make_problem("c4", W=6, nz=4, n_left=1)
    dp = to_device(p)
    with pytest.raises(shiftk.ShiftkError) as e:
        shiftk.Solver(dp.op, "cocg", dp.b, p.z)     # Table 1: COCG on complex Hermitian H
    assert e.value.code == -6
    g = shiftk.Solver(op4, "cocg", b, z)
    g.finalize()
    h = ctypes_null_handle()
    assert shiftk.load().sk_finalize(h) == -5


def ctypes_null_handle():
    import ctypes
    return ctypes.byref(ctypes.c_void_p())


def test_spmv_count_and_memory_invariants():
    """Table 2: 1 SpMV/iteration (COCG), 2 (BiCG), independent of N_z."""
    for nz in (1, 64):
        p = synth.make_problem("c2", L=10, nz=nz)
        g = make_solver(to_device(p))
        g.run(20)
        c = g.coefficients()
        assert c["spmv_count"] == c["iterations"]
        q = synth.make_problem("c4", W=8, nz=nz, n_left=2)
        h = make_solver(to_device(q))
        h.run(20)
        c = h.coefficients()
        assert c["spmv_count"] == 2 * c["iterations"]


@pytest.mark.parametrize("name,kw", [("c2", dict(L=12, nz=64)), ("c4", dict(W=16, nz=16, n_left=6))])
def test_recalc_parity(name, kw):
    """Recalculation at new shifts from the coefficient log: GPU replay vs the run's
    own projections at the original shifts (identity) and vs the oracle's replay at new shifts."""
    p = synth.make_problem(name, **kw)
    dp = to_device(p)
    g = make_solver(dp, flags=shiftk.FLAG_LOG, itermax=5000)
    assert g.run(5000) == shiftk.CONVERGED
    y_id, res_id = g.recalc(p.z)
    assert np.all(proj_err(y_id, g.projections()) <= 1e-12)
    assert np.all(res_id < p.tol)
    o = oracle.Oracle(p.method, p.b, p.z, left=p.left, tol=p.tol, itermax=5000)
    assert o.run(p.op, 5000) == oracle.CONVERGED
    z_new = (p.z[:-1] + p.z[1:]) / 2 + 0.01j       # between the original shifts
    yg, rg = g.recalc(z_new)
    yo, ro = o.recalc(z_new)
    assert np.all(proj_err(yg, yo) <= REL)
    # the two logs are different finite-precision trajectories near convergence (R24): compare
    # the replayed residuals by what they certify, not digit by digit
    # (a new shift nearer the real axis may not be converged when the log ends: both replays
    # then report a residual above tol, of the same size)
    assert np.all((rg < p.tol) == (ro < p.tol)) or np.all(np.abs(np.log10(rg / ro)) < 1)
    assert g.coefficients()["spmv_count"] == g.coefficients()["iterations"] * (2 if p.method == "bicg" else 1)


@pytest.mark.parametrize("name,kw", [("c1", dict(L=10, nz=8)), ("c2", dict(L=14, nz=64)),
                                     ("c4", dict(W=12, nz=8, n_left=4))])
def test_checkpoint_restart_matches_oracle(name, kw):
    """Restart ("restart coefficients supplied at init", P:L575 calctype=restart; SURVEY
    f-4) against the ORACLE: k iterations, checkpoint, the context destroyed, a fresh context
    restored from the blob; the restored state equals the oracle's after k iterations, and the
    restored context then advances in lockstep with the uninterrupted oracle run through the
    rest of the trajectory window (1e-9 on residuals and projections, equal retirement
    iterations, active sets and seed; full x compared in full mode)."""
    p = synth.make_problem(name, **kw)
    n_w = horizon(p, 40)
    assert n_w >= 10, n_w
    k = n_w // 2
    dp = to_device(p)
    a = make_solver(dp)
    a.run(k)
    blob = a.checkpoint()
    a.finalize()
    del a
    g = make_solver(dp)
    g.restore(blob)
    o = oracle.Oracle(p.method, p.b, p.z, left=p.left, full_x=p.full_x, tol=p.tol, itermax=p.itermax)
    for _ in range(k):
        o.step(p.op)
    for n in range(k, n_w + 1):
        if n > k:
            assert g.update() == o.step(p.op), n
        rg, ro = g.residuals(), o.residuals()
        assert np.all(np.abs(rg - ro) <= REL * ro), (n, np.max(np.abs(rg - ro) / ro))
        assert np.all(proj_err(g.projections(), o.projections()) <= REL), n
        c = g.coefficients()
        assert c["iterations"] == o.iterations == n
        if c["seed_index"] != o.seed_index:   # a |pi| tie (conjugate contour pairs): see run_window
            pio = np.abs(o.pi())
            assert abs(pio[c["seed_index"]] / pio[o.seed_index] - 1) < 1e-9, n
        _, act, ret = g.shift_state()
        assert np.array_equal(act, o.active()) and np.array_equal(ret, o.retired_at()), n
        if p.full_x:
            for kk in (0, p.n_shift - 1):
                xo = o.solution(kk)
                assert np.linalg.norm(g.solution(kk) - xo) <= REL * np.linalg.norm(xo), (n, kk)


@pytest.mark.parametrize("name,kw", [("c1", dict(L=10, nz=8)), ("c4", dict(W=12, nz=8, n_left=4))])
def test_checkpoint_restart_bitwise(name, kw):
    """Restart (SURVEY f-4): k iterations, checkpoint, restore into a fresh
    context, continue — bit-identical to the uninterrupted run (full x included)."""
    p = synth.make_problem(name, **kw)
    dp = to_device(p)
    a = make_solver(dp, flags=shiftk.FLAG_LOG, itermax=3000)
    a.run(37)
    blob = a.checkpoint()
    b = make_solver(dp, flags=shiftk.FLAG_LOG, itermax=3000)
    b.restore(blob)
    a.run(3000)
    b.run(3000)
    assert a.coefficients() == b.coefficients()
    assert np.array_equal(a.projections(), b.projections())
    assert np.array_equal(a.residuals(), b.residuals())
    if p.full_x:
        assert np.array_equal(a.solution(3), b.solution(3))
    assert np.array_equal(a.recalc(p.z)[0], b.recalc(p.z)[0])
    c = make_solver(to_device(synth.make_problem(name, **dict(kw, nz=kw["nz"] + 1))))
    with pytest.raises(shiftk.ShiftkError):
        c.restore(blob)
