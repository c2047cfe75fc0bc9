"""The row-sharded multi-rank path on ONE GPU through a loopback group: `world` contexts, each
with its own rows, reading the other ranks' rows in place through the shard tables (the same
kernels and tables the NCCL mode uses with NVLink peer mappings), all-reduces done by the
group.  Parity against the oracle on the global problem, as in test_gpu_parity."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2001_08707_b200 import shiftk  # noqa: E402
from paper_2001_08707_b200.dist import to_device_slice  # noqa: E402

REL = 1e-9


def proj_err(a, b):
    return np.max(np.abs(a - b), axis=1) / np.maximum(np.max(np.abs(b), axis=1), 1e-300)


def make_group(p, world):
    g = shiftk.Group(world)
    keep = []
    for r in range(world):
        dp, s = to_device_slice(p, world, r)
        shiftk.Solver(dp.op, p.method, dp.b, p.z, left=dp.left, full_x=p.full_x, tol=p.tol,
                      itermax=p.itermax, rank=r, world=world, group=g)
        keep.append(dp)
    g.connect()
    return g, keep


@pytest.mark.parametrize("name,kw,world,n_w", [
    ("c2", dict(L=14, nz=64), 2, 25),       # Heisenberg, top spin bit sharded
    ("c5", dict(L=16, nz=64), 8, 20),       # Heisenberg, top 3 spin bits (the C5 layout)
    ("c3", dict(M=1 << 12, nz=16), 4, 20),  # real CSR, random columns: most reads remote
    ("c4", dict(W=32, nz=16, n_left=8), 4, 20),   # complex Hermitian CSR, BiCG, 8 left vectors
])
def test_loopback_group_window(name, kw, world, n_w):
    p = synth.make_problem(name, **kw)
    g, keep = make_group(p, world)
    o = oracle.Oracle(p.method, p.b, p.z, left=p.left, full_x=p.full_x, tol=p.tol, itermax=p.itermax)
    for n in range(n_w):
        sg = g.update()
        so = o.step(p.op)
        assert sg == so, n
        ro = o.residuals()
        yo = o.projections()
        for m in g.members:   # every rank holds the same (replicated) per-shift results
            rg = m.residuals()
            assert np.all(np.abs(rg - ro) <= REL * ro), (n, np.max(np.abs(rg - ro) / ro))
            assert np.all(proj_err(m.projections(), yo) <= REL), n
        if p.full_x:
            for k in (0, p.n_shift - 1):
                xg = np.concatenate([m.solution(k) for m in g.members])
                xo = o.solution(k)
                assert np.linalg.norm(xg - xo) <= REL * np.linalg.norm(xo)
    c0 = g.members[0].coefficients()
    assert all(m.coefficients() == c0 for m in g.members)   # bit-identical replicated scalars
    g.close()


def test_loopback_group_converges_like_single_gpu():
    p = synth.make_problem("c2", L=12, nz=32)
    g, keep = make_group(p, 4)
    assert g.run(p.itermax) == shiftk.CONVERGED
    o = oracle.solve(p)
    assert o.status == oracle.CONVERGED
    assert np.all(proj_err(g.members[2].projections(), o.projections()) <= REL)
    assert np.all(g.members[0].residuals() < p.tol)
    g.close()


def test_unconnected_context_refuses_to_iterate():
    p = synth.make_problem("c2", L=10, nz=4)
    dp, s = to_device_slice(p, 2, 0)
    solver = shiftk.Solver(dp.op, p.method, dp.b, p.z, tol=p.tol, itermax=10, rank=0, world=2)
    with pytest.raises(shiftk.ShiftkError) as e:
        solver.update()
    assert e.value.code == -5


def test_loopback_group_with_the_streaming_kernel():
    """The multi-rank (MULTI) instantiation of the streaming Heisenberg SpMV — shard-table
    partner addresses fed to the bulk copies — forced at a small size in a subprocess
    (SHIFTK_HEIS_STREAM is read once per process)."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, synth, oracle\n"
        "from test_gpu_multirank import make_group, REL, proj_err\n"
        "p = synth.make_problem('c5', L=16, nz=32)\n"
        "g, keep = make_group(p, 4)\n"
        "o = oracle.Oracle(p.method, p.b, p.z, left=p.left, full_x=p.full_x, tol=p.tol, itermax=p.itermax)\n"
        "for n in range(12):\n"
        "    assert g.update() == o.step(p.op)\n"
        "    ro = o.residuals()\n"
        "    for m in g.members:\n"
        "        assert np.all(np.abs(m.residuals() - ro) <= REL * ro), n\n"
        "        assert np.all(proj_err(m.projections(), o.projections()) <= REL), n\n"
        "g.close()\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SHIFTK_HEIS_STREAM="1", PYTHONPATH=root + os.pathsep + os.path.join(root, "tests"))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-3000:]


def test_nccl_plumbing_one_rank_communicator():
    """The NCCL glue of the multi-rank mode (dlopen'ed entry points, ncclCommInitRank, the
    iteration's ncclDouble / ncclSum all-reduce on a user stream, directly and replayed from a
    captured graph) on real hardware: with ONE rank the sum is the input, bit for bit.  (Several
    NCCL ranks need several GPUs; the sharded data plane is covered by the loopback group above and
    by test_gpu_ipc_two_process.)"""
    x = np.random.default_rng(11).standard_normal(2 * (2 + 32))   # C4's update dots: 2 + N_left complex
    o1, o2 = shiftk.nccl_selftest(x)
    assert np.array_equal(o1, x) and np.array_equal(o2, x)
