"""The multi-rank data plane across PROCESSES on one GPU: two
processes, each its own context over half of the rows (world 2), exchange CUDA IPC handles
through a gloo group and map each other's arena (cudaIpcOpenMemHandle — legal between processes
on one device); the SpMV kernels then read the other process's rows in place through the shard
tables (the MULTI kernels of the NVLink path).  The two per-iteration all-reduces go through the
host collective (sk_connect_host + gloo) instead of NCCL, which refuses two ranks on one GPU; so no
kernel of one process ever waits on the other's kernel (the ranks meet only inside the host
all-reduce — see B200_PROFILING.md on ranks sharing a GPU).  Checked against the oracle on the
global problem (1e-9) and for bit-identical scalars on both ranks."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

REL = 1e-9
CASES = [("c2", dict(L=14, nz=32), 20), ("c3", dict(M=1 << 12, nz=16), 15),
         ("c4", dict(W=32, nz=8, n_left=4), 12)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2001_08707_b200 import dist as skdist
        from paper_2001_08707_b200 import shiftk
        torch.cuda.set_device(0)
        out = {}
        for name, kw, n_w in CASES:
            p = synth.make_problem(name, **kw)
            dp, sl = skdist.to_device_slice(p, world, rank, "cuda:0")
            s = shiftk.Solver(dp.op, p.method, dp.b, p.z, left=dp.left, full_x=p.full_x, tol=p.tol,
                              itermax=p.itermax, device=0, rank=rank, world=world)
            skdist.connect_host(s)
            traj = []
            for _ in range(n_w):
                st = s.update()
                traj.append((st, s.residuals(), s.projections(), s.coefficients()))
            out[name] = traj
            s.finalize()
            del dp
        q.put((rank, out))
    except Exception as e:   # surfaced by the test
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_processes_one_gpu_ipc_data_plane():
    import oracle
    import synth
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=900) for _ in procs)
    for pr in procs:
        pr.join(timeout=120)
    for r in range(world):
        assert isinstance(res[r], dict), res[r]
    for name, kw, n_w in CASES:
        p = synth.make_problem(name, **kw)
        o = oracle.Oracle(p.method, p.b, p.z, left=p.left, full_x=p.full_x, tol=p.tol, itermax=p.itermax)
        for n in range(n_w):
            so = o.step(p.op)
            (s0, r0, y0, c0), (s1, r1, y1, c1) = res[0][name][n], res[1][name][n]
            assert s0 == s1 == so, (name, n)
            # every rank holds the same (all-reduced) scalars, bit for bit
            assert np.array_equal(r0, r1) and np.array_equal(y0, y1) and c0 == c1, (name, n)
            ro = o.residuals()
            assert np.all(np.abs(r0 - ro) <= REL * ro), (name, n, np.max(np.abs(r0 - ro) / ro))
            yo = o.projections()
            e = np.max(np.abs(y0 - yo), axis=1) / np.maximum(np.max(np.abs(yo), axis=1), 1e-300)
            assert np.all(e <= REL), (name, n, np.max(e))
        o.close()
