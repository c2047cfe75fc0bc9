"""CPU tests of the multi-rank host logic with real world-size-2 gloo process groups:
the row partition, the per-rank input slices (their union is the global problem, CSR rows
rebased with global column ids), and the connection handshake protocol (IPC handles gathered in
rank order, one NCCL id shared by every rank)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2001_08707_b200 import dist as skdist


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
        out = {}
        # partition + slices of three operator kinds
        for name, kw in [("c3", dict(M=1 << 10, nz=4)), ("c4", dict(W=16, nz=4, n_left=3)),
                         ("c2", dict(L=10, nz=4))]:
            p = synth.make_problem(name, **kw)
            s = skdist.local_slice(p, world, rank)
            got = [None] * world
            dist.all_gather_object(got, (s.row0, s.M_local, s.b, s.left, s.op))
            out[name] = got
        # handshake: fake 64-byte handles, id made by rank 0 only
        calls = []

        def make_id():
            calls.append(1)
            return bytes([7]) * 128

        h, nid = skdist.exchange_handles(bytes([rank + 1]) * 64, make_id)
        out["handshake"] = (h, nid, len(calls))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_shard_rows_rules():
    assert skdist.shard_rows(1 << 20, 8, 3) == (3 << 17, 1 << 17)
    with pytest.raises(ValueError):
        skdist.shard_rows(3 * 1000, 3, 0)         # M_local not a power of two
    with pytest.raises(ValueError):
        skdist.shard_rows(1 << 10, 3, 0)         # world does not divide M


@pytest.mark.parametrize("name,kw", [("c3", dict(M=1 << 10, nz=4)), ("c4", dict(W=16, nz=4, n_left=3)),
                                     ("c2", dict(L=10, nz=4))])
def test_slices_reassemble_the_problem(results, name, kw):
    p = synth.make_problem(name, **kw)
    for rank in (0, 1):
        parts = results[rank][name]          # every rank sees the same gathered slices
        row0s = [pp[0] for pp in parts]
        assert row0s == [0, p.M // 2]
        assert np.array_equal(np.concatenate([pp[2] for pp in parts]), p.b)
        if p.left is not None:
            assert np.array_equal(np.concatenate([pp[3] for pp in parts], axis=1), p.left)
        if p.op["kind"] != "heisenberg":
            rp = np.concatenate([parts[0][4]["row_ptr"][:-1],
                                 parts[1][4]["row_ptr"] + parts[0][4]["row_ptr"][-1]])
            assert np.array_equal(rp, p.op["row_ptr"])
            assert np.array_equal(np.concatenate([pp[4]["col"] for pp in parts]), p.op["col"])
            assert np.array_equal(np.concatenate([pp[4]["val"] for pp in parts]), p.op["val"])
        else:
            assert all(pp[4] == p.op for pp in parts)


def test_handshake_protocol(results):
    h0, id0, calls0 = results[0]["handshake"]
    h1, id1, calls1 = results[1]["handshake"]
    assert h0 == h1 == bytes([1]) * 64 + bytes([2]) * 64     # rank order
    assert id0 == id1 == bytes([7]) * 128                     # one id, shared
    assert calls0 == 1 and calls1 == 0                        # made on rank 0 only


@pytest.mark.parametrize("world", [2, 4, 8])
def test_remote_rows_model_matches_enumeration(world):
    """The NVLink exchange model (dist.remote_rows_per_spmv, reported by bench.py for N > 1)
    against a brute-force count of the off-rank partners of every local row (L = 10 chain; an
    8-rank CSR with random columns)."""
    import numpy as np
    import synth
    from paper_2001_08707_b200 import dist
    p = synth.make_problem("c2", L=10, nz=2)
    L, M = 10, 1 << 10
    ml = M // world
    for rank in range(world):
        n = 0
        for s in range(rank * ml, (rank + 1) * ml):
            for i in range(L):
                j = (i + 1) % L
                if ((s >> i) ^ (s >> j)) & 1:
                    n += ((s ^ (1 << i) ^ (1 << j)) // ml) != rank
        assert dist.remote_rows_per_spmv(p, world, rank) == n
    q = synth.make_problem("c3", M=1 << 12, nz=2)
    for rank in range(world):
        r0, r1 = rank * (q.M // world), (rank + 1) * (q.M // world)
        rp, col = q.op["row_ptr"], q.op["col"]
        n = sum(int(not (r0 <= c < r1)) for c in col[rp[r0]:rp[r1]])
        assert dist.remote_rows_per_spmv(q, world, rank) == n
