"""Host-side logic of the row-sharded multi-GPU path: the partition of the
vector rows over ranks, the per-rank slices of the inputs, and the connection handshake of the
one-process-per-GPU mode (CUDA IPC handles all-gathered, one ncclUniqueId broadcast).

Rank g owns global rows [g M_local, (g + 1) M_local), M_local = M / world a power of two; for the
Heisenberg chain the top log2(world) spin bits select the rank (sites L-3..L-1
for 8 GPUs).  Dot products are all-reduced; the SpMV reads other ranks' rows in place through
peer memory (include/shiftk.h, sk_dist).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np


def shard_rows(M: int, world: int, rank: int):
    """(row0, M_local) of `rank`; raises unless world divides M into power-of-two shards."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if M % world:
        raise ValueError(f"world {world} does not divide M = {M}")
    ml = M // world
    if ml & (ml - 1):
        raise ValueError(f"M_local = {ml} must be a power of two")
    return rank * ml, ml


@dataclasses.dataclass
class LocalSlice:
    row0: int
    M_local: int
    b: np.ndarray                    # [M_local] complex128
    left: Optional[np.ndarray]       # [n_left, M_local] or None (a = b)
    op: dict                         # operator restricted to the rows (CSR: global columns)


def local_slice(problem, world: int, rank: int) -> LocalSlice:
    """This rank's rows of b, of the left vectors and of the operator."""
    row0, ml = shard_rows(problem.M, world, rank)
    sl = slice(row0, row0 + ml)
    b = np.ascontiguousarray(problem.b[sl])
    left = None if problem.left is None else np.ascontiguousarray(problem.left[:, sl])
    op = dict(problem.op)
    if op["kind"] in ("csr_real", "csr_cplx"):
        rp = problem.op["row_ptr"]
        e0, e1 = int(rp[row0]), int(rp[row0 + ml])
        op["row_ptr"] = np.ascontiguousarray(rp[row0:row0 + ml + 1] - e0)
        op["col"] = np.ascontiguousarray(problem.op["col"][e0:e1])       # global column ids
        op["val"] = np.ascontiguousarray(problem.op["val"][e0:e1])
    return LocalSlice(row0=row0, M_local=ml, b=b, left=left, op=op)


def to_device_slice(problem, world: int, rank: int, device: str = "cuda:0"):
    """DeviceProblem of this rank's slice (sk_operator with M_local / row_begin set)."""
    import torch

    from .device import DeviceProblem
    from .shiftk import make_operator
    s = local_slice(problem, world, rank)
    dev = torch.device(device)
    b = torch.from_numpy(s.b).to(dev)
    left = None if s.left is None else torch.from_numpy(s.left).to(dev)
    arrays = None
    if s.op["kind"] in ("csr_real", "csr_cplx"):
        arrays = {k: torch.from_numpy(s.op[k]).to(dev) for k in ("row_ptr", "col", "val")}
    op = make_operator(s.op, problem.M, arrays, M_local=s.M_local, row_begin=s.row0)
    return DeviceProblem(op=op, b=b, left=left, arrays=arrays, problem=problem), s


def exchange_handles(handle: bytes, make_id, pg=None):
    """All-gather every rank's 64-byte IPC handle (rank order) and broadcast one NCCL id made by
    rank 0 (`make_id()` is only called there).  Returns (handles_concatenated, nccl_id)."""
    import torch.distributed as dist
    world = dist.get_world_size(pg)
    rank = dist.get_rank(pg)
    allh = [None] * world
    dist.all_gather_object(allh, bytes(handle), group=pg)
    box = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=pg)
    assert all(len(h) == 64 for h in allh) and len(box[0]) == 128
    return b"".join(allh), box[0]


def connect(solver, pg=None):
    """One-process-per-GPU connection of a Solver created with rank/world (collective)."""
    from .shiftk import nccl_unique_id
    handles, nid = exchange_handles(solver.ipc_handle(), nccl_unique_id, pg)
    solver.connect(handles, nid)


def connect_host(solver, pg=None):
    """Connection with the host collective of a torch.distributed group (e.g. gloo) in place of
    NCCL (sk_connect_host): IPC handles all-gathered through `pg`, the per-iteration all-reduces
    of the dots through `pg` on the host.  Several processes may share one GPU this way (no
    kernel waits on another process's kernel)."""
    import torch
    import torch.distributed as dist
    allh = [None] * dist.get_world_size(pg)
    dist.all_gather_object(allh, solver.ipc_handle(), group=pg)

    def allreduce(send, recv):
        t = torch.from_numpy(send.copy())
        dist.all_reduce(t, group=pg)
        recv[:] = t.numpy()
    solver.connect_host(b"".join(allh), allreduce)


def remote_rows_per_spmv(problem, world: int, rank: int) -> int:
    """Rows of OTHER ranks this rank's SpMV reads per application (each a 16-B complex128 read
    over NVLink; element count, the algorithmic exchange volume of SURVEY §8(e)).

    Heisenberg chain (rank = top log2(world) spin bits): a bond (i, i+1 mod L) reaches another
    rank iff it flips a rank bit; for a bond between a rank bit and a local bit, half of the local
    rows have it anti-aligned; for a bond between two rank bits, all rows or none (fixed by the
    rank).  CSR: the stored entries of the local rows whose column lies outside them."""
    row0, ml = shard_rows(problem.M, world, rank)
    if world == 1:
        return 0
    op = problem.op
    if op["kind"] == "heisenberg":
        L = int(op["L"])
        k = world.bit_length() - 1
        top = set(range(L - k, L))
        g = rank
        n = 0
        for i in range(L):
            a, b = i, (i + 1) % L
            if a not in top and b not in top:
                continue
            if a in top and b in top:
                ga, gb = (g >> (a - (L - k))) & 1, (g >> (b - (L - k))) & 1
                n += ml if ga != gb else 0
            else:
                n += ml // 2
        return n
    if op["kind"] in ("csr_real", "csr_cplx"):
        rp = op["row_ptr"]
        col = op["col"][int(rp[row0]):int(rp[row0 + ml])]
        return int(np.count_nonzero((col < row0) | (col >= row0 + ml)))
    raise ValueError(f"no exchange model for operator kind {op['kind']}")

