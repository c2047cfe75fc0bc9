"""Torch plumbing: put a synth.Problem's inputs in device memory and build the C-ABI objects.

PyTorch is used only for device allocations and host<->device copies here; the solver never
calls torch ops.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

from .shiftk import Solver, make_operator, sk_operator


@dataclasses.dataclass
class DeviceProblem:
    op: sk_operator
    b: object                 # torch complex128 [M] on device
    left: Optional[object]    # torch complex128 [n_left, M] on device, or None (a = b)
    arrays: Optional[dict]    # CSR device arrays (kept alive here)
    problem: object


def to_device(problem, device: str = "cuda:0") -> DeviceProblem:
    import torch
    dev = torch.device(device)
    b = torch.from_numpy(problem.b).to(dev)
    left = None if problem.left is None else torch.from_numpy(np.ascontiguousarray(problem.left)).to(dev)
    arrays = None
    if problem.op["kind"] in ("csr_real", "csr_cplx"):
        arrays = {k: torch.from_numpy(problem.op[k]).to(dev) for k in ("row_ptr", "col", "val")}
    op = make_operator(problem.op, problem.M, arrays)
    return DeviceProblem(op=op, b=b, left=left, arrays=arrays, problem=problem)


def make_solver(dp: DeviceProblem, *, tol: Optional[float] = None, itermax: Optional[int] = None,
                flags: int = 0, full_x: Optional[bool] = None, host_inputs: bool = False) -> Solver:
    p = dp.problem
    b = p.b if host_inputs else dp.b
    left = (p.left if host_inputs else dp.left) if p.left is not None else None
    return Solver(dp.op, p.method, b, p.z, left=left,
                  full_x=p.full_x if full_x is None else full_x,
                  tol=p.tol if tol is None else tol,
                  itermax=p.itermax if itermax is None else itermax, flags=flags,
                  device=dp.b.device.index or 0)
