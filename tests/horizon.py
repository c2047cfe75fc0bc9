"""Self-divergence horizon of the oracle — TEST INFRASTRUCTURE.

Finite-precision Krylov iterates are chaotic beyond some iteration: two CORRECT fp64 orderings
of the same reductions drift apart geometrically once Ritz values converge (SURVEY §0 finding 4,
§8(c.2) R24).  A trajectory window can therefore only demand 1e-9 agreement between the GPU and
the oracle up to the iteration where the oracle still agrees with ITSELF run in another order.

``horizon(problem, n_max)`` runs the oracle twice on the same input — the natural reduction
order and every reduction reversed (OR_FLAG_REVERSE) — and returns the number of leading
iterations over which both runs agree to ``agree`` (default 1e-11) relative, per shift, in the
residual norm and in the normwise projection (R23), with identical status, active sets and
retirement iterations.  Window tests call it to set their length instead of hard-coding it.

Threshold (R30): SURVEY §8(c.4) proposed 1e-12.  On C3's geometry (Im z = 0.02, a
seed switch nearly every iteration) the two orderings differ by ~1e-12 from the second
iteration on and stay there for dozens of iterations, so 1e-12 gives a horizon of 1; 1e-11 keeps
a factor 100 below the 1e-9 parity bar and measures where the drift really starts (C1: 31,
C2 at L=14: 37, C5's shifts at L=18: 56, C3 at M=2^14: > 60).
"""
from __future__ import annotations

import functools

import numpy as np

import oracle


def _proj_err(a, b):
    return np.max(np.abs(a - b), axis=1) / np.maximum(np.max(np.abs(b), axis=1), 1e-300)


def horizon(problem, n_max: int, *, agree: float = 1e-11, flags: int = 0, tol=None,
            omp=None) -> int:
    """Leading iterations (<= n_max) over which the forward and reversed oracle runs agree."""
    t = problem.tol if tol is None else tol
    kw = dict(left=problem.left, full_x=False, tol=t, itermax=problem.itermax, omp=omp)
    a = oracle.Oracle(problem.method, problem.b, problem.z, flags=flags, **kw)
    b = oracle.Oracle(problem.method, problem.b, problem.z, flags=flags | oracle.FLAG_REVERSE, **kw)
    n = 0
    try:
        while n < n_max:
            sa, sb = a.step(problem.op), b.step(problem.op)
            if sa != sb:
                break
            ra, rb = a.residuals(), b.residuals()
            if not np.all(np.abs(ra - rb) <= agree * np.maximum(ra, 1e-300)):
                break
            if not np.all(_proj_err(a.projections(), b.projections()) <= agree):
                break
            if not (np.array_equal(a.active(), b.active())
                    and np.array_equal(a.retired_at(), b.retired_at())):
                break
            n += 1
            if sa != oracle.ITERATING:
                break
    finally:
        a.close()
        b.close()
    return n


@functools.lru_cache(maxsize=None)
def horizon_of(name: str, n_max: int, **kw) -> int:
    """horizon() of synth.make_problem(name, **kw) (cached per test session)."""
    import synth
    return horizon(synth.make_problem(name, **kw), n_max)
