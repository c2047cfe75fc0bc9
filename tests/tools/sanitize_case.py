"""One small solver run per hot-path kernel family, for compute-sanitizer (tests/test_gpu_sanitizer.py).

    python tests/tools/sanitize_case.py CASE

Cases (the SHIFTK_* switches are set by the caller's environment):
  tiled   Heisenberg L=14 (tiled SpMV, update), and full mode L=10 (FULL update)
  stream  Heisenberg L=23 with SHIFTK_HEIS_STREAM=1 SHIFTK_HEIS_SPLIT=0 (TMA-fed streaming SpMV:
          mbarrier rings, tile queue + rewind, per-group w partials)
  pair    Heisenberg L=24 with SHIFTK_HEIS_SPLIT=0 (tile-pair streaming SpMV)
  split   Heisenberg L=20 with SHIFTK_HEIS_SPLIT=1 (H_A tiled SpMV, B-tile update, split init)
  sector  Sz=0 sector L=20 (block sector SpMV: block queue, per-block/group partials)
  csr     real CSR M=2^14 (row kernel, full x) and BiCG lattice W=32 with 6 left vectors
          (2-RHS CSR, projection-heavy update)
Runs a few iterations through the C-ABI and synchronises; exits non-zero on any library error.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2001_08707_b200.device import make_solver, to_device  # noqa: E402


def run(p, n, **kw):
    g = make_solver(to_device(p), **kw)
    for _ in range(n):
        g.update()
    g.run(2, poll_every=2)   # the graph-captured loop too
    g.residuals()
    g.projections()
    g.finalize()


def main(case):
    if case == "tiled":
        run(synth.make_problem("c2", L=14, nz=8), 3)
        run(synth.make_problem("c1", L=10, nz=8), 3)
    elif case == "stream":
        run(synth.make_problem("c2", L=23, nz=8), 2)
    elif case == "pair":
        run(synth.make_problem("c2", L=24, nz=8), 1)
    elif case == "split":
        run(synth.make_problem("c2", L=20, nz=16), 3)
    elif case == "sector":
        run(synth.make_problem("c5sz", L=20, nz=8), 2)
    elif case == "csr":
        run(synth.make_problem("c3", M=1 << 14, nz=8), 2)
        run(synth.make_problem("c4", W=32, nz=4, n_left=6), 2)
    else:
        raise SystemExit(f"unknown case {case}")
    import torch
    torch.cuda.synchronize()
    print("ok", case)


if __name__ == "__main__":
    main(sys.argv[1])
