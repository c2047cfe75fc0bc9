"""The boundary from plain C: examples/spectrum.c (no Python, no torch) is compiled against
include/shiftk.h and libshiftk.so, run, and its spectral function checked against the oracle
on the same right-hand side (the example's LCG, regenerated here)."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def lcg_b(M, seed=12345):
    out = np.empty(M)
    s = seed
    for i in range(M):
        s = (s * 6364136223846793005 + 1442695040888963407) % (1 << 64)
        out[i] = (s >> 11) / 9007199254740992.0 - 0.5
    return (out / np.linalg.norm(out)).astype(np.complex128)


def test_c_program_spectrum_matches_oracle():
    from paper_2001_08707_b200 import build
    lib_dir = os.path.dirname(build.build())
    L, nz = 10, 24
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "spectrum")
        subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"),
                               os.path.join(ROOT, "examples", "spectrum.c"), "-L", lib_dir, "-lshiftk",
                               f"-Wl,-rpath,{lib_dir}", "-lm", "-o", exe])
        out = subprocess.run([exe, str(L), str(nz)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    assert lines[-1].startswith("status 1")
    data = np.array([[float(v) for v in l.split()] for l in lines[:-1]])
    z = synth.spectrum_shifts(nz, -6.0, 2.0, 0.1)   # the example's grid (same arithmetic)
    assert np.allclose(data[:, 0], z.real, atol=1e-6)
    b = lcg_b(1 << L)
    o = oracle.Oracle("cocg", b, z, tol=1e-10, itermax=20000)
    assert o.run({"kind": "heisenberg", "L": L, "J": 1.0}, 20000) == oracle.CONVERGED
    a_or = -o.projections()[:, 0].imag / np.pi
    assert np.max(np.abs(data[:, 1] - a_or)) <= 2 * (1e-10 + 1e-12) / 0.1 / np.pi
    assert np.all(data[:, 2] < 1e-10)
