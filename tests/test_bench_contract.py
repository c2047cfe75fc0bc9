"""CPU check of bench.py's output contract on the reference arm (the CPU oracle; the GPU arm's
line has the same keys plus roofline / clocks / gpu_launches and is checked on the box)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line_with_the_contract_keys():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "3", "--warmup", "3"],
                         capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "impl",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 3 and d["value"] > 0
    assert d["higher_is_better"] is True and d["data"] == "synthetic"
    assert "workload" in d["config"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_byte_model_covers_every_config():
    sys.path.insert(0, ROOT)
    import bench
    import synth
    for name, kw in [("c1", {}), ("c2", dict(L=12)), ("c3", dict(M=1 << 10)), ("c4", dict(W=16)),
                     ("c5", dict(L=12)), ("c5sz", dict(L=12))]:
        p = synth.make_problem(name, **kw)
        assert bench.bytes_per_row(p, "spmv") >= 32
        assert bench.bytes_per_row(p, "update") >= 64
