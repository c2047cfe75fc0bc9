# Full GPU check of a change: the gpu test suite, then the round's measurements (gpu_profiles_r02.sh).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
tail -4 gpurun_out/pytest.log
SHIFTK_SPLIT_LO=1 timeout 900 python bench.py --config c5 --steps 20 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_lo.json 2>/dev/null
python - <<PY
import json; d=json.loads(open("gpurun_out/bench_c5_lo.json").read().strip().splitlines()[-1]); print("c5 split_lo", round(d["ms_per_step"],3), {k: round(v,3) for k,v in d["kernel_ms_per_step"].items()}, round(d["iteration_gbs_model_frac"],3), d["clocks"]["sm_mhz"])
PY
bash tests/tools/gpu_profiles_r02.sh
