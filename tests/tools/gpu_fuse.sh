cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "split" > gpurun_out/pytest_split.log 2>&1; tail -3 gpurun_out/pytest_split.log
for V in "SHIFTK_SPLIT_FUSE=0 SHIFTK_LEFT_REAL=0" "SHIFTK_SPLIT_FUSE=1 SHIFTK_LEFT_REAL=0" "SHIFTK_SPLIT_FUSE=0 SHIFTK_LEFT_REAL=1" "SHIFTK_SPLIT_FUSE=1 SHIFTK_LEFT_REAL=1"; do
  T=$(echo $V | tr ' =' '__')
  env $V timeout 900 python bench.py --config c5 --steps 20 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_$T.json 2> gpurun_out/bench_c5_$T.err
  python - <<PY
import json; d=json.loads(open("gpurun_out/bench_c5_$T.json").read().strip().splitlines()[-1]); print("$V", round(d["ms_per_step"],3), {k: round(v,3) for k,v in d["kernel_ms_per_step"].items()}, round(d["iteration_gbs_model_frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["solver_state"])
PY
done
