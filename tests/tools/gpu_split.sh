cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "split or tile_pairs" > gpurun_out/pytest_split.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_split.log
tail -5 gpurun_out/pytest_split.log
for A in 1 0; do
SHIFTK_HEIS_STREAM=$A timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_split_s$A.json 2> gpurun_out/bench_c5_split_s$A.err
python - <<PY
import json; d=json.loads(open("gpurun_out/bench_c5_split_s$A.json").read().strip().splitlines()[-1]); print("stream=$A", d["ms_per_step"], d["kernel_ms_per_step"], d["iteration_gbs_model_frac"], d["clocks"]["sm_mhz"])
PY
done
