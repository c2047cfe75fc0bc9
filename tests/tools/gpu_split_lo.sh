cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "split" 2>&1 | tail -2
for V in "SHIFTK_SPLIT_LO=0" "SHIFTK_SPLIT_LO=1"; do
env $V timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_q.json 2> gpurun_out/bench_c5_q.err
python - <<PY
import json; d=json.loads(open("gpurun_out/bench_c5_q.json").read().strip().splitlines()[-1]); print("$V", round(d["ms_per_step"],3), {k: round(v,3) for k,v in d["kernel_ms_per_step"].items()}, round(d["iteration_gbs_model_frac"],3), d["clocks"])
PY
env $V timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed --clock-control none -k "regex:heisenberg_tiled|update_split" -s 4 -c 2 python bench.py --config c5 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "duration|inst_executed|wavefronts"
done
