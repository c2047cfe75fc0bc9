cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {  # name, env...
  N=$1; shift
  env "$@" timeout 900 python bench.py --config c5 --steps 20 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_$N.json 2> gpurun_out/bench_c5_$N.err
  python - <<PY
import json; d=json.loads(open("gpurun_out/bench_c5_$N.json").read().strip().splitlines()[-1]); print("$N", round(d["ms_per_step"],3), {k: round(v,3) for k,v in d["kernel_ms_per_step"].items()}, round(d["iteration_gbs_model_frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["plan"])
PY
}
run early X=1
run min3 SHIFTK_LIB=_var/libshiftk_min3.so
run late SHIFTK_LIB=_var/libshiftk_late.so
run early_lo SHIFTK_SPLIT_LO=1
run nofuse SHIFTK_SPLIT_FUSE=0
run early2 X=1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "split or c5" > gpurun_out/pytest_split.log 2>&1; tail -3 gpurun_out/pytest_split.log
for LIB in "" _var/libshiftk_min3.so; do
SHIFTK_LIB=$LIB timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:heisenberg_tiled|update_split" -s 4 -c 2 python bench.py --config c5 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "heisenberg_tiled|update_split|duration|inst_executed|wavefronts|bytes" | sed "s#^#$LIB #"
done
