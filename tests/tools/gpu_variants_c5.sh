# C5 H_A SpMV variants (libs built by tests/tools/build_variant.py into _var/): isolated ncu duration
# of both split kernels, then the event-timed bench step of each.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for LIB in "" $(ls _var/libshiftk_*.so 2>/dev/null); do
SHIFTK_LIB=$LIB timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --clock-control none -k "regex:heisenberg_tiled|update_split" -s 4 -c 2 python bench.py --config c5 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "heisenberg_tiled|update_split|duration|inst_executed|wavefronts|bytes_read" | sed "s#^#$LIB #"
SHIFTK_LIB=$LIB timeout 900 python bench.py --config c5 --steps 30 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_var.json 2>/dev/null
python - <<PY
import json; d=json.loads(open("gpurun_out/bench_c5_var.json").read().strip().splitlines()[-1]); print("$LIB bench", round(d["ms_per_step"],3), {k: round(v,3) for k,v in d["kernel_ms_per_step"].items()}, round(d["iteration_gbs_model_frac"],3), d["clocks"]["sm_mhz"], d["plan"]["spmv_ctas"])
PY
done
