cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "csr_column_blocked or c3 or c4" > gpurun_out/pytest_csr.log 2>&1; tail -3 gpurun_out/pytest_csr.log
run() {  # config, name, env...
  C=$1; N=$2; shift; shift
  env "$@" timeout 900 python bench.py --config $C --steps ${STEPS:-10} --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_${C}_$N.json 2> gpurun_out/bench_${C}_$N.err
  python - <<PY
import json; d=json.loads(open("gpurun_out/bench_${C}_$N.json").read().strip().splitlines()[-1]); print("$C $N", round(d["ms_per_step"],3), {k: round(v,3) for k,v in d["kernel_ms_per_step"].items()}, round(d["iteration_gbs_model_frac"],3), d["clocks"]["sm_mhz"], d["plan"], d["gpu_launches"])
PY
}
run c3 off SHIFTK_CSR_BLOCKED=0
run c3 b22 X=1
run c3 b21 SHIFTK_CSR_BSHIFT=21
run c3 b23 SHIFTK_CSR_BSHIFT=23
run c4 auto X=1
run c4 forced SHIFTK_CSR_BLOCKED=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:csr_" -s 8 -c 4 python bench.py --config c3 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "csr_|duration|bytes"
timeout 1200 python bench.py > gpurun_out/bench_c5_default.json 2> gpurun_out/bench_c5_default.err; echo "c5 default rc=$?"; tail -c 1500 gpurun_out/bench_c5_default.json
