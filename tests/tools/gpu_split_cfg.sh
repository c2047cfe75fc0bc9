cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for C in 512 512s2 256s3 256s2 1024s1; do
SHIFTK_SPLIT_CFG=$C timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_cfg_$C.json 2> gpurun_out/bench_c5_cfg_$C.err
python - <<PY
import json; d=json.loads(open("gpurun_out/bench_c5_cfg_$C.json").read().strip().splitlines()[-1]); print("cfg=$C", round(d["ms_per_step"],3), {k: round(v,3) for k,v in d["kernel_ms_per_step"].items()}, round(d["iteration_gbs_model_frac"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
