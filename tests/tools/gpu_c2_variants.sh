cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for V in "" "SHIFTK_HEIS_SPLIT=1"; do
env $V timeout 900 python bench.py --config c2 --steps 200 --repeats 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_v.json 2> gpurun_out/bench_c2_v.err
python - <<PY
import json; d=json.loads(open("gpurun_out/bench_c2_v.json").read().strip().splitlines()[-1]); print("$V", round(d["ms_per_step"]*1e3,2), "us", {k: round(v*1e3,2) for k,v in d["kernel_ms_per_step"].items()}, d["plan"], d["passes_ms"])
PY
done
