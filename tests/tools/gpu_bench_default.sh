cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
#timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "split" > gpurun_out/pytest_split.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_split.log
#
SECONDS=0; timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench s=$SECONDS"; tail -c 3000 gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
SECONDS=0; timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref s=$SECONDS"; tail -c 1500 gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
