cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; nvidia-smi) > gpurun_out/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=30 > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 600 python bench.py --config c2 --steps 200 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -3 gpurun_out/pytest.log
