cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ipc_two_process.py -x -q > gpurun_out/pytest_ipc.log 2>&1; echo "ipc rc=$?"; tail -15 gpurun_out/pytest_ipc.log
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -q --durations=20 > gpurun_out/pytest_san.log 2>&1; echo "san rc=$?"; tail -40 gpurun_out/pytest_san.log
