cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:heisenberg_tiled" -s 2 -c 1 -o gpurun_out/ncu_c5_split -f python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c5_split.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_c5_split.log
