# Round-2 ncu launch lists (duration + DRAM bytes per launch) of the C2 / C3 / C4 / C5sz benches;
# summarised into profiles/r02/ncu_configs_summary.json by tests/tools/ncu_summary.py.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for C in c2 c3 c4 c5sz; do
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/launches_$C.csv python bench.py --config $C --steps 10 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e > $O/ncu_launch_$C.log 2>&1; echo "$C launches rc=$?"
done
