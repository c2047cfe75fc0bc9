# Round-2 measurements: bench lines, whole-convergence lines, ncu launch list + full captures.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi > $O/nvidia_smi.txt 2>&1
timeout 1200 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --config c2 --steps 200 > $O/bench_c2.json 2> $O/bench_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --config c1 --converge > $O/converge_c1.json 2> $O/converge_c1.err; echo "c1conv rc=$?"
timeout 1200 python bench.py --config c2 --converge > $O/converge_c2.json 2> $O/converge_c2.err; echo "c2conv rc=$?"
timeout 1200 python bench.py --config c3 --steps 10 > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
timeout 1200 python bench.py --config c4 --steps 10 > $O/bench_c4.json 2> $O/bench_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --config c5sz --steps 50 > $O/bench_c5sz.json 2> $O/bench_c5sz.err; echo "c5sz rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv python bench.py --steps 20 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:heisenberg_tiled|update_split" -s 4 -c 2 -o $O/ncu_c5_full -f python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1; echo "full rc=$?"
for f in $O/*.json; do echo "== $f"; tail -c 600 $f; echo; done
