cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for LIB in "" _var/libshiftk_nb4.so _var/libshiftk_nb6.so; do
SHIFTK_LIB=$LIB timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed --clock-control none -k "regex:heisenberg_tiled" -s 2 -c 1 python bench.py --config c5 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "duration|inst_executed|wavefronts" | sed "s#^#$LIB #"
done
