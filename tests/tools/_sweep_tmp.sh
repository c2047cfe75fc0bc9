for d in 0 128 $((128|112)) $((128|112|6<<8)) $((128|112|11<<8)); do
  SHIFTK_SZ_DBG=$d ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:heisenberg_szb -s 1 -c 1 --csv python tests/tools/probe_sz.py 30 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' -v d=$d '{print d, $(NF-2), $(NF-1), $NF}'
done
SHIFTK_SZ_DBG=128 python tests/tools/probe_sz.py 26 28 30
python tests/tools/probe_sz.py 26 28 30
