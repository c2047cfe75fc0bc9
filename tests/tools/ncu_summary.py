"""Summarise ncu reports into profiles/: launch list (per-kernel mean duration + DRAM bytes)
and full-set captures (duration, DRAM bytes, throughput, occupancy, top stall reasons)."""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg[d["Kernel Name"].split("(")[0]][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
    out = {}
    for k, m in agg.items():
        out[k] = {mm: {"mean": sum(v) / len(v), "n": len(v)} for mm, v in m.items()}
    return out


def full(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        stalls = []
        for i, w in enumerate(hdr):
            if w.startswith("smsp__pcsamp_warps_issue_stalled_") and not w.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), w.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                "launch__grid_size", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
                "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                "lts__t_sectors.avg.pct_of_peak_sustained_elapsed"]
        e = {k: (d.get(k), units[hdr.index(k)] if k in hdr else None) for k in keys}
        e["top_stalls_pct"] = {w: round(100 * v / tot, 1) for v, w in sorted(stalls, reverse=True)[:6]}
        res.append(e)
    return res


if __name__ == "__main__":
    out = {}
    for a in sys.argv[2:]:
        if a.endswith(".csv"):
            out["launches:" + a.split("/")[-1]] = launches(a)
        else:
            out["full:" + a.split("/")[-1]] = full(a)
    json.dump(out, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(out, indent=1)[:3000])
