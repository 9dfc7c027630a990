"""Summarise the CSV exports of probes/ncu_full.sh (raw metrics + source page)
into the JSON kept under profiles/.
  python probes/ncu_raw_summary.py gpurun_out/ncu/<tag> "note" > profiles/<name>.json"""
import csv
import json
import sys

tag = sys.argv[1]
rows = list(csv.reader(open(tag + ".raw.csv")))
hdr, units, vals = rows[0], rows[1], rows[2]
get = lambda k: (vals[hdr.index(k)] + " " + units[hdr.index(k)]).strip() if k in hdr else None
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic"]
out = {k: get(k) for k in keys if get(k) is not None}
try:
    src = list(csv.reader(open(tag + ".source.csv")))
    h = src[1]
    body = [r for r in src[2:] if len(r) >= len(h) - 2]
    S = h.index("# Samples")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(int(r[S] or 0) for r in body)
    agg = {}
    for r in body:
        for i in stall_cols:
            agg[h[i][6:]] = agg.get(h[i][6:], 0) + int(r[i] or 0)
    out["warp_samples"] = tot
    out["stall_samples_top"] = dict(sorted(agg.items(), key=lambda kv: -kv[1])[:8])
    hot = sorted(body, key=lambda r: -int(r[S] or 0))[:8]
    out["hottest_instructions"] = [{"sass": r[1].strip()[:60], "samples": int(r[S] or 0)} for r in hot]
except FileNotFoundError:
    pass
out["source"] = "ncu --set full --import-source on --clock-control none -k <kernel> -c 1 (probes/ncu_full.sh), exported on the box"
if len(sys.argv) > 2:
    out["note"] = sys.argv[2]
print(json.dumps(out, indent=1))
