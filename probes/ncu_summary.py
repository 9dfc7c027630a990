"""Summarise one `ncu --set full` capture (first kernel in the report) into the
JSON kept under profiles/: duration, DRAM bytes and throughput, L2 / SM
throughput, occupancy, registers and the dominant warp-stall reasons.
  python probes/ncu_summary.py gpurun_out/full_cfg2.ncu-rep "note" > profiles/<name>.json
"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
get = lambda k: (vals[hdr.index(k)] + " " + units[hdr.index(k)]).strip() if k in hdr else None
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic"]
out = {k: get(k) for k in keys if get(k) is not None}
stalls = {}
for i, h in enumerate(hdr):
    if h.startswith("smsp__average_warp_latency_issue_stalled_") or (
            h.startswith("smsp__warp_issue_stalled_") and h.endswith("_per_warp_active.pct")):
        try:
            stalls[h] = float(vals[i])
        except ValueError:
            pass
out["top_stalls_pct_of_active_warps"] = dict(sorted(((k.replace("smsp__warp_issue_stalled_", "").replace(
    "_per_warp_active.pct", ""), round(v, 1)) for k, v in stalls.items() if k.endswith(".pct")),
    key=lambda kv: -kv[1])[:6])
out["source"] = f"ncu --set full --import-source on --clock-control none (-k <kernel> -s 5 -c 1) {rep.split('/')[-1]}"
if len(sys.argv) > 2:
    out["note"] = sys.argv[2]
print(json.dumps(out, indent=1))
