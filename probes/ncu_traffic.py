"""Summarise an ncu metrics CSV (dram bytes + duration per launch) into the
per-workload DRAM-traffic record bench.py reports as roofline.traffic.

Capture (GPU box, one GPU; numbers taken under ncu are never bench values):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -s SKIP -c COUNT --csv --log-file gpurun_out/t_cfgK.csv \
      python bench.py --workload cfgK --steps 1 --warmup 3 --no-cpu-baseline
Summarise (here):
  python probes/ncu_traffic.py gpurun_out/t_cfgK.csv cfgK [--iters I]

Per kernel name: launches, mean dram bytes / duration per launch.  For the
slot engine (per-phase kernels) the per-PCG-iteration traffic is the sum of
the per-launch means of the slot kernels; the per-solve figure (the unit of
roofline.achieved) is that times the iteration count.  For the persistent
kernel (one launch = one solve) it is the launch's own bytes.
"""

from __future__ import annotations

import csv
import io
import json
import sys
from collections import defaultdict
from pathlib import Path

SLOT_KERNELS = ("k_slot_top", "k_slot_rows", "k_slot_csc", "k_slot_update", "k_slot_hess", "k_slot_hess_sym",
                "k_slot_dense", "k_comb_direct", "k_comb_seg",
                "k_comb_col", "k_slot_panel", "k_panel_comb")


def load(path: str):
    text = Path(path).read_text()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(lambda: defaultdict(dict))
    for r in rows:
        per[r["ID"]][r["Metric Name"]] = (r["Kernel Name"], r["Metric Unit"], r["Metric Value"])
    out = defaultdict(lambda: {"launches": 0, "read": 0.0, "write": 0.0, "ns": 0.0})
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3,
             "ms": 1e6, "msecond": 1e6, "nsecond": 1}
    for _, mets in per.items():
        name = next(iter(mets.values()))[0]
        k = out[name.split("(")[0].split("<")[0].replace("void ", "").strip()]
        k["launches"] += 1
        for met, (_, unit, val) in mets.items():
            v = float(val.replace(",", "")) * scale.get(unit, 1)
            if met == "dram__bytes_read.sum":
                k["read"] += v
            elif met == "dram__bytes_write.sum":
                k["write"] += v
            elif met == "gpu__time_duration.sum":
                k["ns"] += v
    return out


def main():
    path, workload = sys.argv[1], sys.argv[2]
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else None
    ks = load(path)
    summary = {}
    for name, k in ks.items():
        n = max(k["launches"], 1)
        summary[name] = {"launches": k["launches"], "dram_bytes_per_launch": (k["read"] + k["write"]) / n,
                         "dram_read_per_launch": k["read"] / n, "dram_write_per_launch": k["write"] / n,
                         "us_per_launch": k["ns"] / n / 1e3}
    rec = {"workload": workload, "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                                           f"gpu__time_duration.sum --clock-control none ({Path(path).name})",
           "kernels": summary}
    slot = [k for k in summary if k.startswith(SLOT_KERNELS)]
    if slot:
        per_iter = sum(summary[k]["dram_bytes_per_launch"] for k in slot)
        rec["dram_bytes_per_iter"] = per_iter
        rec["slot_kernels"] = slot
        if iters:
            rec["dram_bytes_per_launch"] = per_iter * (iters + 1)
            rec["unit_note"] = f"per solve = per-iteration slot traffic x ({iters} iterations + final apply)"
    else:
        pk = [k for k in summary if k.startswith("pcg_kernel")]
        if pk:
            rec["dram_bytes_per_launch"] = summary[pk[0]]["dram_bytes_per_launch"]
            rec["unit_note"] = "one persistent-kernel launch = one solve"
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()
