"""Per-rank kernel times of the N-rank sharded slot, measured on ONE GPU: the
workload is sharded over N emulated ranks (qpk_multi_create_emulated:
host-mediated collectives) and solved for a few iterations; run under
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file out.csv \
      python probes/emulated_ranks.py cfg4 8 12
the launch list gives every slot kernel's duration on a 1/N shard (ncu
serialises launches, so ranks do not disturb each other).  Summarise with
  python probes/emulated_ranks.py --summarise out.csv N
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def run(name, ranks, iters):
    import numpy as np
    import bench
    from paper_2308_00637_b200.direction import MultiGpuKkt
    problem, op, rhs, meta = bench.make_workload(name, 1.0)
    mk = MultiGpuKkt(problem, op.bmap, devices=[0], emulate_ranks=ranks)
    mk.set_diagonals(op.d_diag, op.q_diag_extra)
    x, info, _ = mk.pcg(rhs, 1e-300, iters, True)
    fmt = [(mk.ctx.query("scatter", r), mk.ctx.query("hess_tiled", r), mk.ctx.query("row_hi", r) - mk.ctx.query("row_lo", r))
           for r in range(ranks)]
    print("ranks", ranks, "iterations", info.iterations, "per-rank (format, H tiles, rows):", fmt, flush=True)
    mk.close()


def summarise(path, ranks):
    import csv
    import io
    import json
    from collections import defaultdict
    text = Path(path).read_text()
    rows = list(csv.DictReader(io.StringIO(text[text.find('"ID"'):])))
    per = defaultdict(list)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1.0)
        per[r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").strip()].append(v)
    # the host replays slots in chunks of 16: launches past the last iteration exit at once
    # (mode DONE); "active" = the launches within 2x of the longest one's half
    out = {}
    for k, v in per.items():
        act = [t for t in v if t >= 0.5 * max(v)]
        out[k] = {"launches": len(v), "active": len(act), "us_active_mean": sum(act) / len(act), "us_max": max(v)}
    print(json.dumps({"ranks": ranks, "kernels": out}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "--summarise":
        summarise(sys.argv[2], int(sys.argv[3]))
    else:
        run(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 12)
