"""Top sampled SASS instructions of an `ncu --page source --csv` export, with the
dominant stall reasons, plus region totals between BAR / SYNCS markers.
  python probes/ncu_source_top.py gpurun_out/ncu/cfg4_tile.source.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
body = [r for r in rows[2:] if len(r) >= len(hdr) - 2]
ix = {h: i for i, h in enumerate(hdr)}
S = ix["# Samples"]
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[S] or 0) for r in body)
print("total samples", tot, "instructions", len(body))


def stalls(r):
    v = sorted(((int(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
    return " ".join(f"{n}:{c}" for c, n in v if c)


order = sorted(range(len(body)), key=lambda k: -int(body[k][S] or 0))[:topn]
for k in sorted(order):
    r = body[k]
    print(f"{k:5d} {r[0][-5:]} {int(r[S] or 0):6d} {100.0 * int(r[S] or 0) / tot:5.1f}%  {r[1][:70]:70s} {stalls(r)}")
# cumulative samples per 50-instruction window
print("-- samples per region (between BAR.SYNC / SYNCS / EXIT markers)")
acc, start = 0, 0
for k, r in enumerate(body):
    acc += int(r[S] or 0)
    if any(m in r[1] for m in ("BAR.SYNC", "SYNCS.PHASECHK", "SYNCS.ARRIVE", "EXIT")):
        if acc:
            print(f"  [{start:5d}..{k:5d}] {acc:7d} {100.0 * acc / tot:5.1f}%  ends at {r[1][:50]}")
        acc, start = 0, k + 1
