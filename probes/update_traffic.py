"""Merge ncu launch-list summaries (gpurun_out/t_<w>.csv) into profiles/traffic.json:
  python probes/update_traffic.py cfg4 [cfg3 ...]   (200 PCG iterations per bench step)"""
import json
import subprocess
import sys

t = json.load(open("profiles/traffic.json"))
for w in sys.argv[1:]:
    out = subprocess.run([sys.executable, "probes/ncu_traffic.py", f"gpurun_out/t_{w}.csv", w, "--iters", "200"],
                         capture_output=True, text=True, check=True).stdout
    t[w] = json.loads(out)
json.dump(t, open("profiles/traffic.json", "w"), indent=1)
