"""profiles/r02/ncu_dominant.json from gpurun_out/prof_c2.ncu-rep (tools/capture_roofline.sh):
per C2 cell-kernel launch, keyed like bench.py's per_degree entries, its DRAM bytes and the
pipe / stall summary (tools/ncu_summary.py)."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summarise  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "prof_c2.ncu-rep")
keys = open(os.path.join(ROOT, "gpurun_out", "roofline_order.txt")).read().split()
rows = summarise(rep)
assert len(rows) == len(keys), (len(rows), keys)
commit = subprocess.run(["git", "rev-parse", "--short=12", "HEAD"], capture_output=True, text=True, cwd=ROOT).stdout.strip()
for k, r in zip(keys, rows):
    r["key"] = k
out = {"what": "ncu --set full --clock-control none, one launch of each C2 cell kernel after a 256 MiB L2 flush "
               "(tools/capture_roofline.sh); dram_bytes_per_launch = dram__bytes_read.sum + dram__bytes_write.sum",
       "commit": commit, "kernels": rows}
os.makedirs(os.path.join(ROOT, "profiles", "r02"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", "r02", "ncu_dominant.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps([{k: r.get(k) for k in ("key", "kernel", "gpu__time_duration.sum", "dram_bytes_per_launch")} for r in rows], indent=1))
