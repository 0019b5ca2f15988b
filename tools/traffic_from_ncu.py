"""Record per-launch DRAM traffic of one kernel from an `ncu --set full` report into
profiles/traffic.json (read by bench.py for roofline.traffic).

  python tools/traffic_from_ncu.py REPORT.ncu-rep WORKLOAD KERNEL_SUBSTRING
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, workload, kname = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
vals = []
for r in rows[2:]:
    d = dict(zip(h, r))
    if kname not in d.get("Kernel Name", ""):
        continue
    u = dict(zip(h, units))
    rd = float(d["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
    wr = float(d["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
    t = float(d["gpu__time_duration.sum"])
    vals.append((rd + wr, rd, wr, t, u["gpu__time_duration.sum"]))
if not vals:
    sys.exit(f"no launch of {kname} in {rep}")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
db[workload] = {"kernel": kname, "dram_bytes_per_launch": sum(v[0] for v in vals) / len(vals),
                "dram_read": vals[0][1], "dram_write": vals[0][2], "launches": len(vals),
                "ncu_duration": [v[3] for v in vals], "duration_unit": vals[0][4],
                "source": f"ncu --set full --clock-control none ({os.path.basename(rep)})"}
json.dump(db, open(path, "w"), indent=1, sort_keys=True)
print(workload, db[workload])
