"""tools/launch_summary.py LAUNCHES.csv [TITLE]: per-kernel launch count, total and mean device time from an
`ncu --metrics gpu__time_duration.sum --csv` launch list, and the share of the per-SpMV kernels taken by the
tile kernel (partition-time kernels -- pack, col_degree, rebase, hot_slot, the transposition -- excluded)."""
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
acc = {}
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].split("<")[0].split("::")[-1]
    v = float(d["Metric Value"]) * (1e-6 if d["Metric Unit"] == "ns" else 1e-3 if d["Metric Unit"] == "us" else 1.0)
    n, t = acc.get(name, (0, 0.0))
    acc[name] = (n + 1, t + v)
tot = sum(t for _, t in acc.values())
if len(sys.argv) > 2:
    print("#", sys.argv[2])
print("# per-launch times are cold-cache and serialised by ncu; the SHARE is what counts")
for k, (n, t) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:30s} launches={n:4d} total_ms={t:9.3f} mean_ms={t / n:8.4f} share_of_all={t / tot:.3f}")
once = ("pack_kernel", "col_degree_kernel", "rebase_kernel", "hot_slot_kernel", "row_span_kernel")
per = {k: v for k, v in acc.items() if k not in once and not k.startswith("rs_") and k not in ("permute_kernel", "row_ptr_kernel", "expand_cols_kernel")}
pt = sum(t for _, t in per.values())
if "rows_kernel" in per and pt > 0:
    print(f"share of the per-SpMV kernel time taken by rows_kernel: {per['rows_kernel'][1] / pt:.3f}")
