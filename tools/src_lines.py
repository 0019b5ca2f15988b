"""Per-CUDA-source-line stall samples from `ncu --page source --csv --print-source sass,cuda`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out, fname, h = [], None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        h = r
    elif h and len(r) == len(h) and r[0].isdigit():
        try:
            s = float(r[4]); e = float(r[7] or 0)
        except ValueError:
            continue
        if s > 0:
            out.append((s, e, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot = sum(o[0] for o in out) or 1
for s, e, loc, src in sorted(out, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% ex={e:11.0f} {loc:18s} {src}")
