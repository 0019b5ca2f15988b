"""Summarise an ncu source page (--page source --csv --print-source sass): stall reasons per instruction."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    tot = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data) or 1.0
    ins = sum(f(d["Instructions Executed"]) for d in data)
    print(f"kernel: {rows[0][1] if len(rows[0]) > 1 else ''}\nsamples {tot:.0f}  warp-instructions executed {ins:.0f}")
    stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    agg = sorted(((sum(f(d[k]) for d in data), k) for k in stalls), reverse=True)[:8]
    print("stalls:", ", ".join(f"{k} {v / tot * 100:.1f}%" for v, k in agg))
    for d in sorted(data, key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))[:top]:
        st = sorted(((f(d[k]), k) for k in stalls), reverse=True)[:2]
        print(f'{f(d["Warp Stall Sampling (All Samples)"]) / tot * 100:5.1f}% ex={f(d["Instructions Executed"]):9.0f} '
              f'{d["Source"][:56]:56s} {[(k[6:], int(v)) for v, k in st]}')


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
