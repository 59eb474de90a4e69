"""Per-source-line summary of an ncu report's source page (warp-state samples
and executed warp instructions), top lines first.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_source.py src.csv [top]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    cur, hdr, agg = None, None, {}
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "":   # SASS rows repeat their source line's totals
            continue
        d = dict(zip(hdr, r))
        try:
            smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            ins = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        a = agg.setdefault((cur, r[0]), [0, 0, r[1].strip()[:100]])
        a[0] += smp
        a[1] += ins
    tot = max(1, sum(v[0] for v in agg.values()))
    toti = max(1, sum(v[1] for v in agg.values()))
    print(f"samples {tot}  warp instructions {toti}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{v[0]:6d} {100 * v[0] / tot:5.1f}%  {100 * v[1] / toti:5.1f}%i  {k[0]}:{k[1]}  {v[2]}")


if __name__ == "__main__":
    main()
