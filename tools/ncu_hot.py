"""Summarise an `ncu --page source --csv --print-source sass` dump: the hottest
SASS instructions by warp-stall samples with their dominant stall reasons."""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
    si = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    tot = sum(float(r[si] or 0) for r in data)
    data.sort(key=lambda r: -float(r[si] or 0))
    print(f"total samples {tot:.0f}")
    for r in data[:top]:
        n = float(r[si] or 0)
        reasons = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
        rs = ", ".join(f"{k}={v:.0f}" for v, k in reasons if v)
        print(f"{100 * n / tot:5.1f}%  {r[1].strip()[:60]:60s} {rs}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
