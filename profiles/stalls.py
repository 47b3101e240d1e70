"""Top SASS stall locations from `ncu -i REP --page source --csv --print-source sass` output."""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    hdr = rows[hi]
    ci, si = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    data = []
    for r in rows[hi + 1:]:
        if len(r) > max(ci, si):
            try:
                data.append((int(float(r[ci] or 0)), r[si]))
            except ValueError:
                pass
    tot = sum(v for v, _ in data) or 1
    for v, s in sorted(data, key=lambda x: -x[0])[:top]:
        print(f"{v:7d} {100 * v / tot:5.1f}%  {s[:120]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
