"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list (serialised,
cold-cache device times).  python profiles/launch_summary.py launches.csv [steps]"""
import collections
import csv
import sys


def main(path, steps=2):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0][:90]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | ms/step | launches/step | us/launch | share |\n|---|---|---|---|---|")
    for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if v / tot < 0.0005:
            continue
        print(f"| `{k}` | {v / 1e6 / steps:.3f} | {n / steps:g} | {v / n / 1e3:.1f} | "
              f"{100 * v / tot:.1f}% |")
    print(f"| total | {tot / 1e6 / steps:.3f} | | | |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2)
