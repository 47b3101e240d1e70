"""Summarise ncu evidence into profiles/ (committed):
  python profiles/summarize.py launches gpurun_out/launches_TAG.csv [--skip N] > profiles/TAG_launches.md
  python profiles/summarize.py full gpurun_out/prof_TAG.ncu-rep > profiles/TAG_full.md
The launch list is cold-cache and serialised: compare SHARES, not absolute times."""
import collections
import csv
import io
import re
import subprocess
import sys


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("<unnamed>::", "").replace("pgti::", "")
    return name[:70]


def launches(path, skip=0):
    rows = [l for l in open(path) if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(rows)))
    per = collections.OrderedDict()
    n = 0
    for r in rd:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        n += 1
        if n <= skip:
            continue
        k = short(r["Kernel Name"])
        t = float(r["Metric Value"]) / (1000.0 if r["Metric Unit"] == "ns" else 1.0)
        c, s = per.get(k, (0, 0.0))
        per[k] = (c + 1, s + t)
    tot = sum(s for _, s in per.values())
    print(f"# ncu launch list: {path}\n")
    print(f"{n - skip} launches, {tot / 1000:.3f} ms total device time (cold-cache, serialised)\n")
    print("| kernel | launches | total us | mean us | share |")
    print("|---|---|---|---|---|")
    for k, (c, s) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {c} | {s:.1f} | {s / c:.2f} | {100 * s / tot:.1f}% |")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "lts__t_bytes.sum",
           "l1tex__t_bytes.sum", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
           "sm__cycles_elapsed.avg.per_second"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        print("no data")
        return
    hdr = rows[0]
    idx = {m: hdr.index(m) for m in METRICS if m in hdr}
    kcol = hdr.index("Kernel Name")
    print(f"# ncu --set full: {path}\n")
    units = rows[1]
    print("| kernel | " + " | ".join(f"{m} [{units[i]}]" if units[i] else m
                                     for m, i in idx.items()) + " |")
    print("|---|" + "---|" * len(idx))
    for r in rows[2:]:
        if len(r) <= kcol:
            continue
        print(f"| `{short(r[kcol])}` | " + " | ".join(r[i] for i in idx.values()) + " |")


def traffic(path):
    """Mean DRAM bytes (read + write) per launch of each kernel class in an ncu --set full report
    (cold cache: ncu flushes caches before every replayed kernel) -> JSON for bench.py."""
    import json
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    k, rd, wr = (hdr.index(c) for c in ("Kernel Name", "dram__bytes_read.sum",
                                         "dram__bytes_write.sum"))
    per = collections.defaultdict(list)
    for r in rows[2:]:
        if len(r) > max(k, rd, wr):
            name = short(r[k])
            cls = ("spmm" if "spmm" in name else "gemm_wgrad" if "wgrad" in name
                   else "gemm" if "tc_fwd" in name else name)
            per[cls].append(float(r[rd]) + float(r[wr]))
    print(json.dumps({c: {"dram_bytes_per_launch": sum(v) / len(v), "launches": len(v),
                          "source": path.rsplit("/", 1)[-1]} for c, v in per.items()}, indent=1))


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    {"launches": lambda: launches(path, skip), "full": lambda: full(path),
     "traffic": lambda: traffic(path)}[mode]()
