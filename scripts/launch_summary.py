"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (per-kernel totals,
counts and shares).  usage: python scripts/launch_summary.py launches.csv [steps]"""
import collections
import csv
import sys


def main(path, steps=1):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = 1e-3 if d["Metric Unit"] == "ns" else (1.0 if d["Metric Unit"] == "us" else 1e3)
        k = d["Kernel Name"][:100]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    print(f"# {path}: {sum(v[0] for v in agg.values())} launches, {tot:.1f} us total (cold-cache, serialised)")
    print(f"{'total_us':>10} {'count':>6} {'avg_us':>9} {'share':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda t: -t[1][1]):
        print(f"{v[1]:10.1f} {v[0]:6d} {v[1] / v[0]:9.1f} {100 * v[1] / tot:5.1f}%  {k}")
    # the library's own kernels (rt::), per step: the shares to compare with bench.py's phases
    # (torch kernels above are the benchmark's data generation / e2e copies, outside the step)
    ours = {k: v for k, v in agg.items() if "rt::" in k}
    tot_ours = sum(v[1] for v in ours.values())
    print(f"\n# library kernels only, per step ({steps} steps in the capture): {tot_ours / steps:.1f} us/step")
    print(f"{'us/step':>10} {'n/step':>6} {'avg_us':>9} {'share':>6}  kernel")
    for k, v in sorted(ours.items(), key=lambda t: -t[1][1]):
        print(f"{v[1] / steps:10.1f} {v[0] / steps:6.1f} {v[1] / v[0]:9.1f} {100 * v[1] / tot_ours:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
