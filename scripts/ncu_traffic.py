"""Summarise an `ncu --set full` report: per kernel, duration and DRAM traffic
(dram__bytes_read.sum + dram__bytes_write.sum) per launch, plus the key pipe/throughput
metrics; merges the traffic into profiles/traffic.json (read by bench.py).
usage: python scripts/ncu_traffic.py report.ncu-rep [summary.txt]"""
import csv
import io
import json
import os
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def short(name):
    m = re.search(r"(\w+_kernel(?:<[^(]*>)?)", name)
    s = m.group(1) if m else name[:60]
    return s.replace("(int)", "").replace("(bool)", "")


def main(rep, out_txt=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines, traffic = [], {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = short(d.get("Kernel Name", "?"))
        vals = {}
        for key in KEYS:
            if key in d and d[key] not in ("", "n/a"):
                v = float(d[key].replace(",", ""))
                vals[key] = v * UNIT.get(u.get(key, ""), 1.0) if key.startswith("dram__bytes") else v
        tb = vals.get("dram__bytes_read.sum", 0) + vals.get("dram__bytes_write.sum", 0)
        base = k.split("<")[0] if k.startswith("sketch_tc") else k
        traffic[base] = {"bytes_per_launch": tb, "duration": vals.get("gpu__time_duration.sum"), "report": os.path.basename(rep)}
        lines.append(f"{k}: " + ", ".join(f"{kk.split('.')[0]}={vals[kk]:.4g}" for kk in vals) + f", traffic_bytes={tb:.4g}")
    text = "\n".join(lines)
    print(text)
    if out_txt:
        with open(out_txt, "w") as f:
            f.write(f"# {rep} (ncu --set full --clock-control none; durations are ncu replay times)\n" + text + "\n")
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    old = {}
    if os.path.exists(path):
        old = json.load(open(path))
    old.update(traffic)
    json.dump(old, open(path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
