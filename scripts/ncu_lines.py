"""Samples and instruction counts per CUDA source line from an ncu capture (needs -lineinfo).
usage: ncu_lines.py report.ncu-rep [min_pct]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
mp = float(sys.argv[2]) if len(sys.argv) > 2 else 0.7
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]; data = rows[hi + 1:]
iS = h.index("# Samples"); iI = h.index("Instructions Executed")
stalls = [(i, k) for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
per = {}
for r in data:
    if len(r) < len(h) or not r[0].isdigit():
        continue  # SASS rows; line rows carry the per-line aggregates
    key = (int(r[0]), r[1].strip()[:70])
    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0
    e = per.setdefault(key, [0, 0, {}])
    e[0] += num(r[iS]); e[1] += num(r[iI])
    for i, k in stalls:
        e[2][k] = e[2].get(k, 0) + num(r[i])
tot = sum(v[0] for v in per.values())
print("total samples", tot)
for (ln, src), (s, n, st) in sorted(per.items()):
    if 100 * s >= mp * tot:
        top = sorted(((v, k[6:]) for k, v in st.items()), reverse=True)[:2]
        print(f"{ln:5d} {100 * s / tot:5.1f}% inst={n:8d} {src:70s} {top}")
