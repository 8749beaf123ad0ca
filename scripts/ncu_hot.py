"""Summarise an ncu --set full capture's source page: samples per 1 KB SASS region and the
hottest instructions with their top stall reasons.  usage: ncu_hot.py report.ncu-rep [N] [kernel-regex]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kf = sys.argv[3:] and ["--kernel-name", "regex:" + sys.argv[3]] or []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"] + kf, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "# Samples" in r)
h = rows[hi]; ci = {k: i for i, k in enumerate(h)}; data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0].startswith("0x")]
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(int(r[ci["# Samples"]]) for r in data)
print("total samples", tot, "warp insts", sum(int(r[ci["Instructions Executed"]]) for r in data))
acc = {}
for r in data:
    a = int(r[0], 16) >> 9
    e = acc.setdefault(a, [0, 0, r[1].strip()[:45], {}])
    e[0] += int(r[ci["# Samples"]]); e[1] += int(r[ci["Instructions Executed"]])
    for k in stalls:
        e[3][k] = e[3].get(k, 0) + int(r[ci[k]])
for a, (s, n, t, st) in sorted(acc.items()):
    if s * 100 >= tot:
        top = sorted(((v, k[6:]) for k, v in st.items()), reverse=True)[:3]
        print(f"{hex(a << 9)[-5:]} {100 * s / tot:5.1f}% inst={n:8d} {t:45s} {top}")
