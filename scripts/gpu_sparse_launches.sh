# Per-kernel launch list of the C5 bench (ncu, cold-cache serialised), last step's sparse kernels.
timeout 1000 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/sparse_launches.csv python bench.py --algo sparse --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-phases > gpurun_out/ncu_sparse.log 2>&1; echo rc=$?
python scripts/launch_summary.py gpurun_out/sparse_launches.csv 4 2>/dev/null | head -14
python - <<'PY'
import csv
hdr=None;data=[]
for r in csv.reader(open('gpurun_out/sparse_launches.csv')):
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
n=len([d for d in data if 'y_from_fixed' in d['Kernel Name']])//4
last=data[-len(data)//4:]
for d in last:
    if float(d['Metric Value'])>20000: print(d['Kernel Name'][:60], d['Metric Value'], d['Metric Unit'])
PY
