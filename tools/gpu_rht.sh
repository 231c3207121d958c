#!/bin/bash
# prefill accuracy/timing + per-kernel launch times of one 28672x8192 b512 forward
TAG=${1:-rht}
mkdir -p gpurun_out/$TAG
timeout 600 python tools/prefill_check.py 2>&1 | tail -12
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/launches.csv \
  python tools/prefill_one.py > /dev/null 2>&1
python - gpurun_out/$TAG/launches.csv <<'PY'
import csv,sys,collections
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value"); idi=h.index("ID")
ks=[(r[ki][:60], float(r[vi])) for r in rows[1:]]
n=len(ks)//3
for k,v in ks[-n:]: print(f"{v/1000:9.1f} us  {k}")
PY
