#!/bin/bash
# sharded bench at N=1: push vs nccl, plus the push launch list
TAG=${1:-sh}
mkdir -p gpurun_out/$TAG
for ag in push nccl; do
  timeout 500 python bench.py --no-cpu --sharded --allgather $ag --steps 20 > gpurun_out/$TAG/$ag.json 2>gpurun_out/$TAG/$ag.err; tail -2 gpurun_out/$TAG/$ag.err
done
python - gpurun_out/$TAG <<'PY'
import json,sys,os
for f in ['push','nccl']:
    d=json.loads(open(os.path.join(sys.argv[1],f+'.json')).read().strip().splitlines()[-1]); print(f, round(d['value']), round(d['ms_per_step']*1e3,1),'us', 'e2e', round(d['e2e']['value']))
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/launches.csv \
  python bench.py --no-cpu --sharded --no-graph --steps 1 --warmup 1 --copies 1 > /dev/null 2>&1
