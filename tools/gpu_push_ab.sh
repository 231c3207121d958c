#!/bin/bash
# sharded N=1 step: push vs nccl (world 1: the NCCL path skips the identity gather)
for ag in push nccl; do
  timeout 300 python bench.py --no-cpu --sharded --allgather $ag --steps 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$ag', round(d['ms_per_step']*1e3,1), 'us', 'e2e', round(d['e2e']['value']), d['config'].get('allgather'))"
done
