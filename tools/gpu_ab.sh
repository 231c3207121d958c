#!/bin/bash
# A/B of the two K2 kernels: GPU parity tests with the default, then the bench line for each.
TAG=${1:-ab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -5 $OUT/pytest_gpu.log
for k in mma tc; do
  Q8P_K2=$k timeout 300 python bench.py --no-cpu > $OUT/bench_$k.json 2> $OUT/bench_$k.err; tail -2 $OUT/bench_$k.err
  python - <<'PY' $OUT/bench_$k.json $k
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(sys.argv[2], 'value tok/s', round(d['value']), 'e2e', round(d['e2e']['value']), 'ms/step', round(d['ms_per_step']*1e3,1),'us',
 'K2 frac', round(r.get('frac',0),3), [(p['layer'], round(p['us'],1), round(p['gbs'])) for p in r.get('per_layer',[])])
PY
done
exit 0
