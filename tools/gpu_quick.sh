#!/bin/bash
# Quick GPU iteration: parity tests + bench (no CPU baseline).
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 300 python bench.py --no-cpu > $OUT/bench.json 2> $OUT/bench.err; tail -2 $OUT/bench.err
python - <<'PY' $OUT/bench.json
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print('value tok/s', round(d['value']), 'e2e', round(d['e2e']['value']), 'ms/step', round(d['ms_per_step']*1e3,1),'us')
print('K2 frac', round(r.get('frac',0),3), [(p['layer'], round(p['us'],1), round(p['gbs'])) for p in r.get('per_layer',[])])
PY
[ -n "$2" ] && timeout 300 python bench.py --no-cpu --workload 7b > $OUT/bench7b.json 2>&1 && tail -c 600 $OUT/bench7b.json
exit 0
