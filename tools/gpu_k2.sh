#!/bin/bash
# K2 iteration: timeline of the warp-MMA kernel + bench line (no CPU), optional GPU tests.
TAG=${1:-k2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
Q8P_K2=mma python tools/k2_timeline.py 2>&1 | tail -9
Q8P_K2=mma timeout 300 python bench.py --no-cpu > $OUT/bench.json 2> $OUT/bench.err; tail -2 $OUT/bench.err
python - <<'PY' $OUT/bench.json
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print('value tok/s', round(d['value']), 'e2e', round(d['e2e']['value']), 'ms/step', round(d['ms_per_step']*1e3,1),'us',
 'K2 frac', round(r.get('frac',0),3), [(p['layer'], round(p['us'],1), round(p['gbs'])) for p in r.get('per_layer',[])])
PY
if [ -n "$2" ]; then Q8P_K2=mma timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 2>&1 | tail -3; fi
exit 0
