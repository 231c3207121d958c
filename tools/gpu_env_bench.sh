#!/bin/bash
# Run the bench under different env settings (args: "VAR=val VAR2=val" strings, "-" = none).
for v in "$@"; do
  echo "== $v"
  if [ "$v" = "-" ]; then v=""; fi
  env $v timeout 300 python bench.py --no-cpu $BENCH_ARGS 2>/tmp/bench_env.err | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline'] or {}
    print('value', round(d['value']), 'tok/s  step', round(d['ms_per_step']*1e3,1), 'us  e2e', round(d['e2e']['value']), ' K2', [round(p['us'],1) for p in r.get('per_layer',[])])
except Exception as e:
    print('failed', e); print(open('/tmp/bench_env.err').read()[-500:])
"
done
