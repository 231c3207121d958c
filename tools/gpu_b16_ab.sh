#!/bin/bash
for lib in "" "$@"; do
  Q8P_LIB=$lib timeout 300 python bench.py --no-cpu --batch 16 --steps 20 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d.get('roofline') or {}
print('${lib:-default}', round(d['value']), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/step frac', round(r.get('frac',0),3), [(p['layer'], round(p['us'],2)) for p in r.get('per_layer',[])])"
done
