#!/bin/bash
# A/B of alternative library builds (exp_so/*.so, Q8P_LIB) on the batch-1 bench line
for lib in "" "$@"; do
  echo "== ${lib:-default}"
  Q8P_LIB=$lib timeout 300 python bench.py --no-cpu --steps 30 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d.get('roofline') or {}
print('us/step', round(d['ms_per_step']*1e3,1), 'e2e', round(d['e2e']['value']), 'frac', round(r.get('frac',0),3), [(p['layer'], round(p['us'],2), round(p['isolated_us'] or 0,2)) for p in r.get('per_layer',[])])"
done
