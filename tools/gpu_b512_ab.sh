#!/bin/bash
# prefill batch-512 bench line (70B set): default lib vs alternatives (exp_so)
for lib in "" "$@"; do
  Q8P_LIB=$lib timeout 300 python bench.py --no-cpu --batch 512 --steps 10 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d.get('roofline') or {}
print('${lib:-default}', round(d['value']), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/step', 'K4 frac', round(r.get('frac',0),3), [(p['layer'], round(p['us'],1)) for p in r.get('per_layer',[])])"
done
