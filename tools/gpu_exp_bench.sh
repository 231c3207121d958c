#!/bin/bash
# Build variants (NVEXTRA flags as args, "-" = none) and report the bench line's value / per-layer K2.
# BENCH_ARGS env: extra bench.py flags.
for v in "$@"; do
  f=$v; [ "$f" = "-" ] && f=""
  make -s -C paper_2402_04396_b200/csrc clean >/dev/null; make -s -j8 -C paper_2402_04396_b200/csrc NVEXTRA="$f" >/dev/null 2>&1
  echo "== $v $BENCH_ARGS"
  timeout 300 python bench.py --no-cpu $BENCH_ARGS 2>/tmp/bench_exp.err | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline'] or {}
    print('value', round(d['value']), 'tok/s  step', round(d['ms_per_step']*1e3,1), 'us  e2e', round(d['e2e']['value']), ' K2', [round(p['us'],1) for p in r.get('per_layer',[])])
except Exception as e:
    print('failed', e)
"
done
