#!/bin/bash
# quick bench line summary (no CPU): value, e2e, K2 chained/isolated per layer, stream ceiling
TAG=${1:-bq}; shift
mkdir -p gpurun_out/$TAG
timeout 600 python bench.py --no-cpu --steps 20 "$@" > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err; tail -2 gpurun_out/$TAG/bench.err
python - gpurun_out/$TAG/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d.get("roofline") or {}
print("value", round(d["value"]), "e2e", round(d["e2e"]["value"]), "us/step", round(d["ms_per_step"]*1e3,1), "frac", round(r.get("frac",0),3))
for p in r.get("per_layer",[]): print(p["layer"], "chained", round(p["us"],2), "iso", round(p["isolated_us"] or 0,2), "GB/s", round(p["gbs"]), "ceil_us", round((p.get("stream_ceiling") or {}).get("us",0),2))
PY
