#!/bin/bash
# A/B on one box: the in-tree build, then a sed-edited variant ($1 = file, $2 = sed expression) rebuilt on the box.
# Prints the batch-$3 bench line of each (default 512).
B=${3:-512}
run() {
  timeout 300 python bench.py --no-cpu --batch $B --steps 10 > /tmp/ab.json 2>/dev/null
  python - /tmp/ab.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d.get("roofline") or {}
print("tok/s", round(d["value"]), "e2e", round(d["e2e"]["value"]), "ms", round(d["ms_per_step"]*1e3,1), [(p["layer"], round(p["us"],1)) for p in r.get("per_layer",[])])
PY
}
echo "== in-tree"; run
sed -i "$2" "$1"
make -s -j16 -C paper_2402_04396_b200/csrc >/dev/null 2>&1 || echo BUILD FAILED
echo "== variant"; run
echo "== in-tree again needs rebuild; variant again"; run
