#!/bin/bash
# K4 A/B: the in-tree build, then a sed-edited variant ($1 = sed expression on gemm_prefill.cu) rebuilt on the box.
mkdir -p gpurun_out/k4ab
run() {
  [ -n "$PROBE" ] && timeout 150 python tools/dbg_k4_repeat.py 2>&1 | tail -5
  timeout 300 python bench.py --no-cpu --batch 512 --steps 10 > gpurun_out/k4ab/b.json 2>/dev/null
  python - gpurun_out/k4ab/b.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d["roofline"]
print("b512 tok/s", round(d["value"]), "ms", round(d["ms_per_step"]*1e3,1), "frac", round(r["frac"],3), [(p["layer"], round(p["us"],1), round(p["tflops"])) for p in r["per_layer"]])
PY
}
echo "== in-tree"; run
sed -i "$1" paper_2402_04396_b200/csrc/gemm_prefill.cu
make -s -j16 -C paper_2402_04396_b200/csrc >/dev/null 2>&1 || echo BUILD FAILED
echo "== variant: $1"; run
