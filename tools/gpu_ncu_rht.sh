#!/bin/bash
# ncu --set full of the prefill K3 passes (28672x8192 b512 forward)
TAG=${1:-ncu_rht}
mkdir -p gpurun_out/$TAG
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KRE:-rht_pass} -c ${KC:-4} \
  -o gpurun_out/$TAG/rht python tools/prefill_one.py > gpurun_out/$TAG/ncu.log 2>&1
tail -3 gpurun_out/$TAG/ncu.log
