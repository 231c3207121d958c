#!/bin/bash
# ncu --set full of K4 (28672x8192 b512 forward)
TAG=${1:-ncu_k4}
mkdir -p gpurun_out/$TAG
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -c 1 \
  -o gpurun_out/$TAG/k4 python tools/prefill_one.py > gpurun_out/$TAG/ncu.log 2>&1
tail -2 gpurun_out/$TAG/ncu.log
