#!/bin/bash
# ncu --set full of one K2 launch (28672x8192 layer) with source; usage: gpu_ncu.sh TAG [kernel-regex] [skip]
TAG=${1:-ncu}; KR=${2:-gemv_tc}; SK=${3:-1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$KR" -s $SK -c 1 \
  -o $OUT/k2_full python bench.py --steps 2 --warmup 3 --no-cpu --no-graph > $OUT/ncu_full.log 2>&1
tail -2 $OUT/ncu_full.log
