#!/bin/bash
# ncu --set full of the K2 launches on the 70B MLP shape (one launch), summaries into gpurun_out/TAG.
TAG=${1:-ncu}
KREG=${2:-gemv_mma}
OUT=gpurun_out/$TAG
mkdir -p $OUT
SHAPES=28672x8192 Q8P_K2=mma timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KREG -s 4 -c 1 \
  -o $OUT/k2 python tools/k2_timeline.py > $OUT/ncu.log 2>&1
python tools/ncu_summary.py $OUT/k2.ncu-rep 30 > $OUT/summary.txt 2>&1
python tools/ncu_stalls.py $OUT/k2.ncu-rep > $OUT/stalls.txt 2>&1
head -16 $OUT/summary.txt; cat $OUT/stalls.txt
exit 0
