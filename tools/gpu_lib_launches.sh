#!/bin/bash
# per-kernel ncu durations of one eager batch-1 step (3 layers): default lib vs $1
mkdir -p gpurun_out/ll
for lib in "" "$@"; do
  tag=$(basename "${lib:-default}" .so)
  Q8P_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll/$tag.csv \
    python bench.py --no-cpu --no-graph --steps 2 --warmup 3 --copies 1 > /dev/null 2>&1
done
