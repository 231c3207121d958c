#!/bin/bash
# One GPU round-trip: parity tests, smoke, bench, launch list, ncu full capture of K2.
# Usage (from this container): gpurun --timeout 1500 -- 'bash tools/gpu_check.sh TAG'
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
cp MEASURED_PEAKS.json $OUT/ 2>/dev/null
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python bench.py --workload 7b --no-cpu > $OUT/bench7b.json 2> $OUT/bench7b.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-graph > $OUT/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_tc -s 6 -c 3 \
  -o $OUT/k2_full python bench.py --steps 2 --warmup 3 --no-cpu --no-graph > $OUT/ncu_full.log 2>&1
tail -3 $OUT/pytest_gpu.log
cat $OUT/smoke.log | tail -2
cat $OUT/bench.json
