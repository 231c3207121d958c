#!/bin/bash
# Round-2 evidence run: bench lines (70B headline with CPU baseline, 7B, configs[0] 4096^2, batch 16,
# prefill batch 512, 3/4-bit), the reference arm, launch list, ncu --set full of the dominant K2 and of K4.
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
for w in 7b 4096; do timeout 300 python bench.py --no-cpu --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err; done
timeout 300 python bench.py --no-cpu --batch 16 > $OUT/bench_b16.json 2> $OUT/bench_b16.err
timeout 300 python bench.py --no-cpu --batch 512 --steps 10 > $OUT/bench_b512.json 2> $OUT/bench_b512.err
timeout 300 python bench.py --no-cpu --workload 7b --bits 3 > $OUT/bench_7b_3bit.json 2> $OUT/bench_7b_3bit.err
timeout 300 python bench.py --no-cpu --workload 7b --bits 4 > $OUT/bench_7b_4bit.json 2> $OUT/bench_7b_4bit.err
timeout 300 python bench.py --no-cpu --sharded > $OUT/bench_sharded_push.json 2> $OUT/bench_sharded_push.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-graph --copies 2 > $OUT/ncu_launch_bench.log 2>&1
SHAPES=28672x8192 NO_TRACE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_tc -s 4 -c 1 \
  -o $OUT/k2_full python tools/k2_timeline.py > $OUT/ncu_k2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 1 -c 1 \
  -o $OUT/k4_full python tools/prefill_one.py > $OUT/ncu_k4.log 2>&1
python tools/ncu_summary.py $OUT/k2_full.ncu-rep 30 > $OUT/k2_summary.txt 2>&1
python tools/ncu_summary.py $OUT/k4_full.ncu-rep 30 > $OUT/k4_summary.txt 2>&1
ncu -i $OUT/k2_full.ncu-rep --page raw --csv > $OUT/k2_raw.csv 2>/dev/null
ncu -i $OUT/k4_full.ncu-rep --page raw --csv > $OUT/k4_raw.csv 2>/dev/null
tail -c 400 $OUT/bench.json; echo; head -12 $OUT/k2_summary.txt
