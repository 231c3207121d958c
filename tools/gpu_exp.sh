#!/bin/bash
# Build variants (NVEXTRA flags given as args, "-" = none); K2 kernel duration by ncu (median over launches).
for v in "$@"; do
  f=$v; [ "$f" = "-" ] && f=""
  make -s -C paper_2402_04396_b200/csrc clean >/dev/null; make -s -j8 -C paper_2402_04396_b200/csrc NVEXTRA="$f" >/dev/null 2>&1
  echo "== $v"
  for sh in 28672x8192 8192x8192; do
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemv_tc --csv \
      python tools/k2_time.py $sh > /tmp/ncu_exp.csv 2>/dev/null
    python - "$sh" <<'PY'
import csv, statistics, sys
v = [float(r[-1]) for r in csv.reader(open('/tmp/ncu_exp.csv')) if len(r) > 5 and r[-3] == 'gpu__time_duration.sum']
m, n = (int(x) for x in sys.argv[1].split('x'))
b = m * n // 4 + 4 * (m + n)
if v:
    t = statistics.median(v) / 1e3
    print(f"{sys.argv[1]}: ncu K2 median {t:.2f} us over {len(v)} launches -> {b / t / 1e3:.0f} GB/s")
PY
  done
done
