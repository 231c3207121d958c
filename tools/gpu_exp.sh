#!/bin/bash
# Build variants (NVEXTRA flags given as args, "-" = none) and time K2 for each.
for v in "$@"; do
  f=$v; [ "$f" = "-" ] && f=""
  make -s -C paper_2402_04396_b200/csrc clean >/dev/null; make -s -j8 -C paper_2402_04396_b200/csrc NVEXTRA="$f" >/dev/null 2>&1
  echo "== $v"; timeout 120 python tools/k2_time.py 28672x8192 8192x8192
done
