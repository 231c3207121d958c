#!/bin/bash
# compute-sanitizer memcheck + initcheck over tools/sanitize_small.py
TAG=${1:-san}
mkdir -p gpurun_out/$TAG
for tool in memcheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/$TAG/sanitizer_$tool.log 2>&1
  tail -3 gpurun_out/$TAG/sanitizer_$tool.log
done
