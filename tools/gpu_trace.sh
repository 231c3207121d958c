#!/bin/bash
# Build with K2 timeline stamps (+ extra NVEXTRA flags in $1), dump CTA 0's timeline, into gpurun_out/${2:-trace}.
make -s -C paper_2402_04396_b200/csrc clean >/dev/null; make -s -j8 -C paper_2402_04396_b200/csrc NVEXTRA="-DQ8P_K2_TRACE $1" >/dev/null 2>&1
rm -rf gpurun_out/trace; python tools/trace_k2.py; SHAPE=8192x8192 python tools/trace_k2.py
[ -n "$2" ] && rm -rf gpurun_out/$2 && mv gpurun_out/trace gpurun_out/$2
exit 0
