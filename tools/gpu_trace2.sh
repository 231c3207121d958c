#!/bin/bash
make -s -C paper_2402_04396_b200/csrc clean >/dev/null; make -s -j8 -C paper_2402_04396_b200/csrc NVEXTRA="-DQ8P_K2_TRACE -DQ8P_K2_TRACE_SYNC $1" >/dev/null 2>&1
rm -rf gpurun_out/trace; python tools/trace_k2.py
