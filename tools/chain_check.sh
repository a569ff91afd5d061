#!/bin/bash
# GPU check of the flag-ordered chain: tests, timeline, small-domain timings
rm -f gpurun_out/pt_chain.log gpurun_out/trace_flags.log gpurun_out/small_timing.log
timeout 600 python -m pytest tests/test_gpu_chain.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/pt_chain.log
LBW_LIB=/root/repo/build/liblbw_trace.so timeout 200 python tools/trace_timeline.py 64 fast > gpurun_out/trace_flags.log 2>&1
timeout 300 python tools/small_timing.py ${SIZES:-64 128} > gpurun_out/small_timing.log 2>&1
