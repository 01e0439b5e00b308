#!/bin/bash
# development iteration on the GPU: sweep-kernel timings, bit-identity against round 1, and (when
# scripts/_prof/libspmesl.so exists) the sweep kernel's per-phase counters
mkdir -p gpurun_out
timeout 300 python scripts/sweep_timing.py > gpurun_out/timing.log 2>&1; echo "timing rc=$?"; cat gpurun_out/timing.log
timeout 400 python scripts/compare_r1.py > gpurun_out/cmp.log 2>&1; echo "cmp rc=$?"; grep -c "True, True, True, True" gpurun_out/cmp.log; grep -v "True, True, True, True\|declined" gpurun_out/cmp.log | tail -5
if [ -f scripts/_prof/libspmesl.so ]; then timeout 300 python scripts/tail_prof_run.py band3 hub 2>&1; fi
