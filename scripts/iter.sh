#!/bin/bash
# development iteration on the GPU: sweep-kernel timings, bit-identity against round 1, parity subset
mkdir -p gpurun_out
python scripts/sweep_timing.py > gpurun_out/timing.log 2>&1; echo "timing rc=$?"; cat gpurun_out/timing.log
python scripts/compare_r1.py > gpurun_out/cmp.log 2>&1; echo "cmp rc=$?"; grep -c "True, True, True, True" gpurun_out/cmp.log; grep -v "True, True, True, True\|declined" gpurun_out/cmp.log | tail -5
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_joint.py -q -x ${PYTEST_ARGS} > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
if [ -n "$PROF" ]; then
python scripts/tail_profile.py $PROF > gpurun_out/tp.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_sweep -s 1 -c 1 -o gpurun_out/prof_tail_$PROF -f python scripts/tail_profile.py $PROF > gpurun_out/ncu_tail.log 2>&1; echo "ncu rc=$?"
fi
