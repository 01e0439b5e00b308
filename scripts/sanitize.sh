TOOL=${TOOL:-memcheck}
SPMESL_CD_DEBUG=${DBG:-1} timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $TOOL --print-limit 20 python scripts/timing_probe.py 5 ${ARGS} > gpurun_out/sanitize_$TOOL.log 2>&1; echo "rc=$?"
tail -40 gpurun_out/sanitize_$TOOL.log
