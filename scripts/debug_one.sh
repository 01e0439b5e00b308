for i in 1 2; do echo "== debug=1 full run $i"; SPMESL_CD_DEBUG=1 timeout 60 python scripts/timing_probe.py 5 2>&1 | tail -2; done
echo "== debug=1 p2000"; SPMESL_CD_DEBUG=1 timeout 60 python scripts/timing_probe.py 4 p=2000 2>&1 | tail -1
echo "== debug=0"; timeout 60 python scripts/timing_probe.py 5 2>&1 | tail -2
timeout 300 python tests/quick_gpu_check.py 2>&1 | cut -c1-200
