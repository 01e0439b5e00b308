for d in 4 5 6; do echo "debug=$d"; SPMESL_CD_DEBUG=$d timeout 60 python scripts/timing_probe.py 5 2>&1 | tail -4; done
