for d in 0 1 2 3; do echo "debug=$d"; SPMESL_CD_DEBUG=$d timeout 60 python scripts/timing_probe.py 5 | tail -1; done
