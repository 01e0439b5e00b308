# dev: tail sweeps with / without the Gram-column prefetch must agree bitwise; timings
SPMESL_TAIL_NOPREFETCH=1 SPMESL_TAIL_EAGER=1 timeout 200 python scripts/lazy_check.py
timeout 200 python scripts/lazy_check.py
