# dev: tail sweeps — register-z kernel vs shared-memory-z kernel without prefetch must agree
# bitwise; timings of both
SPMESL_TAIL_SMEMZ=1 SPMESL_TAIL_NOPREFETCH=1 SPMESL_TAIL_EAGER=1 timeout 200 python scripts/lazy_check.py
timeout 200 python scripts/lazy_check.py
