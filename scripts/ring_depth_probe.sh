# dev: CD-kernel time per sweep wave vs X-ring depth and tile width (config 5)
for nst in 2 4 6; do echo "NST=$nst"; SPMESL_CD_NST=$nst timeout 120 python scripts/sweep_cost_probe.py 2>&1 | grep -E "m=  1|m= 32"; done
echo "skip-gemm"; SPMESL_CD_DEBUG=1 timeout 120 python scripts/sweep_cost_probe.py 2>&1 | grep -E "m=  1|m= 32"
echo "T=16"; PROBE_T=16 timeout 120 python scripts/sweep_cost_probe.py 2>&1 | grep -E "m=  1|m= 16|m= 32"
