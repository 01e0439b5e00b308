# dev: tcgen05 screen kernel vs the mma.sync one (correctness via gram vs gram16 identity, time)
mkdir -p gpurun_out
python -m paper_2203_15031_b200.build > /dev/null 2>&1
for ms in 1 0; do
  echo "== SPMESL_S16_MMA_SYNC=$ms"
  SPMESL_S16_MMA_SYNC=$ms timeout 180 python scripts/gram16_probe.py 2>&1 | grep -A1 "gram16"; echo "rc=$?"
  SPMESL_S16_MMA_SYNC=$ms timeout 180 python scripts/timeline_probe.py 5 2>&1 | grep -E "screen16" | tail -1 | cut -c1-60
  SPMESL_DEV_S16_NOZERO=1 SPMESL_S16_MMA_SYNC=$ms timeout 180 python scripts/timeline_probe.py 5 2>&1 | grep -E "screen16" | tail -1 | cut -c1-60
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 180 python scripts/timeline_probe.py 5 2>&1 | tail -25
