# dev: screen16 kernel time vs ring depth and the fused zero fill
for v in "-DSPMESL_S16_NST=4" "-DSPMESL_S16_NST=6"; do
  SPMESL_NVCC_EXTRA="$v" python -m paper_2203_15031_b200.build --force > /dev/null 2>&1
  for z in 0 1; do
    if [ $z = 1 ]; then export SPMESL_DEV_S16_NOZERO=1; else unset SPMESL_DEV_S16_NOZERO; fi
    echo "$v nozero=$z"; timeout 200 python scripts/timeline_probe.py 5 2>&1 | grep screen16 | tail -1 | cut -c1-40
  done
done
unset SPMESL_DEV_S16_NOZERO
python -m paper_2203_15031_b200.build --force > /dev/null 2>&1
