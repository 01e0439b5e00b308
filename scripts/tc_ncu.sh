mkdir -p gpurun_out
python -m paper_2203_15031_b200.build > /dev/null 2>&1
for ms in 0 1; do
  SPMESL_DEV_S16_NOZERO=1 SPMESL_S16_MMA_SYNC=$ms timeout 600 ncu --set full --clock-control none -k regex:screen16 -s 1 -c 1 -o gpurun_out/prof_s16_$ms -f python scripts/timeline_probe.py 5 > gpurun_out/ncu_s16_$ms.log 2>&1; echo "rc=$?"
done
