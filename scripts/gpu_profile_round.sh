#!/bin/bash
# Round profile capture (run under gpurun): bench line, reference arm, launch list, ncu of the
# dominant kernel (config 5) and of the sweep kernel (config 4 band(3) and hub).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:screen16 -s 3 -c 1 -o gpurun_out/prof_s16 -f $CMD > gpurun_out/ncu2.log 2>&1; echo "ncu screen16 rc=$?"
python scripts/tail_profile.py band3 > gpurun_out/tp_band.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_sweep -s 3 -c 1 -o gpurun_out/prof_tail_band -f python scripts/tail_profile.py band3 > gpurun_out/ncu3.log 2>&1; echo "ncu tail band rc=$?"
python scripts/tail_profile.py hub > gpurun_out/tp_hub.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_sweep -s 2 -c 1 -o gpurun_out/prof_tail_hub -f python scripts/tail_profile.py hub > gpurun_out/ncu4.log 2>&1; echo "ncu tail hub rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_cols -s 3 -c 1 -o gpurun_out/prof_gc -f $CMD > gpurun_out/ncu5.log 2>&1; echo "ncu gram_cols rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:standardize -s 3 -c 1 -o gpurun_out/prof_std -f $CMD > gpurun_out/ncu6.log 2>&1; echo "ncu standardize rc=$?"
python scripts/tail_profile.py univ5 > gpurun_out/tp_univ.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_sweep -s 1 -c 1 -o gpurun_out/prof_tail_univ -f python scripts/tail_profile.py univ5 > gpurun_out/ncu7.log 2>&1; echo "ncu tail univ rc=$?"
