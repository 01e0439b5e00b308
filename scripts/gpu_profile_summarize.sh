#!/bin/bash
# Round profile capture with the summaries made on the GPU box (the .ncu-rep files together
# exceed gpurun's 64 MiB copy-back): bench line, reference arm, launch lists, ncu summaries.
bash scripts/gpu_profile_round.sh
for r in s16 gc std tail_band tail_hub tail_univ; do
  [ -f gpurun_out/prof_$r.ncu-rep ] && python scripts/ncu_summary.py gpurun_out/prof_$r.ncu-rep 16 > gpurun_out/sum_$r.txt 2>&1
done
rm -f gpurun_out/prof_*.ncu-rep gpurun_out/clocks_*.csv
ls -la gpurun_out
