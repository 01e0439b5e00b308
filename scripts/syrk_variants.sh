# dev: Gram-kernel time for compile-time variants (rebuilds gram_full.cu on the box)
for v in "-DSPMESL_SYRK_SMNR=0" "-DSPMESL_SYRK_SMNR=1" "-DSPMESL_SYRK_SMNR=1 -DSPMESL_SYRK_MIG=4" "-DSPMESL_SYRK_SMNR=1 -DSPMESL_SYRK_MIG=8"; do
  SPMESL_NVCC_EXTRA="$v" python -m paper_2203_15031_b200.build --force > /dev/null 2>&1
  echo "$v"; timeout 100 python scripts/screen_probe.py 2>&1 | tail -1; timeout 100 python scripts/timing_probe.py 5 2>&1 | tail -1
done
python -m paper_2203_15031_b200.build --force > /dev/null 2>&1
