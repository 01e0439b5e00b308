for v in "-DSPMESL_GC_GROUP=2" "-DSPMESL_GC_GROUP=3" "-DSPMESL_GC_GROUP=6"; do
  SPMESL_NVCC_EXTRA="$v" python -m paper_2203_15031_b200.build --force > /dev/null 2>&1
  echo "== $v"
  SPMESL_NO_GRAPH=1 timeout 180 python scripts/timeline_probe.py 5 2>&1 | grep gram_cols | tail -1 | cut -c1-40
done
python -m paper_2203_15031_b200.build --force > /dev/null 2>&1
