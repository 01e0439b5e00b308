python -m paper_2203_15031_b200.build > /dev/null 2>&1
for v in "A=1" "SPMESL_TAIL_NPF=0"; do
for cfg in "5" "4" "4 family=hub" "2"; do
  echo "== $v cfg $cfg"
  env $v timeout 200 python scripts/timing_probe.py $cfg 2>&1 | tail -1 | sed 's/.*total/total/'
done
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
