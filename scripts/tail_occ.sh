# dev: sweep-kernel launch shape (default: 2 CTAs/SM when they fit, else 1 with prefetch)
python -m paper_2203_15031_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "4" "4 family=hub" "5" "3" "2"; do
  for v in "A=1" "SPMESL_TAIL_OCC=1"; do
    echo "== $cfg $v"
    env $v timeout 200 python scripts/timing_probe.py $cfg 2>&1 | tail -1 | sed 's/.*total/total/'
  done
done
