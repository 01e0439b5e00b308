python -m paper_2203_15031_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "A=1" "SPMESL_DEV_STD_NOSTAGE=1"; do
  echo "== $v"
  env $v SPMESL_NO_GRAPH=1 timeout 180 python scripts/timeline_probe.py 5 2>&1 | grep -E "standardize" | tail -1 | cut -c1-100
  env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep "^{" | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"
done
