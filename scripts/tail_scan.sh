python -m paper_2203_15031_b200.build > /dev/null 2>&1
for v in "A=1" "SPMESL_TAIL_NT=256"; do
for cfg in "5" "4 family=hub"; do
  echo "== $v cfg $cfg"
  env $v timeout 200 python scripts/timing_probe.py $cfg 2>&1 | tail -1 | sed 's/.*total/total/'
done
done
SPMESL_TAIL_OCC=1 timeout 200 python scripts/timing_probe.py 4 family=hub 2>&1 | tail -1 | sed 's/.*total/total occ1-512: /'
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep "^{" | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"
