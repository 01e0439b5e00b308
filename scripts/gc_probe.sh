python -m paper_2203_15031_b200.build > /dev/null 2>&1
run() {
  echo "== $*"
  env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python3 -c "import json,sys
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), d['graph_replay'])"
}
run A=1
run SPMESL_DEV_SIDE_ZERO=1
run SPMESL_DEV_SIDE_ZERO=1 SPMESL_DEV_PZ_MEMSET=1
run SPMESL_DEV_SIDE_ZERO=1 SPMESL_DEV_PZ_EARLY=1
run SPMESL_DEV_SIDE_ZERO=1 SPMESL_DEV_PZ_EARLY=2
SPMESL_DEV_SIDE_ZERO=1 SPMESL_DEV_PZ_EARLY=2 timeout 180 python scripts/timeline_probe.py 5 2>&1 | tail -22 | cut -c1-110
