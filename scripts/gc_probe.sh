python -m paper_2203_15031_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
run() {
  echo "== $*"
  env "$@" timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python3 -c "import json,sys
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), d['graph_replay'], d['ms_breakdown']['total_device'])"
}
run A=1
SPMESL_NO_GRAPH=1 timeout 180 python scripts/timeline_probe.py 5 2>&1 | tail -16 | cut -c1-110
