python -m paper_2203_15031_b200.build > /dev/null 2>&1
run() {
  echo "== $*"
  env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python3 -c "import json,sys
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), d['roofline']['frac'])"
}
run SPMESL_S16_ZFRAC=1.0
run SPMESL_DEV_SIDE_ZERO=1
run SPMESL_DEV_SIDE_ZERO=1 SPMESL_DEV_PZ_BULK=148
run SPMESL_DEV_SIDE_ZERO=1 SPMESL_DEV_PZ_BULK=64
run SPMESL_S16_ZFRAC=0.5
run SPMESL_S16_ZFRAC=0.3
SPMESL_DEV_SIDE_ZERO=1 SPMESL_DEV_PZ_BULK=148 timeout 180 python scripts/timeline_probe.py 5 2>&1 | tail -20 | cut -c1-110
