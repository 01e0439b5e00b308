# dev: 128x256 tcgen05 screening tiles vs 128x128
python -m paper_2203_15031_b200.build > /dev/null 2>&1
timeout 300 python scripts/gram16_probe.py 2>&1 | grep -A1 "gram16"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
run() {
  echo "== $*"
  env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python3 -c "import json,sys
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), d['roofline']['frac'], d['roofline']['screen_candidates'])"
}
for bn in 128 256; do
run SPMESL_S16_BN=$bn SPMESL_DEV_S16_NOZERO=1
run SPMESL_S16_BN=$bn SPMESL_S16_ZFRAC=1.0
run SPMESL_S16_BN=$bn SPMESL_S16_ZFRAC=0.5
run SPMESL_S16_BN=$bn SPMESL_S16_ZFRAC=0.7
done
timeout 180 python scripts/timeline_probe.py 5 2>&1 | tail -22 | cut -c1-110
