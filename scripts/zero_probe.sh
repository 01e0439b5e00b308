# dev: share of Theta's zero fill fused into the screening kernel vs run beside the later kernels
python -m paper_2203_15031_b200.build > /dev/null 2>&1
for f in 1.0 0.7 0.55 0.4 0.25; do
  export SPMESL_S16_ZFRAC=$f
  echo "== zfrac $f"
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | python3 -c "import json,sys
for l in sys.stdin:
  if l.startswith('{'): d=json.loads(l); print(d['ms_per_step'], d['roofline']['kernel_ms'])
  elif 'step ms' in l: print(l.strip()[:200])"
done
export SPMESL_S16_ZFRAC=0.55
timeout 180 python scripts/timeline_probe.py 5 2>&1 | tail -22 | cut -c1-110
