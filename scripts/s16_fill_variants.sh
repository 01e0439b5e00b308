# dev: screening-kernel ring depth vs zero-fill piece size (the kernel is bound by Theta's fill)
for rep in 1 2; do
for v in "-DSPMESL_T5_NST=4 -DSPMESL_S16_ZPIECE=2048" "-DSPMESL_T5_NST=3 -DSPMESL_S16_ZPIECE=4096" "-DSPMESL_T5_NST=3 -DSPMESL_S16_ZPIECE=2048"; do
  SPMESL_NVCC_EXTRA="$v" python -m paper_2203_15031_b200.build --force > /dev/null 2>&1
  echo "== $v"
  timeout 300 python bench.py --steps 50 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep "^{" | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3))"
done
done
python -m paper_2203_15031_b200.build --force > /dev/null 2>&1
