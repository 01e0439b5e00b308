python -m paper_2203_15031_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_joint.py -x -q 2>&1 | tail -5
for v in "A=1" "SPMESL_DEV_JOINT_RESIDUAL=1"; do
  echo "== $v"
  env $v timeout 600 python bench.py --mode joint --steps 3 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep "^{" | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config']['sweeps_total'], d['config']['max_outer'], d['config']['solver'])"
done
