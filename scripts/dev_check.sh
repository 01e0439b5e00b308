mkdir -p gpurun_out
timeout 300 python tests/quick_gpu_check.py > gpurun_out/quick.log 2>&1; echo "quick rc=$?"; cat gpurun_out/quick.log | cut -c1-400
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_dev.json 2> gpurun_out/bench_dev.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_dev.json'))
print('value %.3e ms/step %.2f cd %.2f frac %.3f clocks %s' % (d['value'], d['ms_per_step'], d['ms_breakdown']['cd'], d['roofline']['frac'], d['clocks']))
"
