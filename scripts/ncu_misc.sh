mkdir -p gpurun_out
python -m paper_2203_15031_b200.build > /dev/null 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:standardize -s 3 -c 1 -o gpurun_out/prof_std -f $CMD > gpurun_out/ncu_std.log 2>&1; echo "std rc=$?"
