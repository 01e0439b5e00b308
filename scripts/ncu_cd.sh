mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline $*"
timeout 300 $CMD > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cd_sweep -s 1 -c 1 -o gpurun_out/prof_cd -f $CMD > gpurun_out/ncu_cd.log 2>&1; echo "ncu rc=$?"
