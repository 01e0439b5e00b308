mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:screen16 -s 3 -c 1 -o gpurun_out/prof_s16 -f $CMD > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
if [ -n "$PROFILE_ALL" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:syrk_screen -s 2 -c 1 -o gpurun_out/prof_syrk -f $CMD --solver gram > gpurun_out/ncu3.log 2>&1; echo "ncu3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cd_sweep -s 2 -c 1 -o gpurun_out/prof_cd -f $CMD --solver residual > gpurun_out/ncu4.log 2>&1; echo "ncu4 rc=$?"
fi
