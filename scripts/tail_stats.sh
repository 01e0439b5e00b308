# dev: per-column tail-solver counters for config 4 hub (lazy and eager)
for e in 0 1; do
  SPMESL_TAIL_EAGER=$e SPMESL_TAIL_STATS=1 timeout 100 python scripts/timing_probe.py 4 family=hub 2>&1 | tail -1
  python - <<'PY'
import csv
r = list(csv.DictReader(open("gpurun_out/tail_stats.csv")))
r.sort(key=lambda x: -int(x["cycles"]))
for x in r[:5]:
    v = int(x["sweeps"]); sw = v & ((1 << 20) - 1); sc = v >> 20
    print(x["col"], "sweeps", sw, "visits", x["visits"], "rounds", x["rounds"], "full", x["full_refresh"], "row", x["row_refresh"],
          "us/sweep %.2f" % (int(x["cycles"]) / 1965.0 / max(sw, 1)), "search us/sweep %.2f" % (sc / 1965.0 / max(sw, 1)))
PY
done
