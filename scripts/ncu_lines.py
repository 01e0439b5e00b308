"""Warp-stall samples per CUDA source line of an ncu report (cuda,sass source view)."""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = defaultdict(float)
src = {}
fname = ""
cur = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 5 or r[0] in ("Line No", "Function Name"):
        continue
    # cuda lines carry a line number in column 0; sass rows under them have an empty column 0
    if r[0].strip():
        cur = (fname, int(r[0]))
        src[cur] = r[1][:110]
        try:
            agg[cur] += float(r[4] or 0)
        except ValueError:
            pass
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100 * v / tot:5.1f}%  {k[0]}:{k[1]:<5d} {src[k]}")
