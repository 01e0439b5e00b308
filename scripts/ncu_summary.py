"""Summarise an ncu report of the CD kernel: key raw metrics + stall breakdown + hot SASS."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
for k in keys:
    for i, name in enumerate(h):
        if name == k or name.endswith(k):
            print(f"{name:80s} {u[i]:>10s} {v[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; data = rows[2:]
idx = {x: i for i, x in enumerate(hdr)}
def f(row, k):
    try: return float(row[idx[k]].replace(",", ""))
    except: return 0.0
stalls = [x for x in hdr if x.startswith("stall_") and "Not Issued" not in x]
tot = {s: sum(f(rw, s) for rw in data) for s in stalls}
T = sum(tot.values()) or 1
print("stalls:", ", ".join(f"{s[6:]} {v/T*100:.1f}%" for s, v in sorted(tot.items(), key=lambda x: -x[1])[:10]))
S = sum(f(rw, "Warp Stall Sampling (All Samples)") for rw in data) or 1
top = sorted(data, key=lambda rw: -f(rw, "Warp Stall Sampling (All Samples)"))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for rw in top:
    dom = max(stalls, key=lambda s: f(rw, s))
    print(f"{rw[0][-5:]} {f(rw,'Warp Stall Sampling (All Samples)')/S*100:5.1f}% {rw[1][:58]:58s} exec {rw[idx['Instructions Executed']]:>10s} {dom[6:]}")
