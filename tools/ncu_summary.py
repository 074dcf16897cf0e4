"""Summarise an ncu report: key metrics, stall reasons and SASS opcode mix per unit of work."""
import csv, subprocess, sys
from collections import Counter

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else None  # e.g. cell-pairs in the captured launch


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(run("--page", "raw", "--csv").splitlines()))
h, v = raw[0], raw[2]
want = ["gpu__time_duration.sum", "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
        "sm__inst_executed_pipe_fp64.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum"]
for k, x in zip(h, v):
    if k in want:
        print(f"{k:70s} {x}")
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(x) for k, x in zip(h, v)
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and x.replace('.', '', 1).isdigit()}
tot = sum(st.values()) or 1
print("stalls:", ", ".join(f"{k} {100*x/tot:.1f}%" for k, x in sorted(st.items(), key=lambda kv: -kv[1]) if x / tot > 0.01))
rows = list(csv.reader(run("--page", "source", "--csv", "--print-source", "sass").splitlines()))
hdr = rows[1]
ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
c = Counter()
for r in rows[2:]:
    tk = r[isrc].split()
    if not tk:
        continue
    op = (tk[1] if tk[0].startswith("@") else tk[0]).split(".")[0]
    c[op] += float(r[ia] or 0)
T = sum(c.values())
if units:
    print(f"thread-instructions per unit: {32*T/units:.2f}")
print("mix:", ", ".join(f"{op} {100*x/T:.1f}%" + (f" ({32*x/units:.2f}/u)" if units else "") for op, x in c.most_common(16)))
