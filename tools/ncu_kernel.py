"""Per-kernel summary of a multi-kernel ncu report: time, DRAM bytes, issue/tensor activity, top
stall reasons and the hottest source lines. Usage: ncu_kernel.py report.ncu-rep [index ...]"""
import csv, subprocess, sys

rep = sys.argv[1]
want = [int(x) for x in sys.argv[2:]]


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(run("--page", "raw", "--csv").splitlines()))
h = raw[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for i in (want or range(len(raw) - 2)):
    v = raw[2 + i]
    print(f"== [{i}] {v[h.index('Kernel Name')][:90]}")
    for k in keys:
        if k in h:
            print(f"   {k:75s} {v[h.index(k)]}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(x) for k, x in zip(h, v)
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and x.replace('.', '', 1).isdigit()}
    tot = sum(st.values()) or 1
    print("   stalls:", ", ".join(f"{k} {100*x/tot:.1f}%" for k, x in sorted(st.items(), key=lambda kv: -kv[1])
                                if x / tot > 0.02))
